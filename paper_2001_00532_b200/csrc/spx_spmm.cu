// SpMM kernels: C(i,k) = A(i,j) * B(j,k), A in CSR ("ds"), B/C dense row-major.
//
//  K4 SPX_K_SPMM_NNZ  -- Appendix A.4:
//      fuse(i,j,f) pos(f,fpos,A) split(fpos,block,fpos1,NNZ_PER_TB)
//      split(fpos1,warp,nnz,NNZ_PER_WARP) split(k,dvu,thread,32)
//      bound(dvu,dense_val,ceil(N/32),MaxExact)
//    Each CTA owns NNZ_PER_TB consecutive nonzeros (the `block` variable),
//    each warp NNZ_PER_WARP of them (`warp`), and the 32 lanes of a warp
//    cover the dense row k (`thread`, `dense_val`).  The warp walks its
//    positions sequentially (`nnz`) while tracking the row with a row-end
//    cache (SPEC.md:364 Track recovery), gathering one 512 B row of B per
//    nonzero with 16 B vector loads.
//
//    Output without a memset of C and without atomics: a row is *owned* by
//    the chunk that holds its first position pos[r] (empty rows included,
//    rows with pos[r]==nnz by the last chunk).  The owner stores its partial
//    sum with a plain (streaming) store.  A chunk's only other row is its
//    *head* row (the row holding the chunk's first position but starting
//    before it); the head partial is parked in shared memory, summed across
//    warps after the barrier and added onto the owner's value when the owner
//    is in the same CTA, or written to a per-CTA carry slot that the fix-up
//    kernel adds in CTA order (deterministic, SURVEY.md §7.3 "carry-out
//    fixup").  This is the `Atomics` race strategy of the schedule realised
//    without atomics.
//
//  K5 SPX_K_SPMM_ROW  -- warp-per-row (A.3/A.10/A.11 shapes and the GPU
//    warp-per-row schedule): split(i,block,block_row,ROWS_PER_TB)
//    split(block_row,warp_row,warp,WARPS) -> warp w of block b handles rows
//    b*ROWS + warp_row*WARPS + w; lanes cover k.
#include <cstdlib>

#include "spx_common.cuh"

#ifndef SPX_SPMM_ROWS8
#define SPX_SPMM_ROWS8 1
#endif
#ifndef SPX_SPMM_MINB
#define SPX_SPMM_MINB 2  // 512-thread blocks per SM the register path is compiled for (<= 64 regs, no spills)
#endif

namespace spx {
namespace {

template <typename T, int VPL>
constexpr int unroll_for() {
  constexpr int words = VPL * (int)sizeof(T) / 4;  // 32-bit registers per fragment
  constexpr int u = 32 / words;
  return u > 8 ? 8 : (u < 2 ? 2 : u);
}

// first s in [lo,hi) with arr[s] >= key (warp-cooperative, 32-ary)
__device__ __forceinline__ int64_t warp_lower_bound(const int32_t* __restrict__ arr, int64_t lo,
                                                    int64_t hi, int64_t key, int lane) {
  int64_t a = lo, b = hi;  // answer in [a, b]
  while (b - a > 32) {
    int64_t stride = (b - a + 31) >> 5;
    int64_t idx = a + (int64_t)lane * stride;
    bool lt = idx < b && (int64_t)__ldg(arr + idx) < key;
    unsigned m = __ballot_sync(kFull, lt);
    if (m == 0) return a;
    int last = 31 - __clz(m);
    int64_t na = a + (int64_t)last * stride + 1;
    int64_t nb = a + (int64_t)(last + 1) * stride;
    if (nb > b) nb = b;
    a = na;
    b = nb;
  }
  int64_t idx = a + lane;
  bool lt = idx < b && (int64_t)__ldg(arr + idx) < key;
  unsigned m = __ballot_sync(kFull, lt);
  return a + __popc(m);
}

template <typename T, int VPL, bool CONTIG>
__device__ __forceinline__ void store_zero_row(T* __restrict__ row, int lane, int ncols) {
  Frag<T, VPL, CONTIG> z;
  z.zero();
  z.store(row, lane, ncols);
}

// One batch of 32 consecutive positions held one per lane: column and value.
template <typename T>
struct Batch {
  int c;
  T v;
  __device__ __forceinline__ void load(const int32_t* __restrict__ crd, const T* __restrict__ vals, int idx, int end,
                                       uint64_t pol) {
    c = 0;
    v = T(0);
    if (idx < end) {
      c = ld_i32_first(crd + idx, pol);
      v = ld_stream_hint(vals + idx, pol);
    }
  }
};

// RING == 0: staged-register path (default; any VPL / mapping).
// RING  > 0: cp.async ring of RING row slots per warp in shared memory
//            (CONTIG rows of 16 or 32 B per lane): each lane copies and later
//            reads back only its own 16 B pieces, so the per-lane
//            cp.async.wait_group is the only synchronisation; no data
//            registers are held for rows in flight, which buys occupancy.
template <typename T, int VPL, bool CONTIG, int U, int RING>
__global__ void __launch_bounds__(kMaxThreads, RING == 0 ? SPX_SPMM_MINB : 1) spmm_nnz_kernel(
    const int32_t* __restrict__ pos, const int32_t* __restrict__ crd, const T* __restrict__ vals,
    const T* __restrict__ B, T* __restrict__ C, int64_t M, int64_t N, int64_t nnz, int64_t TB,
    int64_t W, int32_t* __restrict__ carry_row, T* __restrict__ carry_val, const int32_t* __restrict__ first) {
  using F = Frag<T, VPL, CONTIG>;
  constexpr int PW = 32 * VPL;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nw = blockDim.x >> 5;
  T* sval = reinterpret_cast<T*>(smem_raw);
  int32_t* srow = reinterpret_cast<int32_t*>(sval + nw * PW);
  T* ring_base = reinterpret_cast<T*>(smem_raw + ((nw * (PW * sizeof(T) + sizeof(int32_t)) + 15) & ~size_t(15)));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t cta = blockIdx.x, ncta = gridDim.x;
  const int64_t p0 = cta * TB;
  const int64_t p1 = min(p0 + TB, nnz);
  const int64_t q0 = min(p0 + (int64_t)warp * W, p1);
  const int64_t q1 = min(q0 + W, p1);
  const int64_t col0 = (int64_t)blockIdx.y * PW;
  const int ncols = (int)min((int64_t)PW, N - col0);
  const T* __restrict__ Bp = B + col0;
  T* __restrict__ Cp = C + col0;

  int32_t head = -1;
  if (q0 < q1) {
    int64_t r = __ldg(first + q0 / W);  // row holding q0 (chunk_segments_kernel)
    const int64_t rstart = __ldg(pos + r);
    bool is_head = rstart < q0;
    if (!is_head && r > 0 && __ldg(pos + r - 1) == q0) {
      // empty rows with pos == q0 sit before r and belong to this chunk
      int64_t lb = warp_lower_bound(pos, 0, r, q0, lane);
      for (int64_t rr = lb; rr < r; ++rr) store_zero_row<T, VPL, CONTIG>(Cp + rr * N, lane, ncols);
    }
    // Hot loop.  Positions fit int32 (pos is int32, tensors.py:248).  The
    // next 32 (crd, vals) are fetched one batch ahead; within a batch the B
    // gathers run two groups of U rows ahead of the FMAs (double buffer),
    // so each warp keeps up to 2*U 512 B rows in flight.
    const uint64_t pol_b = l2_evict_last();
    const uint64_t pol_s = l2_evict_first();
    RowEndCache ends;
    ends.fill(pos, r, M, lane);
    int rr32 = (int)r;
    int rend = (int)ends.end(pos, r, M, lane);
    F acc;
    acc.zero();
    const int qe = (int)q1;
    int p = (int)q0;
    auto flush = [&]() {
      if (is_head) {
        acc.store_smem(sval + warp * PW, lane);
        head = rr32;
        is_head = false;
      } else {
        acc.store_hint(Cp + (int64_t)rr32 * N, lane, ncols, pol_s);
      }
      acc.zero();
    };
    if constexpr (RING > 0) {
      static_assert(CONTIG && (VPL * sizeof(T)) % 16 == 0, "ring path needs 16 B lane pieces");
      static_assert(32 % RING == 0 && RING % 4 == 0, "ring depth must divide the 32-position batch");
      constexpr int LB = VPL * (int)sizeof(T);  // bytes per lane per row
      constexpr int ROWB = 32 * LB;
      constexpr int GS = 4;          // positions per cp.async commit group
      constexpr int NG = RING / GS;  // groups resident in the ring
      T* ring = ring_base + (size_t)warp * RING * PW;
      const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring) + lane * LB;
      const T* ring_lane = ring + lane * VPL;
      const char* Bb = reinterpret_cast<const char*>(Bp) + lane * LB;
      const uint32_t rowstride = (uint32_t)(N * (int64_t)sizeof(T));
      const int n = qe - p;
      Batch<T> b0, b1, b2;  // batches k, k+1 (resident) and k+2 (in flight)
      b0.load(crd, vals, p + lane, qe, pol_s);
      b1.load(crd, vals, p + 32 + lane, qe, pol_s);
      b2.load(crd, vals, p + 64 + lane, qe, pol_s);
      auto issue = [&](int c, int slot) {
        const char* src = Bb + (uint64_t)(uint32_t)c * rowstride;
#pragma unroll
        for (int k = 0; k < LB / 16; ++k) cp_async16(ring_s + slot * ROWB + k * 16, src + k * 16, pol_b);
      };
      // prologue: groups 0 .. NG-2 in flight
#pragma unroll
      for (int t = 0; t < RING - GS; ++t) {
        const int c = __shfl_sync(kFull, b0.c, t);
        if (t < n) issue(c, t);
        if (t % GS == GS - 1) cp_async_commit();
      }
      for (int base = 0; base < n; base += 32) {
        const bool full = base + 32 + RING - GS <= n;
#pragma unroll
        for (int j = 0; j < 32 / GS; ++j) {
          // issue group j+NG-1 (may reach into the next batch)
#pragma unroll
          for (int u = 0; u < GS; ++u) {
            const int t = (j + NG - 1) * GS + u;
            const int c = __shfl_sync(kFull, t < 32 ? b0.c : b1.c, t & 31);
            if (full || base + t < n) issue(c, t % RING);
          }
          cp_async_commit();
          cp_async_wait<NG - 1>();  // group j has landed (for this lane's pieces)
          if (!full && base + j * GS >= n) break;
          const int gbase = p + base + j * GS;
          const int cnt = full ? GS : min(GS, n - base - j * GS);
          T vv[GS];
          F bv[GS];
#pragma unroll
          for (int u = 0; u < GS; ++u) {
            vv[u] = __shfl_sync(kFull, b0.v, j * GS + u);
            const float4* sp = reinterpret_cast<const float4*>(ring_lane + ((j * GS + u) % RING) * PW);
#pragma unroll
            for (int k = 0; k < LB / 16; ++k) unpack16(&bv[u].v[k * (16 / sizeof(T))], sp[k]);
          }
          if (cnt == GS && gbase + GS <= rend) {
#pragma unroll
            for (int u = 0; u < GS; ++u) acc.fma(vv[u], bv[u]);
          } else {
#pragma unroll
            for (int u = 0; u < GS; ++u) {
              if (u < cnt) {
                while (gbase + u >= rend) {  // row(s) finished: store, skip empty rows
                  flush();
                  ++rr32;
                  rend = (int)ends.end(pos, rr32, M, lane);
                }
                acc.fma(vv[u], bv[u]);
              }
            }
          }
        }
        b0 = b1;
        b1 = b2;
        b2.load(crd, vals, p + base + 96 + lane, qe, pol_s);
      }
      cp_async_wait<0>();
    } else {
      // Staged-register path: the (column, value) pairs of each 32-position
      // batch stream into a per-warp cp.async ring and come back as 16 B
      // broadcasts (4 columns / 4 values per LDS); the B rows go straight
      // into registers with LDG.128, four rows in flight per warp.  Per
      // nonzero: one 512 B row gather + half a broadcast + VPL/2 FFMA2.
      constexpr int SR = 4;  // ring depth (batches)
      using Ring = LeafRing<T, SR>;
      Ring ring;
      ring.init(reinterpret_cast<unsigned char*>(ring_base) + (size_t)warp * Ring::kBytes, crd, vals, p, qe);
      ring.prologue(lane, pol_s);
      const char* __restrict__ Bl = reinterpret_cast<const char*>(Bp + (CONTIG ? lane * VPL : 0));
      const uint32_t rowb = (uint32_t)(N * (int64_t)sizeof(T));
      auto brow = [&](F& d, int c) {
        if constexpr (CONTIG) {
          d.load_ptr_hint(reinterpret_cast<const T*>(addr_wide(Bl, (uint32_t)c, rowb)), pol_b);
        } else {
          d.load(reinterpret_cast<const T*>(addr_wide(Bl, (uint32_t)c, rowb)), lane, ncols);
        }
      };
      for (int b = 0; b < ring.nb; ++b) {
        ring.acquire(b, lane, pol_s);
        const int pb = p + b * 32;
        const int n = min(32, qe - pb);
        const int32_t* Cs = ring.crd_slot(b);
        const T* Vs = ring.val_slot(b);
        // eight B rows in flight per warp when a row is one 16 B piece per lane
        // (cfg2: 64 registers, no spills): 1.67 -> 1.44 ms, against four rows
        constexpr bool kRows8 = SPX_SPMM_ROWS8 && VPL * (int)sizeof(T) <= 16;
        if constexpr (kRows8) {
#pragma unroll 1
        for (int t8 = 0; t8 < n; t8 += 8) {
          const int4 c4a = *reinterpret_cast<const int4*>(Cs + t8);  // zero-filled past n
          const int4 c4b = *reinterpret_cast<const int4*>(Cs + t8 + 4);
          F a0, a1, a2, a3, e0, e1, e2, e3;
          brow(a0, c4a.x);
          brow(a1, c4a.y);
          brow(a2, c4a.z);
          brow(a3, c4a.w);
          brow(e0, c4b.x);
          brow(e1, c4b.y);
          brow(e2, c4b.z);
          brow(e3, c4b.w);
          if (pb + t8 + 8 <= rend && t8 + 8 <= n) {
            acc.fma(Vs[t8], a0);
            acc.fma(Vs[t8 + 1], a1);
            acc.fma(Vs[t8 + 2], a2);
            acc.fma(Vs[t8 + 3], a3);
            acc.fma(Vs[t8 + 4], e0);
            acc.fma(Vs[t8 + 5], e1);
            acc.fma(Vs[t8 + 6], e2);
            acc.fma(Vs[t8 + 7], e3);
            continue;
          }
          const F* bb[8] = {&a0, &a1, &a2, &a3, &e0, &e1, &e2, &e3};
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (t8 + u < n) {
              while (pb + t8 + u >= rend) {  // row(s) finished: store, skip empty rows
                flush();
                ++rr32;
                rend = (int)ends.end(pos, rr32, M, lane);
              }
              acc.fma(Vs[t8 + u], *bb[u]);
            }
          }
        }
        } else {
#pragma unroll 1
        for (int t = 0; t < n; t += 4) {
          const int4 c4 = *reinterpret_cast<const int4*>(Cs + t);  // zero-filled past n
          F b0, b1, b2, b3;
          brow(b0, c4.x);
          brow(b1, c4.y);
          brow(b2, c4.z);
          brow(b3, c4.w);
          const T v0 = Vs[t], v1 = Vs[t + 1], v2 = Vs[t + 2], v3 = Vs[t + 3];
          if (pb + t + 4 <= rend && t + 4 <= n) {
            acc.fma(v0, b0);
            acc.fma(v1, b1);
            acc.fma(v2, b2);
            acc.fma(v3, b3);
          } else {
            const F* bb[4] = {&b0, &b1, &b2, &b3};
            const T vv[4] = {v0, v1, v2, v3};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (t + u < n) {
                while (pb + t + u >= rend) {  // row(s) finished: store, skip empty rows
                  flush();
                  ++rr32;
                  rend = (int)ends.end(pos, rr32, M, lane);
                }
                acc.fma(vv[u], *bb[u]);
              }
            }
          }
        }
        }
        ring.release();
      }
    }  // RING == 0
    flush();
    r = rr32;
    if (q1 == nnz) {
      // trailing rows with pos[r] == nnz belong to the last chunk
      for (int64_t rr = r + 1; rr < M; ++rr) store_zero_row<T, VPL, CONTIG>(Cp + rr * N, lane, ncols);
    }
  } else if (nnz == 0 && cta == 0) {
    for (int64_t rr = warp; rr < M; rr += nw) store_zero_row<T, VPL, CONTIG>(Cp + rr * N, lane, ncols);
  }
  if (lane == 0) srow[warp] = head;
  __syncthreads();

  const int32_t hr = srow[warp];
  const int64_t slot = (int64_t)blockIdx.y * ncta + cta;
  if (hr >= 0 && (warp == 0 || srow[warp - 1] != hr)) {
    F s;
    s.zero();
    s.add_smem(sval + warp * PW, lane);
    for (int w2 = warp + 1; w2 < nw && srow[w2] == hr; ++w2) s.add_smem(sval + w2 * PW, lane);
    if ((int64_t)__ldg(pos + hr) >= p0) {
      s.add_into(Cp + (int64_t)hr * N, lane, ncols);  // owner stored before the barrier
    } else {
      s.store_smem(carry_val + slot * PW, lane);
      if (lane == 0) carry_row[slot] = hr;
    }
  }
  if (threadIdx.x == 0) {
    const int32_t h0 = srow[0];
    if (!(h0 >= 0 && (int64_t)__ldg(pos + h0) < p0)) carry_row[slot] = -1;
  }
}

// Adds the per-CTA carries onto their rows.  The first CTA of a run of
// equal carry rows sums the run in CTA order and updates C once.
template <typename T, int VPL, bool CONTIG>
__global__ void carry_fixup_kernel(const int32_t* __restrict__ carry_row, const T* __restrict__ carry_val,
                                   T* __restrict__ C, int64_t N, int64_t nslots) {
  using F = Frag<T, VPL, CONTIG>;
  constexpr int PW = 32 * VPL;
  const int lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= nslots) return;
  const int64_t base = (int64_t)blockIdx.y * nslots;
  const int32_t row = carry_row[base + c];
  if (row < 0) return;
  if (c > 0 && carry_row[base + c - 1] == row) return;
  const int64_t col0 = (int64_t)blockIdx.y * PW;
  const int ncols = (int)min((int64_t)PW, N - col0);
  F s;
  s.zero();
  for (int64_t c2 = c; c2 < nslots && carry_row[base + c2] == row; ++c2)
    s.add_smem(carry_val + (base + c2) * PW, lane);
  s.add_into(C + col0 + (int64_t)row * N, lane, ncols);
}

// K5 warp-per-row: the row's (column, value) pairs stream through the
// warp's cp.async LeafRing (three batches ahead) and come back as 16 B
// broadcasts; B rows are gathered U at a time into registers.  A row longer
// than the ring keeps streaming, so one warp on a long row still has ~U rows
// of B and three batches of A in flight.
#ifndef SPX_SPMM_ROW_PF
#define SPX_SPMM_ROW_PF 1  // next-batch L1 prefetch of B rows in K5's row walk (cfg2 K5 6.21 -> 5.30 ms)
#endif
#ifndef SPX_SPMM_ROW_MINB
#define SPX_SPMM_ROW_MINB 1  // K5: the heaviest row is latency-bound; 16 rows in flight beat occupancy
#endif
// acc = sum over positions [a, e) of A[p] * B[crd[p], panel] (one warp)
template <typename T, int VPL, bool CONTIG, int U, bool PF = false>
__device__ __forceinline__ void spmm_row_range(Frag<T, VPL, CONTIG>& acc, const int32_t* __restrict__ crd,
                                               const T* __restrict__ vals, const char* __restrict__ Bl,
                                               uint32_t rowb, int ncols, unsigned char* ring_base, int lane, int a,
                                               int e, uint64_t pol_s) {
  using F = Frag<T, VPL, CONTIG>;
  using Ring = LeafRing<T, 4>;
  Ring ring;
  ring.init(ring_base, crd, vals, a, e);
  ring.prologue(lane, pol_s);
  for (int b = 0; b < ring.nb; ++b) {
    if constexpr (PF) {
      // batches b and b+1 landed: batch b+1's B rows start moving into L1
      // (each lane prefetches the lines of its leaf's row panel) -- a warp
      // alone on a long row is latency-bound on these gathers
      ring.issue(b + 3, lane, pol_s);
      cp_async_wait<2>();
      __syncwarp();
      if (b + 1 < ring.nb && a + (b + 1) * 32 + lane < e) {
        const char* rp = Bl - (CONTIG ? lane * VPL * (int)sizeof(T) : 0) +
                         (size_t)(uint32_t)ring.crd_slot(b + 1)[lane] * rowb;
#pragma unroll
        for (int l = 0; l < (32 * VPL * (int)sizeof(T) + 127) / 128; ++l)
          asm volatile("prefetch.global.L1 [%0];" ::"l"(rp + l * 128));
      }
    } else {
      ring.acquire(b, lane, pol_s);
    }
    const int n = min(32, e - (a + b * 32));
    const int32_t* Cs = ring.crd_slot(b);
    const T* Vs = ring.val_slot(b);
#pragma unroll 1
    for (int t = 0; t < n; t += U) {
      F bb[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = Cs[t + u];  // zero-filled past n
        const T* src = reinterpret_cast<const T*>(addr_wide(Bl, (uint32_t)c, rowb));
        if constexpr (CONTIG) bb[u].load_ptr(src);
        else bb[u].load(src, lane, ncols);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (t + u < n) acc.fma(Vs[t + u], bb[u]);
    }
    ring.release();
  }
}

// CUT (CPU-tagged row schedules, A.3): a row longer than `cut` positions is
// skipped here and appended to heavy_list; spmm_heavy_row_kernel gives it a
// whole CTA.  With the long rows gone the warps are throughput-bound, so the
// kernel trades rows in flight for occupancy (SPX_SPMM_CUT_MINB / _UDIV).
// !CUT: every row on its warp, as a GPU schedule writes it.
#ifndef SPX_SPMM_CUT_MINB
#define SPX_SPMM_CUT_MINB 3  // cfg2 A.3: 3 CTAs/SM with 8 rows in flight 1.92 ms; 2 with 16: 2.07; 4 with 8: 2.02
#endif
#ifndef SPX_SPMM_CUT_UDIV
#define SPX_SPMM_CUT_UDIV 2  // B rows in flight per warp in the cut row kernel: UR / this
#endif
template <typename T, int VPL, bool CONTIG, int U, bool CUT>
__global__ void __launch_bounds__(kMaxThreads, CUT ? SPX_SPMM_CUT_MINB : SPX_SPMM_ROW_MINB) spmm_row_kernel(
    const int32_t* __restrict__ pos, const int32_t* __restrict__ crd, const T* __restrict__ vals,
    const T* __restrict__ B, T* __restrict__ C, int64_t M, int64_t N, int64_t R, int64_t cut,
    int32_t* __restrict__ heavy_list, int32_t* __restrict__ heavy_count) {
  using F = Frag<T, VPL, CONTIG>;
  using Ring = LeafRing<T, 4>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int PW = 32 * VPL;
  const int nw = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t col0 = (int64_t)blockIdx.y * PW;
  const int ncols = (int)min((int64_t)PW, N - col0);
  const T* __restrict__ Bp = B + col0;
  T* __restrict__ Cp = C + col0;
  const uint64_t pol_s = l2_evict_first();
  const char* __restrict__ Bl = reinterpret_cast<const char*>(Bp + (CONTIG ? lane * VPL : 0));
  const uint32_t rowb = (uint32_t)(N * (int64_t)sizeof(T));
  const int64_t rows_lo = (int64_t)blockIdx.x * R;
  const int nwr = (int)((R + nw - 1) / nw);
  for (int wr = 0; wr < nwr; ++wr) {
    const int64_t br = (int64_t)wr * nw + warp;  // block_row = warp_row*WARPS + warp
    if (br >= R) break;
    const int64_t row = rows_lo + br;
    if (row >= M) break;
    const int a = __ldg(pos + row), e = __ldg(pos + row + 1);
    if (CUT && e - a > cut) {
      if (lane == 0 && blockIdx.y == 0) heavy_list[atomicAdd(heavy_count, 1)] = (int32_t)row;
      continue;
    }
    F acc;
    acc.zero();
    spmm_row_range<T, VPL, CONTIG, U, !CUT && SPX_SPMM_ROW_PF>(acc, crd, vals, Bl, rowb, ncols,
                                                               smem_raw + (size_t)warp * Ring::kBytes, lane, a, e,
                                                               pol_s);
    acc.store(Cp + row * N, lane, ncols);
  }
}

// One CTA per heavy row (list order is irrelevant): warp w sums the w-th of
// nw equal position ranges, the partial rows meet in shared memory and warp 0
// adds them in range order -- the row still has one owner and a fixed
// summation order.
// 16 warps per heavy row, 2 CTAs/SM with half the row kernel's B rows in
// flight (tools/gpu_r02_az.sh); 8 / 4 warps per row were 4.20 / 7.05 ms
// (tools/gpu_r02_ae.sh)
constexpr int kHeavyWarps = 16;
#ifndef SPX_SPMM_HEAVY_MINB
#define SPX_SPMM_HEAVY_MINB 2  // cfg2 A.3: 2 CTAs/SM with 8 rows in flight 2.06 ms; 1 CTA/SM with 16: 2.15
#endif
#ifndef SPX_SPMM_HEAVY_UDIV
#define SPX_SPMM_HEAVY_UDIV 2  // B rows in flight per warp: the row kernel's UR / this (/4: 2.36 ms)
#endif
template <typename T, int VPL, bool CONTIG, int U>
__global__ void __launch_bounds__(kHeavyWarps * 32, SPX_SPMM_HEAVY_MINB) spmm_heavy_row_kernel(
    const int32_t* __restrict__ pos, const int32_t* __restrict__ crd, const T* __restrict__ vals,
    const T* __restrict__ B, T* __restrict__ C, int64_t N, const int32_t* __restrict__ heavy_list,
    const int32_t* __restrict__ heavy_count) {
  using F = Frag<T, VPL, CONTIG>;
  using Ring = LeafRing<T, 4>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int PW = 32 * VPL;
  if ((int64_t)blockIdx.x >= (int64_t)*heavy_count) return;
  const int nw = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t col0 = (int64_t)blockIdx.y * PW;
  const int ncols = (int)min((int64_t)PW, N - col0);
  const char* __restrict__ Bl = reinterpret_cast<const char*>(B + col0 + (CONTIG ? lane * VPL : 0));
  const uint32_t rowb = (uint32_t)(N * (int64_t)sizeof(T));
  const int64_t row = heavy_list[blockIdx.x];
  const int a = __ldg(pos + row), e = __ldg(pos + row + 1);
  const int64_t len = e - a;
  const int wa = a + (int)(len * warp / nw), we = a + (int)(len * (warp + 1) / nw);
  F acc;
  acc.zero();
  spmm_row_range<T, VPL, CONTIG, U>(acc, crd, vals, Bl, rowb, ncols, smem_raw + (size_t)warp * Ring::kBytes, lane,
                                    wa, we, l2_evict_first());
  T* part = reinterpret_cast<T*>(smem_raw + (size_t)nw * Ring::kBytes);  // [nw][PW]
  acc.store_smem(part + warp * PW, lane);
  __syncthreads();
  if (warp == 0) {
    F sum;
    sum.zero();
    for (int w = 0; w < nw; ++w) sum.add_smem(part + w * PW, lane);
    sum.store(C + col0 + row * N, lane, ncols);
  }
}

struct SpmmGeom {
  int vpl;
  int pw;
  int npanels;
  bool contig;
};

SpmmGeom spmm_geom(int dtype, int64_t N) {
  const int vmax = dtype == SPX_F32 ? 8 : 4;
  int v = (int)ceil_div(N < 1 ? 1 : N, 32);
  int vpl = 1;
  while (vpl < v && vpl < vmax) vpl <<= 1;
  SpmmGeom g;
  g.vpl = vpl;
  g.pw = 32 * vpl;
  g.npanels = (int)ceil_div(N < 1 ? 1 : N, g.pw);
  g.contig = (N % g.pw) == 0;
  return g;
}

// carry values per (CTA, panel), carry rows per (CTA, panel), and the
// per-warp-chunk start rows (ncta * warps_per_cta + 1)
NnzWorkspace spmm_workspace(int64_t ncta, int64_t wpc, const SpmmGeom& g, size_t es) {
  NnzWorkspace w = nnz_workspace(ncta * g.npanels, es, g.pw);
  const NnzWorkspace f = nnz_workspace(ncta * wpc, 1, 0);
  w.total = w.first + (f.total - f.first);
  return w;
}

int check_bound(const Args& a, int64_t N) {
  const int ws = a.params[2] ? a.params[2] : 32;
  if (ws != 32)
    return fail(SPX_E_UNSUPPORTED, "split of the dense dimension must be WARP_SIZE=32, got %d", ws);
  const int b = a.params[3];
  if (b != 0 && (int64_t)b != ceil_div(N, 32))
    return fail(SPX_E_CONTRACT,
                "MaxExact bound violated: dense_val bound %d but the runtime extent ceil(%lld/32) is %lld",
                b, (long long)N, (long long)ceil_div(N, 32));
  return SPX_OK;
}

// Depth of the cp.async row ring (0 = register pipeline); SPX_SPMM_RING
// overrides the default for tuning sweeps.
int ring_depth() {
  static const int d = [] {
    const char* s = getenv("SPX_SPMM_RING");
    return s ? atoi(s) : -1;
  }();
  return d;
}

// positions above which a CPU-tagged row schedule hands a row to a whole CTA
#ifndef SPX_SPMM_CUT_MIN
#define SPX_SPMM_CUT_MIN 512  // cfg2 A.3: 4096 -> 3.76 ms, 2048 -> 3.24, 1024 -> 3.10, 512 -> 2.95, 256 -> 3.12
#endif
#ifndef SPX_SPMM_CUT_DIV
#define SPX_SPMM_CUT_DIV 131072
#endif
inline int64_t spmm_row_cut(int64_t nnz) { return std::max<int64_t>(SPX_SPMM_CUT_MIN, nnz / SPX_SPMM_CUT_DIV); }
inline size_t ws_spmm_row(int64_t nnz) {
  return (size_t)(4 + std::max<int64_t>(1, nnz / (spmm_row_cut(nnz) + 1))) * sizeof(int32_t);
}

template <typename T, int VPL, bool CONTIG>
int run_spmm(int kid, const Args& a, const SpmmGeom& g) {
  constexpr int U = unroll_for<T, VPL>();
  const int32_t* pos = a.pos[0];
  const int32_t* crd = a.crd[0];
  const T* vals = static_cast<const T*>(a.vals[0]);
  const T* B = static_cast<const T*>(a.vals[1]);
  T* C = static_cast<T*>(a.out);
  const int64_t M = a.dims[0][0], N = a.dims[1][1];
  const int64_t nnz = a.level_sizes[1];
  if (M == 0 || N == 0) return SPX_OK;
  if (kid == SPX_K_SPMM_NNZ) {
    const int64_t TB = a.params[0], W = a.params[1];
    if (TB < 1 || W < 1 || TB % W != 0 || TB / W > kMaxWarps)
      return fail(SPX_E_UNSUPPORTED,
                  "SpMM nnz-split needs NNZ_PER_TB a multiple of NNZ_PER_WARP with <= 16 warps (got %lld, %lld)",
                  (long long)TB, (long long)W);
    const int nw = (int)(TB / W);
    const int64_t ncta = nnz == 0 ? 1 : ceil_div(nnz, TB);
    if (ncta > INT32_MAX) return fail(SPX_E_ARG, "grid too large");
    const NnzWorkspace L = spmm_workspace(ncta, TB / W, g, sizeof(T));
    if (a.ws_bytes < L.total || !a.ws)
      return fail(SPX_E_WORKSPACE, "workspace %zu < %zu bytes", a.ws_bytes, L.total);
    T* carry_val = reinterpret_cast<T*>(static_cast<char*>(a.ws) + L.carry_val);
    int32_t* carry_row = reinterpret_cast<int32_t*>(static_cast<char*>(a.ws) + L.carry_row);
    int32_t* first = reinterpret_cast<int32_t*>(static_cast<char*>(a.ws) + L.first);
    if (nnz > 0)
      if (int e = launch_chunk_segments(pos, M, W, ncta * (TB / W), first, a.stream)) return e;
    const size_t head_smem = ((size_t)nw * (g.pw * sizeof(T) + sizeof(int32_t)) + 15) & ~size_t(15);
    const size_t reg_ring = (size_t)nw * LeafRing<T, 4>::kBytes;  // staged-register path
    dim3 grid((unsigned)ncta, (unsigned)g.npanels);
    // params[5]: B-row transport (0 = default SPX_SPMM_RING or the staged-register path, >0 = cp.async ring depth, <0 = staged-register path)
    const int ring = a.params[5] != 0 ? (a.params[5] < 0 ? 0 : a.params[5]) : ring_depth();
    if constexpr (CONTIG && (VPL * sizeof(T)) % 16 == 0) {
      if (ring > 0) {
        auto launch = [&](auto kern, int depth) -> int {
          const size_t smem = head_smem + (size_t)nw * depth * g.pw * sizeof(T);
          if (int e = check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                                 "cudaFuncSetAttribute"))
            return e;
          kern<<<grid, nw * 32, smem, a.stream>>>(pos, crd, vals, B, C, M, N, nnz, TB, W, carry_row, carry_val, first);
          return SPX_OK;
        };
        int e = ring >= 16 ? launch(spmm_nnz_kernel<T, VPL, CONTIG, U, 16>, 16)
                           : launch(spmm_nnz_kernel<T, VPL, CONTIG, U, 8>, 8);
        if (e) return e;
      } else {
          spmm_nnz_kernel<T, VPL, CONTIG, U, 0><<<grid, nw * 32, head_smem + reg_ring, a.stream>>>(
            pos, crd, vals, B, C, M, N, nnz, TB, W, carry_row, carry_val, first);
      }
    } else {
      spmm_nnz_kernel<T, VPL, CONTIG, U, 0><<<grid, nw * 32, head_smem + reg_ring, a.stream>>>(
          pos, crd, vals, B, C, M, N, nnz, TB, W, carry_row, carry_val, first);
    }
    count_launch();
    if (int e = check_cuda(cudaGetLastError(), "spmm_nnz_kernel")) return e;
    const int fw = 8;
    dim3 fgrid((unsigned)ceil_div(ncta, fw), (unsigned)g.npanels);
    carry_fixup_kernel<T, VPL, CONTIG><<<fgrid, fw * 32, 0, a.stream>>>(carry_row, carry_val, C, N, ncta);
    count_launch();
    return check_cuda(cudaGetLastError(), "carry_fixup_kernel");
  }
  // warp-per-row
  const int64_t R = a.params[0] > 0 ? a.params[0] : 8;
  int64_t nw = a.params[1] > 0 ? a.params[1] : (R < 8 ? R : 8);
  if (nw > kMaxWarps) nw = kMaxWarps;
  dim3 grid((unsigned)ceil_div(M, R), (unsigned)g.npanels);
#ifndef SPX_SPMM_ROW_UR
#define SPX_SPMM_ROW_UR 16
#endif
  // B rows in flight per warp: the register budget holds SPX_SPMM_ROW_UR
  // 4-float (16 B per lane) rows; the heaviest row (one warp, by the schedule) is
  // latency-bound, so deeper is better while nothing spills
  constexpr int UR_MAX = SPX_SPMM_ROW_UR * 16 / (VPL * (int)sizeof(T));  // 32-bit registers per row: VPL*sizeof/4
  constexpr int UR = UR_MAX < 1 ? 1 : (UR_MAX > 16 ? 16 : UR_MAX);
  // params[4] = 1 (CPU-tagged row schedule): rows longer than the cut go to
  // spmm_heavy_row_kernel, one CTA each (workspace: count + row list)
  const int64_t cut = a.params[4] ? spmm_row_cut(nnz) : 0;
  int32_t* heavy_count = nullptr;
  int32_t* heavy_list = nullptr;
  if (cut > 0) {
    const size_t need = ws_spmm_row(nnz);
    if (!a.ws || a.ws_bytes < need) return fail(SPX_E_WORKSPACE, "workspace %zu < %zu bytes", a.ws_bytes, need);
    heavy_count = static_cast<int32_t*>(a.ws);
    heavy_list = heavy_count + 4;
    if (int e = check_cuda(cudaMemsetAsync(heavy_count, 0, sizeof(int32_t), a.stream), "memset")) return e;
  }
  constexpr int URC = UR / SPX_SPMM_CUT_UDIV > 0 ? UR / SPX_SPMM_CUT_UDIV : 1;
  auto rk = cut > 0 ? spmm_row_kernel<T, VPL, CONTIG, URC, true> : spmm_row_kernel<T, VPL, CONTIG, UR, false>;
  rk<<<grid, (unsigned)(nw * 32), (size_t)nw * LeafRing<T, 4>::kBytes, a.stream>>>(pos, crd, vals, B, C, M, N, R, cut,
                                                                                   heavy_list, heavy_count);
  count_launch();
  if (int e = check_cuda(cudaGetLastError(), "spmm_row_kernel")) return e;
  if (cut > 0) {
    const int hw = kHeavyWarps;
    const size_t hsm = (size_t)hw * LeafRing<T, 4>::kBytes + (size_t)hw * 32 * VPL * sizeof(T);
    auto hk = spmm_heavy_row_kernel<T, VPL, CONTIG, (UR / SPX_SPMM_HEAVY_UDIV > 0 ? UR / SPX_SPMM_HEAVY_UDIV : 1)>;
    static thread_local size_t hset = 0;
    if (hsm > 48 * 1024 && hsm > hset) {
      if (int e = check_cuda(cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm),
                             "cudaFuncSetAttribute"))
        return e;
      hset = hsm;
    }
    dim3 hgrid((unsigned)std::max<int64_t>(1, nnz / (cut + 1)), (unsigned)g.npanels);
    hk<<<hgrid, (unsigned)(hw * 32), hsm, a.stream>>>(pos, crd, vals, B, C, N, heavy_list, heavy_count);
    count_launch();
    if (int e = check_cuda(cudaGetLastError(), "spmm_heavy_row_kernel")) return e;
  }
  return SPX_OK;
}

template <typename T>
int dispatch_spmm(int kid, const Args& a, const SpmmGeom& g) {
  switch (g.vpl * 2 + (g.contig ? 1 : 0)) {
    case 2: return run_spmm<T, 1, false>(kid, a, g);
    case 3: return run_spmm<T, 1, true>(kid, a, g);
    case 4: return run_spmm<T, 2, false>(kid, a, g);
    case 5: return run_spmm<T, 2, true>(kid, a, g);
    case 8: return run_spmm<T, 4, false>(kid, a, g);
    case 9: return run_spmm<T, 4, true>(kid, a, g);
    default: break;
  }
  if constexpr (sizeof(T) == 4) {
    if (g.vpl == 8) return g.contig ? run_spmm<T, 8, true>(kid, a, g) : run_spmm<T, 8, false>(kid, a, g);
  }
  return fail(SPX_E_UNSUPPORTED, "no SpMM instantiation for %d values per lane", g.vpl);
}

}  // namespace

size_t ws_spmm(int kid, const Args& a) {
  if (kid == SPX_K_SPMM_ROW) return a.params[4] ? ws_spmm_row(a.level_sizes[1]) : 0;
  if (kid != SPX_K_SPMM_NNZ) return 0;
  const int64_t N = a.dims[1][1];
  const SpmmGeom g = spmm_geom(a.dtype, N);
  const int64_t nnz = a.level_sizes[1];
  const int64_t TB = a.params[0] > 0 ? a.params[0] : 1;
  const int64_t W = a.params[1] > 0 ? a.params[1] : TB;
  const int64_t ncta = nnz == 0 ? 1 : ceil_div(nnz, TB);
  const size_t es = a.dtype == SPX_F32 ? 4 : 8;
  return spmm_workspace(ncta, TB / W > 0 ? TB / W : 1, g, es).total;
}

int launch_spmm(int kid, const Args& a) {
  const int64_t M = a.dims[0][0], K = a.dims[0][1];
  if (a.dims[1][0] != K) return fail(SPX_E_ARG, "SpMM: A is %lld x %lld but B has %lld rows", (long long)M,
                                     (long long)K, (long long)a.dims[1][0]);
  const int64_t N = a.dims[1][1];
  if (int e = check_bound(a, N)) return e;
  const SpmmGeom g = spmm_geom(a.dtype, N);
  return a.dtype == SPX_F32 ? dispatch_spmm<float>(kid, a, g) : dispatch_spmm<double>(kid, a, g);
}

}  // namespace spx
