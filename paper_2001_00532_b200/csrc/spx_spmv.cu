// SpMV kernels: y(i) = A(i,j) * x(j), A in CSR ("ds"), x and y dense.
//
//  K1 SPX_K_SPMV_ROW  -- thread per row: A.7 `split(i,block,thread,ROWS_PER_TB)`
//     (PAPER.md:2004-2016), also the A.1 CPU shape `split(i,i0,i1,CHUNK)`
//      and the unscheduled statement.
//  K2 SPX_K_SPMV_WARP -- warp per row, A.8:
//     split(i,block,block_row,ROWS_PER_TB) split(block_row,warp_row,warp,W)
//     pos(j,jpos,A) split(jpos,thread_nz,thread,32), thread:Temporary -> the
//     lanes stride the row's positions and fold with a shuffle tree.
//  K3 SPX_K_SPMV_NNZ  -- position-split, A.2/A.9 (PAPER.md:1902-1925,
//     2039-2057): fuse(i,j,f) pos(f,fpos,A) split(fpos,block,..,NNZ_PER_TB)
//     split(..,warp,..,NNZ_PER_WARP) split(..,thread,thread_nz,NNZ_PER_THREAD).
//     Thread t of a CTA owns NNZ_PER_THREAD consecutive positions
//     (`thread_nz` innermost, exactly the schedule), loads them with 16 B
//     vector loads, tracks the row through a shared-memory copy of the CTA's
//     slice of pos (Track recovery), stores rows it owns and
//     parks its head partial (the `Atomics` output race) in shared memory;
//     runs of equal head rows are folded after the barrier and CTA-spanning
//     rows go through the deterministic carry fix-up (see spx_spmm.cu).
#include "spx_common.cuh"

namespace spx {
namespace {

constexpr int kPosCache = 4096;  // ints of pos staged per CTA

// Row kernels are bound by their heaviest row (one thread / one warp by the
// schedule), which is a latency chain: the loads in flight per step are
// tuning knobs (SPX_SPMV_ROW_STEP positions per thread, SPX_SPMV_WARP_STEPS
// 32-position steps per warp) traded against occupancy (..._MINB).
#ifndef SPX_SPMV_ROW_STEP
#define SPX_SPMV_ROW_STEP 32  // cfg5 A7 15.1 -> 9.2 ms (one CTA/SM)
#endif
#ifndef SPX_SPMV_ROW_MINB
#define SPX_SPMV_ROW_MINB 1
#endif
#ifndef SPX_SPMV_WARP_STEPS
#define SPX_SPMV_WARP_STEPS 8  // cfg5 A8 2.29 -> 1.70 ms; 16 steps at 1 CTA/SM: 2.47
#endif
#ifndef SPX_SPMV_ROW_PF
#define SPX_SPMV_ROW_PF 4  // L2 prefetch distance (steps) of the thread-per-row streams (cfg5 A.7 9.13 -> 8.02 ms; 16: 8.10)
#endif
#ifndef SPX_SPMV_WARP_MINB
#define SPX_SPMV_WARP_MINB 2
#endif

template <typename T>
__global__ void __launch_bounds__(kMaxThreads, SPX_SPMV_ROW_MINB) spmv_row_kernel(const int32_t* __restrict__ pos,
                                                        const int32_t* __restrict__ crd,
                                                        const T* __restrict__ vals, const T* __restrict__ x,
                                                        T* __restrict__ y, int64_t M, int64_t R) {
  const int64_t lo = (int64_t)blockIdx.x * R;
  for (int64_t t = threadIdx.x; t < R; t += blockDim.x) {
    const int64_t i = lo + t;
    if (i >= M) return;
    const int a = __ldg(pos + i), e = __ldg(pos + i + 1);
    // STEP positions' loads in flight per step (a long row is one thread's
    // serial dependency chain otherwise); sequential fold order kept
    constexpr int STEP = SPX_SPMV_ROW_STEP;
    T acc = T(0);
    int p = a;
    for (; p + STEP <= e; p += STEP) {
      int c[STEP];
      T v[STEP], xv[STEP];
#if SPX_SPMV_ROW_PF
      // a thread alone on a long row is a serial latency chain: pull the
      // (crd, vals) lines SPX_SPMV_ROW_PF steps ahead into L2
      if (p + (SPX_SPMV_ROW_PF + 1) * STEP <= e) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(crd + p + SPX_SPMV_ROW_PF * STEP));
#pragma unroll
        for (int l = 0; l < STEP * (int)sizeof(T); l += 128)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(vals + p + SPX_SPMV_ROW_PF * STEP) + l));
      }
#endif
#pragma unroll
      for (int k = 0; k < STEP; ++k) {
        c[k] = __ldcs(crd + p + k);
        v[k] = __ldcs(vals + p + k);
      }
#pragma unroll
      for (int k = 0; k < STEP; ++k) xv[k] = __ldg(x + c[k]);
#pragma unroll
      for (int k = 0; k < STEP; ++k) acc += v[k] * xv[k];
    }
    for (; p < e; ++p) acc += __ldcs(vals + p) * __ldg(x + __ldcs(crd + p));
    __stcs(y + i, acc);
  }
}

template <typename T>
__global__ void __launch_bounds__(kMaxThreads, SPX_SPMV_WARP_MINB) spmv_warp_kernel(const int32_t* __restrict__ pos,
                                                         const int32_t* __restrict__ crd,
                                                         const T* __restrict__ vals, const T* __restrict__ x,
                                                         T* __restrict__ y, int64_t M, int64_t R) {
  const int nw = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t lo = (int64_t)blockIdx.x * R;
  const int64_t nwr = (R + nw - 1) / nw;
  for (int64_t wr = 0; wr < nwr; ++wr) {
    const int64_t br = wr * nw + warp;
    if (br >= R) break;
    const int64_t i = lo + br;
    if (i >= M) break;
    const int a = __ldg(pos + i), e = __ldg(pos + i + 1);
    // lanes stride the row (thread_nz x thread); S 32-position steps'
    // loads are in flight at once, then the Temporary fold
    constexpr int S = SPX_SPMV_WARP_STEPS;
    T acc = T(0);
    int p = a + lane;
    for (; p + 32 * (S - 1) < e; p += 32 * S) {
      int c[S];
      T v[S], xv[S];
#pragma unroll
      for (int k = 0; k < S; ++k) {
        c[k] = __ldcs(crd + p + 32 * k);
        v[k] = __ldcs(vals + p + 32 * k);
      }
#pragma unroll
      for (int k = 0; k < S; ++k) xv[k] = __ldg(x + c[k]);
#pragma unroll
      for (int k = 0; k < S; ++k) acc += v[k] * xv[k];
    }
    for (; p < e; p += 32) acc += __ldcs(vals + p) * __ldg(x + __ldcs(crd + p));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
    if (lane == 0) __stcs(y + i, acc);
  }
}

// 256-bit streaming loads (LDG.E.256, sm_100): one lane reads one whole
// 32 B sector per instruction.  With 16 B vectors at a 32 B (crd) or 64 B
// (fp64 vals) lane stride every sector is requested from L2 twice -- once per
// half -- which the cfg5 ncu capture showed as ~1.5x the compulsory L2->SM
// sectors.  L1::no_allocate keeps the streams out of L1, which then holds
// only x.  Same-box A/B on cfg5: 1.27 ms (16 B) -> 1.19 (256-bit, L1
// allocating) -> 1.15 ms (256-bit, no_allocate).
#define SPX_LD256 "ld.global.nc.L1::no_allocate"
__device__ __forceinline__ void ld256_stream(const int32_t* p, int32_t* r) {
  asm volatile(SPX_LD256 ".v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "l"(p));
}
__device__ __forceinline__ void ld256_stream(const float* p, float* r) {
  asm volatile(SPX_LD256 ".v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
               : "l"(p));
}
__device__ __forceinline__ void ld256_stream(const double* p, double* r) {
  asm volatile(SPX_LD256 ".v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3])
               : "l"(p));
}

// One thread's NNZ_PER_THREAD consecutive (crd, vals): whole-sector 256-bit
// loads where the per-thread bytes are a multiple of 32 (16 B vectors where
// only of 16), when the chunk is full and the addresses are aligned (always,
// for cudaMalloc'd arrays and NNZ_PER_WARP-aligned chunks); else scalar.
template <typename T, int TPT>
__device__ __forceinline__ void load_thread_chunk(const int32_t* __restrict__ crd, const T* __restrict__ vals,
                                                  int a, int n, int32_t* cc, T* vv) {
  constexpr int kC = TPT * 4, kV = TPT * (int)sizeof(T);  // bytes per thread
  constexpr bool c256 = kC % 32 == 0, v256 = kV % 32 == 0;
  constexpr uintptr_t kAlign = (c256 || v256) ? 31 : 15;
  const bool vec = kC % 16 == 0 && kV % 16 == 0 && n == TPT &&
                   (((reinterpret_cast<uintptr_t>(crd + a) | reinterpret_cast<uintptr_t>(vals + a)) & kAlign) == 0);
  if (vec) {
    if constexpr (c256) {
#pragma unroll
      for (int k = 0; k < TPT / 8; ++k) ld256_stream(crd + a + 8 * k, cc + 8 * k);
    } else {
#pragma unroll
      for (int k = 0; k < TPT / 4; ++k) {
        const int4 q = __ldcs(reinterpret_cast<const int4*>(crd + a) + k);
        cc[4 * k] = q.x;
        cc[4 * k + 1] = q.y;
        cc[4 * k + 2] = q.z;
        cc[4 * k + 3] = q.w;
      }
    }
    if constexpr (v256) {
      constexpr int kPer = 32 / (int)sizeof(T);
#pragma unroll
      for (int k = 0; k < TPT / kPer; ++k) ld256_stream(vals + a + kPer * k, vv + kPer * k);
    } else {
      constexpr int kPer = 16 / (int)sizeof(T);
#pragma unroll
      for (int k = 0; k < TPT / kPer; ++k) {
        const float4 q = __ldcs(reinterpret_cast<const float4*>(vals + a) + k);
        unpack16(&vv[kPer * k], q);
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < TPT; ++k) {
      cc[k] = k < n ? __ldcs(crd + a + k) : 0;
      vv[k] = k < n ? __ldcs(vals + a + k) : T(0);
    }
  }
}

// TPT > 0: compile-time NNZ_PER_THREAD; TPT == 0: runtime `tpt`.
template <typename T, int TPT>
__global__ void __launch_bounds__(kMaxThreads, 2) spmv_nnz_kernel(const int32_t* __restrict__ pos,
                                                        const int32_t* __restrict__ crd,
                                                        const T* __restrict__ vals, const T* __restrict__ x,
                                                        T* __restrict__ y, int64_t M, int64_t nnz, int64_t TB,
                                                        int tpt_rt, int32_t* __restrict__ carry_row,
                                                        T* __restrict__ carry_val,
                                                        const int32_t* __restrict__ first) {
  __shared__ int32_t s_pos[kPosCache];
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* s_hval = reinterpret_cast<T*>(smem_raw);
  int32_t* s_hrow = reinterpret_cast<int32_t*>(s_hval + blockDim.x);

  // positions are int32 (pos/crd are int32, tensors.py:248-249)
  const int tpt = TPT > 0 ? TPT : tpt_rt;
  const int tid = threadIdx.x;
  const int cta = blockIdx.x;
  const int p0 = (int)((int64_t)cta * TB);
  const int p1 = (int)min((int64_t)p0 + TB, nnz);
  const int a = min(p0 + tid * tpt, p1);
  const int e = min(a + tpt, p1);
  const int n = e - a;

  if (p0 >= p1) {
    if (nnz == 0 && cta == 0)
      for (int64_t q = tid; q < M; q += blockDim.x) __stcs(y + q, T(0));
    if (tid == 0) carry_row[cta] = -1;
    return;
  }
  // Issue this thread's (crd, vals) loads and x gathers first so their
  // latency overlaps the staging of pos below.
  int32_t cc[TPT > 0 ? TPT : 1];
  T vv[TPT > 0 ? TPT : 1];
  T xv[TPT > 0 ? TPT : 1];
  if constexpr (TPT > 0) {
    load_thread_chunk<T, TPT>(crd, vals, a, n, cc, vv);
#pragma unroll
    for (int k = 0; k < TPT; ++k) xv[k] = __ldg(x + cc[k]);  // cc = 0 past n: harmless
  }
  // rows of this chunk: [first[cta], first[cta+1]] (chunk_segments_kernel)
  const int rlo = __ldg(first + cta), rhi = __ldg(first + cta + 1);
  const int nstage = rhi - rlo + 2;  // pos[rlo .. rhi+1]
  const bool staged = nstage <= kPosCache;
  if (staged)
    for (int k = tid; k < nstage; k += blockDim.x) s_pos[k] = __ldg(pos + rlo + k);
  __syncthreads();
#define SPX_P(r) (staged ? s_pos[(r) - rlo] : __ldg(pos + (r)))

  int32_t head = -1;
  T hval = T(0);
  if (n > 0) {
    // SearchSegment over the CTA's rows (ir.py:178-190)
    int lo = rlo, hi = rhi + 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (SPX_P(mid) <= a) lo = mid + 1;
      else hi = mid;
    }
    int r = lo - 1;
    bool is_head = SPX_P(r) < a;
    if (!is_head && r > 0) {
      // empty rows with pos == a before r are owned by this thread
      int rr = r - 1;
      while (rr >= rlo && SPX_P(rr) == a) __stcs(y + rr--, T(0));
      if (rr < rlo && rr >= 0 && __ldg(pos + rr) == a) {
        const int lb = (int)lower_bound(pos, 0, rlo, a);
        for (int q = lb; q < rlo; ++q) __stcs(y + q, T(0));
      }
    }
    int rend = SPX_P(r + 1);
    T acc = T(0);
    if constexpr (TPT > 0) {
      if (n == TPT && a + TPT <= rend) {
        // whole chunk inside one row: plain fold, no tracking
#pragma unroll
        for (int k = 0; k < TPT; ++k) acc += vv[k] * xv[k];
      } else {
#pragma unroll
        for (int k = 0; k < TPT; ++k) {
          if (k < n) {
            while (a + k >= rend) {
              if (is_head) {
                head = r;
                hval = acc;
                is_head = false;
              } else {
                __stcs(y + r, acc);
              }
              acc = T(0);
              ++r;
              rend = SPX_P(r + 1);
            }
            acc += vv[k] * xv[k];
          }
        }
      }
    } else {
      for (int p = a; p < e; ++p) {
        const T prod = __ldcs(vals + p) * __ldg(x + __ldcs(crd + p));
        while (p >= rend) {
          if (is_head) {
            head = r;
            hval = acc;
            is_head = false;
          } else {
            __stcs(y + r, acc);
          }
          acc = T(0);
          ++r;
          rend = SPX_P(r + 1);
        }
        acc += prod;
      }
    }
    if (is_head) {
      head = r;
      hval = acc;
    } else {
      __stcs(y + r, acc);
    }
    if (e == nnz)
      for (int64_t q = (int64_t)r + 1; q < M; ++q) __stcs(y + q, T(0));
  }
  // Fold the head partials: threads with equal head rows are contiguous in
  // tid order.  Segmented shuffle reduction inside each warp (the first lane
  // of a run ends with the run's warp-local sum), then runs that cross warps
  // are joined through one partial per warp.
  const int lane = tid & 31, warp = tid >> 5;
  T hv = hval;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_down_sync(kFull, hv, o);
    const int h2 = __shfl_down_sync(kFull, head, o);
    if (lane + o < 32 && h2 == head) hv += y;
  }
  const int hprev = __shfl_up_sync(kFull, head, 1);
  s_hrow[tid] = head;
  if (lane == 0) s_hval[warp] = hv;  // the lane-0 run's warp-local sum
  __syncthreads();
  if (head >= 0 && (lane == 0 || hprev != head) && (tid == 0 || s_hrow[tid - 1] != head)) {
    T s = hv;
    const int nw = blockDim.x >> 5;
    for (int w2 = warp + 1; w2 < nw && s_hrow[w2 * 32] == head; ++w2) s += s_hval[w2];
    if (SPX_P(head) >= p0) {
      y[head] = __ldcg(y + head) + s;
    } else {
      carry_val[cta] = s;
      carry_row[cta] = head;
    }
  }
  if (tid == 0 && !(head >= 0 && SPX_P(head) < p0)) carry_row[cta] = -1;
#undef SPX_P
}

// Atomics variant of K3 (the default): the schedule tags `thread` with the
// Atomics race strategy, and that is what this kernel does -- y is zeroed
// first, a row that lies inside one thread's positions is stored plainly,
// every other partial is added with red.global.add after a segmented
// shuffle fold inside the warp (one atomic per row run per warp).  Warps are
// independent: each stages the pos entries of its own rows in warp-private
// shared memory (chunk table at NNZ_PER_WARP granularity), so there is no
// CTA barrier and no carry fix-up.  fp64 sums of a row split across warps
// may differ in the last bits from run to run (atomic order).
constexpr int kWarpPos = 320;  // pos entries staged per warp
#ifndef SPX_SPMV_CARVEOUT
#define SPX_SPMV_CARVEOUT 20  // percent of 228 KB: 4 CTAs x 8 warps x 1.25 KB of pos slices fit the 64 KB config
#endif

// tuning knob: 3 CTAs/SM forces 40 registers and spills (cfg5 1.32 vs 1.15 ms)
#ifndef SPX_SPMV_MINB
#define SPX_SPMV_MINB 2
#endif
// XS: x is short enough to sit in shared memory (the TTV vector c): it is
// staged once per CTA and the per-position gathers become shared-memory
// reads -- random 4/8 B gathers through L1 cost one L1TEX wavefront each,
// even when they hit.
template <typename T, int TPT, bool XS = false>
__global__ void __launch_bounds__(kMaxThreads, SPX_SPMV_MINB) spmv_nnz_atomic_kernel(
    const int32_t* __restrict__ pos, const int32_t* __restrict__ crd, const T* __restrict__ vals,
    const T* __restrict__ x, T* __restrict__ y, int64_t M, int64_t nnz, int64_t W, int tpt_rt,
    const int32_t* __restrict__ first, int64_t xlen = 0) {
  // dynamic shared memory: [x (XS only)] [pos slices, kWarpPos per warp of this CTA] -- sized by
  // the CTA's actual warps, so the carveout leaves the rest of the SM's 256 KB to L1 (x gathers)
  extern __shared__ __align__(16) unsigned char smem_x[];
  int32_t* s_pos_all = reinterpret_cast<int32_t*>(smem_x + (XS ? ((size_t)xlen * sizeof(T) + 15) / 16 * 16 : 0));
  const T* __restrict__ xr = x;
  if constexpr (XS) {
    T* sx = reinterpret_cast<T*>(smem_x);
    for (int64_t i = threadIdx.x; i < xlen; i += blockDim.x) sx[i] = __ldg(x + i);
    __syncthreads();
    xr = sx;
  }
  const int tpt = TPT > 0 ? TPT : tpt_rt;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t* s_pos = s_pos_all + warp * kWarpPos;
  const int q = (int)blockIdx.x * (int)(blockDim.x >> 5) + warp;  // warp chunk
  const int q0 = (int)((int64_t)q * W);
  if ((int64_t)q0 >= nnz) return;
  const int q1 = (int)min((int64_t)q0 + W, nnz);
  const int a = min(q0 + lane * tpt, q1);
  const int e = min(a + tpt, q1);
  const int n = e - a;
  // loads first: (crd, vals) with 256-bit vectors, then the x gathers
  int32_t cc[TPT > 0 ? TPT : 1];
  T vv[TPT > 0 ? TPT : 1];
  T xv[TPT > 0 ? TPT : 1];
  if constexpr (TPT > 0) {
    load_thread_chunk<T, TPT>(crd, vals, a, n, cc, vv);
#pragma unroll
    for (int k = 0; k < TPT; ++k) xv[k] = XS ? xr[cc[k]] : __ldg(x + cc[k]);  // cc = 0 past n: harmless
  }
  const int rlo = __ldg(first + q), rhi = __ldg(first + q + 1);
  const int nstage = rhi - rlo + 2;  // pos[rlo .. rhi+1]
  const bool staged = nstage <= kWarpPos;
  if (staged)
    for (int k = lane; k < nstage; k += 32) s_pos[k] = __ldg(pos + rlo + k);
  __syncwarp();
#define SPX_P(r) (staged ? s_pos[(r) - rlo] : __ldg(pos + (r)))
  int32_t head = -1;
  T hval = T(0);
  if (n > 0) {
    int lo = rlo, hi = rhi + 1;  // SearchSegment (ir.py:178-190)
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (SPX_P(mid) <= a) lo = mid + 1;
      else hi = mid;
    }
    int r = lo - 1;
    bool is_head = SPX_P(r) < a;
    int rend = SPX_P(r + 1);
    T acc = T(0);
    // a finished row partial: plain store when the row lies inside this
    // thread's positions, else it joins the head fold / an atomic add
    auto close_row = [&]() {
      if (is_head) {
        head = r;
        hval = acc;
        is_head = false;
      } else {
        __stcs(y + r, acc);
      }
    };
    if constexpr (TPT > 0) {
      if (n == TPT && a + TPT <= rend) {
#pragma unroll
        for (int k = 0; k < TPT; ++k) acc += vv[k] * xv[k];
      } else {
#pragma unroll
        for (int k = 0; k < TPT; ++k) {
          if (k < n) {
            while (a + k >= rend) {
              close_row();
              acc = T(0);
              ++r;
              rend = SPX_P(r + 1);
            }
            acc += vv[k] * xv[k];
          }
        }
      }
    } else {
      for (int p = a; p < e; ++p) {
        const int cp = __ldcs(crd + p);
        const T prod = __ldcs(vals + p) * (XS ? xr[cp] : __ldg(x + cp));
        while (p >= rend) {
          close_row();
          acc = T(0);
          ++r;
          rend = SPX_P(r + 1);
        }
        acc += prod;
      }
    }
    // last row of the range: complete here, or shared with later threads
    if (is_head) {
      head = r;
      hval = acc;
    } else if (rend <= e) {
      __stcs(y + r, acc);
    } else {
      atomicAdd(y + r, acc);
    }
  }
  // segmented fold of the head partials (equal heads are contiguous lanes)
  T hv = hval;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T yv = __shfl_down_sync(kFull, hv, o);
    const int h2 = __shfl_down_sync(kFull, head, o);
    if (lane + o < 32 && h2 == head) hv += yv;
  }
  const int hprev = __shfl_up_sync(kFull, head, 1);
  if (head >= 0 && (lane == 0 || hprev != head)) atomicAdd(y + head, hv);
#undef SPX_P
}

template <typename T>
__global__ void spmv_fixup_kernel(const int32_t* __restrict__ carry_row, const T* __restrict__ carry_val,
                                  T* __restrict__ y, int64_t n) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int32_t row = carry_row[c];
  if (row < 0 || (c > 0 && carry_row[c - 1] == row)) return;
  T s = T(0);
  for (int64_t c2 = c; c2 < n && carry_row[c2] == row; ++c2) s += carry_val[c2];
  y[row] = __ldcg(y + row) + s;
}

// The Atomics nnz-split kernel over any segment structure: y[r] =
// sum_{p in [pos[r], pos[r+1])} vals[p] * x[crd[p]] for r < nseg, with y
// zeroed by the caller and `first` the chunk table at W granularity.  SpMV
// (rows) and the nnz-split TTV (fibers of a CSF tensor) share it.
template <typename T>
int segsum_atomic(const int32_t* pos, const int32_t* crd, const T* vals, const T* x, T* y, int64_t nseg,
                  int64_t nnz, int64_t TB, int64_t W, int64_t TPT, const int32_t* first, cudaStream_t st,
                  int64_t xlen = 0) {
  const int threads = (int)(TB / TPT);
  const unsigned g = (unsigned)(nnz == 0 ? 1 : ceil_div(nnz, TB));
  const size_t pbytes = (size_t)((threads + 31) / 32) * kWarpPos * sizeof(int32_t);
  // x in shared memory when it is short (<= 16 KB) and no larger than the
  // (crd, vals) bytes a CTA streams (every CTA stages all of x)
  const size_t xbytes = (size_t)xlen * sizeof(T);
  if (TPT == 8 && xlen > 0 && xbytes <= 16384 && (size_t)TB * (4 + sizeof(T)) >= xbytes) {
    const size_t sm = (xbytes + 15) / 16 * 16 + pbytes;
    spmv_nnz_atomic_kernel<T, 8, true><<<g, threads, sm, st>>>(pos, crd, vals, x, y, nseg, nnz, W, 8, first, xlen);
    count_launch();
    return check_cuda(cudaGetLastError(), "spmv_nnz_atomic_kernel");
  }
  static bool carve = [] {  // shared memory for the resident CTAs' pos slices; the rest is L1
    for (auto k : {spmv_nnz_atomic_kernel<T, 4>, spmv_nnz_atomic_kernel<T, 8>, spmv_nnz_atomic_kernel<T, 16>,
                   spmv_nnz_atomic_kernel<T, 0>})
      cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, SPX_SPMV_CARVEOUT);
    return true;
  }();
  (void)carve;
  switch (TPT) {
    case 4: spmv_nnz_atomic_kernel<T, 4><<<g, threads, pbytes, st>>>(pos, crd, vals, x, y, nseg, nnz, W, 4, first); break;
    case 8: spmv_nnz_atomic_kernel<T, 8><<<g, threads, pbytes, st>>>(pos, crd, vals, x, y, nseg, nnz, W, 8, first); break;
    case 16:
      spmv_nnz_atomic_kernel<T, 16><<<g, threads, pbytes, st>>>(pos, crd, vals, x, y, nseg, nnz, W, 16, first);
      break;
    default:
      spmv_nnz_atomic_kernel<T, 0><<<g, threads, pbytes, st>>>(pos, crd, vals, x, y, nseg, nnz, W, (int)TPT, first);
  }
  count_launch();
  return check_cuda(cudaGetLastError(), "spmv_nnz_atomic_kernel");
}

template <typename T>
int run_spmv(int kid, const Args& a) {
  const int32_t* pos = a.pos[0];
  const int32_t* crd = a.crd[0];
  const T* vals = static_cast<const T*>(a.vals[0]);
  const T* x = static_cast<const T*>(a.vals[1]);
  T* y = static_cast<T*>(a.out);
  const int64_t M = a.dims[0][0];
  const int64_t nnz = a.level_sizes[1];
  if (M == 0) return SPX_OK;
  if (kid == SPX_K_SPMV_ROW) {
    const int64_t R = a.params[0] > 0 ? a.params[0] : 256;
    const int threads = (int)(R < 256 ? (R < 32 ? 32 : R) : 256);
    spmv_row_kernel<T><<<(unsigned)ceil_div(M, R), threads, 0, a.stream>>>(pos, crd, vals, x, y, M, R);
    count_launch();
    return check_cuda(cudaGetLastError(), "spmv_row_kernel");
  }
  if (kid == SPX_K_SPMV_WARP) {
    const int64_t R = a.params[0] > 0 ? a.params[0] : 8;
    int64_t nw = a.params[1] > 0 ? a.params[1] : (R < 8 ? R : 8);
    if (nw > kMaxWarps) nw = kMaxWarps;
    spmv_warp_kernel<T><<<(unsigned)ceil_div(M, R), (unsigned)(nw * 32), 0, a.stream>>>(pos, crd, vals, x, y, M, R);
    count_launch();
    return check_cuda(cudaGetLastError(), "spmv_warp_kernel");
  }
  // nnz-split
  const int64_t TB = a.params[0], W = a.params[1], TPT = a.params[2];
  if (TB < 1 || W < 1 || TPT < 1 || W != 32 * TPT || TB % W != 0 || TB / TPT > kMaxThreads)
    return fail(SPX_E_UNSUPPORTED,
                "SpMV nnz-split needs NNZ_PER_WARP == 32*NNZ_PER_THREAD and NNZ_PER_TB a multiple of "
                "NNZ_PER_WARP with <= 512 threads (got %lld, %lld, %lld)",
                (long long)TB, (long long)W, (long long)TPT);
  const int threads = (int)(TB / TPT);
  const int64_t ncta = nnz == 0 ? 1 : ceil_div(nnz, TB);
  if (a.params[5] == 0) {
    // default: the schedule's Atomics strategy (zeroed y, red.add of partials)
    if (int e = check_cuda(cudaMemsetAsync(y, 0, (size_t)M * sizeof(T), a.stream), "memset")) return e;
    if (nnz == 0) return SPX_OK;
    const int64_t nslots = ncta * (TB / W);
    const size_t need = (size_t)(nslots + 1) * sizeof(int32_t);
    if (!a.ws || a.ws_bytes < need) return fail(SPX_E_WORKSPACE, "workspace %zu < %zu bytes", a.ws_bytes, need);
    int32_t* first = static_cast<int32_t*>(a.ws);
    if (int e = launch_chunk_segments(pos, M, W, nslots, first, a.stream)) return e;
    return segsum_atomic(pos, crd, vals, x, y, M, nnz, TB, W, TPT, first, a.stream, a.dims[1][0]);
  }
  const NnzWorkspace L = nnz_workspace(ncta, sizeof(T));
  if (!a.ws || a.ws_bytes < L.total) return fail(SPX_E_WORKSPACE, "workspace %zu < %zu bytes", a.ws_bytes, L.total);
  T* carry_val = reinterpret_cast<T*>(static_cast<char*>(a.ws) + L.carry_val);
  int32_t* carry_row = reinterpret_cast<int32_t*>(static_cast<char*>(a.ws) + L.carry_row);
  int32_t* first = reinterpret_cast<int32_t*>(static_cast<char*>(a.ws) + L.first);
  if (nnz > 0)
    if (int e = launch_chunk_segments(pos, M, TB, ncta, first, a.stream)) return e;
  const size_t smem = (size_t)threads * (sizeof(T) + sizeof(int32_t));
  const unsigned g = (unsigned)ncta;
  switch (TPT) {
    case 4: spmv_nnz_kernel<T, 4><<<g, threads, smem, a.stream>>>(pos, crd, vals, x, y, M, nnz, TB, 4, carry_row, carry_val, first); break;
    case 8: spmv_nnz_kernel<T, 8><<<g, threads, smem, a.stream>>>(pos, crd, vals, x, y, M, nnz, TB, 8, carry_row, carry_val, first); break;
    case 16: spmv_nnz_kernel<T, 16><<<g, threads, smem, a.stream>>>(pos, crd, vals, x, y, M, nnz, TB, 16, carry_row, carry_val, first); break;
    default:
      spmv_nnz_kernel<T, 0><<<g, threads, smem, a.stream>>>(pos, crd, vals, x, y, M, nnz, TB, (int)TPT, carry_row,
                                                            carry_val, first);
  }
  count_launch();
  if (int e = check_cuda(cudaGetLastError(), "spmv_nnz_kernel")) return e;
  spmv_fixup_kernel<T><<<(unsigned)ceil_div(ncta, 256), 256, 0, a.stream>>>(carry_row, carry_val, y, ncta);
  count_launch();
  return check_cuda(cudaGetLastError(), "spmv_fixup_kernel");
}

}  // namespace

size_t ws_spmv(int kid, const Args& a) {
  if (kid != SPX_K_SPMV_NNZ) return 0;
  const int64_t nnz = a.level_sizes[1];
  const int64_t TB = a.params[0] > 0 ? a.params[0] : 1;
  const int64_t W = a.params[1] > 0 ? a.params[1] : TB;
  const int64_t ncta = nnz == 0 ? 1 : ceil_div(nnz, TB);
  const size_t es = a.dtype == SPX_F32 ? 4 : 8;
  const size_t atomic_ws = (size_t)(ncta * (TB / W > 0 ? TB / W : 1) + 1) * sizeof(int32_t);
  const size_t det_ws = nnz_workspace(ncta, es).total;
  return atomic_ws > det_ws ? atomic_ws : det_ws;
}

int segsum_atomic_f32(const int32_t* pos, const int32_t* crd, const float* vals, const float* x, float* y,
                      int64_t nseg, int64_t nnz, int64_t TB, int64_t W, int64_t TPT, const int32_t* first,
                      cudaStream_t st, int64_t xlen) {
  return segsum_atomic<float>(pos, crd, vals, x, y, nseg, nnz, TB, W, TPT, first, st, xlen);
}
int segsum_atomic_f64(const int32_t* pos, const int32_t* crd, const double* vals, const double* x, double* y,
                      int64_t nseg, int64_t nnz, int64_t TB, int64_t W, int64_t TPT, const int32_t* first,
                      cudaStream_t st, int64_t xlen) {
  return segsum_atomic<double>(pos, crd, vals, x, y, nseg, nnz, TB, W, TPT, first, st, xlen);
}

int launch_spmv(int kid, const Args& a) {
  if (a.dims[1][0] != a.dims[0][1])
    return fail(SPX_E_ARG, "SpMV: A has %lld columns but x has %lld entries", (long long)a.dims[0][1],
                (long long)a.dims[1][0]);
  return a.dtype == SPX_F32 ? run_spmv<float>(kid, a) : run_spmv<double>(kid, a);
}

}  // namespace spx
