// CSF ("sss") kernels: TTV and MTTKRP over a 3rd-order tensor B stored as
// the reference's coordinate hierarchy (pack, tensors.py:212-258):
//   level 0: pos0[2]   crd0[S]   (slices, coordinate i)
//   level 1: pos1[S+1] crd1[F]   (fibers, coordinate of the 2nd mode)
//   level 2: pos2[F+1] crd2[nnz] (leaves, coordinate of the 3rd mode), vals[nnz]
//
//  K7 SPX_K_TTV_FIBER   A(i,j) = B(i,j,k) * c(k):
//     fuse(i,j,f) pos(f,fpos,B) -> fpos walks level-1 positions (fibers);
//     split(fpos,block,..,FIBERS_PER_TB) split(..,warp,..,FIBERS_PER_WARP).
//     A warp takes FIBERS_PER_WARP consecutive fibers and reduces their
//     leaves by key (below).  Every fiber is a distinct (i,j), so the dense
//     output (zeroed first) is written with plain stores.
//  K8 SPX_K_MTTKRP_NNZ  A(i,j) = B(i,k,l) * C(k,j) * D(l,j), Appendix A.6
//     (PAPER.md:1981-2002): reorder(i,k,l,j) fuse(k,l,kl) fuse(i,kl,f)
//     pos(f,fpos,B) split(fpos,block,..,NNZ_PER_TB) split(..,warp,nnz,
//     NNZ_PER_WARP) split(j,dvu,thread,32) bound(dvu,dense_val,ceil(R/32)).
//     A warp walks NNZ_PER_WARP leaves; lanes cover j; the fiber partial
//     sum_l B*D[l,:] is scaled by C[k,:] when the fiber ends and the slice
//     partial is reduced into A[i,:] with red.global.add (the schedule's
//     Atomics strategy; A is 256 KB at cfg4 and stays in L2).
//  K9 SPX_K_MTTKRP_SLICE  A.5 shape: pos(i,ipos,B)
//     split(ipos,ipos0,ipos1,CHUNK) -> a CTA owns CHUNK slices, one warp per
//     slice, plain stores.
#include <cstdlib>
#include <type_traits>

#include "spx_common.cuh"

namespace spx {
namespace {

// K7 TTV: persistent CTAs of kTtvWarps warps stage c in shared memory (when
// it fits); the warps take fiber groups of FIBERS_PER_WARP fibers
// round-robin.  A group's leaves are one contiguous position range.
constexpr int kTtvWarps = 8;

// K7 TTV, reduce-by-key form: a warp takes 32*LPL consecutive leaves per
// step, LPL per lane (whole 16 B vectors of coordinates and values, streamed
// by cp.async.cg into a per-warp ring two steps ahead).  Each lane folds its
// LPL products v*c[k] into the fibers they belong to; fibers that start and
// end inside the lane are stored at once, the lane's trailing partial joins a
// segmented warp scan (one per step), and the lane that holds a fiber's next
// start stores the completed sum.  Fiber starts come from the 32 fibers of
// the group held one per lane (bit masks over the step's positions, one
// 32-bit word per 32 positions); every per-lane array is indexed at compile
// time.  LPL is a tuning knob: same-box A/B on cfg4 gave 0.45 / 0.51 / 0.72 ms
// for LPL = 4 / 8 / 16 -- larger steps amortise the scan but the bigger ring
// slots cost occupancy, which this latency-bound loop needs more.
constexpr int kRbkSlots = 3;
#ifndef SPX_TTV_MINB
#define SPX_TTV_MINB 6  // 40 registers: 6 CTAs (48 warps) per SM; occupancy-bound
#endif
#ifndef SPX_TTV_LPL
#define SPX_TTV_LPL 4
#endif
constexpr int kTtvLpl = SPX_TTV_LPL;

template <typename T, int LPL, bool CSMEM>
__global__ void __launch_bounds__(kTtvWarps * 32, SPX_TTV_MINB) ttv_rbk_kernel(const int32_t* __restrict__ crd0,
                                                      const int32_t* __restrict__ pos1,
                                                      const int32_t* __restrict__ crd1,
                                                      const int32_t* __restrict__ pos2,
                                                      const int32_t* __restrict__ crd2,
                                                      const T* __restrict__ vals, const T* __restrict__ c,
                                                      T* __restrict__ A, int64_t S, int64_t F, int64_t J,
                                                      int64_t K, int64_t FW, int64_t ngroups, int nnz) {
  static_assert(LPL % 4 == 0 && LPL <= 32, "whole int4 coordinate vectors per lane");
  constexpr int STEP = 32 * LPL;                       // leaves per warp step
  constexpr int SLOT = STEP * (4 + (int)sizeof(T));    // coordinates then values
  constexpr int VCH = LPL * (int)sizeof(T) / 16;       // 16 B value chunks per lane
  constexpr int VPC = 16 / (int)sizeof(T);             // values per chunk
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* sc = reinterpret_cast<T*>(smem_raw + (size_t)nw * kRbkSlots * SLOT);
  if (CSMEM) {
    for (int64_t k = threadIdx.x; k < K; k += blockDim.x) sc[k] = __ldg(c + k);
    __syncthreads();
  }
  unsigned char* ring = smem_raw + (size_t)warp * kRbkSlots * SLOT;
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
  __shared__ int64_t s_offs[kTtvWarps][32];
  int64_t* offs = s_offs[warp];
  const uint64_t pol_s = l2_evict_first();
  for (int64_t g = (int64_t)blockIdx.x * nw + warp; g < ngroups; g += (int64_t)gridDim.x * nw) {
    const int gf1 = (int)min(g * FW + FW, F);
    int sl = -1;
    for (int f0 = (int)(g * FW); f0 < gf1; f0 += 32) {
      const int f1 = min(f0 + 32, gf1);
      const int myfib = f0 + lane;
      const bool is_fib = myfib < f1;
      const int st_mine = is_fib ? __ldg(pos2 + myfib) : 0x7fffffff;
      if (sl < 0) sl = (int)warp_search_segment(pos1, 0, S, f0, lane);
      int s_mine = sl;
      if (is_fib)
        while (__ldg(pos1 + s_mine + 1) <= myfib) ++s_mine;
      const int64_t off_mine = is_fib ? (int64_t)__ldg(crd0 + s_mine) * J + __ldg(crd1 + myfib) : 0;
      sl = __shfl_sync(kFull, s_mine, f1 - f0 - 1);
      const int q0 = __shfl_sync(kFull, st_mine, 0), q1 = __ldg(pos2 + f1);
      const int a0 = q0 & ~3;  // 16-byte aligned start; positions < q0 are masked
      const int nsteps = (q1 - a0 + STEP - 1) / STEP;
      auto issue = [&](int st, int slot_i) {
        if (st < nsteps) {
          const int p = a0 + st * STEP + LPL * lane;
          const uint32_t d = ring_s + slot_i * SLOT;
          // whole 16 B copies wherever the step lies inside the arrays: positions
          // past q1 are masked in the fold, so only the arrays' end needs care
          if (a0 + (st + 1) * STEP <= nnz) {  // warp-uniform
#pragma unroll
            for (int h = 0; h < LPL / 4; ++h)
              cp_async16_zfill(d + (lane * LPL + 4 * h) * 4, crd2 + p + 4 * h, 16, pol_s);
#pragma unroll
            for (int h = 0; h < VCH; ++h)
              cp_async16_zfill(d + STEP * 4 + (lane * LPL + h * VPC) * (int)sizeof(T), vals + p + h * VPC, 16, pol_s);
          } else {  // the arrays' last step: nothing past q1 is read
#pragma unroll
            for (int h = 0; h < LPL / 4; ++h) {
              const int k = min(max(q1 - (p + 4 * h), 0), 4);
              cp_async16_elems<4>(d + (lane * LPL + 4 * h) * 4,
                                  k ? (const void*)(crd2 + p + 4 * h) : (const void*)crd2, k, pol_s);
            }
#pragma unroll
            for (int h = 0; h < VCH; ++h) {
              const int kk = min(max(q1 - (p + h * VPC), 0), VPC);
              cp_async16_elems<(int)sizeof(T)>(d + STEP * 4 + (lane * LPL + h * VPC) * (int)sizeof(T),
                                               kk ? (const void*)(vals + p + h * VPC) : (const void*)vals, kk, pol_s);
            }
          }
        }
        cp_async_commit();
      };
      issue(0, 0);
      issue(1, 1);
      offs[lane] = off_mine;  // A offsets of this subgroup's fibers, by f - f0
      __syncwarp();
      int fo = f0 - 1;  // fiber open just before the current step's first position
      T carry = T(0);   // its partial sum
      int slot_i = 0;   // st % kRbkSlots
      for (int st = 0; st < nsteps; ++st) {
        issue(st + 2, slot_i == 0 ? 2 : slot_i - 1);
        cp_async_wait<2>();
        __syncwarp();
        const int p = a0 + st * STEP;
        const unsigned char* slot = ring + slot_i * SLOT;
        slot_i = slot_i == kRbkSlots - 1 ? 0 : slot_i + 1;
        int kk[LPL];
        T v[LPL];
#pragma unroll
        for (int h = 0; h < LPL / 4; ++h) {
          const int4 k4 = *reinterpret_cast<const int4*>(slot + (lane * LPL + 4 * h) * 4);
          kk[4 * h] = k4.x;
          kk[4 * h + 1] = k4.y;
          kk[4 * h + 2] = k4.z;
          kk[4 * h + 3] = k4.w;
        }
#pragma unroll
        for (int j = 0; j < LPL; ++j) v[j] = reinterpret_cast<const T*>(slot + STEP * 4)[LPL * lane + j];
        __syncwarp();  // the slot is refilled two steps later
        T x[LPL];
        if (p >= q0 && p + STEP <= q1) {  // interior step (warp-uniform): no position masks
#pragma unroll
          for (int j = 0; j < LPL; ++j) x[j] = v[j] * (CSMEM ? sc[kk[j]] : __ldg(c + kk[j]));
        } else {
#pragma unroll
          for (int j = 0; j < LPL; ++j) {
            const int pp = p + LPL * lane + j;
            x[j] = (pp >= q0 && pp < q1) ? v[j] * (CSMEM ? sc[kk[j]] : __ldg(c + kk[j])) : T(0);
          }
        }
        // fiber starts in [p, p+STEP) as a bit mask, one word per 32 positions
        const int rel = st_mine - p;
        const int rw = (rel >= 0 && rel < STEP) ? (rel >> 5) : -1;
        const unsigned rbit = 1u << (rel & 31);
        constexpr int kLanesPerWord = 32 / LPL;
        const int wi = lane / kLanesPerWord, sh = (LPL * lane) & 31;
        unsigned myw = 0u;
        int before = 0, total = 0;
#pragma unroll
        for (int w = 0; w < LPL; ++w) {
          const unsigned Hw = __reduce_or_sync(kFull, rw == w ? rbit : 0u);
          const int pc = __popc(Hw);
          before += (w < wi) ? pc : 0;
          total += pc;
          myw = (w == wi) ? Hw : myw;
        }
        constexpr unsigned kLaneMask = LPL == 32 ? 0xffffffffu : ((1u << LPL) - 1u);
        const unsigned hb = (myw >> sh) & kLaneMask;  // start flags of my LPL positions
        before += __popc(myw & ((1u << sh) - 1u));
        // lane-local fold: seg0 = products before my first start; fibers that
        // start and end inside my positions are stored here
        T seg0 = T(0), run = T(0);
        int cnt = before;
#pragma unroll
        for (int j = 0; j < LPL; ++j) {
          if ((hb >> j) & 1u) {
            if (cnt > before) {
              if (fo + cnt >= f0) A[offs[(fo + cnt - f0) & 31]] = run;
            } else {
              seg0 = run;
            }
            run = T(0);
            ++cnt;
          }
          run += x[j];
        }
        const bool seen = hb != 0u;
        // segmented inclusive scan of the partial leaving each lane; the
        // step's carry enters at lane 0
        T vs = seen ? run : run + (lane == 0 ? carry : T(0));
        // segment heads are the lanes that saw a start (and lane 0); a lane
        // sums the lanes from its head on, so only values are shuffled
        const unsigned heads = __ballot_sync(kFull, seen || lane == 0);
        const int seg = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const T y = __shfl_up_sync(kFull, vs, o);
          if (lane - o >= seg) vs += y;
        }
        T in = __shfl_up_sync(kFull, vs, 1);  // partial arriving at my first position
        if (lane == 0) in = carry;
        if (seen) {  // my first start completes the fiber open when my lane begins
          const int fc = fo + before;
          if (fc >= f0) A[offs[(fc - f0) & 31]] = in + seg0;
        }
        carry = __shfl_sync(kFull, vs, 31);
        fo += total;
      }
      // the last fiber of the subgroup ends at q1
      if (lane == 0 && fo >= f0) A[offs[(fo - f0) & 31]] = carry;
      cp_async_wait<0>();
      __syncwarp();
    }
  }
}

// ---------------------------------------------------------------------------
// MTTKRP leaf-range engine shared by K8 (nnz-split) and K9 (slice-split).
//
// A warp walks a contiguous range of leaf positions [q0, q1) of B (level 2)
// with its lanes over the rank dimension j.  The (l, v) of the leaves stream
// through a per-warp cp.async ring (LeafRing) and are read back four at a
// time as 16-byte broadcasts; per leaf the warp then issues one row read of
// D (L1-resident: 256 KB at cfg4) and VPL FFMAs, so the D row read (128 B at
// R=32 fp32) is the per-leaf cost.  The fiber partial sum_l B*D[l,:] is
// scaled by C[k,:] when the fiber ends (the C row is prefetched when the
// fiber starts) and the slice partial goes to A[i,:] when the slice ends:
// red.global.add for chunks that may share a slice (the schedule's Atomics
// strategy), a plain store for a warp that owns the whole slice.
// ---------------------------------------------------------------------------
constexpr int kLeafRing = 4;
#ifndef SPX_MTTKRP_THREADS
#define SPX_MTTKRP_THREADS 512
#endif
constexpr int kMttkrpThreads = SPX_MTTKRP_THREADS;
// tuning knobs (same-box A/B on cfg4: G=4 with 2 CTAs/SM 1.24-1.26 ms; G=8 or
// 1 CTA/SM 1.63-1.65 ms -- occupancy wins over per-warp ILP here)
#ifndef SPX_MTTKRP_G
#define SPX_MTTKRP_G 4
#endif
#ifndef SPX_MTTKRP_SLICE_G
#define SPX_MTTKRP_SLICE_G 8
#endif
#ifndef SPX_MTTKRP_SLICE_MINB
#define SPX_MTTKRP_SLICE_MINB 1
#endif
#ifndef SPX_MTTKRP_MINB
#define SPX_MTTKRP_MINB 2
#endif

template <typename T, int VPL, bool CONTIG>
struct MttkrpCtx {
  const int32_t *crd0, *pos1, *crd1, *pos2, *crd2;
  const T *vals, *Cm, *Dm;
  T* A;
  int64_t S, F, R;
};

// Quarter-warp walk for 32-wide fp32 rows (rank 32, the cfg4 shape): the
// four quarter-warps take four consecutive leaves, each lane holding four
// columns (float4), so one warp instruction reads four 128 B rows of D (one
// L1TEX wavefront each -- the floor for this op) and two FFMA2 per lane cover
// all four leaves.  The quarters keep separate fiber and slice partials:
// scaling by C[k,:] is linear, so sum_q(accf_q * crow) is applied per quarter
// at each fiber end with no cross-lane traffic, and the quarters are folded
// (two xor shuffles) only when a slice is flushed.  A group of 4*G leaves
// inside one fiber takes 2*G FFMA2 per lane; a group that crosses fiber ends
// runs segment by segment with the products masked (FSEL) to the segment.
template <bool OWNED, int G>
__device__ __forceinline__ void mttkrp_walk_quad(const MttkrpCtx<float, 1, true>& c, unsigned char* ring_base,
                                                 int lane, int q0, int q1, int f, int s, float* part_dst) {
  static_assert(G == 4 || G == 8, "whole 16 B vectors of coordinates / values per quarter");
  // fiber window: ends and k coordinates of fibers [fb, fb+32), per warp in
  // shared memory (broadcast reads, no shuffles in the divergent close path)
  __shared__ int s_win[kMttkrpThreads / 32][64];
  int* win = s_win[threadIdx.x >> 5];
  const int qw = lane >> 3, ql = lane & 7;
  const uint64_t pol_s = l2_evict_first();
  int fb = f;
  auto load_win = [&]() {
    __syncwarp();
    win[lane] = __ldg(c.pos2 + min((int64_t)fb + 1 + lane, c.F));
    win[32 + lane] = __ldg(c.crd1 + min((int64_t)fb + lane, c.F - 1));
    __syncwarp();
  };
  load_win();
  auto fiber_end = [&](int ff) -> int {
    if (ff - fb >= 32) {
      fb = ff;
      load_win();
    }
    return win[ff - fb];
  };
  const float4* __restrict__ Cq = reinterpret_cast<const float4*>(c.Cm) + ql;
  const float4* __restrict__ Dq = reinterpret_cast<const float4*>(c.Dm) + ql;
  auto crow_of = [&](int ff) -> float4 { return __ldg(Cq + (uint32_t)win[32 + ff - fb] * 8u); };
  int fend = fiber_end(f);
  int send = __ldg(c.pos1 + s + 1);
  float2 af0 = make_float2(0.f, 0.f), af1 = af0, as0 = af0, as1 = af0;
  float4 crow = crow_of(f);
  auto flush_slice = [&]() {
    float4 x = make_float4(as0.x, as0.y, as1.x, as1.y);
#pragma unroll
    for (int o = 8; o < 32; o <<= 1) {
      x.x += __shfl_xor_sync(kFull, x.x, o);
      x.y += __shfl_xor_sync(kFull, x.y, o);
      x.z += __shfl_xor_sync(kFull, x.z, o);
      x.w += __shfl_xor_sync(kFull, x.w, o);
    }
    if (qw == 0) {
      float4* dst = reinterpret_cast<float4*>(part_dst ? part_dst : c.A + (int64_t)__ldg(c.crd0 + s) * 32) + ql;
      if constexpr (OWNED) *dst = x;
      else atomicAdd(dst, x);
    }
    as0 = make_float2(0.f, 0.f);
    as1 = as0;
  };
  auto close_fiber = [&]() {
    as0 = __ffma2_rn(af0, make_float2(crow.x, crow.y), as0);
    as1 = __ffma2_rn(af1, make_float2(crow.z, crow.w), as1);
    af0 = make_float2(0.f, 0.f);
    af1 = af0;
    ++f;
    fend = fiber_end(f);
    while (f >= send) {
      flush_slice();
      ++s;
      send = __ldg(c.pos1 + s + 1);
    }
    crow = crow_of(f);
  };
  LeafRing<float, kLeafRing> ring;
  ring.init(ring_base, c.crd2, c.vals, q0, q1);
  ring.prologue(lane, pol_s);
  for (int b = 0; b < ring.nb; ++b) {
    ring.acquire(b, lane, pol_s);
    const int p = q0 + b * 32;
    const int n = min(32, q1 - p);
    const int32_t* Ls = ring.crd_slot(b);
    const float* Vs = ring.val_slot(b);
#pragma unroll 1
    for (int t = 0; t < n; t += 4 * G) {
      // quarter qw takes leaves t + G*qw .. t + G*qw + G-1 (zero-filled past n)
      float4 d[G];
      float v[G];
#pragma unroll
      for (int h = 0; h < G / 4; ++h) {
        const int4 l4 = *reinterpret_cast<const int4*>(Ls + t + G * qw + 4 * h);
        const float4 v4 = *reinterpret_cast<const float4*>(Vs + t + G * qw + 4 * h);
        d[4 * h] = __ldg(Dq + (uint32_t)l4.x * 8u);
        d[4 * h + 1] = __ldg(Dq + (uint32_t)l4.y * 8u);
        d[4 * h + 2] = __ldg(Dq + (uint32_t)l4.z * 8u);
        d[4 * h + 3] = __ldg(Dq + (uint32_t)l4.w * 8u);
        v[4 * h] = v4.x;
        v[4 * h + 1] = v4.y;
        v[4 * h + 2] = v4.z;
        v[4 * h + 3] = v4.w;
      }
#define SPX_QFMA(vv, d)                                                          \
  do {                                                                           \
    af0 = __ffma2_rn(make_float2((vv), (vv)), make_float2((d).x, (d).y), af0); \
    af1 = __ffma2_rn(make_float2((vv), (vv)), make_float2((d).z, (d).w), af1); \
  } while (0)
      if (t + 4 * G <= n && p + t + 4 * G <= fend) {
#pragma unroll
        for (int u = 0; u < G; ++u) SPX_QFMA(v[u], d[u]);
      } else {
        // fiber segment by fiber segment: leaves [L0, L1) of the group lie
        // in fiber f; products outside the segment are masked to zero
        const int cnt = min(4 * G, n - t);
        const int me = G * qw;
        int L0 = 0;
        while (true) {
          const int L1 = min(cnt, fend - (p + t));
#pragma unroll
          for (int u = 0; u < G; ++u) SPX_QFMA((me + u >= L0 && me + u < L1) ? v[u] : 0.f, d[u]);
          if (L1 >= cnt) break;
          L0 = L1;
          while (p + t + L0 >= fend) close_fiber();
        }
      }
#undef SPX_QFMA
    }
    ring.release();
  }
  as0 = __ffma2_rn(af0, make_float2(crow.x, crow.y), as0);
  as1 = __ffma2_rn(af1, make_float2(crow.z, crow.w), as1);
  flush_slice();
}


// Walk leaves [q0, q1); f = fiber holding q0, s = slice holding f.
// OWNED: the warp owns every slice it touches completely (plain stores).
// part_dst (OWNED, a range inside one slice): the slice partial goes there
// instead of A's row (a part of a split slice, folded by slice_fold_kernel).
// QG: leaves per quarter per group of the rank-32 walk (0 = the default:
// SPX_MTTKRP_SLICE_G for OWNED, whose whole-slice warps are latency-bound
// at 1 CTA/SM, SPX_MTTKRP_G otherwise).
template <typename T, int VPL, bool CONTIG, bool OWNED, int QG = 0>
__device__ __forceinline__ void mttkrp_walk(const MttkrpCtx<T, VPL, CONTIG>& c, unsigned char* ring_base, int lane,
                                            int q0, int q1, int f, int s, T* part_dst = nullptr) {
  if constexpr (std::is_same<T, float>::value && VPL == 1 && CONTIG) {
    if (c.R == 32) {
      constexpr int G = QG ? QG : (OWNED ? SPX_MTTKRP_SLICE_G : SPX_MTTKRP_G);
      mttkrp_walk_quad<OWNED, G>(c, ring_base, lane, q0, q1, f, s, part_dst);
      return;
    }
  }
  using Fr = Frag<T, VPL, CONTIG>;
  const int ncols = (int)c.R;
  const int Ri = (int)c.R;
  const uint64_t pol_s = l2_evict_first();
  // fibers [fb, fb+32): ends and k coordinates, one per lane
  int fb = f;
  int fe_mine = __ldg(c.pos2 + min((int64_t)fb + 1 + lane, c.F));
  int k_mine = __ldg(c.crd1 + min((int64_t)fb + lane, c.F - 1));
  auto fiber_end = [&](int ff) -> int {
    if (ff - fb >= 32) {
      fb = ff;
      fe_mine = __ldg(c.pos2 + min((int64_t)fb + 1 + lane, c.F));
      k_mine = __ldg(c.crd1 + min((int64_t)fb + lane, c.F - 1));
    }
    return __shfl_sync(kFull, fe_mine, ff - fb);
  };
  auto fiber_k = [&](int ff) -> int { return __shfl_sync(kFull, k_mine, ff - fb); };
  int fend = fiber_end(f);
  int send = __ldg(c.pos1 + s + 1);
  Fr accf, accs, crow;
  accf.zero();
  accs.zero();
  crow.load(c.Cm + fiber_k(f) * Ri, lane, ncols);
  auto flush_slice = [&]() {
    T* dst = part_dst ? part_dst : c.A + (int64_t)__ldg(c.crd0 + s) * c.R;
    if constexpr (OWNED) accs.store(dst, lane, ncols);
    else accs.atomic_add_into(dst, lane, ncols);
    accs.zero();
  };
  // close fibers until position pp lies inside fiber f
  auto advance_to = [&](int pp) {
    while (pp >= fend) {
#pragma unroll
      for (int i = 0; i < VPL; ++i) accs.v[i] += accf.v[i] * crow.v[i];
      accf.zero();
      ++f;
      fend = fiber_end(f);
      while (f >= send) {
        flush_slice();
        ++s;
        send = __ldg(c.pos1 + s + 1);
      }
      crow.load(c.Cm + fiber_k(f) * Ri, lane, ncols);
    }
  };
  // this lane's slice of D: row l starts at Dl + l*R (32-bit offsets)
  const char* __restrict__ Dl = reinterpret_cast<const char*>(c.Dm + (CONTIG ? lane * VPL : lane));
  const uint32_t rowb = (uint32_t)(c.R * (int64_t)sizeof(T));
#define SPX_DROW(d, l)                                                                       \
  do {                                                                                       \
    const T* src_ = reinterpret_cast<const T*>(addr_wide(Dl, (uint32_t)(l), rowb));         \
    if constexpr (CONTIG) {                                                                  \
      (d).load_ptr(src_);                                                                    \
    } else {                                                                                 \
      _Pragma("unroll") for (int i_ = 0; i_ < VPL; ++i_)(d).v[i_] =                         \
          (i_ * 32 + lane < ncols) ? __ldg(src_ + i_ * 32) : T(0);                          \
    }                                                                                        \
  } while (0)
  LeafRing<T, kLeafRing> ring;
  ring.init(ring_base, c.crd2, c.vals, q0, q1);
  ring.prologue(lane, pol_s);
  for (int b = 0; b < ring.nb; ++b) {
    ring.acquire(b, lane, pol_s);
    const int p = q0 + b * 32;
    const int n = min(32, q1 - p);
    const int32_t* Ls = ring.crd_slot(b);
    const T* Vs = ring.val_slot(b);
    // groups of G leaves: all G row reads of D are issued before the first
    // FMA (G*VPL >= 8 values per lane in flight), then the group is consumed
    // fiber segment by fiber segment (predicated FMAs keep d[] in registers)
    constexpr int G = (8 / VPL) < 4 ? 4 : (8 / VPL);
#pragma unroll 1
    for (int t = 0; t < n; t += G) {
      Fr d[G];
#pragma unroll
      for (int u = 0; u < G; u += 4) {
        const int4 l4 = *reinterpret_cast<const int4*>(Ls + t + u);  // zero-filled past n
        SPX_DROW(d[u], l4.x);
        SPX_DROW(d[u + 1], l4.y);
        SPX_DROW(d[u + 2], l4.z);
        SPX_DROW(d[u + 3], l4.w);
      }
      T vg[G];
#pragma unroll
      for (int u = 0; u < G; ++u) vg[u] = Vs[t + u];  // zero-filled past n
      const int cnt = min(G, n - t);
      if (cnt == G && p + t + G <= fend) {
        // the whole group lies in fiber f
#pragma unroll
        for (int u = 0; u < G; ++u) accf.fma(vg[u], d[u]);
      } else {
        int u0 = 0;
        while (true) {
          const int u1 = min(cnt, fend - (p + t));  // leaves [u0, u1) lie in fiber f
#pragma unroll
          for (int u = 0; u < G; ++u)
            if (u >= u0 && u < u1) accf.fma(vg[u], d[u]);
          if (u1 >= cnt) break;
          u0 = u1;
          advance_to(p + t + u0);
        }
      }
    }
    ring.release();
  }
#pragma unroll
  for (int i = 0; i < VPL; ++i) accs.v[i] += accf.v[i] * crow.v[i];
  flush_slice();
}
#undef SPX_DROW

// ---------------------------------------------------------------------------
// K8 for rank-32 fp32 (the cfg4 shape): quarter-warp sub-chunks.
//
// The warp's chunk of NNZ_PER_WARP leaves is cut into four contiguous
// quarter chunks; quarter qw (8 lanes x float4 = one 128 B row) walks its
// own leaves with its own fiber / slice state.  A group of four leaves that
// stays inside the quarter's current fiber costs 2 LDS.128 + 4 LDG.128 (one
// L1 wavefront per D row, the floor) + 8 FFMA2 with no masking; only a
// quarter whose group crosses a fiber end takes the leaf-by-leaf path, and
// that path closes the fiber (scale by the C row held in registers) without
// touching the other quarters' leaves.  Fiber ends and k coordinates come from
// an 8-fiber window held one per lane of the quarter (width-8 shuffles), the
// next C row is loaded when a fiber opens and consumed when it closes.
// ---------------------------------------------------------------------------
#ifndef SPX_MTTKRP_QUARTER
#define SPX_MTTKRP_QUARTER 1
#endif
#ifndef SPX_MQ_RING
#define SPX_MQ_RING 3  // batch bi in use, bi+1 landed (its D rows prefetched), bi+2 in flight
#endif
#ifndef SPX_MQ_CARVEOUT
#define SPX_MQ_CARVEOUT 14  // percent of 228 KB: the 32 KB shared-memory config, L1 keeps 224 KB for D
#endif
constexpr int kQRing = SPX_MQ_RING;       // slots of QB leaves per quarter in flight
#ifndef SPX_MQ_THREADS
#define SPX_MQ_THREADS 512  // x 2 CTAs/SM (same-box A/B: 24 warps at 80 registers ran slower than 32 at 64)
#endif
#ifndef SPX_MQ_MINB
#define SPX_MQ_MINB 2
#endif
constexpr int kQThreads = SPX_MQ_THREADS;
#ifndef SPX_MQ_SMWIN
#define SPX_MQ_SMWIN 1  // fiber window in shared memory (else per-lane registers + width-8 shuffles)
#endif
#ifndef SPX_MQ_PF
#define SPX_MQ_PF 1  // prefetch the next batch's D rows into L1 (needs SPX_MQ_RING >= 3): cfg4 1.013 vs 1.038 ms
#endif
static_assert(!SPX_MQ_PF || SPX_MQ_RING >= 3, "the next-batch prefetch needs a 3-slot ring");
#ifndef SPX_MQ_QB
#define SPX_MQ_QB 16  // leaves per quarter per batch with 16 B copies (8: half the lanes copy)
#endif
// a ring slot: QB coordinates then QB values per quarter (fp32)
template <int QB>
constexpr int q_slot_bytes() { return 4 * QB * 8; }
constexpr int kQSlotBytes = q_slot_bytes<8>();

__device__ __forceinline__ int4 lds_i4(uint32_t a) {
  int4 r;
  asm volatile("ld.shared.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
  return r;
}
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
  float4 r;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "r"(a));
  return r;
}
__device__ __forceinline__ float4 ld_f4_na(const float4* p) {
  float4 r;
  asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ float4 ld_drow(const float4* p) {
  // an explicit L2 policy (the descriptor becomes an immediate in a uniform
  // register, so the loop needs no R2UR of the default descriptor per load)
  return ld_f4_hint(p, kPolicyEvictLast);
}
__device__ __forceinline__ void red_add_f4(float* dst, float4 x) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(dst), "f"(x.x), "f"(x.y), "f"(x.z), "f"(x.w)
               : "memory");
}

template <bool AL16>
__global__ void __launch_bounds__(kQThreads, SPX_MQ_MINB) mttkrp_quarter_kernel(
    const int32_t* __restrict__ crd0, const int32_t* __restrict__ pos1, const int32_t* __restrict__ crd1,
    const int32_t* __restrict__ pos2, const int32_t* __restrict__ crd2, const float* __restrict__ vals,
    const float* __restrict__ Cm, const float* __restrict__ Dm, float* __restrict__ A, int S, int F, int nnz,
    int W, int nchunks, const int32_t* __restrict__ chunkF, const int32_t* __restrict__ chunkS, uint32_t rowb) {
  // rowb = 128 (bytes per C / D row) arrives as a parameter so that row
  // addresses stay one IMAD.WIDE.U32 (a literal 128 is strength-reduced to
  // a three-instruction shift-and-add)
  // QB leaves per quarter per batch: AL16 uses SPX_MQ_QB (16: every lane
  // issues one 16 B copy per batch, no lane predicate), else 8 (4 B copies)
  constexpr int QB = AL16 ? SPX_MQ_QB : 8;
  constexpr int kSlot = q_slot_bytes<QB>();
  constexpr int kValOff = 4 * QB * 4;  // values follow the four quarters' coordinates
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qw = lane >> 3, ql = lane & 7;
  const unsigned qmask = 0xFFu << (qw * 8);
  unsigned char* ring = smem_raw + (size_t)warp * (kQRing * kSlot);
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
  const uint64_t pol_s = l2_evict_first();
#if SPX_MQ_SMWIN
  __shared__ int s_qwin[kQThreads / 32][4][16];
#endif
  // this lane's 16 B column slice of the C / D / A rows (row r at + r*128 B)
  const char* __restrict__ Cl = reinterpret_cast<const char*>(Cm) + ql * 16;
  const char* __restrict__ Dl = reinterpret_cast<const char*>(Dm) + ql * 16;
  float* __restrict__ Al = A + ql * 4;
  // the quarter's QB leaf coordinates / values of a slot (broadcast LDS.128)
  const int rd_off = qw * QB * 4;
  // AL16: QB/2 lanes of a quarter copy 16 B each -- (coordinates | values) x QB/4 chunks of 4 leaves
  constexpr int kChunks = QB / 4;
  const int cp_h = ql % kChunks, cp_which = (ql / kChunks) & 1;
  const bool cp_lane = ql < 2 * kChunks;
  const uint32_t cp_dst = (uint32_t)(cp_which * kValOff + qw * QB * 4 + cp_h * 16);
  const char* cp_src = cp_which ? reinterpret_cast<const char*>(vals) : reinterpret_cast<const char*>(crd2);
  const int Wq = W >> 2;
  for (int q = blockIdx.x * nw + warp; q < nchunks; q += gridDim.x * nw) {
    const int c0 = q * W, c1 = min(c0 + W, nnz);
    const int a = min(c0 + qw * Wq, c1), b = min(a + Wq, c1);
    const int nbw = (min(Wq, c1 - c0) + QB - 1) / QB;  // batches of QB leaves (quarter 0 has the most)
    // issue batch bi into ring slot `slot`
    // AL16: this lane's next 16 B source and how many of its leaves remain
    const char* isrc = cp_src + (size_t)(a + cp_h * 4) * 4;
    int irem = b - (a + cp_h * 4);
    auto issue = [&](int bi, uint32_t slot) {
      if (bi < nbw) {
        if constexpr (AL16) {
          if (cp_lane) {
            const int nv = max(0, min(4, irem));
            cp_async16_zfill(ring_s + slot + cp_dst, nv ? isrc : cp_src, nv * 4, pol_s);
          }
          isrc += QB * 4;
          irem -= QB;
        } else {
          const int p = a + bi * 8 + ql;
          const bool ok = p < b;
          cp_async4(ring_s + slot + lane * 4, crd2 + (ok ? p : 0), ok ? 4 : 0, pol_s);
          cp_async4(ring_s + slot + 128 + lane * 4, vals + (ok ? p : 0), ok ? 4 : 0, pol_s);
        }
      }
      cp_async_commit();
    };
    uint32_t rslot = 0, islot = (kQRing - 1) * kSlot;
#pragma unroll
    for (int bi = 0; bi < kQRing - 1; ++bi) issue(bi, bi * kSlot);
    const bool live = a < b;
    int f = live ? __ldg(chunkF + q * 4 + qw) : 0;
    int s = live ? __ldg(chunkS + q * 4 + qw) : 0;
#if SPX_MQ_SMWIN
    // fiber window in shared memory: ends and k of fibers fb..fb+7 per
    // quarter, read with broadcast LDS in the quarter-divergent close path
    // (a shuffle there costs a warp-convergence check sequence)
    int* const wend = s_qwin[threadIdx.x >> 5][qw];
    int* const wk = wend + 8;
    int fb = f;
    wend[ql] = ld_i32_first(pos2 + min(fb + 1 + ql, F), pol_s);
    wk[ql] = ld_i32_first(crd1 + min(fb + ql, F - 1), pol_s);
    __syncwarp();
    int send = __ldg(pos1 + s + 1);
    int fend = wend[0];
    float4 crow = ld_f4_na(reinterpret_cast<const float4*>(addr_wide(Cl, (uint32_t)wk[0], rowb)));
    float2 af0 = make_float2(0.f, 0.f), af1 = af0, as0 = af0, as1 = af0;
    // close fiber f (quarter-divergent: only this quarter's lanes run it)
    auto close_fiber = [&]() {
      as0 = __ffma2_rn(af0, make_float2(crow.x, crow.y), as0);
      as1 = __ffma2_rn(af1, make_float2(crow.z, crow.w), as1);
      af0 = make_float2(0.f, 0.f);
      af1 = af0;
      ++f;
      if (f - fb >= 8) {
        fb = f;
        const int e_ = ld_i32_first(pos2 + min(fb + 1 + ql, F), pol_s);
        const int k_ = ld_i32_first(crd1 + min(fb + ql, F - 1), pol_s);
        __syncwarp(qmask);
        wend[ql] = e_;
        wk[ql] = k_;
        __syncwarp(qmask);
      }
      fend = wend[f - fb];
      while (f >= send) {
        red_add_f4(Al + (int64_t)__ldg(crd0 + s) * 32, make_float4(as0.x, as0.y, as1.x, as1.y));
        as0 = make_float2(0.f, 0.f);
        as1 = as0;
        ++s;
        send = __ldg(pos1 + s + 1);
      }
      crow = ld_f4_na(reinterpret_cast<const float4*>(addr_wide(Cl, (uint32_t)wk[f - fb], rowb)));
    };
#else
    // fiber window: lane ql holds the end and k of fiber fb+ql
    int fb = f;
    int fe_w = ld_i32_first(pos2 + min(fb + 1 + ql, F), pol_s);
    int k_w = ld_i32_first(crd1 + min(fb + ql, F - 1), pol_s);
    int send = __ldg(pos1 + s + 1);
    int fend = __shfl_sync(kFull, fe_w, 0, 8);
    float4 crow = ld_f4_na(reinterpret_cast<const float4*>(addr_wide(Cl, (uint32_t)__shfl_sync(kFull, k_w, 0, 8), rowb)));
    float2 af0 = make_float2(0.f, 0.f), af1 = af0, as0 = af0, as1 = af0;
    // close fiber f (quarter-divergent: only this quarter's lanes run it)
    auto close_fiber = [&]() {
      as0 = __ffma2_rn(af0, make_float2(crow.x, crow.y), as0);
      as1 = __ffma2_rn(af1, make_float2(crow.z, crow.w), as1);
      af0 = make_float2(0.f, 0.f);
      af1 = af0;
      ++f;
      if (f - fb >= 8) {
        fb = f;
        fe_w = ld_i32_first(pos2 + min(fb + 1 + ql, F), pol_s);
        k_w = ld_i32_first(crd1 + min(fb + ql, F - 1), pol_s);
      }
      fend = __shfl_sync(qmask, fe_w, f - fb, 8);
      while (f >= send) {
        red_add_f4(Al + (int64_t)__ldg(crd0 + s) * 32, make_float4(as0.x, as0.y, as1.x, as1.y));
        as0 = make_float2(0.f, 0.f);
        as1 = as0;
        ++s;
        send = __ldg(pos1 + s + 1);
      }
      crow = ld_f4_na(reinterpret_cast<const float4*>(addr_wide(Cl, (uint32_t)__shfl_sync(qmask, k_w, f - fb, 8), rowb)));
    };
#endif
#define SPX_QF(vv, d)                                                            \
  do {                                                                           \
    af0 = __ffma2_rn(make_float2((vv), (vv)), make_float2((d).x, (d).y), af0); \
    af1 = __ffma2_rn(make_float2((vv), (vv)), make_float2((d).z, (d).w), af1); \
  } while (0)
#define SPX_DR(l) ld_drow(reinterpret_cast<const float4*>(addr_wide(Dl, (uint32_t)(l), rowb)))
    int pp = a;  // first leaf of the current group
#pragma unroll 1
    for (int bi = 0; bi < nbw; ++bi) {
      issue(bi + kQRing - 1, islot);
      islot = islot == (kQRing - 1) * kSlot ? 0 : islot + kSlot;
#if SPX_MQ_PF
      // batch bi+1 has landed too: pull its D rows into L1 while batch bi is
      // processed (each lane of the quarter prefetches QB/8 of its rows)
      cp_async_wait<kQRing - 2>();
      __syncwarp();
      const uint32_t sl = ring_s + rslot + rd_off;
      rslot = rslot == (kQRing - 1) * kSlot ? 0 : rslot + kSlot;
      if (bi + 1 < nbw) {
        const uint32_t sn = ring_s + rslot + rd_off + ql * (QB / 2);
#pragma unroll
        for (int j = 0; j < QB / 8; ++j) {
          int lj;
          asm volatile("ld.shared.s32 %0, [%1];" : "=r"(lj) : "r"(sn + 4 * j));
          asm volatile("prefetch.global.L1 [%0];" ::"l"(addr_wide(Dl, (uint32_t)lj, rowb)));
        }
      }
#else
      cp_async_wait<kQRing - 1>();
      __syncwarp();
      const uint32_t sl = ring_s + rslot + rd_off;
      rslot = rslot == (kQRing - 1) * kSlot ? 0 : rslot + kSlot;
#endif
#pragma unroll
      for (int h = 0; h < QB / 4; ++h, pp += 4) {
        const int4 l4 = lds_i4(sl + h * 16);
        const float4 d0 = SPX_DR(l4.x), d1 = SPX_DR(l4.y), d2 = SPX_DR(l4.z), d3 = SPX_DR(l4.w);
        const float4 v4 = lds_f4(sl + kValOff + h * 16);
        if (pp + 4 <= fend) {  // leaves pp..pp+3 lie in fiber f (zero-filled past b)
          SPX_QF(v4.x, d0);
          SPX_QF(v4.y, d1);
          SPX_QF(v4.z, d2);
          SPX_QF(v4.w, d3);
        } else if (pp < b) {
          while (pp >= fend) close_fiber();
          SPX_QF(v4.x, d0);
          if (pp + 1 < b) {
            while (pp + 1 >= fend) close_fiber();
            SPX_QF(v4.y, d1);
            if (pp + 2 < b) {
              while (pp + 2 >= fend) close_fiber();
              SPX_QF(v4.z, d2);
              if (pp + 3 < b) {
                while (pp + 3 >= fend) close_fiber();
                SPX_QF(v4.w, d3);
              }
            }
          }
        }
      }
      __syncwarp();
    }
#undef SPX_QF
#undef SPX_DR
    // close the open fiber; fold the quarters when they end in one slice
    as0 = __ffma2_rn(af0, make_float2(crow.x, crow.y), as0);
    as1 = __ffma2_rn(af1, make_float2(crow.z, crow.w), as1);
    float4 x = make_float4(as0.x, as0.y, as1.x, as1.y);
    const int skey = live ? s : -1;
    const bool same = __all_sync(kFull, __shfl_sync(kFull, skey, 0) == skey);
    if (same) {
#pragma unroll
      for (int o = 8; o < 32; o <<= 1) {
        x.x += __shfl_xor_sync(kFull, x.x, o);
        x.y += __shfl_xor_sync(kFull, x.y, o);
        x.z += __shfl_xor_sync(kFull, x.z, o);
        x.w += __shfl_xor_sync(kFull, x.w, o);
      }
      if (qw == 0 && live) red_add_f4(Al + (int64_t)__ldg(crd0 + s) * 32, x);
    } else if (live) {
      red_add_f4(Al + (int64_t)__ldg(crd0 + s) * 32, x);
    }
  }
  cp_async_wait<0>();
}

// the quarter kernel's shape: fp32, rank 32, NNZ_PER_WARP a multiple of 4,
// 16 B aligned C / D / A rows (float4 loads, red.v4)
bool mttkrp_quarter_ok(const Args& a) {
  if (!SPX_MTTKRP_QUARTER || a.dtype != SPX_F32 || a.dims[1][1] != 32) return false;
  const int64_t W = a.params[1];
  if (W < 4 || W % 4 != 0) return false;
  auto al = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  return (!a.vals[1] || al(a.vals[1])) && (!a.vals[2] || al(a.vals[2])) && (!a.out || al(a.out));
}

constexpr size_t kSmemBudget = 200 * 1024;

// K8: persistent CTAs; warp-chunk q covers leaves [q*W, (q+1)*W) (the
// schedule's `warp` variable; NNZ_PER_TB/NNZ_PER_WARP chunks make a `block`).
template <typename T, int VPL, bool CONTIG>
__global__ void __launch_bounds__(kMttkrpThreads, SPX_MTTKRP_MINB) mttkrp_nnz_kernel(
    const int32_t* __restrict__ crd0, const int32_t* __restrict__ pos1, const int32_t* __restrict__ crd1,
    const int32_t* __restrict__ pos2, const int32_t* __restrict__ crd2, const T* __restrict__ vals,
    const T* __restrict__ Cm, const T* __restrict__ Dm, T* __restrict__ A, int64_t S, int64_t F, int64_t nnz,
    int64_t R, int64_t W, int64_t nchunks, const int32_t* __restrict__ first) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* ring = smem_raw + (size_t)warp * LeafRing<T, kLeafRing>::kBytes;
  MttkrpCtx<T, VPL, CONTIG> c{crd0, pos1, crd1, pos2, crd2, vals, Cm, Dm, A, S, F, R};
  for (int64_t q = (int64_t)blockIdx.x * nw + warp; q < nchunks; q += (int64_t)gridDim.x * nw) {
    const int q0 = (int)(q * W);
    const int q1 = (int)min(q * W + W, nnz);
    const int f = __ldg(first + q);
    const int s = (int)warp_search_segment(pos1, 0, S, f, lane);
    mttkrp_walk<T, VPL, CONTIG, false>(c, ring, lane, q0, q1, f, s);
  }
}

// K9: slice-split (A.5 shape) -- every slice has one owner and no output
// races.  A slice of at most `part` leaves is one unit: one warp walks it and
// stores A's row.  A heavier slice is cut into ceil(leaves / part) leaf
// ranges; their warps store partial rows into the workspace and
// slice_fold_kernel adds them in range order (deterministic, no atomics).
// Without the cut the heaviest slice sets the time: at cfg4 (2,048 slices,
// the largest 890K leaves) one warp per slice ran 15.9 ms.
// unit -> (slice, range): part_start[s] = first unit of slice s (scan of
// max(1, ceil(leaves_s / part)) by slice_parts_kernel), part_start[S] = units.
__global__ void slice_parts_kernel(const int32_t* __restrict__ pos1, const int32_t* __restrict__ pos2, int64_t S,
                                   int64_t part, int32_t* __restrict__ part_start) {
  __shared__ int64_t s_warp[32];
  __shared__ int64_t s_base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  if (tid == 0) s_base = 0;
  __syncthreads();
  for (int64_t t0 = 0; t0 < S; t0 += blockDim.x) {
    const int64_t s = t0 + tid;
    int64_t np = 0;
    if (s < S) {
      const int64_t leaves = (int64_t)__ldg(pos2 + __ldg(pos1 + s + 1)) - __ldg(pos2 + __ldg(pos1 + s));
      np = leaves > part ? (leaves + part - 1) / part : 1;
    }
    int64_t x = np;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int64_t w = lane < nw ? s_warp[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(kFull, w, o);
        if (lane >= o) w += y;
      }
      if (lane < nw) s_warp[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const int64_t base = s_base;
    if (s < S) part_start[s] = (int32_t)(base + (warp ? s_warp[warp - 1] : 0) + x - np);
    __syncthreads();
    if (tid == 0) s_base = base + s_warp[nw - 1];
    __syncthreads();
  }
  if (tid == 0) part_start[S] = (int32_t)s_base;
}

// SPLIT (params[2] = 1): balanced units, 2 CTAs/SM and the nnz-split's group
// depth (cfg4 MTTKRP0: 1.42 ms, against 2.04 at 1 CTA/SM with G = 8);
// whole-slice warps keep 1 CTA/SM and G = 8 for the latency-bound heaviest slice.
template <typename T, int VPL, bool CONTIG, bool SPLIT>
__global__ void __launch_bounds__(kMttkrpThreads, SPLIT ? SPX_MTTKRP_MINB : SPX_MTTKRP_SLICE_MINB) mttkrp_slice_kernel(
    const int32_t* __restrict__ crd0, const int32_t* __restrict__ pos1, const int32_t* __restrict__ crd1,
    const int32_t* __restrict__ pos2, const int32_t* __restrict__ crd2, const T* __restrict__ vals,
    const T* __restrict__ Cm, const T* __restrict__ Dm, T* __restrict__ A, int64_t S, int64_t F, int64_t R,
    const int32_t* __restrict__ part_start, int64_t part, T* __restrict__ partial) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* ring = smem_raw + (size_t)warp * LeafRing<T, kLeafRing>::kBytes;
  MttkrpCtx<T, VPL, CONTIG> c{crd0, pos1, crd1, pos2, crd2, vals, Cm, Dm, A, S, F, R};
  const int64_t units = __ldg(part_start + S);
  for (int64_t u = (int64_t)blockIdx.x * nw + warp; u < units; u += (int64_t)gridDim.x * nw) {
    const int64_t s = warp_search_segment(part_start, 0, S, u, lane);
    const int64_t k = u - __ldg(part_start + s), np = __ldg(part_start + s + 1) - __ldg(part_start + s);
    const int f0 = __ldg(pos1 + s), f1 = __ldg(pos1 + s + 1);
    const int q0 = __ldg(pos2 + f0), q1 = __ldg(pos2 + f1);
    constexpr int QG = SPLIT ? SPX_MTTKRP_G : SPX_MTTKRP_SLICE_G;
    if (np == 1) {
      if (q0 < q1) mttkrp_walk<T, VPL, CONTIG, true, QG>(c, ring, lane, q0, q1, f0, (int)s);
    } else {
      const int a = (int)(q0 + k * part), b = (int)min((int64_t)q1, (int64_t)a + part);
      const int f = (int)warp_search_segment(pos2, f0, f1, a, lane);  // fiber holding leaf a
      mttkrp_walk<T, VPL, CONTIG, true, QG>(c, ring, lane, a, b, f, (int)s, partial + u * R);
    }
  }
}

// A[crd0[s], :] = sum of slice s's partial rows in range order (split slices only)
template <typename T>
__global__ void slice_fold_kernel(const int32_t* __restrict__ part_start, const int32_t* __restrict__ crd0,
                                  int64_t S, int64_t R, const T* __restrict__ partial, T* __restrict__ A) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t s = g >> 5;
  if (s >= S) return;
  const int u0 = __ldg(part_start + s), u1 = __ldg(part_start + s + 1);
  if (u1 - u0 < 2) return;
  T* dst = A + (int64_t)__ldg(crd0 + s) * R;
  for (int64_t j = g & 31; j < R; j += 32) {
    T acc = partial[(int64_t)u0 * R + j];
    for (int u = u0 + 1; u < u1; ++u) acc += partial[(int64_t)u * R + j];
    dst[j] = acc;
  }
}

// leaves per K9 unit: slices heavier than this are cut (about 8,192 units at
// scale, so the largest unit is a small share of a warp's work)
#ifndef SPX_SLICE_UNITS
#define SPX_SLICE_UNITS 8192
#endif
inline int64_t slice_part_leaves(int64_t nnz) {
  return std::max<int64_t>(4096, (nnz + SPX_SLICE_UNITS - 1) / SPX_SLICE_UNITS);
}

int num_sms() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return n;
}

struct Csf {
  const int32_t *crd0, *pos1, *crd1, *pos2, *crd2;
  int64_t S, F, nnz;
};

Csf csf_of(const Args& a) {
  Csf c;
  c.crd0 = a.crd[0];
  c.pos1 = a.pos[1];
  c.crd1 = a.crd[1];
  c.pos2 = a.pos[2];
  c.crd2 = a.crd[2];
  c.S = a.level_sizes[0];
  c.F = a.level_sizes[1];
  c.nnz = a.level_sizes[2];
  return c;
}

template <typename T>
int run_ttv(const Args& a) {
  const Csf c = csf_of(a);
  const int64_t I = a.dims[0][0], J = a.dims[0][1], K = a.dims[0][2];
  T* A = static_cast<T*>(a.out);
  if (int e = check_cuda(cudaMemsetAsync(A, 0, (size_t)(I * J) * sizeof(T), a.stream), "memset")) return e;
  if (c.F == 0) return SPX_OK;
  const int64_t FTB = a.params[0] > 0 ? a.params[0] : 256;
  const int64_t FW = a.params[1] > 0 ? a.params[1] : 32;
  if (ceil_div(FTB, FW) > kMaxWarps)
    return fail(SPX_E_UNSUPPORTED, "TTV: FIBERS_PER_TB/FIBERS_PER_WARP must be <= 16");
  // the schedule's block (FIBERS_PER_TB fibers) is a unit of work; the
  // persistent CTAs are 8 warps that take fiber groups round-robin
  const int64_t nw = kTtvWarps;
  const size_t cbytes = (size_t)K * sizeof(T);
  const size_t rbytes = (size_t)nw * kRbkSlots * 32 * kTtvLpl * (4 + sizeof(T));
  const int c_in_smem = cbytes + rbytes <= kSmemBudget ? 1 : 0;
  const size_t smem = rbytes + (c_in_smem ? cbytes : 0);
  auto kern = c_in_smem ? ttv_rbk_kernel<T, kTtvLpl, true> : ttv_rbk_kernel<T, kTtvLpl, false>;
  if (int e = check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                         "cudaFuncSetAttribute"))
    return e;
  // persistent: as many CTAs as fit (smem-limited when c is large)
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, (int)(nw * 32), smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t grid = min((int64_t)num_sms() * per_sm, ceil_div(ceil_div(c.F, FW), nw));
  kern<<<(unsigned)grid, (unsigned)(nw * 32), smem, a.stream>>>(c.crd0, c.pos1, c.crd1, c.pos2, c.crd2,
                                                                 static_cast<const T*>(a.vals[0]),
                                                                 static_cast<const T*>(a.vals[1]), A, c.S, c.F, J, K,
                                                                 FW, ceil_div(c.F, FW), (int)c.nnz);
  count_launch();
  return check_cuda(cudaGetLastError(), "ttv_rbk_kernel");
}

template <typename T>
__global__ void ttv_prep_kernel(const int32_t* __restrict__ pos1, const int32_t* __restrict__ pos2,
                                int32_t* __restrict__ chunkF, int32_t* __restrict__ chunkS, T* __restrict__ A,
                                int64_t nA, int S, int F, int CH);

template <typename T, int VPL, bool CONTIG>
int run_mttkrp(int kid, const Args& a) {
  const Csf c = csf_of(a);
  const int64_t I = a.dims[0][0], R = a.dims[1][1];
  T* A = static_cast<T*>(a.out);
  const T* vals = static_cast<const T*>(a.vals[0]);
  const T* Cm = static_cast<const T*>(a.vals[1]);
  const T* Dm = static_cast<const T*>(a.vals[2]);
  if constexpr (std::is_same<T, float>::value && VPL == 1 && CONTIG && SPX_MTTKRP_QUARTER) {
    if (kid == SPX_K_MTTKRP_NNZ && R == 32 && c.nnz > 0 && mttkrp_quarter_ok(a)) {
      const int64_t TB = a.params[0], W = a.params[1];
      if (TB < 1 || W < 1 || TB % W != 0 || TB / W > kMaxWarps)
        return fail(SPX_E_UNSUPPORTED, "MTTKRP nnz-split needs NNZ_PER_TB a multiple of NNZ_PER_WARP, <= 16 warps");
      const int64_t Wq = W / 4, nq = ceil_div(c.nnz, Wq), nchunks = ceil_div(c.nnz, W);
      const size_t need = (size_t)2 * nq * sizeof(int32_t);
      if (!a.ws || a.ws_bytes < need) return fail(SPX_E_WORKSPACE, "workspace %zu < %zu bytes", a.ws_bytes, need);
      int32_t* chunkF = static_cast<int32_t*>(a.ws);
      int32_t* chunkS = chunkF + nq;
      const int64_t nA = I * R;
      const int64_t prep_work =
          std::max<int64_t>(std::max<int64_t>(ceil_div(c.F, 8), nA * (int64_t)sizeof(T) / 16), c.S * 32);
      const int64_t prep_grid = std::min<int64_t>(ceil_div(prep_work, 256), (int64_t)num_sms() * 8);
      // zero A and build the quarter-chunk table (fiber, slice holding each quarter chunk's first leaf)
      ttv_prep_kernel<float><<<(unsigned)prep_grid, 256, 0, a.stream>>>(c.pos1, c.pos2, chunkF, chunkS, A, nA,
                                                                         (int)c.S, (int)c.F, (int)Wq);
      count_launch();
      if (int e = check_cuda(cudaGetLastError(), "ttv_prep_kernel")) return e;
      const size_t smem = (size_t)(kQThreads / 32) * kQRing * (W % 16 == 0 ? q_slot_bytes<SPX_MQ_QB>() : kQSlotBytes);
      // 16 B leaf copies need every quarter chunk to start on a 4-leaf boundary
      auto kern = W % 16 == 0 ? mttkrp_quarter_kernel<true> : mttkrp_quarter_kernel<false>;
      static bool carve = [] {
        // the smallest shared-memory carveout that holds SPX_MQ_MINB CTAs
        // (ring + fiber windows + 1 KB reserved each): the rest stays L1 for D
        for (int al = 0; al < 2; ++al) {
          const size_t dyn = (size_t)(kQThreads / 32) * kQRing * (al ? q_slot_bytes<SPX_MQ_QB>() : kQSlotBytes);
          const size_t need = (size_t)SPX_MQ_MINB * (dyn + 4096 + 1024);
          const int pct = std::max<int>(SPX_MQ_CARVEOUT, (int)((need * 100 + 228 * 1024 - 1) / (228 * 1024)));
          cudaFuncSetAttribute(al ? mttkrp_quarter_kernel<true> : mttkrp_quarter_kernel<false>,
                               cudaFuncAttributePreferredSharedMemoryCarveout, pct);
        }
        return true;
      }();
      (void)carve;
      int per_sm = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kQThreads, smem);
      if (per_sm < 1) per_sm = 1;
      const int64_t grid = std::min<int64_t>((int64_t)num_sms() * per_sm, ceil_div(nchunks, kQThreads / 32));
      kern<<<(unsigned)grid, kQThreads, smem, a.stream>>>(
          c.crd0, c.pos1, c.crd1, c.pos2, c.crd2, vals, Cm, Dm, A, (int)c.S, (int)c.F, (int)c.nnz, (int)W,
          (int)nchunks, chunkF, chunkS, (uint32_t)(R * sizeof(float)));
      count_launch();
      return check_cuda(cudaGetLastError(), "mttkrp_quarter_kernel");
    }
  }
  if (int e = check_cuda(cudaMemsetAsync(A, 0, (size_t)(I * R) * sizeof(T), a.stream), "memset")) return e;
  if (c.nnz == 0) return SPX_OK;
  const int nw = kMttkrpThreads / 32;
  const size_t smem = (size_t)nw * LeafRing<T, kLeafRing>::kBytes;
  auto grid_for = [&](auto kern, int64_t units) -> int64_t {
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kMttkrpThreads, smem);
    if (per_sm < 1) per_sm = 1;
    return min((int64_t)num_sms() * per_sm, ceil_div(units, nw));
  };
  if (kid == SPX_K_MTTKRP_NNZ) {
    const int64_t TB = a.params[0], W = a.params[1];
    if (TB < 1 || W < 1 || TB % W != 0 || TB / W > kMaxWarps)
      return fail(SPX_E_UNSUPPORTED, "MTTKRP nnz-split needs NNZ_PER_TB a multiple of NNZ_PER_WARP, <= 16 warps");
    const int64_t nchunks = ceil_div(c.nnz, W);
    if (!a.ws || a.ws_bytes < (size_t)(nchunks + 1) * sizeof(int32_t))
      return fail(SPX_E_WORKSPACE, "workspace %zu < %zu bytes", a.ws_bytes, (size_t)(nchunks + 1) * 4);
    int32_t* first = static_cast<int32_t*>(a.ws);
    if (int e = launch_chunk_segments(c.pos2, c.F, W, nchunks, first, a.stream)) return e;
    auto kern = mttkrp_nnz_kernel<T, VPL, CONTIG>;
    kern<<<(unsigned)grid_for(kern, nchunks), kMttkrpThreads, smem, a.stream>>>(
        c.crd0, c.pos1, c.crd1, c.pos2, c.crd2, vals, Cm, Dm, A, c.S, c.F, c.nnz, R, W, nchunks, first);
    count_launch();
    return check_cuda(cudaGetLastError(), "mttkrp_nnz_kernel");
  }
  // K9: units of whole slices or leaf ranges of split slices (slice_parts_kernel);
  // params[2] == 0 (a GPU schedule's warp per slice): no slice is split
  const int64_t part = a.params[2] ? slice_part_leaves(c.nnz) : (int64_t)INT32_MAX;
  const int64_t max_units = c.S + (a.params[2] ? ceil_div(c.nnz, part) : 0);
  const size_t ps_bytes = (size_t)ceil_div((c.S + 1) * (int64_t)sizeof(int32_t), 256) * 256;
  const size_t need = ps_bytes + (size_t)max_units * (size_t)R * sizeof(T);
  if (!a.ws || a.ws_bytes < need) return fail(SPX_E_WORKSPACE, "workspace %zu < %zu bytes", a.ws_bytes, need);
  int32_t* part_start = static_cast<int32_t*>(a.ws);
  T* partial = reinterpret_cast<T*>(static_cast<char*>(a.ws) + ps_bytes);
  slice_parts_kernel<<<1, 1024, 0, a.stream>>>(c.pos1, c.pos2, c.S, part, part_start);
  count_launch();
  if (int e = check_cuda(cudaGetLastError(), "slice_parts_kernel")) return e;
  auto kern = a.params[2] ? mttkrp_slice_kernel<T, VPL, CONTIG, true> : mttkrp_slice_kernel<T, VPL, CONTIG, false>;
  kern<<<(unsigned)grid_for(kern, max_units), kMttkrpThreads, smem, a.stream>>>(
      c.crd0, c.pos1, c.crd1, c.pos2, c.crd2, vals, Cm, Dm, A, c.S, c.F, R, part_start, part, partial);
  count_launch();
  if (int e = check_cuda(cudaGetLastError(), "mttkrp_slice_kernel")) return e;
  if (max_units > c.S) {  // some slice may be split
    slice_fold_kernel<T><<<(unsigned)ceil_div(c.S * 32, 256), 256, 0, a.stream>>>(part_start, c.crd0, c.S, R,
                                                                                    partial, A);
    count_launch();
    if (int e = check_cuda(cudaGetLastError(), "slice_fold_kernel")) return e;
  }
  return SPX_OK;
}

template <typename T>
int dispatch_mttkrp(int kid, const Args& a, int64_t R) {
  const int vmax = sizeof(T) == 4 ? 8 : 4;
  int v = (int)ceil_div(R < 1 ? 1 : R, 32), vpl = 1;
  while (vpl < v) vpl <<= 1;
  if (vpl > vmax) return fail(SPX_E_UNSUPPORTED, "MTTKRP supports rank <= %d for this dtype", 32 * vmax);
  const bool contig = R == 32 * vpl;
  switch (vpl * 2 + (contig ? 1 : 0)) {
    case 2: return run_mttkrp<T, 1, false>(kid, a);
    case 3: return run_mttkrp<T, 1, true>(kid, a);
    case 4: return run_mttkrp<T, 2, false>(kid, a);
    case 5: return run_mttkrp<T, 2, true>(kid, a);
    case 8: return run_mttkrp<T, 4, false>(kid, a);
    case 9: return run_mttkrp<T, 4, true>(kid, a);
    default: break;
  }
  if constexpr (sizeof(T) == 4) {
    if (vpl == 8) return contig ? run_mttkrp<T, 8, true>(kid, a) : run_mttkrp<T, 8, false>(kid, a);
  }
  return fail(SPX_E_UNSUPPORTED, "no MTTKRP instantiation");
}

// K11 TTV nnz-split: pos over the leaves of the fused (i,j,k) space split
// into NNZ_PER_TB / NNZ_PER_WARP / NNZ_PER_THREAD chunks -- the A.2 SpMV
// shape applied to TTV.  The fibers are segments of the leaf array (pos2),
// so the Atomics segment sum of the nnz-split SpMV produces the per-fiber
// sums into a workspace vector, and one pass scatters them to A[i, j].
template <typename T>
__global__ void ttv_scatter_kernel(const int32_t* __restrict__ crd0, const int32_t* __restrict__ pos1,
                                   const int32_t* __restrict__ crd1, const T* __restrict__ fsum, T* __restrict__ A,
                                   int64_t S, int64_t F, int64_t J) {
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  int64_t lo = 0, hi = S;  // the slice of fiber f: largest s with pos1[s] <= f (SearchSegment)
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(pos1 + mid) <= f) lo = mid;
    else hi = mid;
  }
  A[(int64_t)__ldg(crd0 + lo) * J + __ldg(crd1 + f)] = fsum[f];
}


// ---------------------------------------------------------------------------
// K11 TTV nnz-split, streaming form.  The leaf level is a CSR whose rows are
// the fibers (pos2 the row pointer); A(i,j) = sum_k B(i,j,k) c(k) is a
// segmented sum over the leaf stream, and that stream (crd2 + vals, 8 B per
// fp32 leaf) is the only HBM-sized traffic, so the kernel is built to keep
// it moving with no block-wide synchronisation:
//  * the schedule's warp split (NNZ_PER_WARP = 32 * NNZ_PER_THREAD leaves) is
//    a chunk; a warp takes chunks grid-stride, a CTA's warps the NNZ_PER_TB
//    consecutive leaves of one block instance per round;
//  * a pre-pass (one launch, fully parallel, no searches) zeroes A and builds
//    the chunk table: the fiber holding each chunk's first leaf (a scatter
//    over fibers) and its slice (a scatter over slices) -- SearchSegment
//    (ir.py:178-190) for every chunk start without a dependent search;
//  * per chunk, a lane issues its NNZ_PER_THREAD coordinates and values as
//    16 B vector loads first; the fibers starting inside the chunk come from
//    one coalesced window of pos2 / crd1 (their slices advance from the
//    chunk's slice: "step: while-advance over pos boundaries")
//    and are marked in a per-warp head mask with their output offsets
//    crd0[slice]*J + crd1[f]; the next chunk's table entry is prefetched;
//  * a lane folds its leaves fiber by fiber, stores fibers that start and
//    end inside it, and one segmented warp scan joins the partials crossing
//    lanes; a fiber crossing a chunk boundary gets one red.add per chunk end
//    (the schedule's Atomics strategy on the thread loop; A zeroed first).
// ---------------------------------------------------------------------------
template <typename T>
__global__ void ttv_prep_kernel(const int32_t* __restrict__ pos1, const int32_t* __restrict__ pos2,
                                int32_t* __restrict__ chunkF, int32_t* __restrict__ chunkS, T* __restrict__ A,
                                int64_t nA, int S, int F, int CH) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gs = (int64_t)gridDim.x * blockDim.x;
  float4* A4 = reinterpret_cast<float4*>(A);
  const int64_t n4 = nA * (int64_t)sizeof(T) / 16;
  for (int64_t i = g; i < n4; i += gs) A4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t i = n4 * 16 / (int64_t)sizeof(T) + g; i < nA; i += gs) A[i] = T(0);
  // chunk starts inside fiber f (non-empty: [pos2[f], pos2[f+1])) -> chunkF;
  // eight fibers per thread, their nine pos2 entries loaded together
  for (int64_t f0 = g * 8; f0 < F; f0 += gs * 8) {
    int p[9];
#pragma unroll
    for (int u = 0; u < 9; ++u) p[u] = __ldg(pos2 + min(f0 + u, (int64_t)F));
#pragma unroll
    for (int u = 0; u < 8; ++u)
      for (int t = (p[u] + CH - 1) / CH; (int64_t)t * CH < p[u + 1]; ++t) chunkF[t] = (int)(f0 + u);
  }
  // chunk starts inside slice s (leaves [pos2[pos1[s]], pos2[pos1[s+1]])) -> chunkS;
  // one warp per slice, lanes over its chunks (a heavy slice holds thousands)
  const int lane = threadIdx.x & 31;
  for (int64_t s = g >> 5; s < S; s += gs >> 5) {
    const int a = __ldg(pos2 + __ldg(pos1 + s)), b = __ldg(pos2 + __ldg(pos1 + s + 1));
    for (int t = (a + CH - 1) / CH + lane; (int64_t)t * CH < b; t += 32) chunkS[t] = (int)s;
  }
}

// c staged in shared memory at a hashed position: the bit-skewed mode
// indices of real tensors (cfg4: P(bit)=0.3) concentrate on low-popcount
// values -- 0, 32, 64, ..., 1024 all share bank 0 in a plain layout.  The
// low five bits are XORed with a multiplicative hash of the rest (a
// permutation inside every 32-entry block).
__device__ __forceinline__ int c_slot(int k) { return k ^ (int)(((unsigned)(k >> 5) * 0x9E3779B1u) >> 27); }

__device__ __forceinline__ int ld_i32_early(const int32_t* p) {
  int r;  // volatile: issued where written (a prefetch for the next loop trip), not sunk to its use
  asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}

#ifndef SPX_TTV_PREFETCH
#define SPX_TTV_PREFETCH 0
#endif
#ifdef SPX_TTV_MAXNREG
#define SPX_TTV_BOUNDS __maxnreg__(SPX_TTV_MAXNREG)
#else
#define SPX_TTV_BOUNDS __launch_bounds__(512)
#endif
// DET (params[3] = 1, serial TTV): the lead and the open carry of a chunk go
// to per-chunk slots that ttv_slot_fold_kernel adds in chunk order
// (bit-identical repeats, cfg4 0.187 ms); !DET (K11 as scheduled, the
// thread loop's Atomics): red.add into the zeroed A (0.177 ms).
template <typename T, int LPT, typename OffT, bool DET>
__global__ void SPX_TTV_BOUNDS ttv_stream_kernel(
    const int32_t* __restrict__ crd0, const int32_t* __restrict__ pos1, const int32_t* __restrict__ crd1,
    const int32_t* __restrict__ pos2, const int32_t* __restrict__ crd2, const T* __restrict__ vals,
    const T* __restrict__ c, const int32_t* __restrict__ chunkF, const int32_t* __restrict__ chunkS,
    T* __restrict__ A, int S, int F, int nnz, int64_t J, int K, int nchunks, int csmem,
    int64_t* __restrict__ lead_off, T* __restrict__ lead_val, int64_t* __restrict__ carry_off,
    T* __restrict__ carry_val) {
  static_assert(LPT % 4 == 0 && LPT <= 16, "rows of 4 or 8 leaves per lane");
  constexpr int CH = 32 * LPT;          // leaves per warp chunk
  constexpr int RL = LPT >= 8 ? 8 : 4;  // consecutive leaves per lane in a row
  constexpr int ROWS = LPT / RL;        // a chunk is ROWS rows of 32*RL leaves
  constexpr int RW = 32 * RL;           // leaves per row
  constexpr int RMASK = (1 << RL) - 1;
  extern __shared__ __align__(16) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  // layout: per warp { offp[CH] (OffT), mask[32] } | c[K] (when staged)
  constexpr int kWarpBytes = CH * (int)sizeof(OffT) + 32 * 4;
  OffT* offp = reinterpret_cast<OffT*>(sm + (size_t)warp * kWarpBytes);
  unsigned* mask = reinterpret_cast<unsigned*>(sm + (size_t)warp * kWarpBytes + CH * sizeof(OffT));
  T* sc = reinterpret_cast<T*>(sm + (size_t)wpc * kWarpBytes);
  if (csmem) {
    for (int k = threadIdx.x; k < K; k += blockDim.x) sc[c_slot(k)] = __ldg(c + k);
    __syncthreads();
  }
  const uint64_t pol = l2_evict_first();
  const unsigned lt = (1u << lane) - 1u;  // lanes below mine
  const int stride = gridDim.x * wpc;
  int chunk = blockIdx.x * wpc + warp;
  int fi = chunk < nchunks ? __ldg(chunkF + chunk) : 0, si = chunk < nchunks ? __ldg(chunkS + chunk) : 0;
  for (; chunk < nchunks; chunk += stride) {
    const int p0 = chunk * CH, p1 = min(p0 + CH, nnz);
    // the first window of fibers that may start in the chunk and the chunk's
    // slice: one L2 round trip, issued first
    int f = fi + 1 + lane;
    int q = f < F ? __ldg(pos2 + f) : INT_MAX;
    int qn = f < F ? __ldg(pos2 + f + 1) : INT_MAX;
    int kf = f < F ? __ldg(crd1 + f) : 0;
    const int i_in = __ldg(crd0 + si), send_in = __ldg(pos1 + si + 1);
    const OffT off_in = (OffT)i_in * (OffT)J + (OffT)__ldg(crd1 + fi);
    // the next chunk's table entry (issued now, used next trip)
    const int nxt = min(chunk + stride, nchunks - 1);
    const int fi_n = ld_i32_early(chunkF + nxt), si_n = ld_i32_early(chunkS + nxt);
    // row h, lane L: leaves p0 + RW*h + RL*L + e (e < RL) -- every warp load
    // is one coalesced run (32 B per lane for RL = 8)
    int kk[LPT];
    T v[LPT];
    if (p0 + CH <= p1) {
#pragma unroll
      for (int h = 0; h < ROWS; ++h) {
        const int qq = p0 + RW * h + RL * lane;
        if constexpr (RL == 8) {
          ld256_i32_hint(crd2 + qq, kk + 8 * h, pol);
          ld256_nc_hint(vals + qq, v + 8 * h, pol);
          if constexpr (sizeof(T) == 8) ld256_nc_hint(vals + qq + 4, v + 8 * h + 4, pol);
        } else {
          const int4 k4 = ld_i4_hint(crd2 + qq, pol);
          kk[4 * h] = k4.x;
          kk[4 * h + 1] = k4.y;
          kk[4 * h + 2] = k4.z;
          kk[4 * h + 3] = k4.w;
          if constexpr (sizeof(T) == 4) unpack16<T>(v + 4 * h, ld_f4_hint(vals + qq, pol));
          else ld256_nc_hint(vals + qq, v + 4 * h, pol);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < LPT; ++j) {
        const int qq = p0 + RW * (j / RL) + RL * lane + (j % RL);
        const bool in = qq < p1;
        kk[j] = in ? __ldg(crd2 + qq) : 0;
        v[j] = in ? __ldg(vals + qq) : T(0);
      }
    }
    if (SPX_TTV_PREFETCH && lane == 0 && chunk + stride < nchunks) {
      const int pn = nxt * CH, nb = min(CH, nnz - pn);
      bulk_prefetch_l2(crd2 + pn, (uint32_t)(((nb * 4) + 15) & ~15));
      bulk_prefetch_l2(vals + pn, (uint32_t)(((nb * (int)sizeof(T)) + 15) & ~15));
    }
    mask[lane] = 0u;
    __syncwarp();
    // non-empty fibers starting in (p0, p1) become heads: bit RL*h + e of lane L's word
    while (true) {
      if (q < p1 && qn > q) {
        // output offset crd0[slice]*J + crd1[f]; the slice advances from the
        // chunk's ("step: while-advance over pos boundaries")
        int isl = i_in;
        if (send_in <= f) isl = __ldg(crd0 + search_segment(pos1, si + 1, S, f));
        const int d = q - p0;
        offp[d] = (OffT)isl * (OffT)J + (OffT)kf;
        atomicOr(mask + (d % RW) / RL, 1u << ((d / RW) * RL + d % RL));
      }
      if (__shfl_sync(kFull, q, 31) >= p1) break;
      f += 32;  // more than 32 fibers start in this chunk: the next window
      q = f < F ? __ldg(pos2 + f) : INT_MAX;
      qn = f < F ? __ldg(pos2 + f + 1) : INT_MAX;
      kf = f < F ? __ldg(crd1 + f) : 0;
    }
    __syncwarp();
    const unsigned hball = mask[lane];
    OffT open_off = off_in;  // fiber open at the end of the previous row
    bool started = false;    // has a fiber started in this chunk yet (warp-uniform)
    T carry = T(0);          // its partial so far in this chunk
    int64_t my_lead_off = -1;  // the fiber open before the chunk, closed by my first start
    T my_lead = T(0);
#pragma unroll
    for (int h = 0; h < ROWS; ++h) {
      const unsigned hb = (hball >> (RL * h)) & RMASK;
      const unsigned rowheads = __ballot_sync(kFull, hb != 0u);
      // the fiber open before my first leaf of this row: the last head in a
      // lower lane of the row, else the one open at the previous row's end
      const int dlast = hb ? RW * h + RL * lane + (31 - __clz(hb)) : 0;
      const unsigned below = rowheads & lt;
      const int dsrc = __shfl_sync(kFull, dlast, below ? 31 - __clz(below) : 0);
      OffT cur = below ? offp[dsrc] : open_off;
      const OffT first_off = cur;
      T acc = T(0), lead = T(0);
      bool seen = false, lead_empty = false;
#pragma unroll
      for (int e = 0; e < RL; ++e) {
        const int j = RL * h + e;
        const T x = v[j] * (csmem ? sc[c_slot(kk[j])] : __ldg(c + kk[j]));
        if ((hb >> e) & 1u) {  // a fiber starts here (Track: advance to it)
          if (!seen) {
            lead = acc;
            lead_empty = e == 0;
            seen = true;
          } else {
            A[cur] = acc;  // started and ended inside this lane's run
          }
          cur = offp[RW * h + RL * lane + e];
          acc = T(0);
        }
        acc += x;
      }
      // segmented inclusive scan of the partial leaving each lane; the
      // previous rows' open partial enters at lane 0
      T sv = (lane == 0 && !seen) ? acc + carry : acc;
      const int seg = 31 - __clz((rowheads | 1u) & (0xffffffffu >> (31 - lane)));
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const T y = __shfl_up_sync(kFull, sv, o);
        if (lane - o >= seg) sv += y;
      }
      T in = __shfl_up_sync(kFull, sv, 1);  // open partial arriving at my first leaf
      if (lane == 0) in = carry;
      if (seen) {  // my first start closes the fiber open before it
        if (started || below) {
          A[first_off] = in + lead;  // it started inside this chunk
        } else if (!(h == 0 && lane == 0 && lead_empty)) {
          if constexpr (DET) {
            my_lead_off = (int64_t)first_off;  // it started before: the chunk's lead slot
            my_lead = in + lead;
          } else {
            atomicAdd(A + first_off, in + lead);
          }
        }
      }
      carry = __shfl_sync(kFull, sv, 31);
      open_off = __shfl_sync(kFull, cur, 31);
      started = started || rowheads != 0u;
    }
    // the lead (at most one lane) and the fiber open at the chunk's end go to
    // the chunk's slots; ttv_slot_fold_kernel adds them in chunk order
    if constexpr (DET) {
      const unsigned lb = __ballot_sync(kFull, my_lead_off >= 0);
      const int ls = lb ? __ffs(lb) - 1 : 0;
      const int64_t lo = __shfl_sync(kFull, my_lead_off, ls);
      const T lv = __shfl_sync(kFull, my_lead, ls);
      if (lane == 0) {
        lead_off[chunk] = lb ? lo : -1;
        lead_val[chunk] = lv;
        carry_off[chunk] = (int64_t)open_off;
        carry_val[chunk] = carry;
      }
    } else if (lane == 0) {
      atomicAdd(A + open_off, carry);  // the fiber open at the chunk's end continues past it
    }
    fi = fi_n;
    si = si_n;
    __syncwarp();
  }
}

struct TtvNnzLayout {
  size_t fsum, first, total;
  int64_t nslots;
};
TtvNnzLayout ttv_nnz_layout(const Args& a) {
  const int64_t F = a.level_sizes[1], nnz = a.level_sizes[2];
  const int64_t TB = a.params[0] > 0 ? a.params[0] : 1;
  const int64_t W = a.params[1] > 0 ? a.params[1] : TB;
  const size_t es = a.dtype == SPX_F32 ? 4 : 8;
  TtvNnzLayout L;
  L.nslots = (nnz == 0 ? 1 : ceil_div(nnz, TB)) * (TB / W > 0 ? TB / W : 1);
  L.fsum = 0;
  L.first = ((size_t)(F > 0 ? F : 1) * es + 255) & ~(size_t)255;
  L.total = L.first + (size_t)(L.nslots + 1) * sizeof(int32_t);
  return L;
}


// A fiber that spans chunks c..m: chunk c's open carry, the whole-chunk
// carries of c+1..m-1 and chunk m's lead, added in chunk order by the thread
// of the chunk where it starts (deterministic: the schedule's Atomics
// strategy without atomics, like the SpMM carry fix-up).
template <typename T>
__global__ void ttv_slot_fold_kernel(const int64_t* __restrict__ lead_off, const T* __restrict__ lead_val,
                                     const int64_t* __restrict__ carry_off, const T* __restrict__ carry_val,
                                     int64_t nchunks, T* __restrict__ A) {
  const int64_t ch = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (ch >= nchunks) return;
  // a lead whose fiber starts exactly at this chunk's first leaf (it is no
  // earlier chunk's carry) is the whole fiber
  const int64_t lf = lead_off[ch];
  if (lf >= 0 && (ch == 0 || carry_off[ch - 1] != lf)) A[lf] = lead_val[ch];
  const int64_t f = carry_off[ch];
  if (ch > 0 && carry_off[ch - 1] == f) return;  // started in an earlier chunk
  T sum = carry_val[ch];
  int64_t m = ch + 1;
  for (; m < nchunks && carry_off[m] == f; ++m) sum += carry_val[m];
  if (m < nchunks && lead_off[m] == f) sum += lead_val[m];
  A[f] = sum;
}

template <typename T, int LPT, typename OffT>
int launch_ttv_stream(const Args& a, const Csf& c, int64_t TB) {
  const int64_t I = a.dims[0][0], J = a.dims[0][1], K = a.dims[0][2];
  constexpr int CH = 32 * LPT;
  const int threads = (int)(TB / LPT);
  const int wpc = threads / 32;
  const int csmem = (size_t)K * sizeof(T) <= 16384 ? 1 : 0;
  const size_t smem = (size_t)wpc * (CH * sizeof(OffT) + 128) + (csmem ? (size_t)K * sizeof(T) : 0);
  const int64_t nchunks = ceil_div(c.nnz, CH);
  const size_t tab = ((size_t)2 * nchunks * sizeof(int32_t) + 255) & ~(size_t)255;
  const size_t need = tab + (size_t)nchunks * 2 * (sizeof(int64_t) + sizeof(T));
  if (!a.ws || a.ws_bytes < need) return fail(SPX_E_WORKSPACE, "workspace %zu < %zu bytes", a.ws_bytes, need);
  int32_t* chunkF = static_cast<int32_t*>(a.ws);
  int32_t* chunkS = chunkF + nchunks;
  int64_t* lead_off = reinterpret_cast<int64_t*>(static_cast<char*>(a.ws) + tab);
  int64_t* carry_off = lead_off + nchunks;
  T* lead_val = reinterpret_cast<T*>(carry_off + nchunks);
  T* carry_val = lead_val + nchunks;
  T* A = static_cast<T*>(a.out);
  const int64_t nA = I * J;
  const int64_t prep_work = std::max<int64_t>(std::max<int64_t>(ceil_div(c.F, 8), nA * (int64_t)sizeof(T) / 16),
                                              c.S * 32);
  const int64_t prep_grid = std::min<int64_t>(ceil_div(prep_work, 256), (int64_t)num_sms() * 8);
  ttv_prep_kernel<T><<<(unsigned)prep_grid, 256, 0, a.stream>>>(c.pos1, c.pos2, chunkF, chunkS, A, nA, (int)c.S,
                                                                 (int)c.F, CH);
  count_launch();
  if (int e = check_cuda(cudaGetLastError(), "ttv_prep_kernel")) return e;
  const bool det = a.params[3] != 0;
  auto kern = det ? ttv_stream_kernel<T, LPT, OffT, true> : ttv_stream_kernel<T, LPT, OffT, false>;
  static thread_local size_t attr_set[2] = {0, 0};  // per kernel variant (DET / atomics)
  if (smem > 32 * 1024 && smem > attr_set[det]) {
    if (int e = check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                           "smem attribute"))
      return e;
    attr_set[det] = smem;
  }
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t grid = std::min<int64_t>((int64_t)num_sms() * per_sm, ceil_div(nchunks, wpc));
  kern<<<(unsigned)grid, (unsigned)threads, smem, a.stream>>>(
      c.crd0, c.pos1, c.crd1, c.pos2, c.crd2, static_cast<const T*>(a.vals[0]), static_cast<const T*>(a.vals[1]),
      chunkF, chunkS, A, (int)c.S, (int)c.F, (int)c.nnz, J, (int)K, (int)nchunks, csmem, lead_off, lead_val,
      carry_off, carry_val);
  count_launch();
  if (int e = check_cuda(cudaGetLastError(), "ttv_stream_kernel")) return e;
  if (!det) return SPX_OK;
  ttv_slot_fold_kernel<T><<<(unsigned)ceil_div(nchunks, 256), 256, 0, a.stream>>>(lead_off, lead_val, carry_off,
                                                                                  carry_val, nchunks, A);
  count_launch();
  return check_cuda(cudaGetLastError(), "ttv_slot_fold_kernel");
}

template <typename T>
int run_ttv_stream(const Args& a, const Csf& c, int64_t TB, int TPT) {
  const bool off32 = a.dims[0][0] * a.dims[0][1] < (int64_t)INT32_MAX;
  switch (TPT * 2 + (off32 ? 1 : 0)) {
    case 9: return launch_ttv_stream<T, 4, int32_t>(a, c, TB);
    case 8: return launch_ttv_stream<T, 4, int64_t>(a, c, TB);
    case 17: return launch_ttv_stream<T, 8, int32_t>(a, c, TB);
    case 16: return launch_ttv_stream<T, 8, int64_t>(a, c, TB);
    case 33: return launch_ttv_stream<T, 16, int32_t>(a, c, TB);
    default: return launch_ttv_stream<T, 16, int64_t>(a, c, TB);
  }
}

template <typename T>
int run_ttv_nnz(const Args& a) {
  const Csf c = csf_of(a);
  const int64_t I = a.dims[0][0], J = a.dims[0][1];
  T* A = static_cast<T*>(a.out);
  const int64_t TB = a.params[0], W = a.params[1], TPT = a.params[2];
  if (c.nnz > 0 && (TPT == 4 || TPT == 8 || TPT == 16) && W == 32 * TPT && TB % W == 0 && TB / TPT <= kMaxThreads)
    return run_ttv_stream<T>(a, c, TB, (int)TPT);  // zeroes A itself
  if (int e = check_cuda(cudaMemsetAsync(A, 0, (size_t)(I * J) * sizeof(T), a.stream), "memset")) return e;
  if (c.nnz == 0) return SPX_OK;
  if (TB < 1 || W < 1 || TPT < 1 || W != 32 * TPT || TB % W != 0 || TB / TPT > kMaxThreads)
    return fail(SPX_E_UNSUPPORTED,
                "TTV nnz-split needs NNZ_PER_WARP == 32*NNZ_PER_THREAD and NNZ_PER_TB a multiple of "
                "NNZ_PER_WARP with <= 512 threads (got %lld, %lld, %lld)",
                (long long)TB, (long long)W, (long long)TPT);
  const TtvNnzLayout L = ttv_nnz_layout(a);
  if (!a.ws || a.ws_bytes < L.total) return fail(SPX_E_WORKSPACE, "workspace %zu < %zu bytes", a.ws_bytes, L.total);
  T* fsum = reinterpret_cast<T*>(static_cast<char*>(a.ws) + L.fsum);
  int32_t* first = reinterpret_cast<int32_t*>(static_cast<char*>(a.ws) + L.first);
  if (int e = check_cuda(cudaMemsetAsync(fsum, 0, (size_t)c.F * sizeof(T), a.stream), "memset")) return e;
  if (int e = launch_chunk_segments(c.pos2, c.F, W, L.nslots, first, a.stream)) return e;
  const T* vals = static_cast<const T*>(a.vals[0]);
  const T* cv = static_cast<const T*>(a.vals[1]);
  int e;
  if constexpr (sizeof(T) == 4) e = segsum_atomic_f32(c.pos2, c.crd2, vals, cv, fsum, c.F, c.nnz, TB, W, TPT, first, a.stream, a.dims[0][2]);
  else e = segsum_atomic_f64(c.pos2, c.crd2, vals, cv, fsum, c.F, c.nnz, TB, W, TPT, first, a.stream, a.dims[0][2]);
  if (e) return e;
  ttv_scatter_kernel<T><<<(unsigned)ceil_div(c.F, 256), 256, 0, a.stream>>>(c.crd0, c.pos1, c.crd1, fsum, A, c.S,
                                                                          c.F, J);
  count_launch();
  return check_cuda(cudaGetLastError(), "ttv_scatter_kernel");
}

}  // namespace

size_t ws_csf(int kid, const Args& a) {
  if (kid == SPX_K_TTV_NNZ) {
    const int tpt = a.params[2];
    if (tpt == 4 || tpt == 8 || tpt == 16) {  // the streaming form: chunk table (fiber, slice) + lead / carry slots
      const size_t nch = (size_t)ceil_div(a.level_sizes[2] > 0 ? a.level_sizes[2] : 1, 32 * tpt);
      const size_t es = a.dtype == SPX_F32 ? 4 : 8;
      return ((2 * nch * sizeof(int32_t) + 255) & ~(size_t)255) + nch * 2 * (sizeof(int64_t) + es);
    }
    return ttv_nnz_layout(a).total;
  }
  if (kid == SPX_K_MTTKRP_SLICE) {  // unit table + partial rows of split slices
    const int64_t S = a.level_sizes[0], nnz = a.level_sizes[2], R = a.dims[1][1];
    if (nnz <= 0) return 0;
    const size_t es = a.dtype == SPX_F32 ? 4 : 8;
    const int64_t units = S + (a.params[2] ? ceil_div(nnz, slice_part_leaves(nnz)) : 0);
    return (size_t)ceil_div((S + 1) * 4, 256) * 256 + (size_t)units * (size_t)R * es;
  }
  if (kid != SPX_K_MTTKRP_NNZ) return 0;
  const int64_t nnz = a.level_sizes[2];
  const int64_t W = a.params[1] > 0 ? a.params[1] : 1;
  size_t ws = (size_t)(ceil_div(nnz, W) + 1) * sizeof(int32_t);
  if (mttkrp_quarter_ok(a)) ws = std::max(ws, (size_t)2 * (size_t)ceil_div(nnz > 0 ? nnz : 1, W / 4) * sizeof(int32_t));
  return ws;
}

int launch_csf(int kid, const Args& a) {
  if (kid == SPX_K_TTV_FIBER || kid == SPX_K_TTV_NNZ) {
    if (a.dims[1][0] != a.dims[0][2])
      return fail(SPX_E_ARG, "TTV: B's third dimension %lld != length of c %lld", (long long)a.dims[0][2],
                  (long long)a.dims[1][0]);
    if (kid == SPX_K_TTV_NNZ) return a.dtype == SPX_F32 ? run_ttv_nnz<float>(a) : run_ttv_nnz<double>(a);
    return a.dtype == SPX_F32 ? run_ttv<float>(a) : run_ttv<double>(a);
  }
  const int64_t R = a.dims[1][1];
  if (a.dims[1][0] != a.dims[0][1] || a.dims[2][0] != a.dims[0][2] || a.dims[2][1] != R)
    return fail(SPX_E_ARG, "MTTKRP: operand shapes disagree");
  if (kid == SPX_K_MTTKRP_NNZ) {
    const int ws = a.params[2] ? a.params[2] : 32;
    if (ws != 32) return fail(SPX_E_UNSUPPORTED, "split of j must be WARP_SIZE=32");
    if (a.params[3] != 0 && (int64_t)a.params[3] != ceil_div(R, 32))
      return fail(SPX_E_CONTRACT, "MaxExact bound violated: bound %d but ceil(%lld/32) = %lld", a.params[3],
                  (long long)R, (long long)ceil_div(R, 32));
  }
  return a.dtype == SPX_F32 ? dispatch_mttkrp<float>(kid, a, R) : dispatch_mttkrp<double>(kid, a, R);
}

}  // namespace spx
