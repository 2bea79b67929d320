// SDDMM kernels: A(i,j) = B(i,j) * C(i,k) * D(j,k) with B in CSR ("ds") and
// C (M x K), D (N x K) dense row-major.  The result lives on B's pattern:
// out[p] = B_vals[p] * <C[i,:], D[crd[p],:]>  (nnz-aligned, the sparse-output
// extension of SURVEY.md §0.6 / §8(f) row 4); params[7]=1 scatters it into a
// dense M x N output instead (the reference's dense-output semantics,
// notation.py:156).
//
//  K6 SPX_K_SDDMM_NNZ: fuse(i,j,f) pos(f,fpos,B) split(fpos,block,..,NNZ_PER_TB)
//     split(..,warp,nnz,NNZ_PER_WARP) split(k,dvu,thread,32)
//     bound(dvu,dense_val,ceil(K/32),MaxExact), thread:Temporary.
//     A warp walks NNZ_PER_WARP positions; lanes cover k; each group of eight
//     dot products is folded with an eight-wide transpose-reduction and lane t
//     ends with nonzero t's value, so the store is coalesced.  Each position
//     writes its own output: no races, no carries.
//  K10 SPX_K_SDDMM_ROW: warp per row (row-split / unscheduled shapes), the
//     same batch pipeline one row at a time.
#include "spx_common.cuh"

// tuning knob: 3 CTAs/SM forces 40 registers and spills 48-280 B per thread
#ifndef SPX_SDDMM_ROW_MINB
#define SPX_SDDMM_ROW_MINB 1  // the heaviest row is latency-bound: more rows in flight beat occupancy
#endif
#ifndef SPX_SDDMM_ROW_UR
#define SPX_SDDMM_ROW_UR 4   // cfg3 K10: 7.8 ms (2 rows, 2 CTAs/SM) -> 5.7 ms
#endif
#ifndef SPX_SDDMM_ROW_PF
#define SPX_SDDMM_ROW_PF 1  // next-batch L1 prefetch of D rows in K10's row walk (cfg3 5.42 -> 4.67 ms)
#endif
#ifndef SPX_SDDMM_UN
#define SPX_SDDMM_UN 2  // D rows (1 KB) in flight per warp; 4 spills at 64 registers (cfg3 1.68 vs 1.57 ms)
#endif
#ifndef SPX_SDDMM_MINB
#define SPX_SDDMM_MINB 2
#endif

namespace spx {
namespace {

template <typename T, int VPL, bool CONTIG>
__device__ __forceinline__ T dot(const Frag<T, VPL, CONTIG>& a, const Frag<T, VPL, CONTIG>& b) {
  T s = T(0);
#pragma unroll
  for (int i = 0; i < VPL; ++i) s += a.v[i] * b.v[i];
  return s;
}

template <typename T>
__device__ __forceinline__ void emit(T* __restrict__ out, bool dense, int64_t N, int64_t p, int64_t r, int32_t c,
                                     T val) {
  if (dense) out[r * N + c] = val;
  else __stcs(out + p, val);
}

// part[i] (i < 8) on every lane -> lanes with (lane & 3) == 0 hold the sum
// over all lanes of part[lane >> 2]: 3 halving exchange steps + 2 folds.
template <typename T>
__device__ __forceinline__ T transpose_reduce8(T (&part)[8], int lane) {
#pragma unroll
  for (int o = 16, h = 4; o >= 4; o >>= 1, h >>= 1) {
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const T send = upper ? part[i] : part[i + h];
      const T keep = upper ? part[i + h] : part[i];
      part[i] = keep + __shfl_xor_sync(kFull, send, o);
    }
  }
  T v = part[0];
  v += __shfl_xor_sync(kFull, v, 2);
  v += __shfl_xor_sync(kFull, v, 1);
  return v;
}

// K6: warp chunk q covers positions [q*W, q*W+W).  The (column, value) pairs
// stream through a per-warp cp.async ring; the warp takes the chunk eight
// positions at a time: U rows of D in flight, each dotted with the current
// C row (held in registers while the row lasts), the eight partial dot
// products folded by transpose_reduce8, and the 32 results of a batch
// stored coalesced by the lanes that own them.
template <typename T, int VPL, bool CONTIG, int U>
__global__ void __launch_bounds__(kMaxThreads, SPX_SDDMM_MINB) sddmm_nnz_kernel(const int32_t* __restrict__ pos,
                                                            const int32_t* __restrict__ crd,
                                                            const T* __restrict__ vals, const T* __restrict__ Cm,
                                                            const T* __restrict__ Dm, T* __restrict__ out, int64_t M,
                                                            int64_t N, int64_t K, int64_t nnz, int64_t W,
                                                            int wpc, bool dense, const int32_t* __restrict__ first) {
  using F = Frag<T, VPL, CONTIG>;
  using Ring = LeafRing<T, 4>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = (int)blockIdx.x * wpc + warp;
  const int q0 = (int)((int64_t)q * W);
  const int q1 = (int)min((int64_t)q0 + W, nnz);
  if (q0 >= q1) return;
  const int ncols = (int)K;
  const uint64_t pol_s = l2_evict_first();
  int64_t r = __ldg(first + q);  // row holding q0 (chunk_segments_kernel)
  RowEndCache ends;
  ends.fill(pos, r, M, lane);
  int rend = (int)ends.end(pos, r, M, lane);
  F crow;
  crow.load(Cm + r * K, lane, ncols);
  const char* __restrict__ Dl = reinterpret_cast<const char*>(Dm + (CONTIG ? lane * VPL : lane));
  const uint32_t rowb = (uint32_t)(K * (int64_t)sizeof(T));
  auto drow = [&](F& d, int c) {
    const T* src = reinterpret_cast<const T*>(addr_wide(Dl, (uint32_t)c, rowb));
    if constexpr (CONTIG) {
      d.load_ptr(src);
    } else {
#pragma unroll
      for (int i = 0; i < VPL; ++i) d.v[i] = (i * 32 + lane < ncols) ? __ldg(src + i * 32) : T(0);
    }
  };
  Ring ring;
  ring.init(smem_raw + (size_t)warp * Ring::kBytes, crd, vals, q0, q1);
  ring.prologue(lane, pol_s);
  for (int b = 0; b < ring.nb; ++b) {
    ring.acquire(b, lane, pol_s);
    const int p = q0 + b * 32;
    const int n = min(32, q1 - p);
    const int32_t* Cs = ring.crd_slot(b);
    const T* Vs = ring.val_slot(b);
    T res = T(0);
    int64_t myr = r;  // row of position p + lane (dense scatter)
#pragma unroll 1
    for (int g = 0; g < 4 && g * 8 < n; ++g) {
      T part[8];
#pragma unroll
      for (int u0 = 0; u0 < 8; u0 += U) {
        F d[U];
#pragma unroll
        for (int uu = 0; uu < U; ++uu) drow(d[uu], Cs[g * 8 + u0 + uu]);  // zero-filled past n
#pragma unroll
        for (int uu = 0; uu < U; ++uu) {
          const int t = g * 8 + u0 + uu;
          if (t < n) {
            if (p + t >= rend) {
              do {
                ++r;
                rend = (int)ends.end(pos, r, M, lane);
              } while (p + t >= rend);
              crow.load(Cm + r * K, lane, ncols);
            }
            if (lane == t) myr = r;
            part[u0 + uu] = dot(crow, d[uu]);
          } else {
            part[u0 + uu] = T(0);
          }
        }
      }
      const T sum = transpose_reduce8(part, lane);
      const T got = __shfl_sync(kFull, sum, (lane & 7) * 4);
      if ((lane >> 3) == g) res = got;
    }
    if (lane < n) emit(out, dense, N, (int64_t)p + lane, myr, Cs[lane], Vs[lane] * res);
    ring.release();
  }
}

// K10 warp-per-row: the same batch pipeline as K6 over one row at a time
// (C row loaded once per row, (column, value) pairs on the warp's LeafRing,
// eight dot products per transpose_reduce8, coalesced stores).
template <typename T, int VPL, bool CONTIG, int U>
__global__ void __launch_bounds__(kMaxThreads, SPX_SDDMM_ROW_MINB) sddmm_row_kernel(const int32_t* __restrict__ pos,
                                                            const int32_t* __restrict__ crd,
                                                            const T* __restrict__ vals, const T* __restrict__ Cm,
                                                            const T* __restrict__ Dm, T* __restrict__ out, int64_t M,
                                                            int64_t N, int64_t K, int64_t R, bool dense) {
  using F = Frag<T, VPL, CONTIG>;
  using Ring = LeafRing<T, 4>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nw = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncols = (int)K;
  const uint64_t pol_s = l2_evict_first();
  const char* __restrict__ Dl = reinterpret_cast<const char*>(Dm + (CONTIG ? lane * VPL : lane));
  const uint32_t rowb = (uint32_t)(K * (int64_t)sizeof(T));
  const int64_t lo = (int64_t)blockIdx.x * R;
  const int nwr = (int)((R + nw - 1) / nw);
  for (int wr = 0; wr < nwr; ++wr) {
    const int64_t br = (int64_t)wr * nw + warp;
    if (br >= R) break;
    const int64_t r = lo + br;
    if (r >= M) break;
    const int a = __ldg(pos + r), e = __ldg(pos + r + 1);
    if (a == e) continue;
    F crow;
    crow.load(Cm + r * K, lane, ncols);
    Ring ring;
    ring.init(smem_raw + (size_t)warp * Ring::kBytes, crd, vals, a, e);
    ring.prologue(lane, pol_s);
    for (int b = 0; b < ring.nb; ++b) {
#if SPX_SDDMM_ROW_PF
      // batches b and b+1 landed: batch b+1's D rows start moving into L1
      // (a lane per leaf, one prefetch per 128 B line) -- the warp alone on
      // the heaviest row is latency-bound on these gathers
      ring.issue(b + 3, lane, pol_s);
      cp_async_wait<2>();
      __syncwarp();
      if (b + 1 < ring.nb && a + (b + 1) * 32 + lane < e) {
        const char* rp = reinterpret_cast<const char*>(Dm) + (size_t)(uint32_t)ring.crd_slot(b + 1)[lane] * rowb;
        for (uint32_t l = 0; l < rowb; l += 128) asm volatile("prefetch.global.L1 [%0];" ::"l"(rp + l));
      }
#else
      ring.acquire(b, lane, pol_s);
#endif
      const int p = a + b * 32;
      const int n = min(32, e - p);
      const int32_t* Cs = ring.crd_slot(b);
      const T* Vs = ring.val_slot(b);
      T res = T(0);
#pragma unroll 1
      for (int g = 0; g < 4 && g * 8 < n; ++g) {
        T part[8];
#pragma unroll
        for (int u0 = 0; u0 < 8; u0 += U) {
          F d[U];
#pragma unroll
          for (int uu = 0; uu < U; ++uu) {
            const T* src = reinterpret_cast<const T*>(addr_wide(Dl, (uint32_t)Cs[g * 8 + u0 + uu], rowb));
            if constexpr (CONTIG) {
              d[uu].load_ptr(src);
            } else {
#pragma unroll
              for (int i = 0; i < VPL; ++i) d[uu].v[i] = (i * 32 + lane < ncols) ? __ldg(src + i * 32) : T(0);
            }
          }
#pragma unroll
          for (int uu = 0; uu < U; ++uu) part[u0 + uu] = (g * 8 + u0 + uu < n) ? dot(crow, d[uu]) : T(0);
        }
        const T sum = transpose_reduce8(part, lane);
        const T got = __shfl_sync(kFull, sum, (lane & 7) * 4);
        if ((lane >> 3) == g) res = got;
      }
      if (lane < n) emit(out, dense, N, (int64_t)p + lane, r, Cs[lane], Vs[lane] * res);
      ring.release();
    }
  }
}

template <typename T, int VPL, bool CONTIG>
int run_sddmm(int kid, const Args& a) {
  const int32_t* pos = a.pos[0];
  const int32_t* crd = a.crd[0];
  const T* vals = static_cast<const T*>(a.vals[0]);
  const T* Cm = static_cast<const T*>(a.vals[1]);
  const T* Dm = static_cast<const T*>(a.vals[2]);
  T* out = static_cast<T*>(a.out);
  const int64_t M = a.dims[0][0], N = a.dims[0][1], K = a.dims[1][1];
  const int64_t nnz = a.level_sizes[1];
  const bool dense = a.params[7] != 0;
  if (dense) {
    if (int e = check_cuda(cudaMemsetAsync(out, 0, (size_t)(M * N) * sizeof(T), a.stream), "memset")) return e;
  }
  if (M == 0 || nnz == 0) return SPX_OK;
  if (kid == SPX_K_SDDMM_NNZ) {
    const int64_t TB = a.params[0], W = a.params[1];
    if (TB < 1 || W < 1 || TB % W != 0 || TB / W > kMaxWarps)
      return fail(SPX_E_UNSUPPORTED, "SDDMM nnz-split needs NNZ_PER_TB a multiple of NNZ_PER_WARP, <= 16 warps");
    const int64_t wpc = TB / W, ncta = ceil_div(nnz, TB), nchunks = ncta * wpc;
    if (!a.ws || a.ws_bytes < (size_t)(nchunks + 1) * sizeof(int32_t))
      return fail(SPX_E_WORKSPACE, "workspace %zu < %zu bytes", a.ws_bytes, (size_t)(nchunks + 1) * 4);
    int32_t* first = static_cast<int32_t*>(a.ws);
    if (int e = launch_chunk_segments(pos, M, W, nchunks, first, a.stream)) return e;
    constexpr int UN = VPL * (int)sizeof(T) >= 32 ? SPX_SDDMM_UN : 4;  // D rows in flight per warp
    sddmm_nnz_kernel<T, VPL, CONTIG, UN><<<(unsigned)ncta, (unsigned)(wpc * 32), wpc * LeafRing<T, 4>::kBytes,
                                           a.stream>>>(pos, crd, vals, Cm, Dm, out, M, N, K, nnz, W, (int)wpc,
                                                       dense, first);
    count_launch();
    return check_cuda(cudaGetLastError(), "sddmm_nnz_kernel");
  }
  const int64_t R = a.params[0] > 0 ? a.params[0] : 8;
  int64_t nw = a.params[1] > 0 ? a.params[1] : (R < 8 ? R : 8);
  if (nw > kMaxWarps) nw = kMaxWarps;
  constexpr int UR = VPL * (int)sizeof(T) >= 32 ? SPX_SDDMM_ROW_UR : 4;  // D rows in flight per warp
  sddmm_row_kernel<T, VPL, CONTIG, UR><<<(unsigned)ceil_div(M, R), (unsigned)(nw * 32),
                                         (size_t)nw * LeafRing<T, 4>::kBytes, a.stream>>>(pos, crd, vals, Cm, Dm, out,
                                                                                          M, N, K, R, dense);
  count_launch();
  return check_cuda(cudaGetLastError(), "sddmm_row_kernel");
}

template <typename T>
int dispatch_sddmm(int kid, const Args& a, int64_t K) {
  const int vmax = 8;
  int v = (int)ceil_div(K < 1 ? 1 : K, 32), vpl = 1;
  while (vpl < v) vpl <<= 1;
  if (vpl > vmax)
    return fail(SPX_E_UNSUPPORTED, "SDDMM supports K <= %d for this dtype, got %lld", 32 * vmax, (long long)K);
  const bool contig = K == 32 * vpl;
  switch (vpl * 2 + (contig ? 1 : 0)) {
    case 2: return run_sddmm<T, 1, false>(kid, a);
    case 3: return run_sddmm<T, 1, true>(kid, a);
    case 4: return run_sddmm<T, 2, false>(kid, a);
    case 5: return run_sddmm<T, 2, true>(kid, a);
    case 8: return run_sddmm<T, 4, false>(kid, a);
    case 9: return run_sddmm<T, 4, true>(kid, a);
    default: break;
  }
  if (vpl == 8) return contig ? run_sddmm<T, 8, true>(kid, a) : run_sddmm<T, 8, false>(kid, a);
  return fail(SPX_E_UNSUPPORTED, "no SDDMM instantiation");
}

}  // namespace

size_t ws_sddmm(int kid, const Args& a) {
  if (kid != SPX_K_SDDMM_NNZ) return 0;
  const int64_t nnz = a.level_sizes[1];
  const int64_t TB = a.params[0] > 0 ? a.params[0] : 1;
  const int64_t W = a.params[1] > 0 ? a.params[1] : TB;
  const int64_t nchunks = ceil_div(nnz > 0 ? nnz : 1, TB) * (TB / W > 0 ? TB / W : 1);
  return (size_t)(nchunks + 1) * sizeof(int32_t);
}

int launch_sddmm(int kid, const Args& a) {
  const int64_t M = a.dims[0][0], N = a.dims[0][1], K = a.dims[1][1];
  if (a.dims[1][0] != M || a.dims[2][0] != N || a.dims[2][1] != K)
    return fail(SPX_E_ARG, "SDDMM: operand shapes disagree (B %lldx%lld, C %lldx%lld, D %lldx%lld)", (long long)M,
                (long long)N, (long long)a.dims[1][0], (long long)K, (long long)a.dims[2][0],
                (long long)a.dims[2][1]);
  const int ws = a.params[2] ? a.params[2] : 32;
  if (ws != 32) return fail(SPX_E_UNSUPPORTED, "split of k must be WARP_SIZE=32");
  if (a.params[3] != 0 && (int64_t)a.params[3] != ceil_div(K, 32))
    return fail(SPX_E_CONTRACT, "MaxExact bound violated: bound %d but ceil(%lld/32) = %lld", a.params[3],
                (long long)K, (long long)ceil_div(K, 32));
  return a.dtype == SPX_F32 ? dispatch_sddmm<float>(kid, a, K) : dispatch_sddmm<double>(kid, a, K);
}

}  // namespace spx
