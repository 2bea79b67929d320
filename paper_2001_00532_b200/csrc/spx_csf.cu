// CSF ("sss") kernels: TTV and MTTKRP over a 3rd-order tensor B stored as
// the reference's coordinate hierarchy (pack, tensors.py:212-258):
//   level 0: pos0[2]   crd0[S]   (slices, coordinate i)
//   level 1: pos1[S+1] crd1[F]   (fibers, coordinate of the 2nd mode)
//   level 2: pos2[F+1] crd2[nnz] (leaves, coordinate of the 3rd mode), vals[nnz]
//
//  K7 SPX_K_TTV_FIBER   A(i,j) = B(i,j,k) * c(k):
//     fuse(i,j,f) pos(f,fpos,B) -> fpos walks level-1 positions (fibers);
//     split(fpos,block,..,FIBERS_PER_TB) split(..,warp,..,FIBERS_PER_WARP).
//     A warp takes consecutive fibers; its lanes stride the fiber's leaves
//     and fold with a shuffle tree.  Every fiber is a distinct (i,j), so the
//     dense output (zeroed first) is written with plain stores.
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
#include "spx_common.cuh"

namespace spx {
namespace {

template <typename T>
__global__ void __launch_bounds__(kMaxThreads) ttv_fiber_kernel(const int32_t* __restrict__ crd0,
                                                         const int32_t* __restrict__ pos1,
                                                         const int32_t* __restrict__ crd1,
                                                         const int32_t* __restrict__ pos2,
                                                         const int32_t* __restrict__ crd2,
                                                         const T* __restrict__ vals, const T* __restrict__ c,
                                                         T* __restrict__ A, int64_t S, int64_t F, int64_t J,
                                                         int64_t FTB, int64_t FW) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t f0 = min((int64_t)blockIdx.x * FTB + (int64_t)warp * FW, F);
  const int64_t f1 = min(min(f0 + FW, (int64_t)(blockIdx.x + 1) * FTB), F);
  if (f0 >= f1) return;
  int64_t s = warp_search_segment(pos1, 0, S, f0, lane);
  int64_t send = __ldg(pos1 + s + 1);
  for (int64_t f = f0; f < f1; ++f) {
    while (f >= send) {
      ++s;
      send = __ldg(pos1 + s + 1);
    }
    const int64_t a = __ldg(pos2 + f), e = __ldg(pos2 + f + 1);
    T acc = T(0);
    for (int64_t p = a + lane; p < e; p += 32) acc += __ldcs(vals + p) * __ldg(c + __ldcs(crd2 + p));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
    if (lane == 0) A[(int64_t)__ldg(crd0 + s) * J + __ldg(crd1 + f)] = acc;
  }
}

template <typename T, int VPL, bool CONTIG, int U>
__global__ void __launch_bounds__(kMaxThreads) mttkrp_nnz_kernel(
    const int32_t* __restrict__ crd0, const int32_t* __restrict__ pos1, const int32_t* __restrict__ crd1,
    const int32_t* __restrict__ pos2, const int32_t* __restrict__ crd2, const T* __restrict__ vals,
    const T* __restrict__ Cm, const T* __restrict__ Dm, T* __restrict__ A, int64_t S, int64_t F, int64_t nnz,
    int64_t R, int64_t TB, int64_t W) {
  using Fr = Frag<T, VPL, CONTIG>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p0 = (int64_t)blockIdx.x * TB;
  const int64_t p1 = min(p0 + TB, nnz);
  const int64_t q0 = min(p0 + (int64_t)warp * W, p1);
  const int64_t q1 = min(q0 + W, p1);
  if (q0 >= q1) return;
  const int ncols = (int)R;
  int64_t f = warp_search_segment(pos2, 0, F, q0, lane);
  int64_t s = warp_search_segment(pos1, 0, S, f, lane);
  RowEndCache fends;
  fends.fill(pos2, f, F, lane);
  int64_t fend = fends.end(pos2, f, F, lane);
  int64_t send = __ldg(pos1 + s + 1);
  Fr accf, accs, crow;
  accf.zero();
  accs.zero();
  for (int64_t p = q0; p < q1; p += 32) {
    const int n = (int)min((int64_t)32, q1 - p);
    int my_l = 0;
    T my_v = T(0);
    if (lane < n) {
      my_l = __ldcs(crd2 + p + lane);
      my_v = __ldcs(vals + p + lane);
    }
    for (int t0 = 0; t0 < n; t0 += U) {
      Fr d[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int l = __shfl_sync(kFull, my_l, (t0 + u) & 31);
        if (t0 + u < n) d[u].load(Dm + (int64_t)l * R, lane, ncols);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (t0 + u < n) {
          const T v = __shfl_sync(kFull, my_v, (t0 + u) & 31);
          const int64_t pp = p + t0 + u;
          while (pp >= fend) {
            crow.load(Cm + (int64_t)__ldg(crd1 + f) * R, lane, ncols);
#pragma unroll
            for (int i = 0; i < VPL; ++i) accs.v[i] += accf.v[i] * crow.v[i];
            accf.zero();
            ++f;
            fend = fends.end(pos2, f, F, lane);
            while (f >= send) {
              accs.atomic_add_into(A + (int64_t)__ldg(crd0 + s) * R, lane, ncols);
              accs.zero();
              ++s;
              send = __ldg(pos1 + s + 1);
            }
          }
          accf.fma(v, d[u]);
        }
      }
    }
  }
  crow.load(Cm + (int64_t)__ldg(crd1 + f) * R, lane, ncols);
#pragma unroll
  for (int i = 0; i < VPL; ++i) accs.v[i] += accf.v[i] * crow.v[i];
  accs.atomic_add_into(A + (int64_t)__ldg(crd0 + s) * R, lane, ncols);
}

template <typename T, int VPL, bool CONTIG, int U>
__global__ void __launch_bounds__(kMaxThreads) mttkrp_slice_kernel(
    const int32_t* __restrict__ crd0, const int32_t* __restrict__ pos1, const int32_t* __restrict__ crd1,
    const int32_t* __restrict__ pos2, const int32_t* __restrict__ crd2, const T* __restrict__ vals,
    const T* __restrict__ Cm, const T* __restrict__ Dm, T* __restrict__ A, int64_t S, int64_t R, int64_t CH) {
  using Fr = Frag<T, VPL, CONTIG>;
  const int nw = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncols = (int)R;
  const int64_t lo = (int64_t)blockIdx.x * CH;
  for (int64_t k = warp; k < CH; k += nw) {
    const int64_t s = lo + k;
    if (s >= S) return;
    Fr accs, accf, crow;
    accs.zero();
    for (int64_t f = __ldg(pos1 + s); f < __ldg(pos1 + s + 1); ++f) {
      accf.zero();
      const int64_t a = __ldg(pos2 + f), e = __ldg(pos2 + f + 1);
      for (int64_t p = a; p < e; p += 32) {
        const int n = (int)min((int64_t)32, e - p);
        int my_l = 0;
        T my_v = T(0);
        if (lane < n) {
          my_l = __ldcs(crd2 + p + lane);
          my_v = __ldcs(vals + p + lane);
        }
        for (int t0 = 0; t0 < n; t0 += U) {
          Fr d[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int l = __shfl_sync(kFull, my_l, (t0 + u) & 31);
            if (t0 + u < n) d[u].load(Dm + (int64_t)l * R, lane, ncols);
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const T v = __shfl_sync(kFull, my_v, (t0 + u) & 31);
            if (t0 + u < n) accf.fma(v, d[u]);
          }
        }
      }
      crow.load(Cm + (int64_t)__ldg(crd1 + f) * R, lane, ncols);
#pragma unroll
      for (int i = 0; i < VPL; ++i) accs.v[i] += accf.v[i] * crow.v[i];
    }
    accs.store(A + (int64_t)__ldg(crd0 + s) * R, lane, ncols);
  }
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
  const int64_t I = a.dims[0][0], J = a.dims[0][1];
  T* A = static_cast<T*>(a.out);
  if (int e = check_cuda(cudaMemsetAsync(A, 0, (size_t)(I * J) * sizeof(T), a.stream), "memset")) return e;
  if (c.F == 0) return SPX_OK;
  const int64_t FTB = a.params[0] > 0 ? a.params[0] : 256;
  const int64_t FW = a.params[1] > 0 ? a.params[1] : 32;
  const int64_t nw = ceil_div(FTB, FW);
  if (nw > kMaxWarps) return fail(SPX_E_UNSUPPORTED, "TTV: FIBERS_PER_TB/FIBERS_PER_WARP must be <= 16");
  ttv_fiber_kernel<T><<<(unsigned)ceil_div(c.F, FTB), (unsigned)(nw * 32), 0, a.stream>>>(
      c.crd0, c.pos1, c.crd1, c.pos2, c.crd2, static_cast<const T*>(a.vals[0]), static_cast<const T*>(a.vals[1]), A,
      c.S, c.F, J, FTB, FW);
  count_launch();
  return check_cuda(cudaGetLastError(), "ttv_fiber_kernel");
}

template <typename T, int VPL, bool CONTIG>
int run_mttkrp(int kid, const Args& a) {
  constexpr int words = VPL * (int)sizeof(T) / 4;
  constexpr int U = words >= 8 ? 4 : 8;
  const Csf c = csf_of(a);
  const int64_t I = a.dims[0][0], R = a.dims[1][1];
  T* A = static_cast<T*>(a.out);
  const T* vals = static_cast<const T*>(a.vals[0]);
  const T* Cm = static_cast<const T*>(a.vals[1]);
  const T* Dm = static_cast<const T*>(a.vals[2]);
  if (int e = check_cuda(cudaMemsetAsync(A, 0, (size_t)(I * R) * sizeof(T), a.stream), "memset")) return e;
  if (c.nnz == 0) return SPX_OK;
  if (kid == SPX_K_MTTKRP_NNZ) {
    const int64_t TB = a.params[0], W = a.params[1];
    if (TB < 1 || W < 1 || TB % W != 0 || TB / W > kMaxWarps)
      return fail(SPX_E_UNSUPPORTED, "MTTKRP nnz-split needs NNZ_PER_TB a multiple of NNZ_PER_WARP, <= 16 warps");
    mttkrp_nnz_kernel<T, VPL, CONTIG, U><<<(unsigned)ceil_div(c.nnz, TB), (unsigned)(TB / W * 32), 0, a.stream>>>(
        c.crd0, c.pos1, c.crd1, c.pos2, c.crd2, vals, Cm, Dm, A, c.S, c.F, c.nnz, R, TB, W);
    count_launch();
    return check_cuda(cudaGetLastError(), "mttkrp_nnz_kernel");
  }
  const int64_t CH = a.params[0] > 0 ? a.params[0] : 8;
  int64_t nw = a.params[1] > 0 ? a.params[1] : (CH < 8 ? CH : 8);
  if (nw > kMaxWarps) nw = kMaxWarps;
  mttkrp_slice_kernel<T, VPL, CONTIG, U><<<(unsigned)ceil_div(c.S, CH), (unsigned)(nw * 32), 0, a.stream>>>(
      c.crd0, c.pos1, c.crd1, c.pos2, c.crd2, vals, Cm, Dm, A, c.S, R, CH);
  count_launch();
  return check_cuda(cudaGetLastError(), "mttkrp_slice_kernel");
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

}  // namespace

int launch_csf(int kid, const Args& a) {
  if (kid == SPX_K_TTV_FIBER) {
    if (a.dims[1][0] != a.dims[0][2])
      return fail(SPX_E_ARG, "TTV: B's third dimension %lld != length of c %lld", (long long)a.dims[0][2],
                  (long long)a.dims[1][0]);
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
