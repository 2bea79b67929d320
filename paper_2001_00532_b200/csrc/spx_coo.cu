// Device-resident COO container support (formats.DeviceCoo): the checks and
// conversions the reference performs on the host in tensors.py, as sm_100a
// kernels over HBM-resident arrays.
//
//   spx_coo_check        CooTensor.validate bounds (tensors.py:75-81): the
//                        first entry (in input order) with a coordinate
//                        outside [0, dim).
//   spx_unpack           Tensor.walk_stored (tensors.py:190-206): the
//                        coordinates of every stored leaf slot, in storage
//                        order (dense levels expand every slot).
//   spx_check_invariants Tensor.check_invariants (tensors.py:147-163), first
//                        violation in the reference's check order.
//   spx_scatter_dense    Tensor.to_dense (tensors.py:181-188).
//
// All are HBM-streaming integer kernels (grid-stride, 4-8 B per element
// per level, binary searches over pos for the parent of a slot).
#include "spx_internal.h"

namespace spx {
namespace {

constexpr int kMaxOrder = 8;

struct LevelTab {
  const int32_t* pos[kMaxOrder];
  const int32_t* crd[kMaxOrder];
  int64_t dims[kMaxOrder];
  int64_t parents[kMaxOrder];  // slot count of the level above (1 for level 0)
  int32_t compressed[kMaxOrder];
  int32_t order;
};

struct CoordTab {
  const int32_t* c[kMaxOrder];
  int64_t stride;
  int64_t dims[kMaxOrder];
  int32_t order;
};

__global__ void coo_check_kernel(CoordTab t, int64_t n, unsigned long long* first_bad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    bool bad = false;
    for (int l = 0; l < t.order; ++l) {
      const int64_t x = t.c[l][i * t.stride];
      bad |= x < 0 || x >= t.dims[l];
    }
    if (bad) atomicMin(first_bad, (unsigned long long)i);
  }
}

// largest s in [0, n) with pos[s] <= key (the segment holding position key)
__device__ __forceinline__ int64_t seg_of(const int32_t* __restrict__ pos, int64_t n, int64_t key) {
  int64_t lo = 0, hi = n, r = 0;
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    if ((int64_t)pos[m] <= key) {
      r = m;
      lo = m + 1;
    } else {
      hi = m;
    }
  }
  return r;
}

__global__ void unpack_kernel(LevelTab t, int64_t nleaves, int32_t* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nleaves; q += stride) {
    int64_t slot = q;
    for (int l = t.order - 1; l >= 0; --l) {
      int64_t c;
      if (t.compressed[l]) {
        c = t.crd[l][slot];
        slot = seg_of(t.pos[l], t.parents[l], slot);
      } else {
        c = slot % t.dims[l];
        slot /= t.dims[l];
      }
      out[(int64_t)l * nleaves + q] = (int32_t)c;
    }
  }
}

// result: min over violations of (level << 40) | (code << 36) | segment
//   code 1: malformed pos (pos[0] != 0 or pos[count] != len(crd))
//   code 2: pos not nondecreasing
//   code 3: segment `segment` coordinates not strictly increasing
__global__ void invariants_kernel(const int32_t* __restrict__ pos, const int32_t* __restrict__ crd, int64_t count,
                                  int64_t ncrd, int level, unsigned long long* result) {
  const unsigned long long lv = (unsigned long long)level << 40;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  if (g == 0 && (pos[0] != 0 || (int64_t)pos[count] != ncrd)) atomicMin(result, lv | (1ull << 36));
  for (int64_t s = g; s < count; s += stride)
    if (pos[s] > pos[s + 1]) atomicMin(result, lv | (2ull << 36));
  // a position p > pos[seg] inside its segment must have crd[p-1] < crd[p]
  for (int64_t p = g + 1; p < ncrd; p += stride) {
    const int64_t s = seg_of(pos, count, p);
    if (p > (int64_t)pos[s] && p < (int64_t)pos[s + 1] && crd[p - 1] >= crd[p])
      atomicMin(result, lv | (3ull << 36) | (unsigned long long)s);
  }
}

template <typename T>
__global__ void scatter_dense_kernel(CoordTab t, int64_t n, const T* __restrict__ vals, T* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    int64_t lin = 0;
    for (int l = 0; l < t.order; ++l) lin = lin * t.dims[l] + t.c[l][i * t.stride];
    out[lin] = vals[i];
  }
}

unsigned grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g < 1) g = 1;
  if (g > 148 * 16) g = 148 * 16;
  return (unsigned)g;
}

}  // namespace
}  // namespace spx

using namespace spx;

extern "C" {

int spx_coo_check(const int32_t* const* coords_host, int64_t coord_stride, int32_t order, const int64_t* dims,
                  int64_t n, uint64_t* first_bad, void* stream) {
  if (order < 1 || order > kMaxOrder) return fail(SPX_E_ARG, "spx_coo_check: order %d outside 1..8", order);
  if (!first_bad || (n > 0 && !coords_host)) return fail(SPX_E_ARG, "spx_coo_check: null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (int e = check_cuda(cudaMemsetAsync(first_bad, 0xff, sizeof(uint64_t), st), "memset")) return e;
  if (n == 0) return SPX_OK;
  CoordTab t{};
  t.order = order;
  t.stride = coord_stride;
  for (int l = 0; l < order; ++l) {
    t.c[l] = coords_host[l];
    t.dims[l] = dims[l];
  }
  coo_check_kernel<<<grid_for(n), 256, 0, st>>>(t, n, reinterpret_cast<unsigned long long*>(first_bad));
  count_launch();
  return check_cuda(cudaGetLastError(), "coo_check_kernel");
}

int spx_unpack(int32_t order, const char* levels, const int64_t* dims, const int32_t* const* pos_host,
               const int32_t* const* crd_host, const int64_t* level_sizes, int64_t nleaves, int32_t* coords_out,
               void* stream) {
  if (order < 1 || order > kMaxOrder) return fail(SPX_E_ARG, "spx_unpack: order %d outside 1..8", order);
  if (nleaves == 0) return SPX_OK;
  if (!levels || !dims || !level_sizes || !coords_out) return fail(SPX_E_ARG, "spx_unpack: null argument");
  LevelTab t{};
  t.order = order;
  for (int l = 0; l < order; ++l) {
    t.compressed[l] = levels[l] == 's';
    t.dims[l] = dims[l];
    t.parents[l] = l == 0 ? 1 : level_sizes[l - 1];
    if (t.compressed[l]) {
      if (!pos_host || !crd_host || !pos_host[l] || !crd_host[l])
        return fail(SPX_E_ARG, "spx_unpack: level %d is compressed but has no pos/crd", l);
      t.pos[l] = pos_host[l];
      t.crd[l] = crd_host[l];
    }
  }
  unpack_kernel<<<grid_for(nleaves), 256, 0, static_cast<cudaStream_t>(stream)>>>(t, nleaves, coords_out);
  count_launch();
  return check_cuda(cudaGetLastError(), "unpack_kernel");
}

int spx_check_invariants(const int32_t* pos, const int32_t* crd, int64_t count, int64_t ncrd, int32_t level,
                         uint64_t* result, void* stream) {
  if (!pos || !result) return fail(SPX_E_ARG, "spx_check_invariants: null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (int e = check_cuda(cudaMemsetAsync(result, 0xff, sizeof(uint64_t), st), "memset")) return e;
  invariants_kernel<<<grid_for(count > ncrd ? count : ncrd), 256, 0, st>>>(
      pos, crd, count, ncrd, level, reinterpret_cast<unsigned long long*>(result));
  count_launch();
  return check_cuda(cudaGetLastError(), "invariants_kernel");
}

int spx_scatter_dense(const int32_t* const* coords_host, int64_t coord_stride, int32_t order, const int64_t* dims,
                      int64_t n, const void* vals, int32_t dtype, void* out, void* stream) {
  if (order < 1 || order > kMaxOrder) return fail(SPX_E_ARG, "spx_scatter_dense: order %d outside 1..8", order);
  if (n == 0) return SPX_OK;
  if (!coords_host || !vals || !out) return fail(SPX_E_ARG, "spx_scatter_dense: null argument");
  CoordTab t{};
  t.order = order;
  t.stride = coord_stride;
  for (int l = 0; l < order; ++l) {
    t.c[l] = coords_host[l];
    t.dims[l] = dims[l];
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == SPX_F32)
    scatter_dense_kernel<float><<<grid_for(n), 256, 0, st>>>(t, n, static_cast<const float*>(vals),
                                                            static_cast<float*>(out));
  else
    scatter_dense_kernel<double><<<grid_for(n), 256, 0, st>>>(t, n, static_cast<const double*>(vals),
                                                             static_cast<double*>(out));
  count_launch();
  return check_cuda(cudaGetLastError(), "scatter_dense_kernel");
}

}  // extern "C"
