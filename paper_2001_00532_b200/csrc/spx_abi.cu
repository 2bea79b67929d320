// C-ABI entry points of libspx.so (declared in include/spx.h).
//
// spx_launch resolves the Manifest-ordered argument tables (ir.py:237-263)
// into role-ordered operands and hands them to the per-family launchers.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "spx_common.cuh"

namespace spx {

namespace {
thread_local char g_err[1024] = "";
std::atomic<uint64_t> g_launches{0};

struct Family {
  int nroles;
  int order[3];       // tensor order per role
  int sparse_levels;  // compressed levels of role 0 (pos/crd pairs)
  int (*launch)(int, const Args&);
};

bool family_of(int kid, Family* f) {
  switch (kid) {
    case SPX_K_SPMV_ROW:
    case SPX_K_SPMV_WARP:
    case SPX_K_SPMV_NNZ:
      *f = {2, {2, 1, 0}, 1, launch_spmv};
      return true;
    case SPX_K_SPMM_NNZ:
    case SPX_K_SPMM_ROW:
      *f = {2, {2, 2, 0}, 1, launch_spmm};
      return true;
    case SPX_K_SDDMM_NNZ:
    case SPX_K_SDDMM_ROW:
      *f = {3, {2, 2, 2}, 1, launch_sddmm};
      return true;
    case SPX_K_TTV_FIBER:
    case SPX_K_TTV_NNZ:
      *f = {2, {3, 1, 0}, 3, launch_csf};
      return true;
    case SPX_K_MTTKRP_NNZ:
    case SPX_K_MTTKRP_SLICE:
      *f = {3, {3, 2, 2}, 3, launch_csf};
      return true;
    default:
      return false;
  }
}

int resolve(const spx_plan* plan, const void* const* vals, const int32_t* const* pos, const int32_t* const* crd,
            const int32_t* dims, Family* fam, Args* a) {
  if (!plan) return fail(SPX_E_ARG, "null plan");
  if (!family_of(plan->kernel_id, fam)) return fail(SPX_E_UNSUPPORTED, "unknown kernel id %d", plan->kernel_id);
  if (plan->dtype != SPX_F32 && plan->dtype != SPX_F64) return fail(SPX_E_ARG, "unknown dtype %d", plan->dtype);
  if (!dims) return fail(SPX_E_ARG, "null dims");
  std::memset(a, 0, sizeof(*a));
  a->dtype = plan->dtype;
  a->params = plan->params;
  // manifest index -> role
  int role_at[3] = {-1, -1, -1};
  for (int r = 0; r < fam->nroles; ++r) {
    const int m = plan->slot[r];
    if (m < 0 || m >= fam->nroles || role_at[m] != -1) return fail(SPX_E_ARG, "bad operand slot table");
    role_at[m] = r;
  }
  int off = 0;
  for (int m = 0; m < fam->nroles; ++m) {
    const int r = role_at[m];
    for (int d = 0; d < fam->order[r]; ++d) {
      if (dims[off + d] < 0) return fail(SPX_E_ARG, "negative dimension");
      a->dims[r][d] = dims[off + d];
    }
    off += fam->order[r];
    if (vals) a->vals[r] = vals[m];
  }
  for (int l = 0; l < fam->sparse_levels; ++l) {
    if (pos) a->pos[l] = pos[l];
    if (crd) a->crd[l] = crd[l];
  }
  for (int l = 0; l < 4; ++l) a->level_sizes[l] = plan->level_sizes[l];
  const int64_t nnz = a->level_sizes[fam->sparse_levels == 1 ? 1 : 2];
  if (nnz < 0 || nnz > INT32_MAX) return fail(SPX_E_ARG, "nnz %lld outside int32 positions", (long long)nnz);
  if (vals) {
    // a null buffer is only acceptable for an operand with no elements
    for (int r = 0; r < fam->nroles; ++r) {
      int64_t n = 1;
      if (r == 0) n = nnz;
      else
        for (int d = 0; d < fam->order[r]; ++d) n *= a->dims[r][d];
      if (!a->vals[r] && n > 0) return fail(SPX_E_ARG, "null vals pointer for operand role %d", r);
    }
  }
  return SPX_OK;
}

}  // namespace

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return SPX_OK;
  return fail(SPX_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

__global__ void partition_kernel(const int32_t* __restrict__ seg_start, int64_t nseg, int64_t nnz, int32_t ndev,
                                 int64_t* __restrict__ out) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g > ndev) return;
  if (g == 0) {
    out[0] = 0;
    return;
  }
  if (g == ndev) {
    out[ndev] = nseg;
    return;
  }
  const int64_t chunk = (nnz + ndev - 1) / ndev;
  int64_t target = (int64_t)g * chunk;
  if (target > nnz) target = nnz;
  out[g] = lower_bound(seg_start, 0, nseg, target);
}

__global__ void chunk_segments_kernel(const int32_t* __restrict__ pos, int64_t nseg, int64_t chunk, int64_t nchunks,
                                      int32_t* __restrict__ first) {
  // positions are int32 (tensors.py:248-249): 32-bit arithmetic throughout
  const uint32_t ch = (uint32_t)chunk;
  const int stride = (int)(gridDim.x * blockDim.x);
  for (int r = (int)(blockIdx.x * blockDim.x + threadIdx.x); r < (int)nseg; r += stride) {
    const uint32_t a = (uint32_t)__ldcs(pos + r), e = (uint32_t)__ldcs(pos + r + 1);
    if (a == e) continue;
    // chunks c with a <= c*chunk < e start inside segment r; later segments
    // start after e and earlier ones end at or before a, so r is the largest
    // segment with pos[r] <= c*chunk
    for (uint32_t c = (a + ch - 1) / ch; (uint64_t)c * ch < e; ++c) first[c] = r;
  }
  // chunks starting at or past the last position (and the sentinel entry
  // nchunks) map to the last segment
  if (blockIdx.x == 0) {
    const int64_t nnz = nseg > 0 ? (int64_t)__ldg(pos + nseg) : 0;
    for (int64_t c = (nnz + chunk - 1) / chunk + threadIdx.x; c <= nchunks; c += blockDim.x)
      first[c] = (int32_t)(nseg > 0 ? nseg - 1 : 0);
  }
}

int launch_chunk_segments(const int32_t* pos, int64_t nseg, int64_t chunk, int64_t nchunks, int32_t* first,
                          cudaStream_t stream) {
  int64_t blocks = ceil_div(nseg > 0 ? nseg : 1, 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  chunk_segments_kernel<<<(unsigned)blocks, 256, 0, stream>>>(pos, nseg, chunk, nchunks, first);
  count_launch();
  return check_cuda(cudaGetLastError(), "chunk_segments_kernel");
}

}  // namespace spx

using namespace spx;

extern "C" {

int spx_version(void) { return SPX_ABI_VERSION; }

const char* spx_last_error(void) { return g_err; }

uint64_t spx_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

size_t spx_workspace_size(const spx_plan* plan, const int32_t* dims) {
  Family fam;
  Args a;
  if (resolve(plan, nullptr, nullptr, nullptr, dims, &fam, &a) != SPX_OK) return 0;
  switch (plan->kernel_id) {
    case SPX_K_SPMV_NNZ: return ws_spmv(plan->kernel_id, a);
    case SPX_K_SPMM_NNZ:
    case SPX_K_SPMM_ROW: return ws_spmm(plan->kernel_id, a);
    case SPX_K_MTTKRP_NNZ:
    case SPX_K_MTTKRP_SLICE:
    case SPX_K_TTV_NNZ: return ws_csf(plan->kernel_id, a);
    case SPX_K_SDDMM_NNZ: return ws_sddmm(plan->kernel_id, a);
    default: return 0;
  }
}

int spx_launch(const spx_plan* plan, void* out, const void* const* vals, const int32_t* const* pos,
               const int32_t* const* crd, const int32_t* dims, void* workspace, size_t ws_bytes, void* stream) {
  Family fam;
  Args a;
  if (int e = resolve(plan, vals, pos, crd, dims, &fam, &a)) return e;
  if (!vals || !pos || !crd) return fail(SPX_E_ARG, "null argument table");
  for (int l = 0; l < fam.sparse_levels; ++l) {
    const int64_t lsize = a.level_sizes[fam.sparse_levels == 1 ? 1 : l];
    if (!a.pos[l] || (!a.crd[l] && lsize > 0)) return fail(SPX_E_ARG, "null pos/crd for level %d", l);
  }
  if (!out) return fail(SPX_E_ARG, "null output");
  a.out = out;
  a.ws = workspace;
  a.ws_bytes = ws_bytes;
  a.stream = static_cast<cudaStream_t>(stream);
  return fam.launch(plan->kernel_id, a);
}

int spx_partition(const int32_t* seg_start, int64_t nseg, int64_t nnz, int32_t ndev, int64_t* bounds_out) {
  if (ndev < 1) return fail(SPX_E_ARG, "ndev must be >= 1");
  if (nseg < 0 || nnz < 0 || (!seg_start && nseg > 0) || !bounds_out) return fail(SPX_E_ARG, "bad partition args");
  const int64_t chunk = (nnz + ndev - 1) / ndev;
  bounds_out[0] = 0;
  for (int g = 1; g < ndev; ++g) {
    int64_t target = (int64_t)g * chunk;
    if (target > nnz) target = nnz;
    int64_t lo = 0, hi = nseg;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)seg_start[mid] < target) lo = mid + 1;
      else hi = mid;
    }
    bounds_out[g] = lo;
  }
  bounds_out[ndev] = nseg;
  return SPX_OK;
}

int spx_partition_device(const int32_t* seg_start, int64_t nseg, int64_t nnz, int32_t ndev, int64_t* bounds_out,
                         void* stream) {
  if (ndev < 1) return fail(SPX_E_ARG, "ndev must be >= 1");
  if (nseg < 0 || nnz < 0 || (!seg_start && nseg > 0) || !bounds_out) return fail(SPX_E_ARG, "bad partition args");
  partition_kernel<<<(ndev + 1 + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(seg_start, nseg, nnz, ndev,
                                                                                          bounds_out);
  count_launch();
  return check_cuda(cudaGetLastError(), "partition_kernel");
}

}  // extern "C"

namespace spx {
__global__ void policy_probe_kernel(uint64_t* out) {
  out[0] = createpolicy_evict_last();
  out[1] = createpolicy_evict_first();
  out[2] = kPolicyEvictLast;
  out[3] = kPolicyEvictFirst;
}
}  // namespace spx

extern "C" int spx_selftest(uint64_t* out4, void* stream) {
  if (!out4) return spx::fail(SPX_E_ARG, "null output");
  spx::policy_probe_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(out4);
  spx::count_launch();
  return spx::check_cuda(cudaGetLastError(), "policy_probe_kernel");
}
