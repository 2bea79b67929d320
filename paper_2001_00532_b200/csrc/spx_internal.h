// Host-side internals shared by the libspx translation units.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/spx.h"

namespace spx {

// Set the thread-local error message and return `code`.
int fail(int code, const char* fmt, ...);
// Map a CUDA error (if any) to SPX_E_CUDA with context.
int check_cuda(cudaError_t e, const char* what);
// Count one kernel launch (exported through spx_launch_count).
void count_launch(int n = 1);

// Resolved launch arguments: operands addressed by role.
struct Args {
  int dtype;
  const int32_t* pos[3];
  const int32_t* crd[3];
  const void* vals[3];     // role-ordered
  int64_t dims[3][3];      // role-ordered dims
  int64_t level_sizes[4];
  const int32_t* params;
  void* out;
  void* ws;
  size_t ws_bytes;
  cudaStream_t stream;
};

// Per-family launchers (return SPX_* status).
int launch_spmv(int kernel_id, const Args& a);
int launch_spmm(int kernel_id, const Args& a);
int launch_sddmm(int kernel_id, const Args& a);
int launch_csf(int kernel_id, const Args& a);

size_t ws_spmv(int kernel_id, const Args& a);
size_t ws_spmm(int kernel_id, const Args& a);
size_t ws_csf(int kernel_id, const Args& a);
size_t ws_sddmm(int kernel_id, const Args& a);

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Workspace of the nnz-split kernels: per-CTA carry values (`vals_per_cta`
// elements of `es` bytes), per-CTA carry rows, and the chunk->segment table
// (ncta + 1 int32).  Offsets are 256 B aligned.
struct NnzWorkspace {
  size_t carry_val, carry_row, first, total;
};
inline NnzWorkspace nnz_workspace(int64_t ncta, size_t es, int64_t vals_per_cta = 1) {
  auto up = [](size_t b) { return (b + 255) & ~(size_t)255; };
  NnzWorkspace w;
  w.carry_val = 0;
  w.carry_row = up((size_t)ncta * vals_per_cta * es);
  w.first = w.carry_row + up((size_t)ncta * sizeof(int32_t));
  w.total = w.first + up((size_t)(ncta + 1) * sizeof(int32_t));
  return w;
}

// first[c] = SearchSegment(pos, 0, nseg, c*chunk) (ir.py:178-190) for every
// chunk c in [0, nchunks) of `chunk` consecutive leaf positions, computed by
// one coalesced pass over pos (each nonempty segment writes the chunks whose
// first position it holds); chunks at or past the last position and the
// sentinel first[nchunks] get nseg - 1.  Replaces a serial
// binary search at the start of every CTA/warp of the nnz-split kernels.
// the Atomics nnz-split segment sum of spx_spmv.cu (y zeroed by the caller)
int segsum_atomic_f32(const int32_t* pos, const int32_t* crd, const float* vals, const float* x, float* y,
                      int64_t nseg, int64_t nnz, int64_t TB, int64_t W, int64_t TPT, const int32_t* first,
                      cudaStream_t st, int64_t xlen);
int segsum_atomic_f64(const int32_t* pos, const int32_t* crd, const double* vals, const double* x, double* y,
                      int64_t nseg, int64_t nnz, int64_t TB, int64_t W, int64_t TPT, const int32_t* first,
                      cudaStream_t st, int64_t xlen);
int launch_chunk_segments(const int32_t* pos, int64_t nseg, int64_t chunk, int64_t nchunks, int32_t* first,
                          cudaStream_t stream);

}  // namespace spx
