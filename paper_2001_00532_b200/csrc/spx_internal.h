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

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace spx
