// Gather microbenchmark (tooling, not product): how fast can an sm_100a warp
// population gather 512 B rows of a dense operand for a given column stream?
// Each warp walks a contiguous chunk of `cols`, loads row cols[p] (16 B per
// lane) and accumulates; one float4 per warp is written.  This bounds the
// SpMM nnz-split kernel from above for the same column sequence.
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 ldh(const void* p, uint64_t pol) {
  float4 r;
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

template <int U>
__global__ void __launch_bounds__(256) gather_kernel(const int* __restrict__ cols, long n, const float4* __restrict__ B,
                                                     int rowvec, float4* __restrict__ out, long per_warp, int mode) {
  const int lane = threadIdx.x & 31;
  const long w = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  long p0 = w * per_warp, p1 = p0 + per_warp;
  if (p1 > n) p1 = n;
  const uint64_t pl = mode == 1 ? pol_last() : pol_first();
  float4 acc = make_float4(0, 0, 0, 0);
  for (long p = p0; p < p1; p += 32) {
    int my = 0;
    if (p + lane < p1) my = __ldcs(cols + p + lane);
    const int cnt = (int)min((long)32, p1 - p);
    for (int t = 0; t < cnt; t += U) {
      float4 b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        int c = __shfl_sync(0xffffffffu, my, (t + u) & 31);
        if (t + u < cnt) {
          const float4* src = B + (long)c * rowvec + lane;
          b[u] = mode == 0 ? __ldg(src) : ldh(src, pl);
        } else {
          b[u] = make_float4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        acc.x += b[u].x;
        acc.y += b[u].y;
        acc.z += b[u].z;
        acc.w += b[u].w;
      }
    }
  }
  out[w * 32 + lane] = acc;
}

__global__ void stream_kernel(const float4* __restrict__ a, long n4, float4* __restrict__ out) {
  float4 acc = make_float4(0, 0, 0, 0);
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
    float4 v = __ldcs(a + i);
    acc.x += v.x;
    acc.y += v.y;
    acc.z += v.z;
    acc.w += v.w;
  }
  out[(long)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

extern "C" int gbench_gather(const int* cols, long n, const void* B, int ncols, void* out, long per_warp, int mode,
                             int unroll, void* stream) {
  const long warps = (n + per_warp - 1) / per_warp;
  const long threads = warps * 32;
  const int bs = 256;
  const long grid = (threads + bs - 1) / bs;
  cudaStream_t s = (cudaStream_t)stream;
  if (unroll == 16)
    gather_kernel<16><<<grid, bs, 0, s>>>(cols, n, (const float4*)B, ncols / 4, (float4*)out, per_warp, mode);
  else if (unroll == 4)
    gather_kernel<4><<<grid, bs, 0, s>>>(cols, n, (const float4*)B, ncols / 4, (float4*)out, per_warp, mode);
  else
    gather_kernel<8><<<grid, bs, 0, s>>>(cols, n, (const float4*)B, ncols / 4, (float4*)out, per_warp, mode);
  return (int)cudaGetLastError();
}

extern "C" int gbench_stream(const void* a, long bytes, void* out, int grid, void* stream) {
  stream_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>((const float4*)a, bytes / 16, (float4*)out);
  return (int)cudaGetLastError();
}
