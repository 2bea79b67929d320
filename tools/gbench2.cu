// Gather microbenchmark 2 (tooling, not product): the 512 B-row gather of
// SpMM through three sm_100a data paths, to find which one the nnz-split
// kernel should use.
//   path 0: LDG.128 into registers (each lane 16 B of the row)
//   path 1: cp.async (LDGSTS) 16 B per lane into a per-warp smem ring, LDS back
//   path 2: cp.async.bulk (TMA bulk copy, UBLKCP) of whole rows into a
//           per-warp smem ring, completion on an mbarrier, LDS back
// Each warp walks a contiguous chunk of `cols` and accumulates the gathered
// rows; one float4 per lane is written.
#include <cuda_runtime.h>
#include <stdint.h>

#define FULL 0xffffffffu

__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 ldh(const void* p, uint64_t pol) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ void add4(float4& a, const float4& b) {
  a.x += b.x;
  a.y += b.y;
  a.z += b.z;
  a.w += b.w;
}

// ---- path 0: registers ------------------------------------------------------
template <int U>
__global__ void __launch_bounds__(256) g_reg(const int* __restrict__ cols, long n, const float4* __restrict__ B,
                                             float4* __restrict__ out, long per_warp) {
  const int lane = threadIdx.x & 31;
  const long w = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  long p0 = w * per_warp, p1 = min(p0 + per_warp, n);
  const uint64_t pl = pol_last();
  float4 acc = make_float4(0, 0, 0, 0);
  for (long p = p0; p < p1; p += 32) {
    int my = p + lane < p1 ? __ldcs(cols + p + lane) : 0;
    const int cnt = (int)min((long)32, p1 - p);
#pragma unroll 1
    for (int t = 0; t < cnt; t += U) {
      float4 b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        int c = __shfl_sync(FULL, my, (t + u) & 31);
        b[u] = (t + u < cnt) ? ldh(B + (long)c * 32 + lane, pl) : make_float4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) add4(acc, b[u]);
    }
  }
  out[w * 32 + lane] = acc;
}

// ---- path 2: TMA bulk row copies ------------------------------------------
__device__ __forceinline__ void mbar_init(uint32_t bar, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(bar),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}

// R rows per stage, S stages per warp; NW warps per CTA.
template <int R, int S>
__global__ void __launch_bounds__(256) g_tma(const int* __restrict__ cols, long n, const float4* __restrict__ B,
                                             float4* __restrict__ out, long per_warp) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long w = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  long p0 = w * per_warp, p1 = min(p0 + per_warp, n);
  float4* ring = reinterpret_cast<float4*>(sm) + (size_t)warp * S * R * 32;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)(blockDim.x >> 5) * S * R * 512) + warp * S;
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
  const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(bars);
  if (lane == 0)
    for (int s = 0; s < S; ++s) mbar_init(bar_s + 8 * s, 1);
  __syncwarp();
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const uint64_t pl = pol_last();
  float4 acc = make_float4(0, 0, 0, 0);
  const long total = p1 - p0;
  const long nst = (total + R - 1) / R;  // stages of R rows
  auto issue = [&](long st) {
    const int s = (int)(st % S);
    const long base = p0 + st * R;
    const int cnt = (int)min((long)R, p1 - base);
    if (lane == 0) mbar_expect(bar_s + 8 * s, cnt * 512u);
    __syncwarp();
    if (lane < cnt) {
      const int c = __ldcs(cols + base + lane);
      bulk_g2s(ring_s + (s * R + lane) * 512, B + (long)c * 32, 512, bar_s + 8 * s, pl);
    }
  };
  for (long st = 0; st < S - 1 && st < nst; ++st) issue(st);
  for (long st = 0; st < nst; ++st) {
    if (st + S - 1 < nst) issue(st + S - 1);
    const int s = (int)(st % S);
    mbar_wait(bar_s + 8 * s, (uint32_t)((st / S) & 1));
    const int cnt = (int)min((long)R, p1 - (p0 + st * R));
    const float4* src = ring + (size_t)s * R * 32 + lane;
#pragma unroll
    for (int u = 0; u < R; ++u)
      if (u < cnt) add4(acc, src[u * 32]);
    __syncwarp();
  }
  out[w * 32 + lane] = acc;
}

// ---- path 3: 8 B scalar gathers (SpMV x[crd[p]]), 8 per thread ---------------
__global__ void __launch_bounds__(256) g_scalar(const int* __restrict__ cols, long n, const double* __restrict__ x,
                                                double* __restrict__ out) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long a = t * 8;
  double acc = 0.0;
  if (a + 8 <= n) {
    const int4 c0 = __ldcs(reinterpret_cast<const int4*>(cols + a));
    const int4 c1 = __ldcs(reinterpret_cast<const int4*>(cols + a) + 1);
    acc = __ldg(x + c0.x) + __ldg(x + c0.y) + __ldg(x + c0.z) + __ldg(x + c0.w) + __ldg(x + c1.x) +
          __ldg(x + c1.y) + __ldg(x + c1.z) + __ldg(x + c1.w);
  }
  out[t] = acc;
}

extern "C" int gb2_scalar(const int* cols, long n, const void* x, void* out, void* stream) {
  const long threads = n / 8;
  g_scalar<<<(threads + 255) / 256, 256, 0, (cudaStream_t)stream>>>(cols, n, (const double*)x, (double*)out);
  return (int)cudaGetLastError();
}

extern "C" int gb2_gather(int path, const int* cols, long n, const void* B, void* out, long per_warp, int variant,
                          void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const long warps = (n + per_warp - 1) / per_warp;
  if (path == 0) {
    const long grid = (warps * 32 + 255) / 256;
    if (variant == 16)
      g_reg<16><<<grid, 256, 0, s>>>(cols, n, (const float4*)B, (float4*)out, per_warp);
    else
      g_reg<8><<<grid, 256, 0, s>>>(cols, n, (const float4*)B, (float4*)out, per_warp);
  } else {
    // variant: 0 -> R16 S4 (4 warps/CTA), 1 -> R32 S2 (4 warps), 2 -> R8 S4 (8 warps), 3 -> R16 S3 (4 warps)
    int R = 16, S = 4, nw = 4;
    if (variant == 1) R = 32, S = 2;
    if (variant == 2) R = 8, S = 4, nw = 8;
    if (variant == 3) R = 16, S = 3;
    const size_t smem = (size_t)nw * S * R * 512 + nw * S * 8;
    const long grid = (warps + nw - 1) / nw;
    auto go = [&](auto kern) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kern<<<grid, nw * 32, smem, s>>>(cols, n, (const float4*)B, (float4*)out, per_warp);
    };
    if (variant == 1)
      go(g_tma<32, 2>);
    else if (variant == 2)
      go(g_tma<8, 4>);
    else if (variant == 3)
      go(g_tma<16, 3>);
    else
      go(g_tma<16, 4>);
  }
  return (int)cudaGetLastError();
}
