// Gather microbenchmark 3 (tooling, not product): the two Blackwell levers
// round 1 did not try for SpMM's 512 B-row gathers of B.
//   g4:    cp.async.bulk.tensor.2d ... tile::gather4 -- one TMA instruction
//          moves four B rows (4 x 128 fp32) into shared memory; per-warp
//          mbarrier ring, lanes read the rows back with LDS.128.
//   dsm:   hot rows of B resident in the shared memory of a thread-block
//          cluster (each CTA holds H rows, the cluster C*H).  Stream entries
//          tagged hot (bit 31 | slot) are read with ld.shared::cluster.v4
//          from the owning CTA, the others with LDG.128 from L2/HBM.
// Both accumulate every gathered row (no arithmetic beyond the adds) and
// write one float4 per lane, like tools/gbench2.cu.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>

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
__device__ __forceinline__ float4 ld_dsm(uint32_t addr) {
  float4 r;
  asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "r"(addr));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void add4(float4& a, const float4& b) {
  a.x += b.x;
  a.y += b.y;
  a.z += b.z;
  a.w += b.w;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
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
__device__ __forceinline__ void g4_load(uint32_t dst, const CUtensorMap* map, int col, int r0, int r1, int r2, int r3,
                                        uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2], %8;" ::"r"(dst),
      "l"(map), "r"(bar), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "l"(pol)
      : "memory");
}

// ---- gather4: G gather4 ops (4G rows) per stage, S stages per warp --------
template <int G, int S>
__global__ void __launch_bounds__(128) g_g4(const __grid_constant__ CUtensorMap map, const int* __restrict__ cols,
                                            long n, float4* __restrict__ out, long per_warp) {
  extern __shared__ __align__(1024) unsigned char sm[];
  constexpr int R = 4 * G;  // rows per stage
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long w = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long p0 = w * per_warp, p1 = min(p0 + per_warp, n);
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
  const long nst = total / R;  // whole stages only (tail ignored: benchmark)
  auto issue = [&](long st) {
    const int s = (int)(st % S);
    const long base = p0 + st * R;
    int my = lane < R ? __ldcs(cols + base + lane) : 0;
    if (lane == 0) {
      mbar_expect(bar_s + 8 * s, R * 512u);
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int c0 = __shfl_sync(FULL, my, 4 * g), c1 = __shfl_sync(FULL, my, 4 * g + 1);
      const int c2 = __shfl_sync(FULL, my, 4 * g + 2), c3 = __shfl_sync(FULL, my, 4 * g + 3);
      if (lane == 0) g4_load(ring_s + (s * R + 4 * g) * 512, &map, 0, c0, c1, c2, c3, bar_s + 8 * s, pl);
    }
  };
  for (long st = 0; st < S - 1 && st < nst; ++st) issue(st);
  for (long st = 0; st < nst; ++st) {
    if (st + S - 1 < nst) issue(st + S - 1);
    const int s = (int)(st % S);
    mbar_wait(bar_s + 8 * s, (uint32_t)((st / S) & 1));
    const float4* src = ring + (size_t)s * R * 32 + lane;
#pragma unroll
    for (int u = 0; u < R; ++u) add4(acc, src[u * 32]);
    __syncwarp();
  }
  out[w * 32 + lane] = acc;
}

// ---- cluster DSMEM hot rows + LDG for the rest -----------------------------
// H rows per CTA held in smem; enc[p] = (1u<<31) | owner<<20 | offset for hot entries.
template <int U>
__global__ void __launch_bounds__(1024, 1) g_dsm(const uint32_t* __restrict__ enc, long n,
                                                const float4* __restrict__ B, const int* __restrict__ hot_rows,
                                                int H, int csize, float4* __restrict__ out, long per_warp) {
  extern __shared__ __align__(128) float4 rows[];
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  // stage this CTA's hot rows: slots [rank*H, rank*H + H)
  for (int i = threadIdx.x; i < H * 32; i += blockDim.x) {
    const int r = hot_rows[rank * H + (i >> 5)];
    rows[i] = B[(long)r * 32 + (i & 31)];
  }
  cluster_sync();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(rows) + lane * 16;
  const long w = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long p0 = w * per_warp, p1 = min(p0 + per_warp, n);
  const uint64_t pl = pol_last();
  float4 acc = make_float4(0, 0, 0, 0);
  for (long p = p0; p < p1; p += 32) {
    const uint32_t my = p + lane < p1 ? __ldcs(enc + p + lane) : 0u;
    const int cnt = (int)min((long)32, p1 - p);
#pragma unroll 1
    for (int t = 0; t < cnt; t += U) {
      float4 b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t c = __shfl_sync(FULL, my, (t + u) & 31);
        if (t + u >= cnt) {
          b[u] = make_float4(0, 0, 0, 0);
        } else if (c >> 31) {
          // enc = 1<<31 | owner<<20 | row offset in the owner's smem
          b[u] = ld_dsm(mapa(base + (c & 0xfffffu) * 512u, (c >> 20) & 0x7ffu));
        } else {
          b[u] = ldh(B + (long)c * 32 + lane, pl);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) add4(acc, b[u]);
    }
  }
  out[w * 32 + lane] = acc;
  cluster_sync();  // no CTA leaves while a peer may still read its rows
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

extern "C" int gb3_g4(const int* cols, long n, const void* B, long K, void* out, long per_warp, int variant,
                      void* stream) {
  CUtensorMap map;
  cuuint64_t gdim[2] = {128, (cuuint64_t)K};
  cuuint64_t gstride[1] = {128 * 4};
  cuuint32_t box[2] = {128, 1};
  cuuint32_t estride[2] = {1, 1};
  CUresult r = get_encode()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(B), gdim, gstride, box,
                            estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    fprintf(stderr, "encode failed %d\n", (int)r);
    return 1000 + (int)r;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const long warps = (n + per_warp - 1) / per_warp;
  const int nw = 4;
  const long grid = (warps + nw - 1) / nw;
  auto go = [&](auto kern, int R, int S) {
    const size_t smem = (size_t)nw * S * R * 512 + nw * S * 8;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, nw * 32, smem, s>>>(map, cols, n, (float4*)out, per_warp);
  };
  // variant: 0 -> G2 S4 (8 rows/stage), 1 -> G4 S3 (16 rows), 2 -> G4 S4, 3 -> G8 S2 (32 rows), 4 -> G1 S8
  switch (variant) {
    case 0: go(g_g4<2, 4>, 8, 4); break;
    case 1: go(g_g4<4, 3>, 16, 3); break;
    case 2: go(g_g4<4, 4>, 16, 4); break;
    case 3: go(g_g4<8, 2>, 32, 2); break;
    default: go(g_g4<1, 8>, 4, 8); break;
  }
  return (int)cudaGetLastError();
}

// enc: encoded stream; hot_rows: csize*H row ids; grid = active clusters * csize
extern "C" int gb3_dsm(const uint32_t* enc, long n, const void* B, const int* hot_rows, int H, int csize,
                       void* out, long per_warp_unused, int* grid_out, void* stream) {
  const size_t smem = (size_t)H * 512;
  auto kern = g_dsm<8>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (csize > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(1024);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nclusters = 0;
  cfg.gridDim = dim3(csize);
  cudaError_t e = cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg);
  if (e != cudaSuccess || nclusters <= 0) {
    fprintf(stderr, "occupancy: %s n=%d\n", cudaGetErrorString(e), nclusters);
    return 2000 + (int)e;
  }
  const long ctas = (long)nclusters * csize;
  const long warps = ctas * 32;
  const long per_warp = (n + warps - 1) / warps;
  cfg.gridDim = dim3((unsigned)ctas);
  *grid_out = (int)ctas;
  e = cudaLaunchKernelEx(&cfg, kern, enc, n, (const float4*)B, hot_rows, H, csize, (float4*)out, per_warp);
  if (e != cudaSuccess) return 3000 + (int)e;
  return (int)cudaGetLastError();
}
