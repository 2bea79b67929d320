// Shared device helpers for the libspx kernels (sm_100a).
//
// Search semantics follow the reference IR exactly (ir.py:178-205):
//   SearchSegment: largest s in [lo, hi) with arr[s] <= key, clamped to lo
//   SearchCoord:   first s in [lo, hi) with arr[s] >= key, else hi
// The oracle restates both in oracle/spx_oracle.c and tests compare them
// bit for bit.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "spx_internal.h"

namespace spx {

constexpr unsigned kFull = 0xffffffffu;
// Largest CTA any kernel is launched with; keeps the per-thread register
// budget at 128 so the unrolled gathers stay in registers.
constexpr int kMaxThreads = 512;
constexpr int kMaxWarps = kMaxThreads / 32;

// ---------------------------------------------------------------------------
// cache-hinted loads/stores.  Streaming data (pos/crd/vals of the sparse
// operand, outputs) is marked evict-first so the gathered dense operand keeps
// its L2 residency (126 MB L2 vs 512 MB B at cfg2).
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T ld_stream(const T* p) { return __ldcs(p); }
template <typename T>
__device__ __forceinline__ T ld_ro(const T* p) { return __ldg(p); }
template <typename T>
__device__ __forceinline__ void st_stream(T* p, T v) { __stcs(p, v); }

// ---------------------------------------------------------------------------
// L2 residency control (createpolicy + .L2::cache_hint).  The gathered dense
// operand is tagged evict_last so that the streamed sparse arrays and the
// output (tagged evict_first) do not push its hot rows out of the 126 MB L2.
// ---------------------------------------------------------------------------
// The 64-bit cache-policy descriptors createpolicy.fractional.L2::evict_*
// 1.0 produces (the constants CUTLASS uses for its TMA/LDG hints).  Using
// immediates lets ptxas keep the policy in a uniform register instead of
// re-deriving it (R2UR) at every cp.async; tests/test_gpu_kernels.py checks
// they equal what createpolicy returns on the device.
constexpr uint64_t kPolicyEvictNormal = 0x1000000000000000ull;
constexpr uint64_t kPolicyEvictFirst = 0x12F0000000000000ull;
constexpr uint64_t kPolicyEvictLast = 0x14F0000000000000ull;
__device__ __forceinline__ uint64_t l2_evict_last() { return kPolicyEvictLast; }
__device__ __forceinline__ uint64_t l2_evict_first() { return kPolicyEvictFirst; }
__device__ __forceinline__ uint64_t createpolicy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t createpolicy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 ld_f4_hint(const void* p, uint64_t pol) {
  float4 r;
  asm("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
      : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
      : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ int4 ld_i4_hint(const void* p, uint64_t pol) {
  int4 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ void st_f4_hint(void* p, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ int ld_i32_first(const int32_t* p, uint64_t pol) {
  int r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ float ld_f32_first(const float* p, uint64_t pol) {
  float r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ double ld_f64_first(const double* p, uint64_t pol) {
  double r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ float ld_stream_hint(const float* p, uint64_t pol) { return ld_f32_first(p, pol); }
__device__ __forceinline__ double ld_stream_hint(const double* p, uint64_t pol) { return ld_f64_first(p, pol); }

// cp.async (LDGSTS) 16 B global -> shared, L1 bypass, with an L2 policy.
__device__ __forceinline__ void cp_async16(uint32_t smem_addr, const void* gptr, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_addr), "l"(gptr),
               "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// base + a*b with one IMAD.WIDE.U32 (32-bit row index times row bytes)
template <typename P>
__device__ __forceinline__ const P* addr_wide(const P* base, uint32_t a, uint32_t b) {
  uint64_t r;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(a), "r"(b), "l"(reinterpret_cast<uint64_t>(base)));
  return reinterpret_cast<const P*>(r);
}

// cp.async.cg of 16 bytes, zero-filling past src_bytes (0..16)
__device__ __forceinline__ void cp_async16_zfill(uint32_t smem_addr, const void* gptr, int src_bytes, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;" ::"r"(smem_addr), "l"(gptr),
               "r"(src_bytes), "l"(pol)
               : "memory");
}

// cp.async of 4 / 8 bytes (L1-allocating .ca form, the only one these sizes
// allow) with zero-fill when src_bytes == 0 and an L2 policy.
__device__ __forceinline__ void cp_async4(uint32_t smem_addr, const void* gptr, int src_bytes, uint64_t pol) {
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2, %3;" ::"r"(smem_addr), "l"(gptr),
               "r"(src_bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t smem_addr, const void* gptr, int src_bytes, uint64_t pol) {
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2, %3;" ::"r"(smem_addr), "l"(gptr),
               "r"(src_bytes), "l"(pol)
               : "memory");
}

// 16 bytes of ELEM-byte elements of which the first `nvalid` exist: one
// 16 B cp.async when the chunk is whole, else one cp.async per element with
// zero-fill, so no byte past the last element is read (compute-sanitizer
// initcheck counts a partial 16 B copy as a 16 B read of the tail).
template <int ELEM>
__device__ __forceinline__ void cp_async16_elems(uint32_t smem_addr, const void* gptr, int nvalid, uint64_t pol) {
  static_assert(ELEM == 4 || ELEM == 8, "4 or 8 byte elements");
  if (nvalid * ELEM >= 16) {
    cp_async16_zfill(smem_addr, gptr, 16, pol);
  } else {
    const char* g = static_cast<const char*>(gptr);
#pragma unroll
    for (int e = 0; e < 16 / ELEM; ++e) {
      const bool ok = e < nvalid;
      if constexpr (ELEM == 4) cp_async4(smem_addr + 4 * e, ok ? g + 4 * e : g, ok ? 4 : 0, pol);
      else cp_async8(smem_addr + 8 * e, ok ? g + 8 * e : g, ok ? 8 : 0, pol);
    }
  }
}

// ---------------------------------------------------------------------------
// Per-warp ring of leaf batches: (crd, val) of 32 consecutive positions per
// slot, streamed from HBM into shared memory by cp.async RING-1 batches
// ahead of use, so a single warp keeps ~RING*32*(4+sizeof(T)) bytes of the
// sparse operand in flight without holding registers for them.  Slot layout:
// 32 int32 coordinates then 32 values, so four leaves are read back as one
// 16-byte broadcast of coordinates and one (or two) of values.
// ---------------------------------------------------------------------------
template <typename T, int RING>
struct LeafRing {
  static constexpr int kSlotBytes = 32 * (4 + (int)sizeof(T));
  static constexpr int kBytes = RING * kSlotBytes;
  unsigned char* base;  // this warp's RING slots
  const int32_t* crd;
  const T* vals;
  int q0, q1, nb;

  __device__ __forceinline__ void init(unsigned char* warp_base, const int32_t* c, const T* v, int a, int b) {
    base = warp_base;
    crd = c;
    vals = v;
    q0 = a;
    q1 = b;
    nb = (b - a + 31) >> 5;
  }
  __device__ __forceinline__ const int32_t* crd_slot(int b) const {
    return reinterpret_cast<const int32_t*>(base + (b % RING) * kSlotBytes);
  }
  __device__ __forceinline__ const T* val_slot(int b) const {
    return reinterpret_cast<const T*>(base + (b % RING) * kSlotBytes + 128);
  }
  __device__ __forceinline__ void issue(int b, int lane, uint64_t pol) {
    if (b < nb) {
      const int p = q0 + b * 32 + lane;
      const bool ok = p < q1;
      const int pp = ok ? p : q0;
      const uint32_t s = (uint32_t)__cvta_generic_to_shared(base + (b % RING) * kSlotBytes);
      cp_async4(s + lane * 4, crd + pp, ok ? 4 : 0, pol);
      if constexpr (sizeof(T) == 8)
        cp_async8(s + 128 + lane * 8, vals + pp, ok ? 8 : 0, pol);
      else
        cp_async4(s + 128 + lane * 4, vals + pp, ok ? 4 : 0, pol);
    }
    cp_async_commit();
  }
  __device__ __forceinline__ void prologue(int lane, uint64_t pol) {
#pragma unroll
    for (int b = 0; b < RING - 1; ++b) issue(b, lane, pol);
  }
  // make batch b readable by the whole warp (issues batch b+RING-1)
  __device__ __forceinline__ void acquire(int b, int lane, uint64_t pol) {
    issue(b + RING - 1, lane, pol);
    cp_async_wait<RING - 1>();
    __syncwarp();
  }
  // all lanes are done reading batch b's slot
  __device__ __forceinline__ void release() { __syncwarp(); }
};


// 256-bit read-only loads (LDG.E.256): a lane's 32 B run is one whole sector,
// so a warp's request touches each sector once.  Two 16 B loads at a 32 B
// lane stride request every sector twice (once per half), which doubles the
// L1TEX traffic of an 8-float-per-lane row read.
__device__ __forceinline__ void ld256_nc(const float* p, float* r) {
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
               : "l"(p));
}
__device__ __forceinline__ void ld256_nc(const double* p, double* r) {
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3]) : "l"(p));
}
__device__ __forceinline__ void ld256_nc_hint(const float* p, float* r, uint64_t pol) {
  asm volatile("ld.global.nc.L2::cache_hint.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
               : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
               : "l"(p), "l"(pol));
}
__device__ __forceinline__ void ld256_nc_hint(const double* p, double* r, uint64_t pol) {
  asm volatile("ld.global.nc.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
               : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3])
               : "l"(p), "l"(pol));
}

// cp.async.bulk.prefetch.L2: pull [p, p + bytes) into L2 (bytes % 16 == 0, p 16 B aligned)
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void ld256_i32_hint(const int32_t* p, int* r, uint64_t pol) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.s32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "l"(p), "l"(pol));
}

#ifndef SPX_FRAG_LD256
#define SPX_FRAG_LD256 1
#endif

// 16 B / 8 B vectors <-> T elements through register bit casts (no type-punned
// stores into the per-lane arrays, which force them into local memory for fp64)
template <typename T>
__device__ __forceinline__ void unpack16(T* d, const float4& q) {
  if constexpr (sizeof(T) == 4) {
    d[0] = q.x; d[1] = q.y; d[2] = q.z; d[3] = q.w;
  } else {
    d[0] = __hiloint2double(__float_as_int(q.y), __float_as_int(q.x));
    d[1] = __hiloint2double(__float_as_int(q.w), __float_as_int(q.z));
  }
}
template <typename T>
__device__ __forceinline__ float4 pack16(const T* s) {
  if constexpr (sizeof(T) == 4) {
    return make_float4(s[0], s[1], s[2], s[3]);
  } else {
    return make_float4(__int_as_float(__double2loint(s[0])), __int_as_float(__double2hiint(s[0])),
                       __int_as_float(__double2loint(s[1])), __int_as_float(__double2hiint(s[1])));
  }
}
template <typename T>
__device__ __forceinline__ void unpack8(T* d, const float2& q) {
  if constexpr (sizeof(T) == 4) {
    d[0] = q.x; d[1] = q.y;
  } else {
    d[0] = __hiloint2double(__float_as_int(q.y), __float_as_int(q.x));
  }
}
template <typename T>
__device__ __forceinline__ float2 pack8(const T* s) {
  if constexpr (sizeof(T) == 4) {
    return make_float2(s[0], s[1]);
  } else {
    return make_float2(__int_as_float(__double2loint(s[0])), __int_as_float(__double2hiint(s[0])));
  }
}

// ---------------------------------------------------------------------------
// Per-lane row fragments: a lane owns VPL values of a dense row.
// CONTIG: lane owns columns [lane*VPL, lane*VPL+VPL) -> vector loads.
// !CONTIG: lane owns columns {v*32 + lane} (the literal `split(k, dv,
// thread, 32)` mapping of Appendix A.4) with a guard k < ncols.
// ---------------------------------------------------------------------------
template <typename T, int VPL, bool CONTIG>
struct Frag {
  T v[VPL];

  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < VPL; ++i) v[i] = T(0);
  }

  __device__ __forceinline__ void load(const T* __restrict__ row, int lane, int ncols) {
    if (CONTIG) {
      const T* p = row + lane * VPL;
      constexpr int BYTES = VPL * (int)sizeof(T);
      if constexpr (BYTES % 32 == 0 && SPX_FRAG_LD256) {
#pragma unroll
        for (int c = 0; c < BYTES / 32; ++c) ld256_nc(p + c * (32 / sizeof(T)), &v[c * (32 / sizeof(T))]);
      } else if constexpr (BYTES % 16 == 0) {
#pragma unroll
        for (int c = 0; c < BYTES / 16; ++c) {
          float4 q = __ldg(reinterpret_cast<const float4*>(p) + c);
          unpack16(&v[c * (16 / sizeof(T))], q);
        }
      } else if constexpr (BYTES % 8 == 0) {
#pragma unroll
        for (int c = 0; c < BYTES / 8; ++c) {
          float2 q = __ldg(reinterpret_cast<const float2*>(p) + c);
          unpack8(&v[c * (8 / sizeof(T))], q);
        }
      } else {
#pragma unroll
        for (int i = 0; i < VPL; ++i) v[i] = __ldg(p + i);
      }
    } else {
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        int k = i * 32 + lane;
        v[i] = k < ncols ? __ldg(row + k) : T(0);
      }
    }
  }

  // CONTIG: load this lane's VPL contiguous values starting at p (p already
  // includes the lane offset), vectorised
  __device__ __forceinline__ void load_ptr(const T* __restrict__ p) {
    constexpr int BYTES = VPL * (int)sizeof(T);
    if constexpr (BYTES % 32 == 0 && SPX_FRAG_LD256) {
#pragma unroll
      for (int c = 0; c < BYTES / 32; ++c) ld256_nc(p + c * (32 / sizeof(T)), &v[c * (32 / sizeof(T))]);
    } else if constexpr (BYTES % 16 == 0) {
#pragma unroll
      for (int c = 0; c < BYTES / 16; ++c) {
        float4 q = __ldg(reinterpret_cast<const float4*>(p) + c);
        unpack16(&v[c * (16 / sizeof(T))], q);
      }
    } else if constexpr (BYTES % 8 == 0) {
#pragma unroll
      for (int c = 0; c < BYTES / 8; ++c) {
        float2 q = __ldg(reinterpret_cast<const float2*>(p) + c);
        unpack8(&v[c * (8 / sizeof(T))], q);
      }
    } else {
#pragma unroll
      for (int i = 0; i < VPL; ++i) v[i] = __ldg(p + i);
    }
  }

  // load_ptr with an L2 eviction-priority policy on the 16 B vector path
  __device__ __forceinline__ void load_ptr_hint(const T* __restrict__ p, uint64_t pol) {
    constexpr int BYTES = VPL * (int)sizeof(T);
    if constexpr (BYTES % 32 == 0 && SPX_FRAG_LD256) {
#pragma unroll
      for (int c = 0; c < BYTES / 32; ++c) ld256_nc_hint(p + c * (32 / sizeof(T)), &v[c * (32 / sizeof(T))], pol);
    } else if constexpr (BYTES % 16 == 0) {
#pragma unroll
      for (int c = 0; c < BYTES / 16; ++c) {
        float4 q = ld_f4_hint(reinterpret_cast<const float4*>(p) + c, pol);
        unpack16(&v[c * (16 / sizeof(T))], q);
      }
    } else {
      load_ptr(p);
    }
  }

  // gather with an L2 eviction-priority policy (16 B vector path)
  __device__ __forceinline__ void load_hint(const T* __restrict__ row, int lane, int ncols, uint64_t pol) {
    constexpr int BYTES = VPL * (int)sizeof(T);
    if constexpr (CONTIG && BYTES % 32 == 0 && SPX_FRAG_LD256) {
      const T* p = row + lane * VPL;
#pragma unroll
      for (int c = 0; c < BYTES / 32; ++c) ld256_nc_hint(p + c * (32 / sizeof(T)), &v[c * (32 / sizeof(T))], pol);
    } else if constexpr (CONTIG && BYTES % 16 == 0) {
      const T* p = row + lane * VPL;
#pragma unroll
      for (int c = 0; c < BYTES / 16; ++c) {
        float4 q = ld_f4_hint(reinterpret_cast<const float4*>(p) + c, pol);
        unpack16(&v[c * (16 / sizeof(T))], q);
      }
    } else {
      load(row, lane, ncols);
    }
  }

  __device__ __forceinline__ void store_hint(T* __restrict__ row, int lane, int ncols, uint64_t pol) const {
    constexpr int BYTES = VPL * (int)sizeof(T);
    if constexpr (CONTIG && BYTES % 16 == 0) {
      T* p = row + lane * VPL;
#pragma unroll
      for (int c = 0; c < BYTES / 16; ++c)
        st_f4_hint(reinterpret_cast<float4*>(p) + c, pack16(&v[c * (16 / sizeof(T))]),
                   pol);
    } else {
      store(row, lane, ncols);
    }
  }

  __device__ __forceinline__ void store(T* __restrict__ row, int lane, int ncols) const {
    if (CONTIG) {
      T* p = row + lane * VPL;
      constexpr int BYTES = VPL * (int)sizeof(T);
      if constexpr (BYTES % 16 == 0) {
#pragma unroll
        for (int c = 0; c < BYTES / 16; ++c)
          __stcs(reinterpret_cast<float4*>(p) + c,
                 pack16(&v[c * (16 / sizeof(T))]));
      } else if constexpr (BYTES % 8 == 0) {
#pragma unroll
        for (int c = 0; c < BYTES / 8; ++c)
          __stcs(reinterpret_cast<float2*>(p) + c,
                 pack8(&v[c * (8 / sizeof(T))]));
      } else {
#pragma unroll
        for (int i = 0; i < VPL; ++i) __stcs(p + i, v[i]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        int k = i * 32 + lane;
        if (k < ncols) __stcs(row + k, v[i]);
      }
    }
  }

  // read-modify-write add (used by the carry fix-ups; reads via L2 so a
  // value written by another CTA/warp before the barrier/kernel boundary is
  // observed)
  __device__ __forceinline__ void add_into(T* __restrict__ row, int lane, int ncols) const {
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      int k = CONTIG ? lane * VPL + i : i * 32 + lane;
      if (CONTIG || k < ncols) row[k] = __ldcg(row + k) + v[i];
    }
  }

  __device__ __forceinline__ void atomic_add_into(T* __restrict__ row, int lane, int ncols) const {
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      int k = CONTIG ? lane * VPL + i : i * 32 + lane;
      if (CONTIG || k < ncols) atomicAdd(row + k, v[i]);
    }
  }

  // shared-memory staging uses the same per-lane layout as global memory
  __device__ __forceinline__ void store_smem(T* row, int lane) const {
#pragma unroll
    for (int i = 0; i < VPL; ++i) row[CONTIG ? lane * VPL + i : i * 32 + lane] = v[i];
  }
  __device__ __forceinline__ void add_smem(const T* row, int lane) {
#pragma unroll
    for (int i = 0; i < VPL; ++i) v[i] += row[CONTIG ? lane * VPL + i : i * 32 + lane];
  }

  __device__ __forceinline__ void fma(T s, const Frag& b) {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000
    if constexpr (sizeof(T) == 4 && VPL % 2 == 0) {
      // packed FFMA2: half the issue slots of scalar FFMA, same rounding
      const float2 ss = make_float2(s, s);
#pragma unroll
      for (int i = 0; i < VPL; i += 2) {
        const float2 r = __ffma2_rn(ss, make_float2(b.v[i], b.v[i + 1]), make_float2(v[i], v[i + 1]));
        v[i] = r.x;
        v[i + 1] = r.y;
      }
    } else
#endif
    {
#pragma unroll
      for (int i = 0; i < VPL; ++i) v[i] = s * b.v[i] + v[i];
    }
  }
};

// ---------------------------------------------------------------------------
// Searches over nondecreasing int32 arrays (pos).
// ---------------------------------------------------------------------------

// ir.py:178-190 SearchSegment: largest s in [lo,hi) with arr[s] <= key,
// clamped into [lo, hi).
__device__ __forceinline__ int64_t search_segment(const int32_t* __restrict__ arr, int64_t lo,
                                                  int64_t hi, int64_t key) {
  if (hi <= lo) return lo;
  int64_t a = lo, b = hi;  // find first index with arr[idx] > key in [lo,hi)
  while (a < b) {
    int64_t mid = (a + b) >> 1;
    if ((int64_t)__ldg(arr + mid) <= key) a = mid + 1;
    else b = mid;
  }
  int64_t s = a - 1;
  return s < lo ? lo : s;
}

// first s in [lo,hi) with arr[s] >= key, else hi  (ir.py:193-205 semantics)
__device__ __forceinline__ int64_t lower_bound(const int32_t* __restrict__ arr, int64_t lo,
                                               int64_t hi, int64_t key) {
  int64_t a = lo, b = hi;
  while (a < b) {
    int64_t mid = (a + b) >> 1;
    if ((int64_t)__ldg(arr + mid) < key) a = mid + 1;
    else b = mid;
  }
  return a;
}

// Warp-cooperative 32-ary SearchSegment: every lane returns the same result.
// ceil(log32(hi-lo)) dependent steps instead of log2 (4 steps for 1M rows).
__device__ __forceinline__ int64_t warp_search_segment(const int32_t* __restrict__ arr, int64_t lo,
                                                       int64_t hi, int64_t key, int lane) {
  if (hi <= lo) return lo;
  int64_t a = lo, b = hi;  // answer in [a, b) if arr[a] <= key
  while (b - a > 32) {
    int64_t stride = (b - a + 31) >> 5;
    int64_t idx = a + (int64_t)lane * stride;
    bool ok = idx < b && (int64_t)__ldg(arr + idx) <= key;
    unsigned m = __ballot_sync(kFull, ok);
    if (m == 0) return lo == a ? lo : a;  // clamp: nothing <= key
    int last = 31 - __clz(m);
    int64_t na = a + (int64_t)last * stride;
    int64_t nb = na + stride < b ? na + stride : b;
    a = na;
    b = nb;
  }
  int64_t idx = a + lane;
  bool ok = idx < b && (int64_t)__ldg(arr + idx) <= key;
  unsigned m = __ballot_sync(kFull, ok);
  if (m == 0) return a;
  return a + (31 - __clz(m));
}

// Per-warp cache of 32 consecutive row ends pos[base+1 .. base+32] held one
// per lane, so row tracking ("step: while-advance over pos boundaries",
// SPEC.md:364) costs a shuffle instead of a dependent global load.
struct RowEndCache {
  int64_t base;
  int32_t mine;
  __device__ __forceinline__ void fill(const int32_t* __restrict__ pos, int64_t r, int64_t nseg, int lane) {
    base = r;
    int64_t idx = r + 1 + lane;
    mine = __ldg(pos + (idx < nseg ? idx : nseg));
  }
  // end of segment r (= pos[r+1]); r must be >= base
  __device__ __forceinline__ int64_t end(const int32_t* __restrict__ pos, int64_t r, int64_t nseg, int lane) {
    if (r - base >= 32) fill(pos, r, nseg, lane);
    return (int64_t)__shfl_sync(kFull, mine, (int)(r - base));
  }
};

}  // namespace spx
