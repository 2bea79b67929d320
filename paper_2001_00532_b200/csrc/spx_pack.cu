// Device-side pack: COO -> the reference's coordinate hierarchy on the GPU
// (SURVEY.md §8(f) row 1), bit-exact with spindle.tensors.pack
// (tensors.py:212-258) and CooTensor.normalized (tensors.py:83-90):
//
//   1. keys:    linearised coordinate key = ((c0*d1 + c1)*d2 + c2)...,
//               bounds check (validate, tensors.py:75-81), idx = input order
//   2. sort:    stable LSD radix sort of (key, idx) -- equal keys keep their
//               input order, so duplicates fold left to right as the dict in
//               normalized() does
//   3. unique:  run starts; each run's values summed sequentially from +0.0
//               in input order (`merged.get(c, 0.0) + value`)
//   4. levels:  per level, the prefix-change flag of the sorted unique
//               entries; Dense: slot = parent*dim + c; Compressed: slot =
//               running count of first entries, crd = c at first entries,
//               pos[p] = #first entries whose parent < p (the add.at/cumsum
//               of tensors.py:241-243)
//   5. vals:    zeros(parent_count) with the folded values at the leaf slots
//
// Every array is caller-allocated (the Python host in formats.py sizes them
// between phases from the counts this file reports); nothing here allocates.
#include <cmath>
#include <utility>

#include "spx_common.cuh"

namespace spx {
namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;  // 2048

// ---------------------------------------------------------------------------
// Exclusive scan of int64 (recursive over tile sums).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t* s_warp, int64_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    int64_t w = lane < nw ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(kFull, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) s_warp[lane] = w;
  }
  __syncthreads();
  total = s_warp[(blockDim.x >> 5) - 1];
  const int64_t before = warp > 0 ? s_warp[warp - 1] : 0;
  __syncthreads();
  return before + x - v;
}

// Single-pass scan with decoupled look-back: tiles are taken in launch order
// from a counter, each publishes its aggregate, then its inclusive prefix once
// the predecessors' prefixes are known (status word = flag << 62 | value;
// flag 1 = aggregate, 2 = inclusive).  One read and one write of the data,
// against two of each for the recursive tile-sum scan (cfg2 pack: the 12.5M-entry
// radix offsets x 4 passes plus the 50M-entry run and level flags).
constexpr uint64_t kStAgg = 1ull << 62, kStIncl = 2ull << 62, kStMask = (1ull << 62) - 1;

__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(kScanThreads) scan_lookback_kernel(const int64_t* __restrict__ in,
                                                                     int64_t* __restrict__ out, int64_t n,
                                                                     unsigned long long* __restrict__ status,
                                                                     unsigned int* __restrict__ tile_ctr) {
  __shared__ int64_t s_warp[32];
  __shared__ int64_t s_prefix;
  __shared__ unsigned int s_tile;
  __shared__ int64_t s_x[kScanTile];  // warp-striped <-> thread-blocked transpose
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int wl = threadIdx.x & 31, wbase = (threadIdx.x >> 5) * 32 * kScanItems;
  const int64_t gw = tile * kScanTile + wbase;  // this warp's 32 * kScanItems elements
  // coalesced loads (element k*32 + lane of the warp's run), then each thread
  // takes kScanItems consecutive elements from shared memory
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t g = gw + k * 32 + wl;
    s_x[wbase + k * 32 + wl] = g < n ? in[g] : 0;
  }
  __syncwarp();
  int64_t v[kScanItems];
  int64_t t = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = s_x[wbase + wl * kScanItems + k];
    t += v[k];
  }
  int64_t total;
  int64_t run = block_exclusive_scan(t, s_warp, total);
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int64_t excl = 0;
    if (tile == 0) {
      if (lane == 0) st_release(status, kStIncl | (unsigned long long)total);
    } else {
      if (lane == 0) st_release(status + tile, kStAgg | (unsigned long long)total);
      int64_t j = tile - 1;
      while (true) {
        const int64_t idx = j - lane;
        unsigned long long st;
        do {
          st = idx >= 0 ? ld_acquire(status + idx) : kStIncl;
        } while (__any_sync(kFull, (st >> 62) == 0));
        const unsigned incl = __ballot_sync(kFull, (st >> 62) == 2);
        const int stop = incl ? __ffs(incl) - 1 : 31;  // the nearest inclusive prefix ends the walk
        int64_t x = lane <= stop ? (int64_t)(st & kStMask) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
        excl += x;
        if (incl) break;
        j -= 32;
      }
      if (lane == 0) st_release(status + tile, kStIncl | (unsigned long long)(excl + total));
    }
    if (lane == 0) s_prefix = excl;
  }
  __syncthreads();
  run += s_prefix;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    s_x[wbase + wl * kScanItems + k] = run;
    run += v[k];
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t g = gw + k * 32 + wl;
    if (g < n) out[g] = s_x[wbase + k * 32 + wl];
  }
}

size_t scan_ws_bytes(int64_t n) {
  const int64_t tiles = ceil_div(n > 0 ? n : 1, kScanTile);
  return (size_t)(tiles + 1) * sizeof(unsigned long long) + 256;
}

// out[i] = sum(in[0..i)) ; returns SPX status.  ws holds the tile status words
// and the tile counter.
int exclusive_scan(const int64_t* in, int64_t* out, int64_t n, int64_t* ws, cudaStream_t s) {
  if (n <= 0) return SPX_OK;
  const int64_t tiles = ceil_div(n, kScanTile);
  unsigned long long* status = reinterpret_cast<unsigned long long*>(ws);
  unsigned int* ctr = reinterpret_cast<unsigned int*>(status + tiles);
  if (int e = check_cuda(cudaMemsetAsync(ws, 0, (size_t)tiles * 8 + 8, s), "memset")) return e;
  scan_lookback_kernel<<<(unsigned)tiles, kScanThreads, 0, s>>>(in, out, n, status, ctr);
  count_launch();
  return check_cuda(cudaGetLastError(), "scan_lookback_kernel");
}

// ---------------------------------------------------------------------------
// Stable LSD radix sort of (uint64 key, uint32 idx), kRadixBits-bit digits.
// ---------------------------------------------------------------------------
constexpr int kSortThreads = 256;
constexpr int kSortRounds = 16;
constexpr int kSortTile = kSortThreads * kSortRounds;  // 4096 keys per tile
#ifndef SPX_RADIX_BITS
#define SPX_RADIX_BITS 10  // 40-bit cfg2 keys: 4 passes (8-bit digits: 5)
#endif
constexpr int kRadixBits = SPX_RADIX_BITS;
constexpr int kBins = 1 << kRadixBits;
constexpr uint64_t kDigitMask = (uint64_t)kBins - 1;
constexpr int kDPT = kBins / kSortThreads;  // digits per thread in the tile scans
static_assert(kBins % kSortThreads == 0, "whole digits per thread");

__global__ void __launch_bounds__(kSortThreads) radix_hist_kernel(const uint64_t* __restrict__ keys, int64_t n,
                                                                  int shift, int64_t ntiles,
                                                                  int64_t* __restrict__ hist) {
  __shared__ int s_hist[kBins];
#pragma unroll
  for (int j = 0; j < kDPT; ++j) s_hist[j * kSortThreads + threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kSortTile;
#pragma unroll 4
  for (int r = 0; r < kSortRounds; ++r) {
    const int64_t i = base + (int64_t)r * kSortThreads + threadIdx.x;
    if (i < n) atomicAdd(&s_hist[(int)((keys[i] >> shift) & kDigitMask)], 1);
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kDPT; ++j) {
    const int d = j * kSortThreads + threadIdx.x;
    hist[(int64_t)d * ntiles + blockIdx.x] = s_hist[d];  // digit-major
  }
}

// Stable scatter through shared memory.  Element order inside a tile is
// warp-major (warp w owns tile elements [w*512, w*512+512), loaded 32 at a
// time, coalesced).  Pass 1 ranks every key inside its warp by digit
// (__match_any_sync per round plus a per-warp running count); a block scan
// over (digit, warp) turns the counts into tile-local positions, so pass 2
// places the tile in shared memory sorted by digit, and pass 3 writes it out
// in that order: consecutive threads store consecutive slots of one digit's
// bucket, whole sectors instead of one scattered 8 B and 4 B store per key
// (the previous direct scatter: 0.93 ms per pass at cfg2).
constexpr int kScatterSmem = kSortTile * 12 + (kSortThreads / 32) * kBins * 4 + kBins * 8 + kBins * 4;

__global__ void __launch_bounds__(kSortThreads) radix_scatter_kernel(
    const uint64_t* __restrict__ keys, const uint32_t* __restrict__ idx, int64_t n, int shift, int64_t ntiles,
    const int64_t* __restrict__ offs, uint64_t* __restrict__ keys_out, uint32_t* __restrict__ idx_out) {
  constexpr int NW = kSortThreads / 32;
  constexpr int PER_WARP = kSortTile / NW;  // 512
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* s_keys = reinterpret_cast<uint64_t*>(smem_raw);
  uint32_t* s_idx = reinterpret_cast<uint32_t*>(s_keys + kSortTile);
  int* s_wcnt = reinterpret_cast<int*>(s_idx + kSortTile);        // [NW][kBins]
  int64_t* s_gbase = reinterpret_cast<int64_t*>(s_wcnt + NW * kBins);  // [kBins] global bucket base
  int* s_dstart = reinterpret_cast<int*>(s_gbase + kBins);          // [kBins] tile-local digit start
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t base = (int64_t)blockIdx.x * kSortTile;
  const int tile_n = (int)min((int64_t)kSortTile, n - base);
  for (int j = threadIdx.x; j < NW * kBins; j += kSortThreads) s_wcnt[j] = 0;
#pragma unroll
  for (int j = 0; j < kDPT; ++j) {
    const int d = j * kSortThreads + threadIdx.x;
    s_gbase[d] = offs[(int64_t)d * ntiles + blockIdx.x];
  }
  __syncthreads();
  // pass 1: load, rank inside the warp
  constexpr int R = PER_WARP / 32;  // 16 rounds
  uint64_t k[R];
  uint32_t v[R];
  int rk[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int t = warp * PER_WARP + r * 32 + lane;
    const bool ok = t < tile_n;
    k[r] = ok ? keys[base + t] : 0;
    v[r] = ok ? idx[base + t] : 0;
    const int d = ok ? (int)((k[r] >> shift) & kDigitMask) : kBins;  // kBins: no digit
    const unsigned peers = __match_any_sync(kFull, d);
    const int before = __popc(peers & lt);
    int cnt = 0;
    if (ok) cnt = s_wcnt[warp * kBins + d];
    rk[r] = cnt + before;
    __syncwarp();
    if (ok && before == 0) s_wcnt[warp * kBins + d] = cnt + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // (digit, warp) counts -> tile-local positions; thread t owns digits
  // [t*kDPT, t*kDPT + kDPT)
  {
    int tot[kDPT];
    int mine = 0;
#pragma unroll
    for (int j = 0; j < kDPT; ++j) {
      const int d = threadIdx.x * kDPT + j;
      tot[j] = 0;
#pragma unroll
      for (int w = 0; w < NW; ++w) tot[j] += s_wcnt[w * kBins + d];
      mine += tot[j];
    }
    // block exclusive scan of the per-thread sums
    int x = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    __shared__ int s_wsum[NW];
    if (lane == 31) s_wsum[warp] = x;
    __syncthreads();
    int wpre = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) wpre += (w < warp) ? s_wsum[w] : 0;
    int start = wpre + x - mine;
#pragma unroll
    for (int j = 0; j < kDPT; ++j) {
      const int d = threadIdx.x * kDPT + j;
      s_dstart[d] = start;
      int acc = start;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const int c = s_wcnt[w * kBins + d];
        s_wcnt[w * kBins + d] = acc;
        acc += c;
      }
      start += tot[j];
    }
  }
  __syncthreads();
  // pass 2: place the tile in shared memory sorted by digit
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int t = warp * PER_WARP + r * 32 + lane;
    if (t < tile_n) {
      const int d = (int)((k[r] >> shift) & kDigitMask);
      const int pos = s_wcnt[warp * kBins + d] + rk[r];
      s_keys[pos] = k[r];
      s_idx[pos] = v[r];
    }
  }
  __syncthreads();
  // pass 3: write out in sorted order (runs of one digit are contiguous)
  for (int t = threadIdx.x; t < tile_n; t += kSortThreads) {
    const uint64_t kk = s_keys[t];
    const int d = (int)((kk >> shift) & kDigitMask);
    const int64_t dst = s_gbase[d] + (t - s_dstart[d]);
    keys_out[dst] = kk;
    idx_out[dst] = s_idx[t];
  }
}

// Workspace carve-up of spx_pack_sort (one definition for sizing and use).
struct PackLayout {
  size_t dcoords, keys, idx, keys2, idx2, flags, ex, hist, offs, scan, total;
};
PackLayout pack_layout(int64_t n) {
  PackLayout L;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t at = off;
    off += (bytes + 255) & ~(size_t)255;
    return at;
  };
  const size_t nn = (size_t)(n > 0 ? n : 1);
  const int64_t ntiles = ceil_div(n > 0 ? n : 1, kSortTile);
  L.dcoords = take(8 * sizeof(void*));
  L.keys = take(nn * 8);
  L.idx = take(nn * 4);
  L.keys2 = take(nn * 8);
  L.idx2 = take(nn * 4);
  L.flags = take(nn * 8);
  L.ex = take(nn * 8);
  L.hist = take((size_t)kBins * ntiles * 8);
  L.offs = take((size_t)kBins * ntiles * 8);
  L.scan = take(scan_ws_bytes((int64_t)nn > kBins * ntiles ? (int64_t)nn : kBins * ntiles));
  L.total = off;
  return L;
}

// ---------------------------------------------------------------------------
// pack phases
// ---------------------------------------------------------------------------
struct DimsArg {
  int64_t d[8];
  int order;
};

__global__ void pack_keys_kernel(DimsArg dims, const int32_t* const* __restrict__ coords, int64_t stride,
                                 int64_t n, uint64_t* __restrict__ keys, uint32_t* __restrict__ idx,
                                 unsigned long long* __restrict__ first_bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t k = 0;
  bool bad = false;
#pragma unroll
  for (int l = 0; l < 8; ++l) {  // static indices: DimsArg stays in the parameter bank
    if (l < dims.order) {
      const int64_t c = coords[l][i * stride];
      bad |= c < 0 || c >= dims.d[l];
      k = k * (uint64_t)dims.d[l] + (uint64_t)c;
    }
  }
  keys[i] = k;
  idx[i] = (uint32_t)i;
  if (bad) atomicMin(first_bad, (unsigned long long)i);
}

// flags[i] = 1 at the first entry of each equal-key run
__global__ void run_flags_kernel(const uint64_t* __restrict__ keys, int64_t n, int64_t* __restrict__ flags) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flags[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// run starts: fold the run's values in input order from +0.0 and emit the
// unique entry's per-level coordinates (original input coordinates of the
// run's first element)
__global__ void unique_fold_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ idx,
                                   const int64_t* __restrict__ flags, const int64_t* __restrict__ ex, int64_t n,
                                   const double* __restrict__ vals, DimsArg dims, int32_t* __restrict__ ucoords,
                                   double* __restrict__ uvals, int64_t* __restrict__ nuniq) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i == n - 1) *nuniq = ex[i] + flags[i];
  if (!flags[i]) return;
  const int64_t u = ex[i];
  const uint64_t key = keys[i];
  double acc = 0.0;
  int64_t j = i;
  do {
    acc = acc + vals[idx[j]];
    ++j;
  } while (j < n && keys[j] == key);
  uvals[u] = acc;
  // the key is the row-major linearisation of the (validated) coordinates,
  // so they decode from it instead of being gathered from the inputs
  uint64_t rest = key;
#pragma unroll
  for (int l = 7; l >= 0; --l) {
    if (l < dims.order) {
      const uint64_t dl = (uint64_t)dims.d[l];
      const uint64_t q = rest / dl;
      ucoords[(int64_t)l * n + u] = (int32_t)(rest - q * dl);
      rest = q;
    }
  }
}

// prefix-change flags for level L: diff |= (c_L[i] != c_L[i-1]); diff[0] = 1
__global__ void level_flags_kernel(const int32_t* __restrict__ c, int64_t n, int64_t* __restrict__ diff) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i == 0) diff[0] = 1;
  else if (c[i] != c[i - 1]) diff[i] = 1;
}

__global__ void dense_slot_kernel(const int32_t* __restrict__ c, int64_t n, int64_t dim, int64_t* __restrict__ slot) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) slot[i] = slot[i] * dim + c[i];
}

// compressed level: ex = exclusive scan of diff.  slot_new = ex + diff - 1;
// first entries write crd and the compacted parent
__global__ void compressed_fill_kernel(const int32_t* __restrict__ c, const int64_t* __restrict__ diff,
                                       const int64_t* __restrict__ ex, int64_t n, int64_t* __restrict__ slot,
                                       int32_t* __restrict__ crd_out, int64_t* __restrict__ cpar) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t k = ex[i] + diff[i] - 1;
  if (diff[i]) {
    crd_out[k] = c[i];
    cpar[k] = slot[i];
  }
  slot[i] = k;
}

// pos[p] = #{k : cpar[k] < p} for p in [0, parent_count]
__global__ void pos_fill_kernel(const int64_t* __restrict__ cpar, int64_t count, int64_t parent_count,
                                int32_t* __restrict__ pos) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p > parent_count) return;
  int64_t lo = 0, hi = count;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (cpar[mid] < p) lo = mid + 1;
    else hi = mid;
  }
  pos[p] = (int32_t)lo;
}

__global__ void count_kernel(const int64_t* __restrict__ ex, const int64_t* __restrict__ flags, int64_t n,
                             int64_t* __restrict__ out) {
  *out = ex[n - 1] + flags[n - 1];
}

__global__ void vals_scatter_kernel(const int64_t* __restrict__ slot, const double* __restrict__ uvals, int64_t n,
                                    double* __restrict__ out_f64, float* __restrict__ out_f32) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (out_f64) out_f64[slot[i]] = uvals[i];
  else out_f32[slot[i]] = (float)uvals[i];
}

unsigned blocks_for(int64_t n) { return (unsigned)ceil_div(n > 0 ? n : 1, 256); }

}  // namespace
}  // namespace spx

using namespace spx;

extern "C" {

size_t spx_pack_workspace_size(int64_t n, int32_t order) {
  if (n < 0 || order < 1 || order > 8) return 0;
  return pack_layout(n).total;
}

int spx_pack_sort_strided(const int32_t* const* coords_host, int64_t coord_stride, int32_t order,
                          const int64_t* dims, int64_t n, const double* vals, void* ws, size_t ws_bytes,
                          int32_t* ucoords, double* uvals, int64_t* info, void* stream) {
  if (coord_stride < 1) return fail(SPX_E_ARG, "spx_pack_sort: coordinate stride %lld", (long long)coord_stride);
  if (order < 1 || order > 8 || n < 0 || !dims || !info) return fail(SPX_E_ARG, "spx_pack_sort: bad arguments");
  if (n > 0 && (!coords_host || !vals || !ucoords || !uvals)) return fail(SPX_E_ARG, "spx_pack_sort: null buffer");
  if (n > (int64_t)UINT32_MAX) return fail(SPX_E_UNSUPPORTED, "spx_pack_sort: more than 2^32 entries");
  if (ws_bytes < spx_pack_workspace_size(n, order) || !ws) return fail(SPX_E_WORKSPACE, "pack workspace too small");
  DimsArg da;
  da.order = order;
  double logsize = 0.0;
  for (int l = 0; l < order; ++l) {
    if (dims[l] < 1) return fail(SPX_E_ARG, "spx_pack_sort: dimension %d is %lld", l, (long long)dims[l]);
    da.d[l] = dims[l];
    logsize += log2((double)dims[l]);
  }
  if (logsize > 63.0) return fail(SPX_E_UNSUPPORTED, "spx_pack_sort: coordinate space exceeds 2^63 keys");
  int bits = 0;
  {
    uint64_t total = 1;
    for (int l = 0; l < order; ++l) total *= (uint64_t)dims[l];
    while (bits < 64 && (total - 1) >> bits) ++bits;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // info[0] = unique count, info[1] = first out-of-bounds input index (or -1)
  if (int e = check_cuda(cudaMemsetAsync(info, 0xff, 2 * sizeof(int64_t), s), "memset")) return e;
  if (n == 0) return check_cuda(cudaMemsetAsync(info, 0, sizeof(int64_t), s), "memset");

  const PackLayout L = pack_layout(n);
  char* w = static_cast<char*>(ws);
  const int32_t** dcoords = reinterpret_cast<const int32_t**>(w + L.dcoords);
  uint64_t* keys = reinterpret_cast<uint64_t*>(w + L.keys);
  uint32_t* idx = reinterpret_cast<uint32_t*>(w + L.idx);
  uint64_t* keys2 = reinterpret_cast<uint64_t*>(w + L.keys2);
  uint32_t* idx2 = reinterpret_cast<uint32_t*>(w + L.idx2);
  int64_t* flags = reinterpret_cast<int64_t*>(w + L.flags);
  int64_t* ex = reinterpret_cast<int64_t*>(w + L.ex);
  const int64_t ntiles = ceil_div(n, kSortTile);
  int64_t* hist = reinterpret_cast<int64_t*>(w + L.hist);
  int64_t* offs = reinterpret_cast<int64_t*>(w + L.offs);
  int64_t* scan_ws = reinterpret_cast<int64_t*>(w + L.scan);
  if (int e = check_cuda(cudaMemcpyAsync(dcoords, coords_host, order * sizeof(void*), cudaMemcpyHostToDevice, s),
                         "cudaMemcpyAsync"))
    return e;
  pack_keys_kernel<<<blocks_for(n), 256, 0, s>>>(da, dcoords, coord_stride, n, keys, idx,
                                                 reinterpret_cast<unsigned long long*>(info + 1));
  count_launch();
  if (int e = check_cuda(cudaGetLastError(), "pack_keys_kernel")) return e;
  if (int e = check_cuda(cudaFuncSetAttribute(radix_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              kScatterSmem),
                         "cudaFuncSetAttribute"))
    return e;
  for (int shift = 0; shift < bits; shift += kRadixBits) {
    radix_hist_kernel<<<(unsigned)ntiles, kSortThreads, 0, s>>>(keys, n, shift, ntiles, hist);
    count_launch();
    if (int e = check_cuda(cudaGetLastError(), "radix_hist_kernel")) return e;
    if (int e = exclusive_scan(hist, offs, (int64_t)kBins * ntiles, scan_ws, s)) return e;
    radix_scatter_kernel<<<(unsigned)ntiles, kSortThreads, kScatterSmem, s>>>(keys, idx, n, shift, ntiles, offs,
                                                                              keys2, idx2);
    count_launch();
    if (int e = check_cuda(cudaGetLastError(), "radix_scatter_kernel")) return e;
    std::swap(keys, keys2);
    std::swap(idx, idx2);
  }
  run_flags_kernel<<<blocks_for(n), 256, 0, s>>>(keys, n, flags);
  count_launch();
  if (int e = exclusive_scan(flags, ex, n, scan_ws, s)) return e;
  unique_fold_kernel<<<blocks_for(n), 256, 0, s>>>(keys, idx, flags, ex, n, vals, da, ucoords, uvals, info);
  count_launch();
  return check_cuda(cudaGetLastError(), "unique_fold_kernel");
}

int spx_pack_sort(const int32_t* const* coords_host, int32_t order, const int64_t* dims, int64_t n,
                  const double* vals, void* ws, size_t ws_bytes, int32_t* ucoords, double* uvals, int64_t* info,
                  void* stream) {
  return spx_pack_sort_strided(coords_host, 1, order, dims, n, vals, ws, ws_bytes, ucoords, uvals, info, stream);
}

int spx_pack_level(const int32_t* ucoord, int64_t nu, int32_t compressed, int64_t dim, int64_t parent_count,
                   int64_t* diff, int64_t* slot, int64_t* ex, void* ws, size_t ws_bytes, int64_t* count_out,
                   void* stream) {
  if (nu < 0 || (nu > 0 && (!ucoord || !diff || !slot))) return fail(SPX_E_ARG, "spx_pack_level: bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (nu == 0) return count_out ? check_cuda(cudaMemsetAsync(count_out, 0, 8, s), "memset") : SPX_OK;
  level_flags_kernel<<<blocks_for(nu), 256, 0, s>>>(ucoord, nu, diff);
  count_launch();
  if (int e = check_cuda(cudaGetLastError(), "level_flags_kernel")) return e;
  if (!compressed) {
    dense_slot_kernel<<<blocks_for(nu), 256, 0, s>>>(ucoord, nu, dim, slot);
    count_launch();
    return check_cuda(cudaGetLastError(), "dense_slot_kernel");
  }
  if (!ex || !count_out || ws_bytes < scan_ws_bytes(nu)) return fail(SPX_E_WORKSPACE, "pack level workspace");
  if (int e = exclusive_scan(diff, ex, nu, static_cast<int64_t*>(ws), s)) return e;
  count_kernel<<<1, 1, 0, s>>>(ex, diff, nu, count_out);
  count_launch();
  (void)parent_count;
  return check_cuda(cudaGetLastError(), "count_kernel");
}

size_t spx_pack_level_workspace_size(int64_t nu) { return scan_ws_bytes(nu); }

int spx_pack_level_fill(const int32_t* ucoord, int64_t nu, const int64_t* diff, const int64_t* ex, int64_t* slot,
                        int64_t count, int64_t parent_count, int32_t* crd_out, int32_t* pos_out, int64_t* cpar,
                        void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!pos_out) return fail(SPX_E_ARG, "spx_pack_level_fill: null pos");
  if (nu > 0) {
    compressed_fill_kernel<<<blocks_for(nu), 256, 0, s>>>(ucoord, diff, ex, nu, slot, crd_out, cpar);
    count_launch();
    if (int e = check_cuda(cudaGetLastError(), "compressed_fill_kernel")) return e;
  }
  pos_fill_kernel<<<blocks_for(parent_count + 1), 256, 0, s>>>(cpar, nu > 0 ? count : 0, parent_count, pos_out);
  count_launch();
  return check_cuda(cudaGetLastError(), "pos_fill_kernel");
}

int spx_pack_vals(const int64_t* slot, const double* uvals, int64_t nu, void* vals_out, int32_t dtype,
                  void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (nu == 0) return SPX_OK;
  vals_scatter_kernel<<<blocks_for(nu), 256, 0, s>>>(slot, uvals, nu,
                                                     dtype == SPX_F64 ? static_cast<double*>(vals_out) : nullptr,
                                                     dtype == SPX_F32 ? static_cast<float*>(vals_out) : nullptr);
  count_launch();
  return check_cuda(cudaGetLastError(), "vals_scatter_kernel");
}

}  // extern "C"
