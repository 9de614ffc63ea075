// primitives.cu -- errors, launch counter, device-wide exclusive scan and a
// stable LSD radix sort (key, value) used by the graph preprocessing
// (DESIGN.md Sec. 6 "a0"; Sec. 3.6 P:756 "converting COO to CSR",
// P:845 "presorted to enable segment MM").  All integer, bit-exact.
#include <stdarg.h>
#include <stdio.h>

#include <algorithm>

#include "common.cuh"

namespace rgnn {

std::atomic<uint64_t> g_launches{0};
static thread_local char t_err[512] = "";

rgnn_status set_error(rgnn_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(t_err, sizeof(t_err), fmt, ap);
  va_end(ap);
  return s;
}

// ---------------------------------------------------------------- scan
// Three-phase reduce-then-scan over tiles of 4096 int32 (512 threads x 8).
constexpr int kScanThreads = 512, kScanItems = 8, kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int32_t block_exclusive_sum(int32_t v, int32_t* s_warp, int32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int32_t w = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0;
    int32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int32_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < (int)(blockDim.x >> 5)) s_warp[lane] = wi - w;
    if (lane == 31) s_warp[32] = wi;
  }
  __syncthreads();
  int32_t r = s_warp[warp] + x - v;
  if (total) *total = s_warp[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const int32_t* __restrict__ in, int64_t n,
                                                              int32_t* __restrict__ bsum) {
  __shared__ int32_t s_warp[33];
  int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int32_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i)
    if (base + i < n) s += in[base + i];
  int32_t tot;
  block_exclusive_sum(s, s_warp, &tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

// Single block: exclusive scan of bsum[0..nb) in place; total -> *total.
__global__ void __launch_bounds__(1024) k_scan_blocks(int32_t* __restrict__ bsum, int64_t nb,
                                                      int32_t* __restrict__ total) {
  __shared__ int32_t s_warp[33];
  int32_t carry = 0;
  for (int64_t b0 = 0; b0 < nb; b0 += 1024) {
    int64_t i = b0 + threadIdx.x;
    int32_t v = i < nb ? bsum[i] : 0;
    int32_t tot;
    int32_t ex = block_exclusive_sum(v, s_warp, &tot);
    if (i < nb) bsum[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_down(const int32_t* in, int32_t* out, int64_t n,
                                                            const int32_t* __restrict__ bsum) {
  __shared__ int32_t s_warp[33];
  int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int32_t v[kScanItems];
  int32_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = base + i < n ? in[base + i] : 0;
    s += v[i];
  }
  int32_t run = block_exclusive_sum(s, s_warp, nullptr) + bsum[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) out[base + i] = run;
    run += v[i];
  }
}

__global__ void k_set_scalar(int32_t* p, int32_t v) { *p = v; }

size_t scan_scratch_bytes(int64_t n) {
  int64_t nb = (n + kScanTile - 1) / kScanTile;
  return align_up(sizeof(int32_t) * (size_t)(nb + 1));
}

// out[i] = sum_{j<i} in[j]; *total = sum (device pointer, may be null).  in may alias out.
rgnn_status scan_exclusive(const int32_t* in, int32_t* out, int64_t n, int32_t* total, void* scratch,
                           size_t scratch_bytes, cudaStream_t s) {
  if (n == 0) {
    if (total) RGNN_LAUNCH(k_set_scalar, 1, 1, 0, s, total, 0);
    return RGNN_OK;
  }
  int64_t nb = (n + kScanTile - 1) / kScanTile;
  if (scratch_bytes < scan_scratch_bytes(n)) return set_error(RGNN_E_WORKSPACE, "scan scratch too small");
  int32_t* bsum = static_cast<int32_t*>(scratch);
  RGNN_LAUNCH(k_scan_reduce, (unsigned)nb, kScanThreads, 0, s, in, n, bsum);
  RGNN_LAUNCH(k_scan_blocks, 1, 1024, 0, s, bsum, nb, total);
  RGNN_LAUNCH(k_scan_down, (unsigned)nb, kScanThreads, 0, s, in, out, n, bsum);
  return RGNN_OK;
}

// ---------------------------------------------------------------- radix sort
// Stable LSD radix sort, 8-bit digits.  Per pass: (1) per-tile digit
// histogram, stored digit-major [256][nb]; (2) exclusive scan of that array
// gives every (digit, tile) its global offset; (3) per tile, a stable rank of
// each item among equal digits (warp match + per-warp prefix, rounds in
// input order) and a scatter.  Stability: ranks follow the input order.
constexpr int kRsThreads = 256, kRsRounds = 8, kRsTile = kRsThreads * kRsRounds, kRsWarps = kRsThreads / 32;

__global__ void __launch_bounds__(kRsThreads) k_rs_hist(const uint32_t* __restrict__ keys, int64_t n, int shift,
                                                        int64_t nb, int32_t* __restrict__ counts,
                                                        const int32_t* __restrict__ n_dev) {
  if (n_dev) n = min(n, (int64_t)*n_dev);
  __shared__ int32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * kRsTile;
#pragma unroll
  for (int j = 0; j < kRsRounds; ++j) {
    int64_t i = base + j * kRsThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[(keys[i] >> shift) & 255u], 1);
  }
  __syncthreads();
  counts[(int64_t)threadIdx.x * nb + blockIdx.x] = h[threadIdx.x];
}

// Scatter of one tile: the stable per-digit ranks (warp match + per-warp prefix, rounds in input
// order) place every item at its digit-sorted position inside the tile in shared memory first;
// the tile then leaves in that order, so the items of one digit -- consecutive in the output --
// are written by consecutive threads (coalesced runs instead of one scattered 4-byte store each).
__global__ void __launch_bounds__(kRsThreads) k_rs_scatter(const uint32_t* __restrict__ keys,
                                                           const uint32_t* __restrict__ vals, int64_t n, int shift,
                                                           int64_t nb, const int32_t* __restrict__ offsets,
                                                           uint32_t* __restrict__ keys_out,
                                                           uint32_t* __restrict__ vals_out,
                                                           const int32_t* __restrict__ n_dev) {
  if (n_dev) n = min(n, (int64_t)*n_dev);
  if ((int64_t)blockIdx.x * kRsTile >= n) return;  // an empty tile (its histogram is zero)
  __shared__ int32_t s_run[256];
  __shared__ int32_t s_goff[256], s_loff[256];
  __shared__ int32_t s_w[kRsWarps][256];
  __shared__ uint32_t s_k[kRsTile], s_v[kRsTile];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t base = (int64_t)blockIdx.x * kRsTile;
  const int tile_n = (int)min((int64_t)kRsTile, n - base);
  {  // this tile's digit counts (from the scanned offsets) -> local exclusive offsets
    const int64_t idx = (int64_t)t * nb + blockIdx.x;
    const int32_t go = offsets[idx];
    const int32_t cnt = (idx + 1 < 256 * nb ? offsets[idx + 1] : (int32_t)n) - go;
    s_goff[t] = go;
    int32_t x = cnt;  // block-wide exclusive scan of the 256 counts
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_w[0][warp] = x;
    __syncthreads();
    int32_t wofs = 0;
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) wofs += w < warp ? s_w[0][w] : 0;
    s_loff[t] = wofs + x - cnt;
    s_run[t] = wofs + x - cnt;
    __syncthreads();
  }
  const uint32_t lt = (1u << lane) - 1u;
  for (int j = 0; j < kRsRounds; ++j) {
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) s_w[w][t] = 0;
    __syncthreads();
    int64_t i = base + j * kRsThreads + t;
    bool valid = i < n;
    uint32_t k = valid ? keys[i] : 0u;
    uint32_t v = valid ? vals[i] : 0u;
    uint32_t d = valid ? ((k >> shift) & 255u) : 256u;
    uint32_t peers = __match_any_sync(0xffffffffu, d);
    int rank = __popc(peers & lt);
    if (valid && rank == 0) s_w[warp][d] = __popc(peers);
    __syncthreads();
    {  // per digit: exclusive prefix over warps, then advance the running (tile-local) offset
      int32_t run = s_run[t];
#pragma unroll
      for (int w = 0; w < kRsWarps; ++w) {
        int32_t c = s_w[w][t];
        s_w[w][t] = run;
        run += c;
      }
      s_run[t] = run;
    }
    __syncthreads();
    if (valid) {
      const int32_t o = s_w[warp][d] + rank;
      s_k[o] = k;
      s_v[o] = v;
    }
    __syncthreads();
  }
  for (int i = t; i < tile_n; i += kRsThreads) {  // the tile in digit order: coalesced per digit run
    const uint32_t k = s_k[i];
    const uint32_t d = (k >> shift) & 255u;
    const int32_t o = s_goff[d] + (i - s_loff[d]);
    keys_out[o] = k;
    vals_out[o] = s_v[i];
  }
}

size_t radix_scratch_bytes(int64_t n) {
  int64_t nb = (n + kRsTile - 1) / kRsTile;
  size_t cnt = (size_t)256 * (size_t)(nb > 0 ? nb : 1);
  return align_up(sizeof(int32_t) * cnt) + scan_scratch_bytes((int64_t)cnt);
}

rgnn_status radix_sort_pairs(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt, int64_t n,
                             int bits, void* scratch, size_t scratch_bytes, cudaStream_t s, bool* result_in_alt,
                             const int32_t* n_dev) {
  *result_in_alt = false;
  if (n <= 1 || bits <= 0) return RGNN_OK;
  if (scratch_bytes < radix_scratch_bytes(n)) return set_error(RGNN_E_WORKSPACE, "radix scratch too small");
  int64_t nb = (n + kRsTile - 1) / kRsTile;
  int32_t* counts = static_cast<int32_t*>(scratch);
  char* scan_scr = static_cast<char*>(scratch) + align_up(sizeof(int32_t) * 256 * (size_t)nb);
  size_t scan_bytes = scratch_bytes - align_up(sizeof(int32_t) * 256 * (size_t)nb);
  uint32_t *ki = keys, *vi = vals, *ko = keys_alt, *vo = vals_alt;
  for (int shift = 0; shift < bits; shift += 8) {
    RGNN_LAUNCH(k_rs_hist, (unsigned)nb, kRsThreads, 0, s, ki, n, shift, nb, counts, n_dev);
    RGNN_TRY(scan_exclusive(counts, counts, 256 * nb, nullptr, scan_scr, scan_bytes, s));
    RGNN_LAUNCH(k_rs_scatter, (unsigned)nb, kRsThreads, 0, s, ki, vi, n, shift, nb, counts, ko, vo, n_dev);
    uint32_t* t;
    t = ki; ki = ko; ko = t;
    t = vi; vi = vo; vo = t;
    *result_in_alt = !*result_in_alt;
  }
  return RGNN_OK;
}

}  // namespace rgnn

extern "C" {

const char* rgnn_last_error(void) { return rgnn::t_err; }
const char* rgnn_version(void) { return "rgnn-b200 0.1 (sm_100a)"; }
uint64_t rgnn_launch_count(void) { return rgnn::g_launches.load(); }

rgnn_status rgnn_partition_dst(int64_t V, const int64_t* indeg_prefix, int nparts, int64_t* bounds) {
  if (!indeg_prefix || !bounds || nparts < 1 || V < 0)
    return rgnn::set_error(RGNN_E_INVALID_ARG, "rgnn_partition_dst: bad arguments");
  const int64_t E = indeg_prefix[V];
  bounds[0] = 0;
  int64_t v = 0;
  for (int k = 1; k < nparts; ++k) {
    // the cut whose prefix is closest to k*E/P (ties -> smaller v); integer
    // arithmetic on 2*P*prefix vs 2*k*E, so the cut is deterministic
    const int64_t t2 = 2 * k * E;  // target * 2P
    while (v < V && 2 * nparts * indeg_prefix[v + 1] <= t2) ++v;
    if (v < V) {
      int64_t below = t2 - 2 * nparts * indeg_prefix[v], above = 2 * nparts * indeg_prefix[v + 1] - t2;
      if (above < below) ++v;
    }
    bounds[k] = std::max(v, bounds[k - 1]);
  }
  bounds[nparts] = V;
  return RGNN_OK;
}

}  // extern "C"
