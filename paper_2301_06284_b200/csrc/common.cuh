// common.cuh -- internal helpers of librgnn.so (never shared with oracle/).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <vector>

#include "rgnn.h"

namespace rgnn {

// ---------------------------------------------------------------- errors
rgnn_status set_error(rgnn_status s, const char* fmt, ...);
extern std::atomic<uint64_t> g_launches;

#define RGNN_CUDA_TRY(expr)                                                                  \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess)                                                                   \
      return ::rgnn::set_error(RGNN_E_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #expr,        \
                               cudaGetErrorString(_e));                                      \
  } while (0)

// Every launch goes through this macro: counts it and checks the launch.
#define RGNN_LAUNCH(kernel, grid, block, smem, stream, ...)                                  \
  do {                                                                                       \
    ::rgnn::g_launches.fetch_add(1, std::memory_order_relaxed);                              \
    kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);                              \
    cudaError_t _e = cudaGetLastError();                                                     \
    if (_e != cudaSuccess)                                                                   \
      return ::rgnn::set_error(RGNN_E_CUDA, "%s:%d launch %s: %s", __FILE__, __LINE__,        \
                               #kernel, cudaGetErrorString(_e));                             \
  } while (0)

#define RGNN_TRY(expr)                         \
  do {                                         \
    rgnn_status _s = (expr);                   \
    if (_s != RGNN_OK) return _s;              \
  } while (0)

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x, size_t a = kAlign) { return (x + a - 1) / a * a; }

// Sequential carve of a caller buffer; `size` is accumulated even when base
// is null so the same code computes the required bytes.
struct Carver {
  char* base;
  size_t off = 0;
  explicit Carver(void* b) : base(static_cast<char*>(b)) {}
  template <typename T>
  T* take(size_t count) {
    size_t o = off;
    off = align_up(off + count * sizeof(T));
    return base ? reinterpret_cast<T*>(base + o) : nullptr;
  }
};

constexpr int kTileRows = 128;       // GEMM M tile (rows of Z per tile)
constexpr int kPieceRows = 64;       // HGT backward: run pieces hold <= 64 positions
constexpr int kDefaultSplitCap = 256; // max in-edges per traversal work item
constexpr int kMaxRanks = 8;           // peer-memory communicator: ranks (one GPU each)
constexpr int kMaxPeers = kMaxRanks - 1;
#ifndef RGNN_NARROW_CAP
#define RGNN_NARROW_CAP 16  // measured r02 (aggregate ms, AM / ogbn-mag): 4: 0.617 / 1.898; 8: 0.590 / 1.824; 16: 0.585 / 1.789; 32: 0.584 / 1.822
#endif
constexpr int kNarrowCap = RGNN_NARROW_CAP;  // forward walk: rows with <= this many in-edges go one per lane group

// Work item of the destination walk: one CSR row, or one chunk of a long row.
struct Item {
  int32_t row;   // local row i (v = dst_begin + i)
  int32_t q0;    // first slot
  int32_t q1;    // one past the last slot
  int32_t part;  // partial-state slot if the row is split, else -1
};
// A split row: its parts are part0 .. part0+nparts-1 in slot order.
struct SplitRow {
  int32_t row, part0, nparts, pad;
};
// GEMM tile: relation r, rows [row0, row1) of the position space.
struct Tile {
  int32_t r, row0, row1, pad;
};

}  // namespace rgnn

struct rgnn_graph {
  int64_t V, V_own, v0, E_in, E_own, J;
  int32_t R, norm, cap;
  int64_t num_tiles, num_items, num_parts, num_split_rows, num_chunks;
  int32_t *perm, *src_s, *dst_s, *seg, *row_ptr, *pos, *et_slot, *run_ptr, *rseg;
  float* inv_c;
  rgnn::Item* items;
  rgnn::SplitRow* split_rows;
  int32_t* empty_rows;  // rows without in-edges (no work item)
  int64_t num_empty;
  // forward walk: rows with deg <= narrow_cap are walked one lane group per row (row-id order,
  // empty rows included); witems = the work items of the other rows (deg > narrow_cap)
  int32_t narrow_cap;
  rgnn::Item* witems;
  int64_t num_witems;
  // compact materialisation (NEXT-1): Z rows per unique (etype, src)
  // dX tables (NEXT-2; RGNN_GRAPH_DX)
  bool has_dx;
  int32_t *run_of_pos, *run_dst, *run_rel, *spos, *srun, *srel, *srow;
  float* sinvc;
  rgnn::Tile* rtiles;
  int64_t num_rtiles;
  rgnn::Item* sitems;      // source work list (rows = global source nodes with out-edges)
  rgnn::SplitRow* ssplit;
  int64_t num_sitems, num_ssplit, num_sparts;
  // node-type segments (HGT)
  bool has_ntype;
  int32_t num_ntypes;
  int32_t *nperm, *ninv;
  rgnn::Tile* ntiles;
  int64_t num_ntiles;
  rgnn::Tile* nchunks;   // dW split-K chunks over the node-type segments (HGT backward)
  int32_t* nchunk_seg;   // [T+1]
  int64_t num_nchunks;
  // run pieces (HGT backward; node types + RGNN_GRAPH_DX): runs cut at multiples of kPieceRows
  bool has_pieces;
  int32_t* piece_ptr;    // [num_pieces + 1] first position of each piece
  int32_t* prseg;        // [R+1] first piece of relation r
  rgnn::Tile* pchunks;   // dW split-K chunks over the pieces
  int32_t* pchunk_seg;   // [R+1] first piece chunk of relation r
  int64_t num_pieces, num_pchunks;
  // aggregate-first RGCN forward (NEXT-4; RGNN_GRAPH_AGGFIRST): GEMM tiles over the pieces, and per
  // CSR slot its piece and weight (1 for the first slot of a piece in its row, else 0)
  bool has_aggfirst;
  rgnn::Tile* ptiles;
  int64_t num_ptiles;
  int32_t* slot_piece;
  float* slot_w;
  bool has_compact;  // compact tables built (COMPACT or AUTO)
  int mat_mode;      // rgnn_materialization requested
  int64_t num_compact, num_ctiles;
  int32_t *crow_of_pos, *zrow_slot, *csrc, *cseg;
  float* invc_slot;
  rgnn::Tile* ctiles;
  rgnn::Tile* tiles;   // 128-row GEMM tiles (never straddle relations)
  rgnn::Tile* chunks;  // dW split-K chunks (never straddle relations)
  int32_t* chunk_seg;  // [R+1] chunks of relation r
  std::vector<int32_t> seg_host, chunk_seg_host;
  int device, num_sms;
};

// Per-call materialisation choice (include/rgnn.h, rgnn_zrows).
inline bool use_compact(const rgnn_graph* g, int model) {
  if (!g->has_compact) return false;
  if (g->mat_mode == RGNN_MAT_COMPACT) return true;
  // RGCN / HGT forward-only use of the rows: compact whenever it saves rows
  // RGAT: compact when U <= 3/4 E_own (measured r02 with the 4-wave backward: AM, U/E = 0.56, 1.83 ->
  // 1.71 ms/step compact; r01 had the cut at 1/2, when AM measured 0.07 ms slower compact)
  return model == RGNN_RGAT ? 4 * g->num_compact <= 3 * g->E_own : g->num_compact < g->E_own;
}


// ---------------------------------------------------------------- device utils
namespace rgnn {

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T>
__device__ __forceinline__ T from_f(float x);
template <>
__device__ __forceinline__ float from_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

// 16-byte vector of T: 4 floats or 8 bf16.
template <typename T>
struct Vec16 {
  static constexpr int kN = 16 / sizeof(T);
  uint4 raw;
  __device__ __forceinline__ void to_float(float* out) const {
    if constexpr (sizeof(T) == 4) {
      out[0] = __uint_as_float(raw.x); out[1] = __uint_as_float(raw.y);
      out[2] = __uint_as_float(raw.z); out[3] = __uint_as_float(raw.w);
    } else {
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float2 f = __bfloat1622float2(h[i]);
        out[2 * i] = f.x; out[2 * i + 1] = f.y;
      }
    }
  }
  __device__ __forceinline__ void from_float(const float* in) {
    if constexpr (sizeof(T) == 4) {
      raw = make_uint4(__float_as_uint(in[0]), __float_as_uint(in[1]), __float_as_uint(in[2]),
                       __float_as_uint(in[3]));
    } else {
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&raw);
#pragma unroll
      for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(in[2 * i], in[2 * i + 1]);
    }
  }
};

__device__ __forceinline__ uint4 ldg_nc16(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ldg16(const void* p) { return __ldg(reinterpret_cast<const uint4*>(p)); }
__device__ __forceinline__ void stg16(void* p, uint4 v) { *reinterpret_cast<uint4*>(p) = v; }

template <int W>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum of a split row's parts in a fixed order: one block per split row; warp w
// sums parts w, w+8, ... then warp 0 adds the 8 warp sums in warp order.
template <int K, typename TO = float>
__device__ __forceinline__ void merge_parts(const float* __restrict__ part, int32_t part0, int32_t nparts, TO* out,
                                            bool add) {
  constexpr int KL = K / 32;
  __shared__ float red[8][K];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  float acc[KL];
#pragma unroll
  for (int i = 0; i < KL; ++i) acc[i] = 0.f;
  for (int32_t t = wp; t < nparts; t += 8) {
    const float* pr = part + (size_t)(part0 + t) * K + lane;
#pragma unroll
    for (int i = 0; i < KL; ++i) acc[i] += pr[32 * i];
  }
#pragma unroll
  for (int i = 0; i < KL; ++i) red[wp][lane + 32 * i] = acc[i];
  __syncthreads();
  if (wp == 0) {
#pragma unroll
    for (int i = 0; i < KL; ++i) {
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) s += red[w][lane + 32 * i];
      if constexpr (sizeof(TO) == 4) {
        if (add) out[lane + 32 * i] += s;
        else out[lane + 32 * i] = s;
      } else {
        out[lane + 32 * i] = from_f<TO>(s);  // bf16 rows (no accumulation)
      }
    }
  }
  __syncthreads();
}

}  // namespace rgnn

// Host-side entry points shared between translation units.
namespace rgnn {
void* profile_begin(const char* name, cudaStream_t s);
void profile_end(void* tok, cudaStream_t s);
// RAII phase scope: events around everything launched in the scope.
struct Phase {
  void* tok;
  cudaStream_t s;
  Phase(const char* name, cudaStream_t st) : tok(profile_begin(name, st)), s(st) {}
  ~Phase() { profile_end(tok, s); }
};
rgnn_status scan_exclusive(const int32_t* in, int32_t* out, int64_t n, int32_t* total, void* scratch,
                           size_t scratch_bytes, cudaStream_t s);
size_t scan_scratch_bytes(int64_t n);
// n_dev (optional): the number of items is *n_dev (device; <= n), read by the kernels -- the grid
// and scratch are sized for n, so no host synchronisation is needed to learn the count.
rgnn_status radix_sort_pairs(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt, int64_t n,
                             int bits, void* scratch, size_t scratch_bytes, cudaStream_t s, bool* result_in_alt, const int32_t* n_dev = nullptr);
size_t radix_scratch_bytes(int64_t n);
}  // namespace rgnn
