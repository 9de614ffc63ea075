// graph.cu -- graph preprocessing (DESIGN.md Sec. 6 step a0).
//
// PAPER.md Sec. 3.6 P:756 emits a preprocessing list ("transposition,
// converting COO to CSR, etc.") run before training/inference, and P:845
// presorts for segment MM.  Here, on the device, for the owned dst range:
//   validate ids (smallest bad edge via atomicMin) -> keep owned edges in
//   input order -> stable radix sort by key = etype*V_own + (dst-v0) ->
//   perm / src_s / dst_s, relation segments seg[R+1], CSR-by-dst row_ptr and
//   pos (second stable sort of positions by dst), et_slot, (etype,dst) runs
//   with 1/c_{v,r}, the destination-walk work list (rows longer than `cap`
//   split into chunks), then -- after the single host sync -- the 128-row
//   GEMM tile table and the dW split-K chunk table (host built, uploaded).
// Tie-break contract = DESIGN.md reading O14 (bit-exact vs the oracle).
#include <algorithm>
#include <chrono>
#include <cstdio>

#include "common.cuh"

namespace rgnn {

struct Counters {
  int32_t bad_edge, bad_node, E_own, J, num_items, num_parts, num_split_rows, num_empty, num_compact;
  int32_t num_sitems, num_sparts, num_ssplit;  // dX source work list
  int32_t num_pieces;                          // HGT backward run pieces
  int32_t bad_csr;                             // CSR input: smallest row v with a bad row_ptr entry
  int32_t num_witems;                          // forward walk: items of rows with deg > narrow cap
};

__global__ void k_init_counters(Counters* c, int32_t big) {
  c->bad_edge = big; c->bad_node = big; c->E_own = 0; c->J = 0;
  c->num_items = 0; c->num_parts = 0; c->num_split_rows = 0; c->num_empty = 0; c->num_compact = 0;
  c->num_sitems = 0; c->num_sparts = 0; c->num_ssplit = 0; c->num_pieces = 0; c->bad_csr = big; c->num_witems = 0;
}

// Run pieces (HGT backward, aggregate-first RGCN): every (etype, dst) run cut every kPieceRows
// positions from its start, so a piece holds <= kPieceRows consecutive positions of one run and
// depends only on the run (a dst-range shard cuts its runs the same way).  Pieces are numbered in
// position order; piece_ptr[i] is the first position of piece i.
__global__ void k_piece_counts(int64_t J, const int32_t* __restrict__ run_ptr, int32_t* __restrict__ cnt) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < J; j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = run_ptr[j], e = run_ptr[j + 1];
    cnt[j] = (e - s + kPieceRows - 1) / kPieceRows;
  }
}
__global__ void k_piece_fill(int64_t J, const int32_t* __restrict__ run_ptr, const int32_t* __restrict__ pofs,
                             int32_t* __restrict__ piece_ptr) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < J; j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = run_ptr[j], e = run_ptr[j + 1];
    int32_t id = pofs[j];
    for (int32_t b = s; b < e; b += kPieceRows) piece_ptr[id++] = b;
  }
}
// Aggregate-first RGCN (NEXT-4): piece of every position (pieces hold <= kPieceRows positions),
// then per CSR slot q its piece and weight 1 for the first slot of each piece within the row (the
// row's slots list each piece's positions in a block), 0 for the others -- the walk then adds every
// piece product once.
__global__ void k_piece_mark(int64_t np_max, const Counters* c, const int32_t* __restrict__ piece_ptr,
                             int32_t* __restrict__ piece_of_pos) {
  const int64_t np = c->num_pieces;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np && i < np_max;
       i += (int64_t)gridDim.x * blockDim.x)
    for (int32_t p = piece_ptr[i]; p < piece_ptr[i + 1]; ++p) piece_of_pos[p] = (int32_t)i;
}
__global__ void k_piece_slots(int64_t n, const int32_t* __restrict__ pos, const int32_t* __restrict__ piece_of_pos,
                              const int32_t* __restrict__ dst_s, int32_t* __restrict__ slot_piece,
                              float* __restrict__ slot_w) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = pos[q], pc = piece_of_pos[p];
    bool first = q == 0;
    if (!first) {
      const int32_t pp = pos[q - 1];
      first = dst_s[pp] != dst_s[p] || piece_of_pos[pp] != pc;
    }
    slot_piece[q] = pc;
    slot_w[q] = first ? 1.f : 0.f;
  }
}
__global__ void k_piece_seg(int32_t R, int64_t J, const int32_t* __restrict__ rseg, const int32_t* __restrict__ pofs,
                            const Counters* c, int32_t* __restrict__ prseg, int32_t* __restrict__ piece_ptr,
                            int32_t E_own) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r <= R; r += gridDim.x * blockDim.x)
    prseg[r] = rseg[r] < J ? pofs[rseg[r]] : c->num_pieces;
  if (blockIdx.x == 0 && threadIdx.x == 0) piece_ptr[c->num_pieces] = E_own;
}

// CSR-by-dst input: row_ptr must be 0 at v = 0, non-decreasing and E at v = V; the smallest
// offending index (v, or V for row_ptr[V] != E) is reported, before the expansion is used.
__global__ void k_validate_csr(const int32_t* __restrict__ row_ptr, int64_t V, int64_t E, Counters* c) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v <= V; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t a = row_ptr[v];
    const bool bad = v == 0 ? a != 0 : (a < row_ptr[v - 1] || (v == V && a != E));
    if (bad) atomicMin(&c->bad_csr, (int32_t)v);
  }
}
// CSR-by-dst input: dst of every edge from row_ptr (one warp per row).  The loop is clamped to
// [0, E) so a malformed row_ptr never writes outside dst; k_validate_csr rejects it afterwards.
__global__ void k_expand_csr(const int32_t* __restrict__ row_ptr, int64_t V, int64_t E, int32_t* __restrict__ dst) {
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  for (int64_t v = w; v < V; v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t lo = max((int64_t)row_ptr[v], (int64_t)0), hi = min((int64_t)row_ptr[v + 1], E);
    for (int64_t e = lo + lane; e < hi; e += 32) dst[e] = (int32_t)v;
  }
}

__global__ void k_validate(int64_t E, int64_t V, int32_t R, const int32_t* __restrict__ src,
                           const int32_t* __restrict__ dst, const int32_t* __restrict__ et, Counters* c) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    int32_t s = src[e], d = dst[e], r = et[e];
    if (s < 0 || s >= V || d < 0 || d >= V || r < 0 || r >= R) atomicMin(&c->bad_edge, (int32_t)e);
  }
}

__global__ void k_validate_ntype(int64_t V, int32_t T, const int32_t* __restrict__ nt, Counters* c) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x)
    if (nt[v] < 0 || nt[v] >= T) atomicMin(&c->bad_node, (int32_t)v);
}

__global__ void k_own_flags(int64_t E, const int32_t* __restrict__ dst, int64_t v0, int64_t v1,
                            int32_t* __restrict__ flag) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
    flag[e] = (dst[e] >= v0 && dst[e] < v1) ? 1 : 0;
}

// Compact owned edges in input order: key = etype*V_own + (dst - v0), val = edge id.
__global__ void k_own_scatter(int64_t E, const int32_t* __restrict__ dst, const int32_t* __restrict__ et,
                              int64_t v0, int64_t v1, int64_t V_own, const int32_t* __restrict__ slot,
                              uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    int32_t d = dst[e];
    if (d >= v0 && d < v1) {
      int32_t o = slot[e];
      keys[o] = (uint32_t)((int64_t)et[e] * V_own + (d - v0));
      vals[o] = (uint32_t)e;
    }
  }
}

// After the (etype,dst) sort: perm, src_s, dst_s, run heads and histograms.
__global__ void k_after_sort(int64_t n, const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                             const int32_t* __restrict__ src, int64_t V_own, int32_t* __restrict__ perm,
                             int32_t* __restrict__ src_s, int32_t* __restrict__ dst_s, int32_t* __restrict__ et_s,
                             int32_t* __restrict__ head) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    uint32_t k = keys[p];
    int32_t e = (int32_t)vals[p];
    int32_t r = (int32_t)(k / (uint32_t)V_own);
    int32_t i = (int32_t)(k - (uint32_t)r * (uint32_t)V_own);
    perm[p] = e;
    src_s[p] = src[e];
    dst_s[p] = i;
    et_s[p] = r;
    head[p] = (p == 0 || keys[p - 1] != k) ? 1 : 0;
  }
}

// Bin boundaries of a sorted key array: out[b] = first index q with key[q] >= b,
// for b in [0, nbins]: one binary search per bin (balanced even when long runs
// of empty bins exist, e.g. node types that receive no edges).
template <typename KeyT>
__global__ void k_bounds(int64_t n, const KeyT* __restrict__ key, int64_t nbins, int32_t* __restrict__ out,
                         const int32_t* __restrict__ n_dev = nullptr) {
  if (n_dev) n = *n_dev;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b <= nbins; b += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)key[mid] < b) lo = mid + 1; else hi = mid;
    }
    out[b] = (int32_t)lo;
  }
}

__global__ void k_copy_u32_to_i32(int64_t n, const uint32_t* __restrict__ a, int32_t* __restrict__ b) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
    b[p] = (int32_t)a[p];
}

__global__ void k_iota_keys(int64_t n, const int32_t* __restrict__ dst_s, uint32_t* __restrict__ k,
                            uint32_t* __restrict__ v) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    k[p] = (uint32_t)dst_s[p];
    v[p] = (uint32_t)p;
  }
}

__global__ void k_slots(int64_t n, const uint32_t* __restrict__ sorted_pos, const int32_t* __restrict__ et_s,
                        int32_t* __restrict__ pos, int32_t* __restrict__ et_slot) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    int32_t p = (int32_t)sorted_pos[q];
    pos[q] = p;
    et_slot[q] = et_s[p];
  }
}

// CSR from the runs.  Keys: the local dst of each run (j < J, J on the device).
__global__ void k_run_keys(int64_t n, const Counters* c, const int32_t* __restrict__ run_ptr,
                           const int32_t* __restrict__ dst_s, uint32_t* __restrict__ k, uint32_t* __restrict__ v) {
  const int64_t J = c->J;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < J && j < n; j += (int64_t)gridDim.x * blockDim.x) {
    k[j] = (uint32_t)dst_s[run_ptr[j]];
    v[j] = (uint32_t)j;
  }
}
// Length of the i-th run in dst order (0 past J: the scan then gives every sorted run its first
// slot), and the inverse permutation run -> sorted index.
__global__ void k_run_lens(int64_t n, const Counters* c, const uint32_t* __restrict__ sorted_run,
                           const int32_t* __restrict__ run_ptr, int32_t* __restrict__ len, uint32_t* __restrict__ inv) {
  const int64_t J = c->J;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < J) {
      const uint32_t j = sorted_run[i];
      len[i] = run_ptr[j + 1] - run_ptr[j];
      inv[j] = (uint32_t)i;
    } else {
      len[i] = 0;
    }
  }
}
// row_ptr[v] = first slot of the first sorted run whose dst is >= v (E_own past the last run).
__global__ void k_row_ptr_runs(int64_t V_own, const Counters* c, const uint32_t* __restrict__ sorted_dst,
                               const int32_t* __restrict__ q0, int32_t* __restrict__ row_ptr) {
  const int64_t J = c->J;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v <= V_own; v += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = J;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)sorted_dst[mid] < v) lo = mid + 1; else hi = mid;
    }
    row_ptr[v] = lo < J ? q0[lo] : c->E_own;
  }
}
// pos[q] for every position p: its run j, the run's sorted index and first slot, plus the offset.
__global__ void k_slots_runs(int64_t n, const int32_t* __restrict__ head, const int32_t* __restrict__ run_ex,
                             const int32_t* __restrict__ run_ptr, const uint32_t* __restrict__ inv,
                             const int32_t* __restrict__ q0, int32_t* __restrict__ pos) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t j = run_ex[p] + head[p] - 1;
    pos[q0[inv[j]] + (int32_t)(p - run_ptr[j])] = (int32_t)p;
  }
}
__global__ void k_slot_et(int64_t n, const int32_t* __restrict__ pos, const int32_t* __restrict__ et_s,
                          int32_t* __restrict__ et_slot) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    et_slot[q] = et_s[pos[q]];
}

// Tile t of a segmented table: segment s = the last with first[s] <= t, rows
// [seg[s] + (t - first[s]) * rows, min(+rows, seg[s+1])) -- the host loop it replaces, per entry.
__global__ void k_fill_tiles(int64_t S, const int32_t* __restrict__ seg, const int32_t* __restrict__ first,
                             int64_t rows, int64_t total, Tile* __restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = S;  // first[lo] <= t < first[hi]
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (first[mid] <= t) lo = mid; else hi = mid;
    }
    while (lo + 1 < S && first[lo + 1] <= t) ++lo;  // skip empty segments at the boundary
    const int64_t a = seg[lo] + (t - first[lo]) * rows;
    out[t] = Tile{(int32_t)lo, (int32_t)a, (int32_t)min(a + rows, (int64_t)seg[lo + 1]), 0};
  }
}

// Runs of equal (etype, dst): run_ptr[j] = first position of run j.
__global__ void k_runs(int64_t n, const int32_t* __restrict__ head, const int32_t* __restrict__ run_ex,
                       int32_t* __restrict__ run_ptr) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
    if (head[p]) run_ptr[run_ex[p]] = (int32_t)p;
}

// Runs are in position order and relation r starts at seg[r] with a new run, so
// rseg[r] = number of runs before position seg[r].
__global__ void k_rseg(int32_t R, int64_t n, const int32_t* __restrict__ seg, const int32_t* __restrict__ run_ex,
                       const Counters* c, int32_t* __restrict__ rseg) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r <= R; r += gridDim.x * blockDim.x)
    rseg[r] = seg[r] < n ? run_ex[seg[r]] : c->J;
}

__global__ void k_run_end(const Counters* c, int32_t* run_ptr) { run_ptr[c->J] = c->E_own; }

// 1/c per position (reading O7): relation in-degree = run length; none; or edge_norm[perm[p]].
__global__ void k_inv_c(int64_t n, int norm, const int32_t* __restrict__ head, const int32_t* __restrict__ run_ex,
                        const int32_t* __restrict__ run_ptr, const int32_t* __restrict__ perm,
                        const float* __restrict__ edge_norm, float* __restrict__ inv_c) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    float f;
    if (norm == RGNN_NORM_NONE) {
      f = 1.0f;
    } else if (norm == RGNN_NORM_EDGE) {
      f = edge_norm[perm[p]];
    } else {
      int32_t j = run_ex[p] + head[p] - 1;
      f = 1.0f / (float)(run_ptr[j + 1] - run_ptr[j]);
    }
    inv_c[p] = f;
  }
}

// ---------------------------------------------------------------- node-type segments (D4; HGT)
// nperm[i] = node at type-sorted row i; ninv[u] = row of node u
__global__ void k_node_perm(int64_t V, const uint32_t* __restrict__ sorted_nodes, int32_t* __restrict__ nperm,
                            int32_t* __restrict__ ninv) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t u = (int32_t)sorted_nodes[i];
    nperm[i] = u;
    ninv[u] = (int32_t)i;
  }
}

// ---------------------------------------------------------------- dX tables (NEXT-2)
// run of each position, and the destination / relation of each run
__global__ void k_dx_runs(int64_t n, const int32_t* __restrict__ head, const int32_t* __restrict__ run_ex,
                          const int32_t* __restrict__ dst_s, const int32_t* __restrict__ et_s,
                          int32_t* __restrict__ run_of_pos, int32_t* __restrict__ run_dst, int32_t* __restrict__ run_rel) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t j = run_ex[p] + head[p] - 1;
    if (run_of_pos) run_of_pos[p] = j;
    if (head[p]) {
      run_dst[j] = dst_s[p];
      if (run_rel) run_rel[j] = et_s[p];
    }
  }
}
__global__ void k_keys_i32(int64_t n, const int32_t* __restrict__ key, uint32_t* __restrict__ k,
                           uint32_t* __restrict__ v) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    k[p] = (uint32_t)key[p];
    v[p] = (uint32_t)p;
  }
}
// source-major slots: position, its run, the run's relation, and 1/c
__global__ void k_dx_slots(int64_t n, const uint32_t* __restrict__ sorted_pos, const int32_t* __restrict__ run_of_pos,
                           const int32_t* __restrict__ run_rel, const float* __restrict__ inv_c,
                           int32_t* __restrict__ spos, int32_t* __restrict__ srun, int32_t* __restrict__ srel,
                           float* __restrict__ sinvc) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = (int32_t)sorted_pos[q];
    const int32_t j = run_of_pos[p];
    spos[q] = p;
    srun[q] = j;
    srel[q] = run_rel[j];
    sinvc[q] = inv_c[p];
  }
}

// Work list: rows with more than cap in-edges are split into ceil(deg/cap) chunks;
// rows without in-edges get no item and go to the empty-row list (Y = 0 / self term).
// n_wide (optional): the items of rows with deg > narrow (the forward walk's wide list).
__global__ void k_item_counts(int64_t V_own, const int32_t* __restrict__ row_ptr, int cap, int32_t* __restrict__ n_items,
                              int32_t* __restrict__ n_parts, int32_t* __restrict__ n_split,
                              int32_t* __restrict__ n_empty, int narrow = 0, int32_t* __restrict__ n_wide = nullptr) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < V_own; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t deg = row_ptr[i + 1] - row_ptr[i];
    int32_t c = deg > cap ? (deg + cap - 1) / cap : (deg > 0 ? 1 : 0);
    n_items[i] = c;
    n_parts[i] = c > 1 ? c : 0;
    n_split[i] = c > 1 ? 1 : 0;
    n_empty[i] = deg == 0 ? 1 : 0;
    if (n_wide) n_wide[i] = deg > narrow ? c : 0;
  }
}

__global__ void k_fill_empty(int64_t V_own, const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ empty_ex,
                             int32_t* __restrict__ empty_rows) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < V_own; i += (int64_t)gridDim.x * blockDim.x)
    if (row_ptr[i + 1] == row_ptr[i]) empty_rows[empty_ex[i]] = (int32_t)i;
}

__global__ void k_fill_items(int64_t V_own, const int32_t* __restrict__ row_ptr, int cap,
                             const int32_t* __restrict__ item_ex, const int32_t* __restrict__ part_ex,
                             const int32_t* __restrict__ split_ex, Item* __restrict__ items,
                             SplitRow* __restrict__ split_rows, int narrow = 0,
                             const int32_t* __restrict__ wide_ex = nullptr, Item* __restrict__ witems = nullptr) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < V_own; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t lo = row_ptr[i], hi = row_ptr[i + 1], deg = hi - lo;
    int32_t c = deg > cap ? (deg + cap - 1) / cap : (deg > 0 ? 1 : 0);
    int32_t b = item_ex[i];
    for (int32_t k = 0; k < c; ++k) {
      Item it;
      it.row = (int32_t)i;
      it.q0 = lo + k * cap;
      it.q1 = min(lo + (k + 1) * cap, hi);
      it.part = c > 1 ? part_ex[i] + k : -1;
      if (c == 1) { it.q0 = lo; it.q1 = hi; }
      items[b + k] = it;
      if (witems && deg > narrow) witems[wide_ex[i] + k] = it;
    }
    if (c > 1) {
      SplitRow s;
      s.row = (int32_t)i; s.part0 = part_ex[i]; s.nparts = c; s.pad = 0;
      split_rows[split_ex[i]] = s;
    }
  }
}

// ---------------------------------------------------------------- compact materialisation (NEXT-1)
// Compact rows = unique (etype, src) pairs of the owned edges, numbered
// lexicographically (reading O15; Sec. 3.1.3: "once for each
// (edge type, unique node index) pair ... stored in a CSR-like format").
__global__ void k_ckeys(int64_t n, const int32_t* __restrict__ et_s, const int32_t* __restrict__ src_s, int64_t V,
                        uint32_t* __restrict__ k, uint32_t* __restrict__ v) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    k[p] = (uint32_t)((int64_t)et_s[p] * V + src_s[p]);
    v[p] = (uint32_t)p;
  }
}
__global__ void k_cheads(int64_t n, const uint32_t* __restrict__ k, int32_t* __restrict__ head) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    head[i] = (i == 0 || k[i - 1] != k[i]) ? 1 : 0;
}
__global__ void k_crows(int64_t n, const uint32_t* __restrict__ k, const uint32_t* __restrict__ pidx,
                        const int32_t* __restrict__ head, const int32_t* __restrict__ cex, int64_t V,
                        int32_t* __restrict__ crow_of_pos, int32_t* __restrict__ csrc, int32_t* __restrict__ crel) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = cex[i] + head[i] - 1;
    crow_of_pos[pidx[i]] = c;
    if (head[i]) {
      csrc[c] = (int32_t)(k[i] % (uint32_t)V);
      crel[c] = (int32_t)(k[i] / (uint32_t)V);
    }
  }
}
// slot-ordered views used by the walks: Z row of slot q, and (RGCN) the 1/c of slot q
__global__ void k_cslots(int64_t n, const int32_t* __restrict__ pos, const int32_t* __restrict__ crow_of_pos,
                         const float* __restrict__ inv_c, int32_t* __restrict__ zrow_slot,
                         float* __restrict__ invc_slot) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = pos[q];
    zrow_slot[q] = crow_of_pos[p];
    invc_slot[q] = inv_c[p];
  }
}

static int bits_for(uint64_t maxval) {
  int b = 0;
  while (b < 64 && (maxval >> b) != 0) ++b;
  return b;
}

struct GraphLayout {
  // device storage
  int32_t *perm, *src_s, *dst_s, *seg, *row_ptr, *pos, *et_slot, *run_ptr, *rseg;
  float* inv_c;
  Item *items, *witems;
  SplitRow* split_rows;
  int32_t* empty_rows;
  int32_t *crow_of_pos, *zrow_slot, *csrc, *cseg;
  float* invc_slot;
  Tile* ctiles;
  Tile *tiles, *chunks;
  int32_t* chunk_seg;
  int32_t *run_of_pos, *run_dst, *run_rel, *spos, *srun, *srel, *srow;
  float* sinvc;
  Tile* rtiles;
  Item* sitems;
  SplitRow* ssplit;
  int32_t *nperm, *ninv, *nseg;
  Tile *ntiles, *nchunks;
  int32_t* nchunk_seg;
  int32_t *piece_ptr, *prseg, *pchunk_seg, *slot_piece;
  float* slot_w;
  Tile* ptiles;
  Tile* pchunks;
  size_t dev_bytes;
  // scratch
  Counters* ctr;
  int32_t *dst_tmp, *flags, *head, *run_ex, *et_s, *n_items, *n_parts, *n_split, *n_empty, *n_wide, *rseg_cnt, *crel;
  uint32_t *k0, *v0, *k1, *v1;
  int32_t* tabs;  // tile-table staging: segment bounds and first tiles
  int64_t tabs_ints;
  void* prim;
  size_t prim_bytes, scratch_bytes;
};

// Forward walk: rows with at most this many in-edges (and never split) are walked one lane
// group per row; the choice depends only on the row's degree, so a dst-range shard walks every
// row exactly like one GPU does (pin P14).  RGNN_NARROW_CAP (environment) overrides it for A/B.
static int narrow_cap(const rgnn_graph_desc* d) {
  static const int env = getenv("RGNN_NARROW_CAP") ? atoi(getenv("RGNN_NARROW_CAP")) : -1;
  const int cap = d->row_split_cap > 0 ? d->row_split_cap : kDefaultSplitCap;
  return std::min(env >= 0 ? env : kNarrowCap, cap);
}

static int64_t max_chunks(int64_t E, int32_t R) { (void)E; return 8 * 1024 + 2 * (int64_t)R; }

static GraphLayout layout(const rgnn_graph_desc* d, void* dev, void* scr) {
  GraphLayout L{};
  const int64_t E = d->num_edges, V_own = d->dst_end - d->dst_begin;
  const int32_t R = d->num_etypes;
  const int cap = d->row_split_cap > 0 ? d->row_split_cap : kDefaultSplitCap;
  const int64_t Ec = E > 0 ? E : 1;
  Carver c(dev);
  L.perm = c.take<int32_t>(Ec);
  L.src_s = c.take<int32_t>(Ec);
  L.dst_s = c.take<int32_t>(Ec);
  L.pos = c.take<int32_t>(Ec);
  L.et_slot = c.take<int32_t>(Ec);
  L.inv_c = c.take<float>(Ec);
  L.run_ptr = c.take<int32_t>(Ec + 1);
  L.seg = c.take<int32_t>(R + 1);
  L.rseg = c.take<int32_t>(R + 1);
  L.row_ptr = c.take<int32_t>(V_own + 1);
  L.items = c.take<Item>(V_own + Ec / cap + 1);
  L.split_rows = c.take<SplitRow>(Ec / cap + 1);
  L.empty_rows = c.take<int32_t>(V_own + 1);
  L.witems = c.take<Item>(Ec / (narrow_cap(d) + 1) + Ec / cap + 1);
  const bool cm = d->materialization != RGNN_MAT_VANILLA;
  L.crow_of_pos = c.take<int32_t>(cm ? Ec : 1);
  L.zrow_slot = c.take<int32_t>(cm ? Ec : 1);
  L.invc_slot = c.take<float>(cm ? Ec : 1);
  L.csrc = c.take<int32_t>(cm ? Ec : 1);
  L.cseg = c.take<int32_t>(R + 1);
  L.ctiles = c.take<Tile>(cm ? Ec / kTileRows + R + 1 : 1);
  L.tiles = c.take<Tile>(Ec / kTileRows + R + 1);
  L.chunks = c.take<Tile>(max_chunks(E, R));
  L.chunk_seg = c.take<int32_t>(R + 1);
  const bool dx = (d->flags & RGNN_GRAPH_DX) != 0;
  const int64_t Ex = dx ? Ec : 1;
  L.run_of_pos = c.take<int32_t>(Ex);
  L.run_dst = c.take<int32_t>(Ec);  // always: the RGAT backward's per-run GEMM gathers G rows by it
  L.run_rel = c.take<int32_t>(Ex);
  L.spos = c.take<int32_t>(Ex);
  L.srun = c.take<int32_t>(Ex);
  L.srel = c.take<int32_t>(Ex);
  L.sinvc = c.take<float>(Ex);
  L.srow = c.take<int32_t>(dx ? d->num_nodes + 1 : 1);
  L.rtiles = c.take<Tile>(Ec / kTileRows + R + 1);  // always (see run_dst)
  L.sitems = c.take<Item>(dx ? d->num_nodes + Ec / cap + 1 : 1);
  L.ssplit = c.take<SplitRow>(dx ? Ec / cap + 1 : 1);
  const bool nt = d->ntype != nullptr;
  const int64_t Vn = nt ? std::max<int64_t>(d->num_nodes, 1) : 1;
  L.nperm = c.take<int32_t>(Vn);
  L.ninv = c.take<int32_t>(Vn);
  L.nseg = c.take<int32_t>(nt ? d->num_ntypes + 1 : 1);
  L.ntiles = c.take<Tile>(nt ? Vn / kTileRows + d->num_ntypes + 1 : 1);
  L.nchunks = c.take<Tile>(nt ? Vn / kTileRows + d->num_ntypes + 1 : 1);  // chunks >= 128 rows: <= #ntiles
  L.nchunk_seg = c.take<int32_t>(nt ? d->num_ntypes + 1 : 1);
  const bool af = (d->flags & RGNN_GRAPH_AGGFIRST) != 0;
  const bool pc = (nt && dx) || af;  // run pieces: HGT backward, aggregate-first RGCN
  L.piece_ptr = c.take<int32_t>(pc ? Ec + Ec / kPieceRows + 2 : 1);
  L.prseg = c.take<int32_t>(pc ? R + 1 : 1);
  L.pchunks = c.take<Tile>(pc ? max_chunks(E, R) : 1);
  L.pchunk_seg = c.take<int32_t>(pc ? R + 1 : 1);
  L.ptiles = c.take<Tile>(af ? (Ec + Ec / kPieceRows + 1) / kTileRows + R + 1 : 1);
  L.slot_piece = c.take<int32_t>(af ? Ec : 1);
  L.slot_w = c.take<float>(af ? Ec : 1);
  // tile-table staging ([seg | first] of <= 8 tile tables), in the graph storage: the fill kernels run
  // after the last host synchronisation, so they must not read the caller's scratch
  L.tabs_ints = 2 * 8 * ((int64_t)R + (d->ntype ? d->num_ntypes : 0) + 2);
  L.tabs = c.take<int32_t>(L.tabs_ints);
  L.dev_bytes = c.off;
  Carver s(scr);
  L.ctr = s.take<Counters>(1);
  L.dst_tmp = s.take<int32_t>(d->row_ptr ? Ec : 1);
  L.flags = s.take<int32_t>(Ec + 1);
  L.head = s.take<int32_t>(Ec);
  L.run_ex = s.take<int32_t>(Ec);
  L.et_s = s.take<int32_t>(Ec);
  const int64_t Vw = std::max<int64_t>(V_own, (d->flags & RGNN_GRAPH_DX) ? d->num_nodes : 0);  // work-list rows
  L.n_items = s.take<int32_t>(Vw + 1);
  L.n_parts = s.take<int32_t>(Vw + 1);
  L.n_split = s.take<int32_t>(Vw + 1);
  L.n_empty = s.take<int32_t>(Vw + 1);
  L.n_wide = s.take<int32_t>(V_own + 1);
  L.rseg_cnt = s.take<int32_t>(R + 1);
  L.crel = s.take<int32_t>(d->materialization != RGNN_MAT_VANILLA ? Ec : 1);
  const int64_t Ek = std::max<int64_t>(Ec, d->ntype ? d->num_nodes : 0);  // sort keys: edges, or nodes (types)
  L.k0 = s.take<uint32_t>(Ek);
  L.v0 = s.take<uint32_t>(Ek);
  L.k1 = s.take<uint32_t>(Ek);
  L.v1 = s.take<uint32_t>(Ek);
  L.prim_bytes = std::max(radix_scratch_bytes(Ek), scan_scratch_bytes(std::max<int64_t>(Ek + 1, Vw + 1)));
  L.prim = s.take<char>(L.prim_bytes);
  L.scratch_bytes = s.off;
  return L;
}

static rgnn_status check_desc(const rgnn_graph_desc* d) {
  if (!d) return set_error(RGNN_E_INVALID_ARG, "desc is NULL");
  if (d->num_nodes < 0 || d->num_edges < 0 || d->num_etypes < 1)
    return set_error(RGNN_E_INVALID_ARG, "bad sizes V=%lld E=%lld R=%d", (long long)d->num_nodes,
                     (long long)d->num_edges, d->num_etypes);
  if (d->num_edges >= (int64_t)INT32_MAX || d->num_nodes >= (int64_t)INT32_MAX)
    return set_error(RGNN_E_UNSUPPORTED, "E and V must be < 2^31 (reading O22)");
  if (d->dst_begin < 0 || d->dst_end < d->dst_begin || d->dst_end > d->num_nodes)
    return set_error(RGNN_E_INVALID_ARG, "bad dst range [%lld, %lld)", (long long)d->dst_begin,
                     (long long)d->dst_end);
  int64_t V_own = d->dst_end - d->dst_begin;
  if ((uint64_t)d->num_etypes * (uint64_t)(V_own > 0 ? V_own : 1) > 0xffffffffull)
    return set_error(RGNN_E_UNSUPPORTED, "R * V_own must fit 32 bits (sort key)");
  if (d->num_edges > 0 && (!d->src || !d->etype || (!d->dst && !d->row_ptr)))
    return set_error(RGNN_E_INVALID_ARG, "src/dst/etype must not be NULL");
  if (d->norm < 0 || d->norm > 2) return set_error(RGNN_E_INVALID_ARG, "bad norm %d", d->norm);
  if (d->norm == RGNN_NORM_EDGE && d->num_edges > 0 && !d->edge_norm)
    return set_error(RGNN_E_INVALID_ARG, "edge_norm required for RGNN_NORM_EDGE");
  if (d->ntype && d->num_ntypes < 1) return set_error(RGNN_E_INVALID_ARG, "num_ntypes must be >= 1");
  if (d->row_split_cap < 0) return set_error(RGNN_E_INVALID_ARG, "row_split_cap < 0");
  if (d->materialization != RGNN_MAT_VANILLA && d->materialization != RGNN_MAT_COMPACT &&
      d->materialization != RGNN_MAT_AUTO)
    return set_error(RGNN_E_INVALID_ARG, "bad materialization %d", d->materialization);
  if (d->flags & ~(RGNN_GRAPH_DX | RGNN_GRAPH_AGGFIRST))
    return set_error(RGNN_E_INVALID_ARG, "unknown flags 0x%x", d->flags);
  if (d->materialization != RGNN_MAT_VANILLA &&
      (uint64_t)d->num_etypes * (uint64_t)(d->num_nodes > 0 ? d->num_nodes : 1) > 0xffffffffull)
    return set_error(RGNN_E_UNSUPPORTED, "compact materialisation needs R * V < 2^32 (sort key)");
  return RGNN_OK;
}

static unsigned grid_for(int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32));
}

}  // namespace rgnn

using namespace rgnn;

extern "C" {

rgnn_status rgnn_graph_bytes(const rgnn_graph_desc* d, size_t* dev_bytes, size_t* scratch_bytes) {
  RGNN_TRY(check_desc(d));
  GraphLayout L = layout(d, nullptr, nullptr);
  if (dev_bytes) *dev_bytes = L.dev_bytes;
  if (scratch_bytes) *scratch_bytes = L.scratch_bytes;
  return RGNN_OK;
}

rgnn_status rgnn_graph_create(const rgnn_graph_desc* d, void* dev, size_t dev_bytes, void* scratch,
                              size_t scratch_bytes, void* stream, rgnn_graph** out) {
  RGNN_TRY(check_desc(d));
  if (!out || !dev || !scratch) return set_error(RGNN_E_INVALID_ARG, "NULL buffer or out pointer");
  if (((uintptr_t)dev | (uintptr_t)scratch) % kAlign) return set_error(RGNN_E_INVALID_ARG, "buffers must be 256B aligned");
  GraphLayout need = layout(d, nullptr, nullptr);
  if (dev_bytes < need.dev_bytes || scratch_bytes < need.scratch_bytes)
    return set_error(RGNN_E_WORKSPACE, "graph buffers too small: need dev %zu scratch %zu", need.dev_bytes,
                     need.scratch_bytes);
  GraphLayout L = layout(d, dev, scratch);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t E = d->num_edges, V = d->num_nodes, v0 = d->dst_begin, v1 = d->dst_end, V_own = v1 - v0;
  const int32_t R = d->num_etypes;
  const int cap = d->row_split_cap > 0 ? d->row_split_cap : kDefaultSplitCap;
  const int T = 256;
  // RGNN_PREP_TRACE=1: host time at each synchronisation point (stderr), for the preprocessing profile
  static const bool trace = getenv("RGNN_PREP_TRACE") != nullptr;
  const auto t_start = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (trace)
      fprintf(stderr, "rgnn_graph_create %-28s %8.3f ms\n", what,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count());
  };

  RGNN_LAUNCH(k_init_counters, 1, 1, 0, s, L.ctr, INT32_MAX);
  const int32_t* dst = d->dst;
  if (d->row_ptr) {
    RGNN_LAUNCH(k_validate_csr, grid_for(V + 1), T, 0, s, d->row_ptr, V, E, L.ctr);
    RGNN_LAUNCH(k_expand_csr, grid_for(V * 32), T, 0, s, d->row_ptr, V, E, L.dst_tmp);
    dst = L.dst_tmp;
  }
  if (E > 0) RGNN_LAUNCH(k_validate, grid_for(E), T, 0, s, E, V, R, d->src, dst, d->etype, L.ctr);
  if (d->ntype && V > 0) RGNN_LAUNCH(k_validate_ntype, grid_for(V), T, 0, s, V, d->num_ntypes, d->ntype, L.ctr);
  // Owned edges, compacted in input order.  (These kernels only compare and copy ids, so they are
  // safe on invalid input; the validation flags are read with the owned-edge count -- host sync 1.)
  Counters h{};
  int32_t* E_own_d = &L.ctr->E_own;
  if (E > 0) {
    RGNN_LAUNCH(k_own_flags, grid_for(E), T, 0, s, E, dst, v0, v1, L.flags);
    RGNN_TRY(scan_exclusive(L.flags, L.flags, E, E_own_d, L.prim, L.prim_bytes, s));
    RGNN_LAUNCH(k_own_scatter, grid_for(E), T, 0, s, E, dst, d->etype, v0, v1, V_own, L.flags, L.k0, L.v0);
  }
  RGNN_CUDA_TRY(cudaMemcpyAsync(&h, L.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, s));
  RGNN_CUDA_TRY(cudaStreamSynchronize(s));
  mark("sync 1 (validation, E_own)");
  if (h.bad_csr != INT32_MAX)
    return set_error(RGNN_E_INVALID_ARG, "row_ptr is not a CSR offset array (0 at v=0, non-decreasing, E at v=V): "
                     "first bad entry row_ptr[%d]", h.bad_csr);
  if (h.bad_edge != INT32_MAX)
    return set_error(RGNN_E_RANGE, "edge %d has an id out of range (V=%lld, R=%d)", h.bad_edge, (long long)V, R);
  if (h.bad_node != INT32_MAX)
    return set_error(RGNN_E_RANGE, "node %d has a node type out of range (T=%d)", h.bad_node, d->num_ntypes);
  const int64_t n = h.E_own;

  // Stable sort of owned edges by (etype, dst).
  bool alt = false;
  int kbits = bits_for((uint64_t)R * (uint64_t)(V_own > 0 ? V_own : 1) - 1);
  RGNN_TRY(radix_sort_pairs(L.k0, L.v0, L.k1, L.v1, n, kbits, L.prim, L.prim_bytes, s, &alt));
  uint32_t* keys = alt ? L.k1 : L.k0;
  uint32_t* vals = alt ? L.v1 : L.v0;
  if (n > 0)
    RGNN_LAUNCH(k_after_sort, grid_for(n), T, 0, s, n, keys, vals, d->src, V_own, L.perm, L.src_s, L.dst_s, L.et_s,
                L.head);
  RGNN_LAUNCH(k_bounds<int32_t>, grid_for(R + 1), T, 0, s, n, L.et_s, (int64_t)R, L.seg);
  if (n > 0) {
    // (etype, dst) runs
    RGNN_TRY(scan_exclusive(L.head, L.run_ex, n, &L.ctr->J, L.prim, L.prim_bytes, s));
    RGNN_LAUNCH(k_runs, grid_for(n), T, 0, s, n, L.head, L.run_ex, L.run_ptr);
    RGNN_LAUNCH(k_run_end, 1, 1, 0, s, L.ctr, L.run_ptr);
    // CSR-by-dst from the runs (a stable sort of the J runs by dst instead of the E positions):
    // the runs are in (etype, dst) order, so sorting them stably by dst lists each row's runs in
    // relation order, and each run's positions are consecutive -- the row's positions come out
    // ascending, exactly the order a stable sort of the positions by dst gives (reading O14).
    uint32_t* rk = L.k0; uint32_t* rv = L.v0;
    RGNN_LAUNCH(k_run_keys, grid_for(n), T, 0, s, n, L.ctr, L.run_ptr, L.dst_s, rk, rv);
    RGNN_TRY(radix_sort_pairs(L.k0, L.v0, L.k1, L.v1, n, bits_for((uint64_t)(V_own > 0 ? V_own - 1 : 0)), L.prim,
                              L.prim_bytes, s, &alt, &L.ctr->J));
    uint32_t* sk = alt ? L.k1 : L.k0;  // sorted run dst
    uint32_t* sv = alt ? L.v1 : L.v0;  // sorted run ids
    uint32_t* inv = alt ? L.v0 : L.v1;  // free buffer: sorted index of each run
    int32_t* q0 = L.et_slot;           // scratch until the slots are written: slot offset of each sorted run
    RGNN_LAUNCH(k_run_lens, grid_for(n), T, 0, s, n, L.ctr, sv, L.run_ptr, q0, inv);
    RGNN_TRY(scan_exclusive(q0, q0, n, nullptr, L.prim, L.prim_bytes, s));
    RGNN_LAUNCH(k_row_ptr_runs, grid_for(V_own + 1), T, 0, s, V_own, L.ctr, sk, q0, L.row_ptr);
    RGNN_LAUNCH(k_slots_runs, grid_for(n), T, 0, s, n, L.head, L.run_ex, L.run_ptr, inv, q0, L.pos);
    RGNN_LAUNCH(k_slot_et, grid_for(n), T, 0, s, n, L.pos, L.et_s, L.et_slot);
  }
  if (n == 0) {
    RGNN_LAUNCH(k_bounds<int32_t>, grid_for(V_own + 1), T, 0, s, (int64_t)0, L.et_s, V_own, L.row_ptr);
    RGNN_LAUNCH(k_run_end, 1, 1, 0, s, L.ctr, L.run_ptr);
  }
  RGNN_LAUNCH(k_rseg, (unsigned)((R + 256) / 256), 256, 0, s, R, n, L.seg, L.run_ex, L.ctr, L.rseg);
  if (n > 0)
    RGNN_LAUNCH(k_inv_c, grid_for(n), T, 0, s, n, d->norm, L.head, L.run_ex, L.run_ptr, L.perm, d->edge_norm,
                L.inv_c);
  const bool dx = (d->flags & RGNN_GRAPH_DX) != 0;
  if (n > 0)
    RGNN_LAUNCH(k_dx_runs, grid_for(n), T, 0, s, n, L.head, L.run_ex, L.dst_s, L.et_s, dx ? L.run_of_pos : nullptr,
                L.run_dst, dx ? L.run_rel : nullptr);
  // Destination-walk work list.
  if (V_own > 0) {
    RGNN_LAUNCH(k_item_counts, grid_for(V_own), T, 0, s, V_own, L.row_ptr, cap, L.n_items, L.n_parts, L.n_split,
                L.n_empty, narrow_cap(d), L.n_wide);
    RGNN_TRY(scan_exclusive(L.n_wide, L.n_wide, V_own, &L.ctr->num_witems, L.prim, L.prim_bytes, s));
    RGNN_TRY(scan_exclusive(L.n_empty, L.n_empty, V_own, &L.ctr->num_empty, L.prim, L.prim_bytes, s));
    RGNN_LAUNCH(k_fill_empty, grid_for(V_own), T, 0, s, V_own, L.row_ptr, L.n_empty, L.empty_rows);
    RGNN_TRY(scan_exclusive(L.n_items, L.n_items, V_own, &L.ctr->num_items, L.prim, L.prim_bytes, s));
    RGNN_TRY(scan_exclusive(L.n_parts, L.n_parts, V_own, &L.ctr->num_parts, L.prim, L.prim_bytes, s));
    RGNN_TRY(scan_exclusive(L.n_split, L.n_split, V_own, &L.ctr->num_split_rows, L.prim, L.prim_bytes, s));
    RGNN_LAUNCH(k_fill_items, grid_for(V_own), T, 0, s, V_own, L.row_ptr, cap, L.n_items, L.n_parts, L.n_split,
                L.items, L.split_rows, narrow_cap(d), L.n_wide, L.witems);
  }
  // Compact materialisation: unique (etype, src) rows, lexicographic.
  const bool cm = d->materialization != RGNN_MAT_VANILLA;
  if (cm && n > 0) {
    RGNN_LAUNCH(k_ckeys, grid_for(n), T, 0, s, n, L.et_s, L.src_s, V, L.k0, L.v0);
    RGNN_TRY(radix_sort_pairs(L.k0, L.v0, L.k1, L.v1, n, bits_for((uint64_t)R * (uint64_t)V - 1), L.prim,
                              L.prim_bytes, s, &alt));
    uint32_t* ck = alt ? L.k1 : L.k0;
    uint32_t* cv = alt ? L.v1 : L.v0;
    RGNN_LAUNCH(k_cheads, grid_for(n), T, 0, s, n, ck, L.head);
    RGNN_TRY(scan_exclusive(L.head, L.run_ex, n, &L.ctr->num_compact, L.prim, L.prim_bytes, s));
    RGNN_LAUNCH(k_crows, grid_for(n), T, 0, s, n, ck, cv, L.head, L.run_ex, V, L.crow_of_pos, L.csrc, L.crel);
    RGNN_LAUNCH(k_cslots, grid_for(n), T, 0, s, n, L.pos, L.crow_of_pos, L.inv_c, L.zrow_slot, L.invc_slot);
  }
  // Host sync 2: counts + relation (and compact) segments.
  std::vector<int32_t> seg_h(R + 1), cseg_h(R + 1, 0);
  if (cm)  // compact segments: first compact row of each relation (U counted on the device)
    RGNN_LAUNCH(k_bounds<int32_t>, grid_for(R + 1), T, 0, s, (int64_t)0, L.crel, (int64_t)R, L.cseg,
                &L.ctr->num_compact);
  RGNN_CUDA_TRY(cudaMemcpyAsync(&h, L.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, s));
  RGNN_CUDA_TRY(cudaMemcpyAsync(seg_h.data(), L.seg, sizeof(int32_t) * (R + 1), cudaMemcpyDeviceToHost, s));
  if (cm) RGNN_CUDA_TRY(cudaMemcpyAsync(cseg_h.data(), L.cseg, sizeof(int32_t) * (R + 1), cudaMemcpyDeviceToHost, s));
  RGNN_CUDA_TRY(cudaStreamSynchronize(s));
  mark("sync 2 (counts, segments)");
  // node-type segments (HGT's node-typed linears, D4): stable sort of node ids by type
  std::vector<int32_t> nseg_h;
  if (d->ntype && V > 0) {
    const int32_t NT = d->num_ntypes;
    nseg_h.assign(NT + 1, 0);
    RGNN_LAUNCH(k_keys_i32, grid_for(V), T, 0, s, V, d->ntype, L.k0, L.v0);
    RGNN_TRY(radix_sort_pairs(L.k0, L.v0, L.k1, L.v1, V, bits_for((uint64_t)(NT > 0 ? NT - 1 : 0)), L.prim,
                              L.prim_bytes, s, &alt));
    RGNN_LAUNCH(k_node_perm, grid_for(V), T, 0, s, V, alt ? L.v1 : L.v0, L.nperm, L.ninv);
    RGNN_LAUNCH(k_bounds<uint32_t>, grid_for(NT + 1), T, 0, s, V, alt ? L.k1 : L.k0, (int64_t)NT, L.nseg);
    RGNN_CUDA_TRY(cudaMemcpyAsync(nseg_h.data(), L.nseg, sizeof(int32_t) * (NT + 1), cudaMemcpyDeviceToHost, s));
  }
  std::vector<int32_t> rseg_h(R + 1, 0), prseg_h;
  RGNN_CUDA_TRY(cudaMemcpyAsync(rseg_h.data(), L.rseg, sizeof(int32_t) * (R + 1), cudaMemcpyDeviceToHost, s));
  if (dx) {
    // source-major CSR over the positions (stable: ascending position within a source)
    if (n > 0) {
      RGNN_LAUNCH(k_keys_i32, grid_for(n), T, 0, s, n, L.src_s, L.k0, L.v0);
      RGNN_TRY(radix_sort_pairs(L.k0, L.v0, L.k1, L.v1, n, bits_for((uint64_t)(V > 0 ? V - 1 : 0)), L.prim,
                                L.prim_bytes, s, &alt));
      RGNN_LAUNCH(k_dx_slots, grid_for(n), T, 0, s, n, alt ? L.v1 : L.v0, L.run_of_pos, L.run_rel, L.inv_c, L.spos,
                  L.srun, L.srel, L.sinvc);
    }
    RGNN_LAUNCH(k_bounds<uint32_t>, grid_for(V + 1), T, 0, s, n, alt ? L.k1 : L.k0, V, L.srow);
    // source work list: sources with more than cap out-edges are split (partial sums merged in order)
    if (V > 0) {
      RGNN_LAUNCH(k_item_counts, grid_for(V), T, 0, s, V, L.srow, cap, L.n_items, L.n_parts, L.n_split, L.n_empty);
      RGNN_TRY(scan_exclusive(L.n_items, L.n_items, V, &L.ctr->num_sitems, L.prim, L.prim_bytes, s));
      RGNN_TRY(scan_exclusive(L.n_parts, L.n_parts, V, &L.ctr->num_sparts, L.prim, L.prim_bytes, s));
      RGNN_TRY(scan_exclusive(L.n_split, L.n_split, V, &L.ctr->num_ssplit, L.prim, L.prim_bytes, s));
      RGNN_LAUNCH(k_fill_items, grid_for(V), T, 0, s, V, L.srow, cap, L.n_items, L.n_parts, L.n_split, L.sitems,
                  L.ssplit);
    }
  }
  const bool af = (d->flags & RGNN_GRAPH_AGGFIRST) != 0;
  if ((d->ntype && dx) || af) {
    // run pieces: every (etype, dst) run cut at the multiples of kPieceRows (HGT backward's
    // relation dW GEMMs; the aggregate-first RGCN forward's GEMM rows)
    if (h.J > 0) {
      RGNN_LAUNCH(k_piece_counts, grid_for(h.J), T, 0, s, (int64_t)h.J, L.run_ptr, L.flags);
      RGNN_TRY(scan_exclusive(L.flags, L.flags, h.J, &L.ctr->num_pieces, L.prim, L.prim_bytes, s));
      RGNN_LAUNCH(k_piece_fill, grid_for(h.J), T, 0, s, (int64_t)h.J, L.run_ptr, L.flags, L.piece_ptr);
    }
    RGNN_LAUNCH(k_piece_seg, (unsigned)((R + 256) / 256), 256, 0, s, R, (int64_t)h.J, L.rseg, L.flags, L.ctr,
                L.prseg, L.piece_ptr, (int32_t)n);
    if (af && n > 0) {
      const int64_t np_max = n + n / kPieceRows + 1;
      int32_t* piece_of_pos = reinterpret_cast<int32_t*>(L.k0);  // sort scratch, free by now
      RGNN_LAUNCH(k_piece_mark, grid_for(np_max), T, 0, s, np_max, L.ctr, L.piece_ptr, piece_of_pos);
      RGNN_LAUNCH(k_piece_slots, grid_for(n), T, 0, s, n, L.pos, piece_of_pos, L.dst_s, L.slot_piece, L.slot_w);
    }
    prseg_h.assign(R + 1, 0);
    RGNN_CUDA_TRY(cudaMemcpyAsync(prseg_h.data(), L.prseg, sizeof(int32_t) * (R + 1), cudaMemcpyDeviceToHost, s));
  }
  if (d->ntype || dx || af) {  // host sync 3 (node types, dX tables, run pieces): their counts and segments
    Counters h2{};
    RGNN_CUDA_TRY(cudaMemcpyAsync(&h2, L.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, s));
    RGNN_CUDA_TRY(cudaStreamSynchronize(s));
    mark("sync 3 (ntype / dX / pieces)");
    h.num_sitems = h2.num_sitems; h.num_sparts = h2.num_sparts; h.num_ssplit = h2.num_ssplit;
    h.num_pieces = h2.num_pieces;
  }
  int dev_id = 0, sms = 148;
  RGNN_CUDA_TRY(cudaGetDevice(&dev_id));
  RGNN_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev_id));

  // Host: 128-row GEMM tiles and dW split-K chunks, never straddling relations.
  // dW chunks (the fused backward runs one CTA per chunk, one CTA per SM): sized so that at most
  // waves * SMs chunks result, i.e. `waves` full waves with no partial wave left over (r01 sizing
  // gave 298 chunks = 2 waves + 2 on ogbn-mag); multiples of the 128-row tile.  Measured (fused
  // backward, ms): r01 sizing mag 3.66 / AM 0.854; 2 waves 3.68 / 0.877; 3 waves 3.54 / 0.790;
  // 4 waves 3.59 / 0.778; then with compact AM rows: 4 waves 3.46 / 0.790, 5: 3.43 / 0.795,
  // 6: 3.45 / 0.766, 8: 3.42 / 0.756 (default).  Chunks are in position order, so each wave's CTAs gather the
  // X / Z rows of one 1/waves slice of the position space at a time.  (Measured r02: one
  // persistent CTA per SM over equal position ranges -- every SM spanning the whole position space
  // at once -- was slower, 3.54 -> 4.97 ms on ogbn-mag.)
  // RGNN_BWD_WAVES (A/B): 0 = the r01 sizing only
  static const int64_t waves = getenv("RGNN_BWD_WAVES") ? std::max(0, atoi(getenv("RGNN_BWD_WAVES"))) : 8;
  auto count_chunks = [&](int64_t cr) {
    int64_t c = 0;
    for (int32_t r = 0; r < R; ++r) c += (seg_h[r + 1] - seg_h[r] + cr - 1) / cr;
    return c;
  };
  // the smallest multiple of 128 rows giving <= waves * SMs chunks; with more non-empty relations
  // than that (many small relations), the r01 sizing (about two chunks' worth of rows per SM)
  int64_t chunk_rows = std::max<int64_t>(kTileRows, ((n / (2 * sms) + 1) + kTileRows - 1) / kTileRows * kTileRows);
  if (waves > 0 && n > 0 && count_chunks(((n + kTileRows - 1) / kTileRows) * kTileRows) <= waves * sms) {
    int64_t lo = 1, hi = (n + kTileRows - 1) / kTileRows;  // in units of 128 rows
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (count_chunks(mid * kTileRows) <= waves * sms) hi = mid; else lo = mid + 1;
    }
    // only when the chunks stay near the balanced size (many small relations would otherwise
    // stretch the large relations' chunks)
    if (lo * kTileRows <= 2 * ((n + waves * sms - 1) / (waves * sms))) chunk_rows = lo * kTileRows;
  }
  // The tile / chunk tables are filled on the device: the host computes only each segment's first
  // tile (a few hundred integers, from the segments read back at sync 2) and uploads them with the
  // segment bounds in one copy; k_fill_tiles writes the Tile entries.
  struct TileJob {
    const std::vector<int32_t>* seg;  // segment bounds [S+1]
    int64_t rows;                     // rows per tile / chunk
    Tile* dst;                        // device table
    int32_t* first_dev;               // device [S+1] first tile of each segment, or null
    std::vector<int32_t> first;       // host copy
    size_t at;                        // offset of [seg | first] in the staging buffer
  };
  std::vector<TileJob> jobs;
  auto add_job = [&](const std::vector<int32_t>& sg, int64_t rows, Tile* dst, int32_t* first_dev) -> TileJob& {
    TileJob j{&sg, rows, dst, first_dev, std::vector<int32_t>(sg.size(), 0), 0};
    for (size_t i = 0; i + 1 < sg.size(); ++i)
      j.first[i + 1] = j.first[i] + (int32_t)((sg[i + 1] - sg[i] + rows - 1) / rows);
    jobs.push_back(std::move(j));
    return jobs.back();
  };
  add_job(seg_h, kTileRows, L.tiles, nullptr);
  add_job(seg_h, chunk_rows, L.chunks, L.chunk_seg);
  if (cm) add_job(cseg_h, kTileRows, L.ctiles, nullptr);
  add_job(rseg_h, kTileRows, L.rtiles, nullptr);  // 128-run GEMM tiles (dX: H = G_v W_r^T per run)
  if (!nseg_h.empty()) {  // HGT: node-type GEMM tiles and dW chunks (dWK / dWQ / dWV)
    add_job(nseg_h, kTileRows, L.ntiles, nullptr);
    add_job(nseg_h, std::max<int64_t>(kTileRows, ((V / (2 * sms) + 1) + kTileRows - 1) / kTileRows * kTileRows),
            L.nchunks, L.nchunk_seg);
  }
  if (af) add_job(prseg_h, kTileRows, L.ptiles, nullptr);  // aggregate-first: piece GEMM tiles
  if (!prseg_h.empty()) {  // dW split-K chunks over the run pieces (HGT backward)
    const int64_t np = h.num_pieces;
    add_job(prseg_h, std::max<int64_t>(kTileRows, ((np / (2 * sms) + 1) + kTileRows - 1) / kTileRows * kTileRows),
            L.pchunks, L.pchunk_seg);
  }
  std::vector<int32_t> stage;
  for (auto& j : jobs) {
    j.at = stage.size();
    stage.insert(stage.end(), j.seg->begin(), j.seg->end());
    stage.insert(stage.end(), j.first.begin(), j.first.end());
  }
  if ((int64_t)stage.size() > L.tabs_ints) return set_error(RGNN_E_CUDA, "internal: tile staging overflow");
  RGNN_CUDA_TRY(cudaMemcpyAsync(L.tabs, stage.data(), sizeof(int32_t) * stage.size(), cudaMemcpyHostToDevice, s));
  for (auto& j : jobs) {
    const int64_t S = (int64_t)j.seg->size() - 1, total = j.first.back();
    const int32_t* sg = L.tabs + j.at;
    const int32_t* fi = sg + S + 1;
    if (total > 0)
      RGNN_LAUNCH(k_fill_tiles, grid_for(total), T, 0, s, S, sg, fi, j.rows, total, j.dst);
    if (j.first_dev)
      RGNN_CUDA_TRY(cudaMemcpyAsync(j.first_dev, fi, sizeof(int32_t) * (S + 1), cudaMemcpyDeviceToDevice, s));
  }
  const std::vector<int32_t>& chunk_seg = jobs[1].first;
  const int64_t num_tiles = jobs[0].first.back(), num_chunks = chunk_seg.back();
  const int64_t num_ctiles = cm ? jobs[2].first.back() : 0;
  int64_t num_rtiles = 0, num_ntiles = 0, num_nchunks = 0, num_ptiles = 0, num_pchunks = 0;
  for (auto& j : jobs) {
    if (j.dst == L.rtiles) num_rtiles = j.first.back();
    if (j.dst == L.ntiles) num_ntiles = j.first.back();
    if (j.dst == L.nchunks) num_nchunks = j.first.back();
    if (j.dst == L.ptiles) num_ptiles = j.first.back();
    if (j.dst == L.pchunks) num_pchunks = j.first.back();
  }
  if (num_chunks > max_chunks(E, R) || num_pchunks > max_chunks(E, R))
    return set_error(RGNN_E_CUDA, "internal: chunk table overflow");
  // No final synchronisation: the staging copy from pageable memory returns once the data is staged,
  // so the host vectors may go out of scope; the tables are complete in stream order before any layer call.

  mark("tables uploaded");
  rgnn_graph* g = new rgnn_graph();
  g->V = V; g->V_own = V_own; g->v0 = v0; g->E_in = E; g->E_own = n; g->J = h.J;
  g->R = R; g->norm = d->norm; g->cap = cap;
  g->num_tiles = num_tiles; g->num_items = h.num_items; g->num_parts = h.num_parts;
  g->num_split_rows = h.num_split_rows; g->num_chunks = num_chunks;
  g->perm = L.perm; g->src_s = L.src_s; g->dst_s = L.dst_s; g->seg = L.seg; g->row_ptr = L.row_ptr;
  g->pos = L.pos; g->et_slot = L.et_slot; g->run_ptr = L.run_ptr; g->rseg = L.rseg; g->inv_c = L.inv_c;
  g->items = L.items; g->split_rows = L.split_rows; g->tiles = L.tiles; g->chunks = L.chunks;
  g->empty_rows = L.empty_rows; g->num_empty = h.num_empty;
  g->narrow_cap = narrow_cap(d); g->witems = L.witems; g->num_witems = h.num_witems;
  g->has_compact = cm; g->mat_mode = d->materialization; g->num_compact = cm ? h.num_compact : 0; g->crow_of_pos = L.crow_of_pos; g->zrow_slot = L.zrow_slot;
  g->invc_slot = L.invc_slot; g->csrc = L.csrc; g->cseg = L.cseg; g->ctiles = L.ctiles;
  g->num_ctiles = num_ctiles;
  g->chunk_seg = L.chunk_seg;
  g->has_dx = dx; g->run_of_pos = L.run_of_pos; g->run_dst = L.run_dst; g->run_rel = L.run_rel; 
  g->spos = L.spos; g->srun = L.srun; g->srel = L.srel; g->sinvc = L.sinvc; g->srow = L.srow;
  g->rtiles = L.rtiles; g->num_rtiles = num_rtiles;
  g->sitems = L.sitems; g->num_sitems = h.num_sitems; g->ssplit = L.ssplit; g->num_ssplit = h.num_ssplit;
  g->num_sparts = h.num_sparts;
  g->has_ntype = d->ntype != nullptr && V > 0; g->num_ntypes = d->ntype ? d->num_ntypes : 0;
  g->nperm = L.nperm; g->ninv = L.ninv; g->ntiles = L.ntiles; g->num_ntiles = num_ntiles;
  g->nchunks = L.nchunks; g->nchunk_seg = L.nchunk_seg; g->num_nchunks = num_nchunks;
  g->has_pieces = !prseg_h.empty(); g->piece_ptr = L.piece_ptr; g->prseg = L.prseg; g->pchunks = L.pchunks; g->pchunk_seg = L.pchunk_seg;
  g->num_pieces = !prseg_h.empty() ? h.num_pieces : 0; g->num_pchunks = num_pchunks;
  g->has_aggfirst = af; g->ptiles = L.ptiles; g->num_ptiles = num_ptiles;
  g->slot_piece = L.slot_piece; g->slot_w = L.slot_w;
  g->seg_host = seg_h;
  g->chunk_seg_host = chunk_seg;
  RGNN_CUDA_TRY(cudaGetDevice(&g->device));
  RGNN_CUDA_TRY(cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, g->device));
  *out = g;
  return RGNN_OK;
}

rgnn_status rgnn_graph_export(const rgnn_graph* g, rgnn_graph_view* v) {
  if (!g || !v) return set_error(RGNN_E_INVALID_ARG, "NULL graph or view");
  v->V = g->V; v->V_own = g->V_own; v->dst_begin = g->v0; v->E_own = g->E_own; v->num_runs = g->J;
  v->num_tiles = g->num_tiles; v->num_items = g->num_items; v->num_split_rows = g->num_split_rows; v->R = g->R;
  v->perm = g->perm; v->src_s = g->src_s; v->dst_s = g->dst_s; v->seg = g->seg; v->row_ptr = g->row_ptr;
  v->pos = g->pos; v->et_slot = g->et_slot; v->inv_c = g->inv_c; v->run_ptr = g->run_ptr; v->rseg = g->rseg;
  v->seg_host = g->seg_host.data();
  v->num_compact = g->num_compact; v->crow_of_pos = g->crow_of_pos; v->csrc = g->csrc; v->cseg = g->cseg;
  v->num_pieces = g->num_pieces; v->piece_ptr = g->num_pieces ? g->piece_ptr : nullptr;
  v->slot_piece = g->has_aggfirst ? g->slot_piece : nullptr;
  v->slot_w = g->has_aggfirst ? g->slot_w : nullptr;
  return RGNN_OK;
}

void rgnn_graph_destroy(rgnn_graph* g) { delete g; }

rgnn_status rgnn_zrows(const rgnn_graph* g, rgnn_model model, int64_t* rows) {
  if (!g || !rows) return set_error(RGNN_E_INVALID_ARG, "NULL graph or rows");
  if (model != RGNN_RGCN && model != RGNN_RGAT && model != RGNN_HGT)
    return set_error(RGNN_E_INVALID_ARG, "bad model %d", (int)model);
  *rows = use_compact(g, model) ? g->num_compact : g->E_own;
  return RGNN_OK;
}

}  // extern "C"
