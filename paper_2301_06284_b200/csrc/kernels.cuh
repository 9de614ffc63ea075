// kernels.cuh -- declarations of the per-layer launchers (one .cu each).
#pragma once
#include "common.cuh"

namespace rgnn {

// Arguments of the typed grouped GEMM, forward (DESIGN.md Sec. 6 "a2"):
//   Z[p, :] = X[gather(p), :] . W_{r(p)}  for every row p of every tile,
//   then the epilogue: Z *= row_scale[p] (RGCN 1/c, the paper's per-row
//   scalar on GEMM tiles) and s_src[p] = Z_fp32[p] . A[r,0] (RGAT).
struct GemmFwdArgs {
  const Tile* tiles;        // [num_tiles] (r, row0, row1) or null: one segment [0, rows) with weight 0
  int64_t num_tiles;
  int64_t rows;             // used when tiles == null
  const void* X;            // [V, K] T
  const int32_t* gather;    // [rows] X row of output row p, or null: row p -> X[gofs + p]
  int64_t gofs;
  const float* W;           // [R, K, N] fp32 master
  void* Z;                  // [rows, N] T
  const float* row_scale;   // [rows] or null
  const float* A;           // [R, 2, N] or null
  float* s_src;             // [rows] (with A)
  void* wt_bf16;            // workspace for the tcgen05 path: [num_w, N, K] bf16 (transposed W)
  int num_w;                // number of weight matrices in W (R, or 1 for the self-loop W0)
  int64_t x_rows;           // rows of X (V)
  int64_t z_rows;           // rows of Z (E_own) when tiles != null
  int z_bf16;               // tf32 kernel only: store Z as bf16
};

// dW split-K GEMM over chunks (DESIGN.md Sec. 6 "a5"):
//   part[c] = sum_{p in chunk c} X[gather(p)]^T B[p]   (K x N)
//   RGAT extra: bvec = sum dpre_p X[src_p] (K); part row stride K*N + K
// B rows: dZ[p] (T), or (bgather) G[bgather[p]] * bscale[p] (fp32).
struct GemmDwArgs {
  const Tile* chunks;       // [num_chunks] or null: chunk c = rows [c*chunk_rows, ...) of [0, rows)
  int64_t num_chunks, rows, chunk_rows;
  const void* X;
  const int32_t* gather;
  int64_t gofs;
  const void* Bz;           // dZ [rows, N] T, or null
  const float* Bg;          // G [*, N] fp32 when Bz is null
  const int32_t* bgather;   // B row index (null = identity)
  const float* bscale;      // per-row scale (null = 1)
  const float* dpre;        // RGAT: [rows] or null
  const int32_t* dst_local; // RGAT: local dst of row p
  int64_t v0;
  float* part;              // [num_chunks, K*N + K]
  int64_t x_rows;           // rows of X (tensor map bound, tcgen05 path)
};

rgnn_status launch_gemm_fwd(int prec, int K, int N, const GemmFwdArgs& a, cudaStream_t s);
rgnn_status launch_gemm_dw(int prec, int K, int N, const GemmDwArgs& a, cudaStream_t s);
rgnn_status launch_dw_reduce(int prec, int K, int N, int R, int64_t num_chunks, const int32_t* chunk_seg,
                             const float* part, const int32_t* cseg, const float* cpart, const float* A,
                             const float* W, float* dW, float* dA, float* dA_scratch /* [R*2*K] */, cudaStream_t s,
                             const Tile* chunks = nullptr, bool src_term = false);
rgnn_status launch_dst_term(int prec, int K, const rgnn_graph* g, const float* dpre, const void* X, float* cpart,
                            cudaStream_t s);
// U[r] = W_r A[r, half] (half = 1: the destination fold of the forward; 0: the source half, dX)
rgnn_status launch_fold_u(int prec, int R, int K, int N, const float* W, const float* A, float* U, cudaStream_t s,
                          int half = 1);

struct AggArgs {
  const Item* items;
  int64_t num_items;
  const int32_t* pos;
  const int32_t* et_slot;
  const void* Z;
  const float* s_src;
  const void* X;
  int64_t v0;
  const float* U;
  int R;                 // relations (rows of U)
  float slope;
  const void* Z0;        // RGCN self-loop rows [V_own, N] T or null
  const float* slot_scale;  // RGCN compact: 1/c of slot q (Z rows unscaled), or null
  bool cache_dst;        // RGAT: long (etype, dst) runs -> x_dst . U[r] once per run
  float* Y;
  float* lse;
  float* part;           // [num_parts, N+4]
  const SplitRow* split_rows;
  int64_t num_split_rows;
  const int32_t* empty_rows;
  int64_t num_empty;
  // narrow pass (forward walk): rows with deg <= narrow walked one lane group per row in row-id
  // order (empty rows included); witems = the items of the other rows.  row_ptr null: no narrow
  // pass (items cover every row with in-edges, empty_rows the rest).
  const int32_t* row_ptr;
  int64_t V_own;
  int narrow;
  const Item* witems;
  int64_t num_witems;
  // peer-memory gather (rgnn_comm_create_local + attach): every finished Y row is also stored into
  // these ranks' Y_full (global row v0 + row), from the walk's own epilogue
  float* peer_y[kMaxPeers];
  int npeer;
};
rgnn_status launch_aggregate(int prec, int K, int N, bool rgat, const AggArgs& a, cudaStream_t s);
// Aggregate-first RGCN (NEXT-4, aggfirst.cu): A_i = sum_{p in piece i} inv_c[p] X[src_s[p]], fp32 rows.
rgnn_status launch_piece_agg(int prec, int K, int64_t np, const int32_t* piece_ptr, const float* inv_c,
                             const int32_t* src_s, const void* X, void* A, cudaStream_t s);

struct BwdArgs {
  const Item* items;
  int64_t num_items;
  const int32_t* pos;
  const int32_t* zrow;   // compact: Z / s_src row of slot q (null: pos[q])
  const int32_t* et_slot;
  const void* Z;
  const float* s_src;
  const void* X;
  int64_t v0;
  const float* U;
  const float* A;
  float slope;
  const float* Y;
  const float* dY;
  const float* lse;
  void* dZ;
  float* dpre;
  float2* ad;            // dX: (alpha, dpre) per position, or null
};
rgnn_status launch_bwd_traverse(int prec, int K, int N, const BwdArgs& a, cudaStream_t s);

// tcgen05 path (gemm_tc.cu): returns RGNN_E_UNSUPPORTED if the shape is not covered.
rgnn_status launch_gemm_fwd_tc(int K, int N, const GemmFwdArgs& a, cudaStream_t s);
rgnn_status launch_gemm_fwd_tc_f32out(int K, int N, const GemmFwdArgs& a, cudaStream_t s);
rgnn_status launch_gemm_dw_tc(int K, int N, const GemmDwArgs& a, cudaStream_t s);
// fp32 operands (X fp32, Bz fp32 or Bg/bgather/bscale), 3xTF32 tcgen05 (gemm_dw_tf32.cu)
rgnn_status launch_gemm_dw_tf32x3(int K, int N, const GemmDwArgs& a, cudaStream_t s);
// fp32 typed GEMM, 3xTF32 tcgen05 (gemm_fwd_tf32x3.cu); a.wt_bf16 = [2, num_w, N, K] fp32 workspace
rgnn_status launch_gemm_fwd_tf32x3(int K, int N, const GemmFwdArgs& a, cudaStream_t s);
// fp32 operands on the tensor cores (tcgen05 kind::tf32), fp32 output (gemm_tf32.cu).  wt_f32 =
// the GEMM weight transposed, [num_w, N, K] fp32 (K-major B operand); a.W is not read.
rgnn_status launch_gemm_fwd_tf32(int K, int N, const GemmFwdArgs& a, const float* wt_f32, cudaStream_t s);
// zmap (compact): Z / s_src row of position p, null = p.
rgnn_status launch_bwd_fused_tc(int K, int N, const rgnn_graph* g, const void* X, const void* Z, const int32_t* zmap,
                                const float* s_src,
                                const float* lse, const float* Y, const float* dY, const float* U, const float* A,
                                float slope, float* part, float* cpart, float2* ad, cudaStream_t s);
// RGAT backward with Z recomputed on the tensor cores (bwd_tm.cu): bf16 layer, d_in, d_out in {64, 128}.
// zmap (compact): s_src row of position p, null = p; U = W_r A[r,1] (fold); Wt = bf16 workspace [R, N, K].
// Writes part (dW with alpha G_v rows + sum dpre x_src, per chunk), dpre per position and (dX) ad = (alpha,
// dpre) per position.
bool bwd_tm_enabled(int K, int N, int prec);
rgnn_status launch_bwd_rgat_tm(int K, int N, const rgnn_graph* g, const void* X, const float* W, void* Wt,
                               const int32_t* zmap, const float* s_src, const float* U, const float* lse,
                               const float* Y, const float* dY, float slope, float* part, float* dpre, float2* ad,
                               cudaStream_t s);
rgnn_status launch_expand_dz(int64_t E, int N, const int32_t* dst_s, const float* inv_c, const float* G, void* dZ,
                             cudaStream_t s);

// dX (dx.cu, NEXT-2)
struct DxArgs {
  int64_t V, V_own, v0;
  const Item* items;                          // source work list (row = source node)
  int64_t num_items;
  const SplitRow* split;                      // split sources
  int64_t num_split;
  float* part;                                // [num_parts, K] partial rows of split sources
  const int32_t *srow, *spos, *srun, *srel;  // source-major CSR over the positions
  const float* sinvc;                         // RGCN: 1/c per source slot
  const float* wpos;                          // non-RGAT walk: weight per position (HGT), else sinvc
  const float2* ad;                           // RGAT: (alpha, dpre) per position
  const void* H;                              // [J, K] fp32 (or bf16 with h_bf16): G_v W_r^T per (etype, dst) run
  int h_bf16;
  void* outb;                                 // non-RGAT walk: bf16 output rows at orow[row] instead of dX (HGT)
  const int32_t* orow;
  const float* U0;                            // RGAT: [R, K] W_r A[r,0]
  const float* U1;                            // RGAT: [R, K] W_r A[r,1]
  const Item* ditems;                         // RGAT destination terms: the dst work list
  int64_t num_ditems;
  const SplitRow* dsplit;
  int64_t num_dsplit;
  float* dpart;                               // [num_parts, K]
  const int32_t *pos, *et_slot;               // CSR-by-dst slots
  const void* H0;                             // RGCN self loop: [V_own, K] fp32 (G W0^T) or null
  float* dX;                                  // [V, K] fp32
};
rgnn_status launch_transpose_w(int prec, int R, int K, int N, const float* W, float* Wt, cudaStream_t s);
rgnn_status launch_dx_walk(int K, bool rgat, const DxArgs& a, cudaStream_t s);

// HGT (hgt.cu, NEXT-3)
struct HgtAggArgs {
  const Item* items;
  int64_t num_items;
  const int32_t* pos;     // slot -> row of KW / M (compact: zrow_slot)
  const void* KW;         // [zrows, N] fp32: k W_{a,r}
  const void* M;          // [zrows, N] fp32: v W_{m,r}
  const void* Q;          // [V, N] fp32: q rows in node-type order
  const int32_t* ninv;    // node -> its row in Q
  int64_t v0;
  float* Y;
  float* lse;
  float* part;
};
// HGT backward destination walk: per position alpha_e and da_e = alpha_e (G_t . m_e - G_t . Y_t),
// per owned destination dq_t = sum_e da_e kw_e (split rows: partial rows, merged in slot order)
struct HgtBwdArgs {
  const Item* items;
  int64_t num_items;
  const int32_t* pos;     // slot -> position p
  const int32_t* zrow;    // slot -> row of KW / M (compact: zrow_slot), null = pos
  const void* KW;         // [zrows, N] fp32
  const void* M;          // [zrows, N] T
  const void* Q;          // [V, N] fp32, node-type order rows
  const int32_t* ninv;
  int64_t v0;
  const float* Y;         // [V_own, N]
  const float* dY;        // [V_own, N]
  const float* lse;       // [V_own]
  float* alpha;           // [E_own] by position
  float* da;              // [E_own] by position
  float* dQ;              // [V, N] node-id order (owned rows written)
  void* dQb;              // or: bf16 rows in node-type order (ninv), when non-null
  float* part;            // [num_parts, N]
  const SplitRow* split_rows;
  int64_t num_split_rows;
};
rgnn_status launch_hgt_bwd_walk(int prec, int N, const HgtBwdArgs& a, cudaStream_t s);
// Run-piece sums of the HGT relation gradients (pieces: rgnn_graph.piece_ptr):
//   vagg_i = sum_{p in piece i} alpha_p v_src(p),  kagg_i = sum_p da_p k_src(p)
// so that dWm_r = sum_i vagg_i^T G_t(i) and dWa_r = sum_i kagg_i^T q_t(i) are GEMMs over the pieces.
struct HgtPieceArgs {
  int64_t num_pieces;
  const int32_t* piece_ptr;
  const int32_t* vrow;    // position -> node-type row of the source
  const float *alpha, *da;
  const void *Vn, *Kn;    // [V, N] fp32 (type-order rows), or bf16 copies (in_bf16)
  int in_bf16;
  const int32_t* dst_s;   // position -> local dst
  const int32_t* ninv;
  int64_t v0;
  void *vagg, *kagg;      // [num_pieces, N] T (the layer's operand type: bf16 feeds the tcgen05 dW)
  int32_t *pdst, *pq;     // [num_pieces] local dst / node-type row of the dst
};
rgnn_status launch_hgt_piece_agg(int prec, int N, const HgtPieceArgs& a, cudaStream_t s);
rgnn_status launch_f32_to_bf16(int64_t n, const float* a, void* b, cudaStream_t s);
rgnn_status launch_hgt_zero_rows(int64_t V, int N, const int32_t* srow, float* dK, float* dV, int64_t v0, int64_t v1,
                                 const int32_t* empty_rows, int64_t num_empty, float* dQ, cudaStream_t s);
// the same on bf16 rows in node-type order (row of node u = ninv[u])
rgnn_status launch_hgt_zero_rows_b(int64_t V, int N, const int32_t* srow, const int32_t* ninv, void* dK, void* dV,
                                   int64_t v0, int64_t v1, const int32_t* empty_rows, int64_t num_empty, void* dQ,
                                   cudaStream_t s);
// out[i] = ninv[idx[i] + ofs]
rgnn_status launch_map_gather(int64_t n, const int32_t* idx, const int32_t* ninv, int32_t* out, cudaStream_t s,
                              int64_t ofs = 0);
rgnn_status launch_bf16_to_f32(int64_t n, const void* a, float* b, cudaStream_t s);
rgnn_status launch_round_bf16(int64_t n, const float* a, float* b, cudaStream_t s);
rgnn_status launch_aggregate_hgt(int prec, int N, const HgtAggArgs& a, cudaStream_t s);

}  // namespace rgnn

#define RGNN_DISPATCH_KN(K, N, ...)                                                        \
  [&]() -> rgnn_status {                                                                   \
    switch ((K) * 1000 + (N)) {                                                            \
      case 32032: { constexpr int kK = 32, kN = 32; return __VA_ARGS__(); }                \
      case 32064: { constexpr int kK = 32, kN = 64; return __VA_ARGS__(); }                \
      case 32128: { constexpr int kK = 32, kN = 128; return __VA_ARGS__(); }               \
      case 64032: { constexpr int kK = 64, kN = 32; return __VA_ARGS__(); }                \
      case 64064: { constexpr int kK = 64, kN = 64; return __VA_ARGS__(); }                \
      case 64128: { constexpr int kK = 64, kN = 128; return __VA_ARGS__(); }               \
      case 128032: { constexpr int kK = 128, kN = 32; return __VA_ARGS__(); }              \
      case 128064: { constexpr int kK = 128, kN = 64; return __VA_ARGS__(); }              \
      case 128128: { constexpr int kK = 128, kN = 128; return __VA_ARGS__(); }             \
      default: return ::rgnn::set_error(RGNN_E_UNSUPPORTED, "d_in=%d d_out=%d not in {32,64,128}", (K), (N)); \
    }                                                                                      \
  }()
