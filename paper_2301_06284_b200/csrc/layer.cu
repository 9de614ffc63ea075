// layer.cu -- the C-ABI layer entry points: argument checks, workspace
// carving and the launch sequence of one RGCN / RGAT layer:
//   RGAT fwd : fold U -> typed GEMM (Z, s_src) -> fused walk (Y, lse) -> merge
//   RGCN fwd : typed GEMM (Z * 1/c) [-> self-loop GEMM Z0] -> walk -> merge
//   RGAT bwd : fold U -> backward walk (dZ, dpre) -> dW split-K GEMM -> reduce (dW, dA)
//   RGCN bwd : dW split-K GEMM gathering G rows by dst with 1/c -> reduce [-> dW0]
//   then, with a communicator, the NCCL gather of Y / all-reduce of dW, dA, dW0.
#include "kernels.cuh"

namespace rgnn {
bool tc_disabled();
rgnn_status comm_check_range(const rgnn_comm* c, int64_t v0, int64_t v1);
rgnn_status comm_gather_rows(rgnn_comm* c, const float* Y_own, int64_t N, void* Y_full, cudaStream_t s);
rgnn_status comm_reduce_rows(rgnn_comm* c, float* buf, int64_t K, cudaStream_t s);
int comm_peer_rows(const rgnn_comm* c, float** out);
bool comm_is_ipc(const rgnn_comm* c);
rgnn_status comm_peer_gather(rgnn_comm* c, const float* Y_own, int64_t N, float* Y_full, bool fused, cudaStream_t s);
rgnn_status comm_peer_barrier(rgnn_comm* c, cudaStream_t s);
rgnn_status comm_allreduce_sum(rgnn_comm* c, float* const* bufs, const size_t* counts, int n, cudaStream_t s);

struct WsLayout {
  float* U;        // [R, K] fp32 (fold of W_r A[r,1])
  float* part;     // [num_parts, N+4] split-row partial states
  void* Z;         // RGCN: [E_own, N] T (RGAT keeps Z in `saved`)
  void* Z0;        // RGCN self-loop rows [V_own, N] T
  void* dZ;        // RGAT: [E_own, N] T
  float* dpre;     // RGAT: [E_own]
  float* dwpart;   // [num_chunks, K*N + K]
  float* dw0part;  // [n0, K*N + K]
  float* cpart;    // RGAT dst term: [num_chunks, K]
  float* vsum;     // RGAT dA vectors: [R, 2, K]
  void* wt;        // tcgen05: bf16 W^T [R, N, K]
  float *PA, *PZ;  // aggregate-first RGCN: piece sums A [num_pieces, K] and products P [num_pieces, N], fp32
  float *PWt, *PZ0;  // ... W^T [R, N, K] (tf32 GEMM operand) and the fp32 self term [V_own, N]
  // dX (with_dx)
  float2* ad;      // RGAT: (alpha, dpre) per position [E_own]
  float* dpart;    // RGAT: [num_parts, K] split-row partial destination terms
  float* Wt;       // [R, N, K] fp32 W^T (and W0^T after it for RGCN)
  float* Wr;       // [R, K, N] fp32 W (RNE-rounded on the bf16 path), then W0: the tf32 GEMM's W^T^T
  void* H;         // [J, K] fp32
  void* H0;        // RGCN self loop: [V_own, K] fp32
  float* U0;       // RGAT: [R, K]
  float* xpart;    // [num_sparts, K] split-source partial rows
  size_t bytes;
};
struct SavedLayout {
  void* Z;         // RGAT: [E_own, N] T
  float* s_src;    // RGAT: [E_own]
  float* lse;      // RGAT, HGT: [V_own]
  // HGT: the forward's typed-linear outputs, read by the backward
  float *Kf, *Qf, *Vn;  // [V, N] fp32 (node-type order rows)
  float *KWf, *M;       // [zrows, N] fp32
  size_t bytes;
};

static size_t elt(int prec) { return prec == RGNN_BF16 ? 2 : 4; }
// Rows of the per-edge tensors Z / s_src: one per edge position (vanilla) or one
// per unique (etype, src) pair (compact materialisation).
static int64_t zrows(const rgnn_graph* g, int model) {
  return std::max<int64_t>(use_compact(g, model) ? g->num_compact : g->E_own, 1);
}
static int64_t dw0_chunk_rows(const rgnn_graph* g) {
  return std::max<int64_t>(kTileRows, (g->V_own / (2 * g->num_sms) + kTileRows) / kTileRows * kTileRows);
}
static int64_t dw0_chunks(const rgnn_graph* g) {
  int64_t cr = dw0_chunk_rows(g);
  return (g->V_own + cr - 1) / cr;
}

struct HgtWs {
  void* wt;               // bf16 W^T of the tcgen05 node GEMMs (bf16 layer)
  float *Xf, *Wr;         // bf16 path: X as fp32 (SIMT fallback only), RNE-rounded WK | WQ | WV | Wa | Wm
  float* Wtr;             // tf32 GEMM weights: (rounded) WK^T | WQ^T | WV^T | Wa^T | Wm^T
  int32_t* gather;
  float* part;
  // backward (training)
  float *alpha, *da;      // [E_own] by position
  int32_t* vrow;          // [E_own] node-type row of the source of position p
  int32_t* qrun;          // [J] node-type row of the destination of run j
  float *dQ, *dK, *dV;    // [V, N] node-id order (fp32 layer)
  void *dQb, *dKb, *dVb;  // bf16 layer: [V, N] bf16 rows in node-type order (the node dW GEMMs' B operand)
  float* H;               // [J, N] fp32: G_t Wm_r^T, then q_t Wa_r^T
  void* Bb;               // [max(E_own, V), N] bf16 B operand of the tcgen05 dW GEMMs
  float* dwpart;          // dW split-K partials
  float *qpart, *xpart;   // split-row partial rows (dq; dk / dv)
  float *WmT, *WaT, *Wmr, *War;  // [R, N, N]: W^T (SIMT GEMM) and W (tf32 GEMM), rounded on bf16
  void *vagg, *kagg;      // [num_pieces, N] T: run-piece sums (relation dW GEMM operand A)
  int32_t *pdst, *pq;     // [num_pieces]
  size_t bytes;
};
static HgtWs hgt_ws_layout(const rgnn_graph* g, int K, int N, int prec, void* base, bool training = false) {
  HgtWs w{};
  Carver c(base);
  const int64_t V = std::max<int64_t>(g->V, 1);
  const int64_t zr = std::max<int64_t>(use_compact(g, RGNN_HGT) ? g->num_compact : g->E_own, 1);
  const int64_t T = std::max<int64_t>(g->num_ntypes, 1);
  const bool bf = prec == RGNN_BF16;
  w.gather = c.take<int32_t>((size_t)zr);
  w.part = c.take<float>((size_t)std::max<int64_t>(g->num_parts, 1) * (N + 4));
  w.wt = c.take<char>(bf ? (size_t)T * K * N * 2 : 1);
  w.Xf = c.take<float>(bf ? (size_t)V * K : 1);
  w.Wr = c.take<float>(bf ? (size_t)(3 * T * K * N + 2 * (int64_t)g->R * N * N) : 1);
  w.Wtr = c.take<float>((size_t)(3 * T * K * N + 2 * (int64_t)g->R * N * N));
  if (training) {
    const int64_t E = std::max<int64_t>(g->E_own, 1), J = std::max<int64_t>(g->J, 1);
    w.alpha = c.take<float>(E);
    w.da = c.take<float>(E);
    w.vrow = c.take<int32_t>(E);
    w.qrun = c.take<int32_t>(J);
    w.dQ = c.take<float>((size_t)V * N);
    w.dK = c.take<float>((size_t)V * N);
    w.dV = c.take<float>((size_t)V * N);
    w.dQb = c.take<char>(bf ? (size_t)V * N * 2 : 1);
    w.dKb = c.take<char>(bf ? (size_t)V * N * 2 : 1);
    w.dVb = c.take<char>(bf ? (size_t)V * N * 2 : 1);
    w.H = c.take<float>((size_t)J * N);
    const int64_t NP = std::max<int64_t>(g->num_pieces, 1);
    w.Bb = c.take<char>(bf ? (size_t)std::max(std::max(E, 2 * V), NP) * N * 2 : 1);  // also the bf16 v, k copies
    const int64_t dwp = std::max<int64_t>(std::max<int64_t>(g->num_pchunks, 1) * (N * N + N),
                                          std::max<int64_t>(g->num_nchunks, 1) * (K * N + K));
    w.dwpart = c.take<float>((size_t)dwp);
    w.qpart = c.take<float>((size_t)std::max<int64_t>(g->num_parts, 1) * N);
    w.xpart = c.take<float>((size_t)std::max<int64_t>(g->num_sparts, 1) * N);
    const size_t rnn = (size_t)g->R * N * N;
    w.WmT = c.take<float>(rnn);
    w.WaT = c.take<float>(rnn);
    w.Wmr = c.take<float>(rnn);
    w.War = c.take<float>(rnn);
    const size_t e = bf ? 2 : 4;
    w.vagg = c.take<char>((size_t)NP * N * e);
    w.kagg = c.take<char>((size_t)NP * N * e);
    w.pdst = c.take<int32_t>(NP);
    w.pq = c.take<int32_t>(NP);
  }
  w.bytes = c.off;
  return w;
}

static WsLayout ws_layout(const rgnn_graph* g, int model, int K, int N, int prec, void* base, bool with_dx = false) {
  WsLayout w{};
  Carver c(base);
  const size_t e = elt(prec);
  const int64_t E = std::max<int64_t>(g->E_own, 1);
  w.U = c.take<float>((size_t)g->R * K);
  w.part = c.take<float>((size_t)std::max<int64_t>(g->num_parts, 1) * (N + 4));
  w.wt = c.take<char>((size_t)g->R * K * N * (prec == RGNN_BF16 ? 2 : 8));  // bf16 W^T | fp32 W^T hi, lo
  if (model == RGNN_RGCN && g->has_aggfirst) {
    const int64_t NP = std::max<int64_t>(g->num_pieces, 1);
    w.PA = c.take<float>((size_t)NP * K);
    w.PZ = c.take<float>((size_t)NP * N);
    w.PWt = c.take<float>((size_t)g->R * N * K);
    w.PZ0 = c.take<float>((size_t)std::max<int64_t>(g->V_own, 1) * N);
  }
  if (model == RGNN_RGCN) {
    w.Z = c.take<char>((size_t)std::max(zrows(g, model), E) * N * e);  // also the bf16 dZ of the unfused dW path
    w.Z0 = c.take<char>((size_t)std::max<int64_t>(g->V_own, 1) * N * e);
  } else {
    w.dZ = c.take<char>((size_t)E * N * e);
    w.dpre = c.take<float>((size_t)E);
  }
  w.dwpart = c.take<float>((size_t)std::max<int64_t>(g->num_chunks, 1) * (K * N + K));
  w.dw0part = c.take<float>(model == RGNN_RGCN ? (size_t)std::max<int64_t>(dw0_chunks(g), 1) * (K * N + K) : 1);
  w.cpart = c.take<float>((size_t)std::max<int64_t>(g->num_chunks, 1) * K);
  w.vsum = c.take<float>((size_t)g->R * 2 * K);
  if (with_dx) {  // run products H = G_v W_r^T (dX)
    const int64_t J = std::max<int64_t>(g->J, 1);
    w.Wt = c.take<float>((size_t)g->R * N * K + (size_t)N * K);
    w.Wr = c.take<float>((size_t)g->R * N * K + (size_t)N * K);
    w.H = c.take<char>((size_t)J * K * 4);
  }
  if (with_dx) {
    w.ad = c.take<float2>(model == RGNN_RGAT ? (size_t)E : 1);
    w.dpart = c.take<float>(model == RGNN_RGAT ? (size_t)std::max<int64_t>(g->num_parts, 1) * K : 1);
    w.H0 = c.take<char>(model == RGNN_RGCN ? (size_t)std::max<int64_t>(g->V_own, 1) * K * 4 : 1);
    w.U0 = c.take<float>((size_t)g->R * K);
    w.xpart = c.take<float>((size_t)std::max<int64_t>(g->num_sparts, 1) * K);
  }
  w.bytes = c.off;
  return w;
}

static SavedLayout saved_layout(const rgnn_graph* g, int model, int N, int prec, void* base) {
  SavedLayout s{};
  Carver c(base);
  if (model == RGNN_RGAT) {
    s.Z = c.take<char>((size_t)zrows(g, model) * N * elt(prec));
    s.s_src = c.take<float>((size_t)zrows(g, model));
    s.lse = c.take<float>((size_t)std::max<int64_t>(g->V_own, 1));
  } else if (model == RGNN_HGT) {
    const int64_t V = std::max<int64_t>(g->V, 1);
    s.lse = c.take<float>((size_t)std::max<int64_t>(g->V_own, 1));
    s.Kf = c.take<float>((size_t)V * N);
    s.Qf = c.take<float>((size_t)V * N);
    s.KWf = c.take<float>((size_t)zrows(g, model) * N);
    s.Vn = c.take<float>((size_t)V * N);
    s.M = c.take<float>((size_t)zrows(g, model) * N);
  }
  s.bytes = c.off;
  return s;
}

static bool width_ok(int d) { return d == 32 || d == 64 || d == 128; }

static rgnn_status check_common(const rgnn_graph* g, int K, int N, int prec, const void* ws, size_t ws_bytes,
                                const WsLayout& need) {
  if (!g) return set_error(RGNN_E_INVALID_ARG, "graph is NULL");
  if (!width_ok(K) || !width_ok(N)) return set_error(RGNN_E_UNSUPPORTED, "d_in=%d d_out=%d not in {32,64,128}", K, N);
  if (prec != RGNN_F32 && prec != RGNN_BF16) return set_error(RGNN_E_INVALID_ARG, "bad precision %d", prec);
  if (!ws) return set_error(RGNN_E_INVALID_ARG, "workspace is NULL");
  if ((uintptr_t)ws % kAlign) return set_error(RGNN_E_INVALID_ARG, "workspace must be 256B aligned");
  if (ws_bytes < need.bytes) return set_error(RGNN_E_WORKSPACE, "workspace %zu < required %zu", ws_bytes, need.bytes);
  return RGNN_OK;
}

// fp32-output GEMM inside a layer of precision `prec`: on the bf16 layer the tensor cores with
// fp32 operands (tcgen05 kind::tf32; wt_f32 = W^T [num_w, N, K]) -- exact for the bf16-valued
// operands, a 10-bit-mantissa truncation of fp32 ones (G, k), well inside the bf16 bound; on the
// fp32 layer (and without tcgen05) the SIMT fp32 kernel on a.W [num_w, K, N].
static rgnn_status f32_gemm(int prec, int K, int N, const GemmFwdArgs& a, const float* wt_f32, cudaStream_t s) {
  if (prec == RGNN_BF16) {
    rgnn_status st = launch_gemm_fwd_tf32(K, N, a, wt_f32, s);
    if (st != RGNN_E_UNSUPPORTED) return st;
  }
  return launch_gemm_fwd(RGNN_F32, K, N, a, s);
}

// dW GEMM of fp32 operands: 3xTF32 on the tensor cores (gemm_dw_tf32.cu) unless d_in = 32 or
// RGNN_DW_SIMT=1 (the SIMT fp32 kernel, kept for d_in = 32 and as the measured baseline).
static rgnn_status gemm_dw_f32(int xprec, int K, int N, const GemmDwArgs& a, cudaStream_t s) {
  static const bool simt = getenv("RGNN_DW_SIMT") && atoi(getenv("RGNN_DW_SIMT")) != 0;
  if (xprec == RGNN_F32 && !simt) {
    rgnn_status st = launch_gemm_dw_tf32x3(K, N, a, s);
    if (st != RGNN_E_UNSUPPORTED) return st;
  }
  return launch_gemm_dw(xprec, K, N, a, s);
}

static rgnn_status typed_gemm(int prec, int K, int N, const GemmFwdArgs& a, cudaStream_t s) {
  if (prec == RGNN_BF16) {
    rgnn_status st = launch_gemm_fwd_tc(K, N, a, s);
    if (st != RGNN_E_UNSUPPORTED) return st;
  }
  static const bool simt = getenv("RGNN_FWD_SIMT") && atoi(getenv("RGNN_FWD_SIMT")) != 0;
  if (prec == RGNN_F32 && !simt) {  // 3xTF32 tensor cores (W^T hi / lo in a.wt_bf16)
    rgnn_status st = launch_gemm_fwd_tf32x3(K, N, a, s);
    if (st != RGNN_E_UNSUPPORTED) return st;
  }
  return launch_gemm_fwd(prec, K, N, a, s);
}

static rgnn_status forward(const rgnn_graph* g, int model, int K, int N, int prec, const void* X, const float* W,
                           const float* W0, const float* A, float slope, float* Y, void* saved, void* ws,
                           size_t ws_bytes, rgnn_comm* comm, float* Y_full, void* stream) {
  if (!g) return set_error(RGNN_E_INVALID_ARG, "graph is NULL");  // before any layout reads g
  const WsLayout need = ws_layout(g, model, K, N, prec, nullptr);
  RGNN_TRY(check_common(g, K, N, prec, ws, ws_bytes, need));
  if (!X || !W || !Y || (model == RGNN_RGAT && (!A || !saved)))
    return set_error(RGNN_E_INVALID_ARG, "X, W, Y (and A, saved for RGAT) must not be NULL");
  if (comm) RGNN_TRY(comm_check_range(comm, g->v0, g->v0 + g->V_own));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  WsLayout w = ws_layout(g, model, K, N, prec, ws);
  SavedLayout sv = saved_layout(g, model, N, prec, saved);

  GemmFwdArgs ga{};
  ga.tiles = g->tiles; ga.num_tiles = g->num_tiles; ga.X = X; ga.gather = g->src_s; ga.W = W; ga.wt_bf16 = w.wt;
  ga.num_w = g->R; ga.x_rows = g->V; ga.z_rows = g->E_own;
  AggArgs aa{};
  aa.items = g->items; aa.num_items = g->num_items; aa.pos = g->pos; aa.et_slot = g->et_slot; aa.X = X;
  const bool cm = use_compact(g, model);
  if (cm) {  // GEMM over the unique (etype, src) rows; the walk reads Z[zrow_slot[q]]
    ga.tiles = g->ctiles; ga.num_tiles = g->num_ctiles; ga.gather = g->csrc; ga.z_rows = g->num_compact;
    aa.pos = g->zrow_slot;
    if (model == RGNN_RGCN) aa.slot_scale = g->invc_slot;  // 1/c applied per edge in the walk
  }
  aa.v0 = g->v0; aa.R = g->R; aa.slope = slope; aa.Y = Y; aa.part = w.part; aa.split_rows = g->split_rows;
  aa.num_split_rows = g->num_split_rows; aa.empty_rows = g->empty_rows; aa.num_empty = g->num_empty;
  aa.row_ptr = g->row_ptr; aa.V_own = g->V_own; aa.narrow = g->narrow_cap; aa.witems = g->witems;
  aa.num_witems = g->num_witems;
  // peer-memory communicator: the walk stores every finished Y row into the peers' Y_full itself
  const bool peer_fused = comm && Y_full && comm_is_ipc(comm);
  if (peer_fused) {
    aa.npeer = comm_peer_rows(comm, aa.peer_y);
    // entry barrier: every rank has reached this call, so whatever it did with its Y_full before
    // (stream-ordered) is finished before any rank stores into it
    Phase ph("comm", s);
    RGNN_TRY(comm_peer_barrier(comm, s));
  }
  static const int cache_env = getenv("RGNN_DST_CACHE") ? atoi(getenv("RGNN_DST_CACHE")) : -1;
  aa.cache_dst = cache_env >= 0 ? cache_env != 0 : g->E_own >= 4 * std::max<int64_t>(g->J, 1);  // mean run >= 4
  if (model == RGNN_RGAT) {
    { Phase ph("fold_u", s); RGNN_TRY(launch_fold_u(prec, g->R, K, N, W, A, w.U, s)); }
    ga.Z = sv.Z; ga.A = A; ga.s_src = sv.s_src;
    if (ga.num_tiles) { Phase ph("gemm_fwd", s); RGNN_TRY(typed_gemm(prec, K, N, ga, s)); }
    aa.Z = sv.Z; aa.s_src = sv.s_src; aa.U = w.U; aa.lse = sv.lse;
    { Phase ph("aggregate", s); RGNN_TRY(launch_aggregate(prec, K, N, true, aa, s)); }
  } else if (g->has_aggfirst && !getenv("RGNN_AGGFIRST_OFF")) {
    // aggregate-first (NEXT-4, aggfirst.cu): piece sums of x_src, one typed GEMM over the pieces,
    // and the walk adds each row's piece products once (slot weights 1 / 0)
    { Phase ph("piece_agg", s);
      RGNN_TRY(launch_piece_agg(prec, K, g->num_pieces, g->piece_ptr, g->inv_c, g->src_s, X, w.PA, s)); }
    // A and P fp32 on both layers (aggfirst.cu): the piece GEMM on the tf32 tensor cores (bf16 layer:
    // W^T rounded to bf16, exact in tf32) or the SIMT fp32 kernel, the walk in fp32
    GemmFwdArgs gp{};
    gp.tiles = g->ptiles; gp.num_tiles = g->num_ptiles; gp.X = w.PA; gp.gather = nullptr; gp.gofs = 0; gp.W = W;
    gp.Z = w.PZ; gp.num_w = g->R; gp.x_rows = std::max<int64_t>(g->num_pieces, 1); gp.z_rows = g->num_pieces;
    if (gp.num_tiles) {
      Phase ph("gemm_fwd", s);
      RGNN_TRY(launch_transpose_w(prec, g->R, K, N, W, w.PWt, s));
      RGNN_TRY(f32_gemm(prec, K, N, gp, w.PWt, s));
    }
    if (W0 && g->V_own > 0) {  // the self term as fp32 rows (bf16 layer: bf16 tcgen05 GEMM, fp32 epilogue)
      GemmFwdArgs g0{};
      g0.rows = g->V_own; g0.X = X; g0.gofs = g->v0; g0.W = W0; g0.Z = w.PZ0; g0.wt_bf16 = w.wt;
      g0.num_w = 1; g0.x_rows = g->V;
      Phase ph("gemm_self", s);
      rgnn_status st = prec == RGNN_BF16 ? launch_gemm_fwd_tc_f32out(K, N, g0, s) : RGNN_E_UNSUPPORTED;
      if (st == RGNN_E_UNSUPPORTED) {
        if (prec == RGNN_BF16) return set_error(RGNN_E_CUDA, "internal: tcgen05 self-loop GEMM unavailable");
        st = typed_gemm(prec, K, N, g0, s);
      }
      RGNN_TRY(st);
      aa.Z0 = w.PZ0;
    }
    aa.Z = w.PZ; aa.pos = g->slot_piece; aa.slot_scale = g->slot_w;
    { Phase ph("aggregate", s); RGNN_TRY(launch_aggregate(RGNN_F32, K, N, false, aa, s)); }
  } else {
    ga.Z = w.Z; ga.row_scale = cm ? nullptr : g->inv_c;
    if (ga.num_tiles) { Phase ph("gemm_fwd", s); RGNN_TRY(typed_gemm(prec, K, N, ga, s)); }
    if (W0 && g->V_own > 0) {
      GemmFwdArgs g0{};
      g0.rows = g->V_own; g0.X = X; g0.gofs = g->v0; g0.W = W0; g0.Z = w.Z0; g0.wt_bf16 = w.wt;
      g0.num_w = 1; g0.x_rows = g->V;
      { Phase ph("gemm_self", s); RGNN_TRY(typed_gemm(prec, K, N, g0, s)); }
      aa.Z0 = w.Z0;
    }
    aa.Z = w.Z;
    { Phase ph("aggregate", s); RGNN_TRY(launch_aggregate(prec, K, N, false, aa, s)); }
  }
  if (peer_fused) {  // rows already in the peers' Y_full: own slice + device barrier
    Phase ph("comm", s);
    RGNN_TRY(comm_peer_gather(comm, Y, N, Y_full, true, s));
  } else if (comm && Y_full) {
    Phase ph("comm", s);
    RGNN_TRY(comm_gather_rows(comm, Y, N, Y_full, s));
  }
  return RGNN_OK;
}

}  // namespace rgnn

using namespace rgnn;

extern "C" {

rgnn_status rgnn_workspace_bytes(const rgnn_graph* g, rgnn_model model, int d_in, int d_out, rgnn_prec prec,
                                 int training, size_t* ws_bytes, size_t* saved_bytes) {
  if (!g) return set_error(RGNN_E_INVALID_ARG, "graph is NULL");
  if (model != RGNN_RGCN && model != RGNN_RGAT && model != RGNN_HGT)
    return set_error(RGNN_E_INVALID_ARG, "bad model %d", (int)model);
  if (prec != RGNN_F32 && prec != RGNN_BF16) return set_error(RGNN_E_INVALID_ARG, "bad precision %d", (int)prec);
  if (!width_ok(d_in) || !width_ok(d_out)) return set_error(RGNN_E_UNSUPPORTED, "widths not in {32,64,128}");
  if (ws_bytes)
    *ws_bytes = model == RGNN_HGT ? hgt_ws_layout(g, d_in, d_out, prec, nullptr, training != 0).bytes
                                  : ws_layout(g, model, d_in, d_out, prec, nullptr, training == RGNN_WS_DX).bytes;
  if (saved_bytes) *saved_bytes = saved_layout(g, model, d_out, prec, nullptr).bytes;
  return RGNN_OK;
}

rgnn_status rgcn_forward(const rgnn_graph* g, int d_in, int d_out, rgnn_prec prec, const void* X, const float* W,
                         const float* W0, float* Y, void* saved, void* ws, size_t ws_bytes, rgnn_comm* comm,
                         float* Y_full, void* stream) {
  return forward(g, RGNN_RGCN, d_in, d_out, prec, X, W, W0, nullptr, 0.f, Y, saved, ws, ws_bytes, comm, Y_full,
                 stream);
}

rgnn_status rgat_forward(const rgnn_graph* g, int d_in, int d_out, rgnn_prec prec, const void* X, const float* W,
                         const float* A, float slope, float* Y, void* saved, void* ws, size_t ws_bytes,
                         rgnn_comm* comm, float* Y_full, void* stream) {
  return forward(g, RGNN_RGAT, d_in, d_out, prec, X, W, nullptr, A, slope, Y, saved, ws, ws_bytes, comm, Y_full,
                 stream);
}

rgnn_status hgt_forward(const rgnn_graph* g, int K, int N, rgnn_prec prec, const void* X, const float* WK,
                        const float* WQ, const float* WV, const float* Wa, const float* Wm, float* Y, void* saved,
                        void* ws, size_t ws_bytes, rgnn_comm* comm, float* Y_full, void* stream) {
  if (!g) return set_error(RGNN_E_INVALID_ARG, "graph is NULL");
  if (!g->has_ntype) return set_error(RGNN_E_UNSUPPORTED, "HGT needs node types (rgnn_graph_desc.ntype)");
  const HgtWs need = hgt_ws_layout(g, K, N, prec, nullptr);
  if (!width_ok(K) || !width_ok(N)) return set_error(RGNN_E_UNSUPPORTED, "d_in=%d d_out=%d not in {32,64,128}", K, N);
  if (prec != RGNN_F32 && prec != RGNN_BF16) return set_error(RGNN_E_INVALID_ARG, "bad precision %d", prec);
  if (!ws || (uintptr_t)ws % kAlign) return set_error(RGNN_E_INVALID_ARG, "workspace NULL or not 256B aligned");
  if (ws_bytes < need.bytes) return set_error(RGNN_E_WORKSPACE, "workspace %zu < required %zu", ws_bytes, need.bytes);
  if (!X || !WK || !WQ || !WV || !Wa || !Wm || !Y || !saved)
    return set_error(RGNN_E_INVALID_ARG, "X, WK, WQ, WV, Wa, Wm, Y, saved must not be NULL");
  if (comm) RGNN_TRY(comm_check_range(comm, g->v0, g->v0 + g->V_own));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  HgtWs w = hgt_ws_layout(g, K, N, prec, ws);
  SavedLayout sv = saved_layout(g, RGNN_HGT, N, prec, saved);
  // Every per-node and per-edge intermediate (k, q, v, k W_{a,r}, v W_{m,r}) is fp32 on both
  // paths; the bf16 layer takes X and the weights in bf16 (RNE-rounded weights), so its GEMMs run
  // on the tcgen05 kind::tf32 kernel with bf16-exact operands (and a tf32 truncation of the fp32
  // k / v in the relation GEMMs).  bf16 logits lose too much through the exponent, and bf16 v / m
  // rows put the backward's dWa at ~0.9 of the bf16 bound (numpy model; O23).
  // Node-typed linears run over the node-type segments (rows in type order), relation-typed ones
  // per (etype, src) pair (or per edge).
  const bool bf = prec == RGNN_BF16;
  const int64_t T = g->num_ntypes;
  const int64_t tkn = T * K * N, rnn = (int64_t)g->R * N * N;
  const float *WKs = WK, *WQs = WQ, *WVs = WV, *Was = Wa, *Wms = Wm;
  const void* Xs = X;
  // bf16 layer: the node-typed linears read X in bf16 on the bf16 tcgen05 GEMM with fp32 output
  // rows (bf16 x bf16 products are exact, fp32 accumulation: the same values the tf32 GEMM gives on
  // the bf16-valued operands); the fp32 copy of X is made only for the SIMT fallback.
  const bool node_tc = bf && !tc_disabled();
  if (bf) {
    Phase ph("hgt_prep", s);
    if (!node_tc) RGNN_TRY(launch_bf16_to_f32(g->V * K, X, w.Xf, s));
    RGNN_TRY(launch_round_bf16(tkn, WK, w.Wr, s));
    RGNN_TRY(launch_round_bf16(tkn, WQ, w.Wr + tkn, s));
    RGNN_TRY(launch_round_bf16(tkn, WV, w.Wr + 2 * tkn, s));
    RGNN_TRY(launch_round_bf16(rnn, Wa, w.Wr + 3 * tkn, s));
    RGNN_TRY(launch_round_bf16(rnn, Wm, w.Wr + 3 * tkn + rnn, s));
    Xs = w.Xf; WKs = w.Wr; WQs = w.Wr + tkn; WVs = w.Wr + 2 * tkn; Was = w.Wr + 3 * tkn; Wms = Was + rnn;
  }
  {
    Phase ph("hgt_prep", s);
    RGNN_TRY(launch_transpose_w(prec, (int)T, K, N, WK, w.Wtr, s));
    RGNN_TRY(launch_transpose_w(prec, (int)T, K, N, WQ, w.Wtr + tkn, s));
    RGNN_TRY(launch_transpose_w(prec, (int)T, K, N, WV, w.Wtr + 2 * tkn, s));
    RGNN_TRY(launch_transpose_w(prec, g->R, N, N, Wa, w.Wtr + 3 * tkn, s));
    RGNN_TRY(launch_transpose_w(prec, g->R, N, N, Wm, w.Wtr + 3 * tkn + rnn, s));
  }
  if (g->num_ntiles) {
    Phase ph("hgt_node_gemm", s);
    auto node_gemm = [&](const float* Wmaster, const float* Win, const float* Wt32, float* out) -> rgnn_status {
      GemmFwdArgs ga{};
      ga.tiles = g->ntiles; ga.num_tiles = g->num_ntiles; ga.gather = g->nperm; ga.Z = out; ga.num_w = (int)T;
      ga.x_rows = g->V; ga.z_rows = g->V;
      if (node_tc) {
        ga.X = X; ga.W = Wmaster; ga.wt_bf16 = w.wt;  // W rounded to bf16 (RNE) inside
        rgnn_status st = launch_gemm_fwd_tc_f32out(K, N, ga, s);
        if (st != RGNN_E_UNSUPPORTED) return st;
        return set_error(RGNN_E_CUDA, "internal: tcgen05 node GEMM unavailable");
      }
      ga.X = Xs; ga.W = Win;
      return f32_gemm(prec, K, N, ga, Wt32, s);
    };
    RGNN_TRY(node_gemm(WK, WKs, w.Wtr, sv.Kf));
    RGNN_TRY(node_gemm(WQ, WQs, w.Wtr + tkn, sv.Qf));
    RGNN_TRY(node_gemm(WV, WVs, w.Wtr + 2 * tkn, sv.Vn));
  }
  const bool cm = use_compact(g, RGNN_HGT);
  const int64_t zr = cm ? g->num_compact : g->E_own;
  const int64_t nt = cm ? g->num_ctiles : g->num_tiles;
  {
    Phase ph("hgt_rel_gemm", s);
    RGNN_TRY(launch_map_gather(zr, cm ? g->csrc : g->src_s, g->ninv, w.gather, s));
    auto rel_gemm = [&](const float* Xin, const float* Win, const float* Wt32, float* out) -> rgnn_status {
      GemmFwdArgs ga{};
      ga.tiles = cm ? g->ctiles : g->tiles; ga.num_tiles = nt; ga.X = Xin; ga.gather = w.gather; ga.W = Win;
      ga.Z = out; ga.num_w = g->R; ga.x_rows = g->V; ga.z_rows = zr;
      return f32_gemm(prec, N, N, ga, Wt32, s);
    };
    if (nt) {
      RGNN_TRY(rel_gemm(sv.Kf, Was, w.Wtr + 3 * tkn, sv.KWf));
      RGNN_TRY(rel_gemm(sv.Vn, Wms, w.Wtr + 3 * tkn + rnn, sv.M));
    }
  }
  {
    Phase ph("aggregate", s);
    HgtAggArgs ha{};
    ha.items = g->items; ha.num_items = g->num_items; ha.pos = cm ? g->zrow_slot : g->pos; ha.KW = sv.KWf;
    ha.M = sv.M; ha.Q = sv.Qf; ha.ninv = g->ninv; ha.v0 = g->v0; ha.Y = Y; ha.lse = sv.lse; ha.part = w.part;
    RGNN_TRY(launch_aggregate_hgt(RGNN_F32, N, ha, s));
    // zero rows and split-row merges of the shared walk infrastructure (online-softmax states)
    AggArgs aa{};
    aa.num_items = 0; aa.Y = Y; aa.lse = sv.lse; aa.part = w.part; aa.split_rows = g->split_rows;
    aa.num_split_rows = g->num_split_rows; aa.empty_rows = g->empty_rows; aa.num_empty = g->num_empty;
    RGNN_TRY(launch_aggregate(prec, N, N, true, aa, s));
  }
  if (comm && Y_full) { Phase ph("comm", s); RGNN_TRY(comm_gather_rows(comm, Y, N, Y_full, s)); }
  return RGNN_OK;
}

// HGT backward (chain rule of hgt_forward; the formulas of oracle_hgt_backward):
//   walk     : alpha_e, da_e by position; dq_t = sum_e da_e kw_e            (owned rows)
//   runs     : Hm_j = G_t Wm_r^T, Ha_j = q_t Wa_r^T per (etype, dst) run j  (fp32 GEMMs, J << E)
//   sources  : dv_s = sum_{e: src=s} alpha_e Hm_j(e),  dk_s = sum_e da_e Ha_j(e)   (source walk)
//   dW       : dWm_r = sum_i vagg_i^T G_t(i), dWa_r = sum_i kagg_i^T q_t(i) over run pieces i (<= 64
//              positions of one (etype, dst) run): vagg_i = sum_p alpha_p v_src(p), kagg_i = sum_p da_p k_src(p)
//              dWK / dWV / dWQ [tau] = sum_{nodes of type tau} x^T dk / dv / dq    (node-type chunks)
// On the bf16 layer the dW GEMMs run on the tcgen05 segmented dW kernel with the B rows
// materialised in bf16 (like the RGAT dZ); on the fp32 layer on the SIMT dW kernel.
rgnn_status hgt_backward(const rgnn_graph* g, int K, int N, rgnn_prec prec, const void* X, const float* WK,
                         const float* WQ, const float* WV, const float* Wa, const float* Wm, const float* Y,
                         const float* dY, const void* saved, float* dWK, float* dWQ, float* dWV, float* dWa,
                         float* dWm, void* ws, size_t ws_bytes, rgnn_comm* comm, void* stream) {
  (void)WK; (void)WQ; (void)WV;
  if (!g) return set_error(RGNN_E_INVALID_ARG, "graph is NULL");
  if (!g->has_ntype) return set_error(RGNN_E_UNSUPPORTED, "HGT needs node types (rgnn_graph_desc.ntype)");
  if (!g->has_dx || !g->has_pieces)
    return set_error(RGNN_E_UNSUPPORTED, "HGT backward needs a graph built with RGNN_GRAPH_DX");
  if (!width_ok(K) || !width_ok(N)) return set_error(RGNN_E_UNSUPPORTED, "d_in=%d d_out=%d not in {32,64,128}", K, N);
  if (prec != RGNN_F32 && prec != RGNN_BF16) return set_error(RGNN_E_INVALID_ARG, "bad precision %d", prec);
  const HgtWs need = hgt_ws_layout(g, K, N, prec, nullptr, true);
  if (!ws || (uintptr_t)ws % kAlign) return set_error(RGNN_E_INVALID_ARG, "workspace NULL or not 256B aligned");
  if (ws_bytes < need.bytes)
    return set_error(RGNN_E_WORKSPACE, "workspace %zu < required %zu (size it with training=1)", ws_bytes, need.bytes);
  if (!X || !Wa || !Wm || !Y || !dY || !saved || !dWK || !dWQ || !dWV || !dWa || !dWm)
    return set_error(RGNN_E_INVALID_ARG, "X, Wa, Wm, Y, dY, saved and the five gradients must not be NULL");
  if (comm) RGNN_TRY(comm_check_range(comm, g->v0, g->v0 + g->V_own));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  HgtWs w = hgt_ws_layout(g, K, N, prec, ws, true);
  SavedLayout sv = saved_layout(g, RGNN_HGT, N, prec, const_cast<void*>(saved));
  const bool bf = prec == RGNN_BF16;
  const bool cm = use_compact(g, RGNN_HGT);
  const int64_t T = g->num_ntypes, V = g->V, E = g->E_own, J = g->J;
  const size_t rnn = (size_t)g->R * N * N;
  {
    Phase ph("hgt_bwd_prep", s);
    RGNN_TRY(launch_transpose_w(prec, g->R, N, N, Wm, w.WmT, s));
    RGNN_TRY(launch_transpose_w(prec, g->R, N, N, Wa, w.WaT, s));
    if (bf) {
      RGNN_TRY(launch_round_bf16((int64_t)rnn, Wm, w.Wmr, s));
      RGNN_TRY(launch_round_bf16((int64_t)rnn, Wa, w.War, s));
    } else {
      RGNN_CUDA_TRY(cudaMemcpyAsync(w.Wmr, Wm, sizeof(float) * rnn, cudaMemcpyDeviceToDevice, s));
      RGNN_CUDA_TRY(cudaMemcpyAsync(w.War, Wa, sizeof(float) * rnn, cudaMemcpyDeviceToDevice, s));
    }
    RGNN_TRY(launch_map_gather(E, g->src_s, g->ninv, w.vrow, s));
    RGNN_TRY(launch_map_gather(J, g->run_dst, g->ninv, w.qrun, s, g->v0));
    if (bf)
      RGNN_TRY(launch_hgt_zero_rows_b(V, N, g->srow, g->ninv, w.dKb, w.dVb, g->v0, g->v0 + g->V_own, g->empty_rows,
                                      g->num_empty, w.dQb, s));
    else
      RGNN_TRY(launch_hgt_zero_rows(V, N, g->srow, w.dK, w.dV, g->v0, g->v0 + g->V_own, g->empty_rows,
                                    g->num_empty, w.dQ, s));
  }
  {
    Phase ph("hgt_bwd_walk", s);
    HgtBwdArgs hb{};
    hb.items = g->items; hb.num_items = g->num_items; hb.pos = g->pos; hb.zrow = cm ? g->zrow_slot : nullptr;
    hb.KW = sv.KWf; hb.M = sv.M; hb.Q = sv.Qf; hb.ninv = g->ninv; hb.v0 = g->v0; hb.Y = Y; hb.dY = dY;
    hb.lse = sv.lse; hb.alpha = w.alpha; hb.da = w.da; hb.dQ = w.dQ; hb.dQb = bf ? w.dQb : nullptr;
    hb.part = w.qpart;
    hb.split_rows = g->split_rows; hb.num_split_rows = g->num_split_rows;
    RGNN_TRY(launch_hgt_bwd_walk(RGNN_F32, N, hb, s));
  }
  // source sums: dv = sum alpha Hm, dk = sum da Ha over each source's out-edges.  On the bf16 layer
  // the run products H are stored in bf16 by the tf32 GEMM (dk / dv only feed the weight
  // gradients dWK / dWV, sums over nodes; O23), halving the walks' gathered bytes.
  const int h_bf16 = (bf && !tc_disabled() && !getenv("RGNN_HGT_H_F32")) ? 1 : 0;
  auto src_sum = [&](const float* G, const int32_t* gidx, int64_t grows, const float* Wt, const float* Wrr,
                     const float* wpos, float* out, void* outb) -> rgnn_status {
    if (g->num_rtiles) {
      Phase ph("hgt_bwd_runs", s);
      GemmFwdArgs gh{};
      gh.tiles = g->rtiles; gh.num_tiles = g->num_rtiles; gh.X = G; gh.gather = gidx; gh.W = Wt; gh.Z = w.H;
      gh.num_w = g->R; gh.x_rows = std::max<int64_t>(grows, 1); gh.z_rows = J; gh.z_bf16 = h_bf16;
      RGNN_TRY(f32_gemm(prec, N, N, gh, Wrr, s));
    }
    Phase ph("hgt_bwd_src", s);
    DxArgs xa{};
    xa.V = V; xa.V_own = g->V_own; xa.v0 = g->v0;
    xa.items = g->sitems; xa.num_items = g->num_sitems; xa.split = g->ssplit; xa.num_split = g->num_ssplit;
    xa.part = w.xpart; xa.srow = g->srow; xa.spos = g->spos; xa.srun = g->srun; xa.srel = g->srel;
    xa.sinvc = g->sinvc; xa.wpos = wpos; xa.H = w.H; xa.h_bf16 = h_bf16; xa.dX = out;
    xa.outb = outb; xa.orow = g->ninv;  // bf16 layer: rows straight into the node dW GEMM's B layout
    return launch_dx_walk(N, false, xa, s);
  };
  RGNN_TRY(src_sum(dY, g->run_dst, g->V_own, w.WmT, w.Wmr, w.alpha, w.dV, bf ? w.dVb : nullptr));
  RGNN_TRY(src_sum(sv.Qf, w.qrun, V, w.WaT, w.War, w.da, w.dK, bf ? w.dKb : nullptr));
  // dW GEMMs: part = sum_p Xin[gather p]^T (scale_p Gm[gidx p]), reduced per segment in chunk order
  auto dw = [&](int xprec, int Kd, const void* Xin, const int32_t* gather, int64_t xrows, const Tile* chunks,
                int64_t nch, const int32_t* cseg, int nseg, int64_t rows, const float* Gm, const int32_t* gidx,
                const float* scale, float* out) -> rgnn_status {
    if (nch == 0) {
      RGNN_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(float) * (size_t)nseg * Kd * N, s));
      return RGNN_OK;
    }
    GemmDwArgs a{};
    a.chunks = chunks; a.num_chunks = nch; a.rows = rows; a.X = Xin; a.gather = gather; a.x_rows = xrows;
    a.part = w.dwpart;
    rgnn_status st = RGNN_E_UNSUPPORTED;
    if (bf && xprec == RGNN_BF16 && (Kd == 64 || Kd == 128)) {
      RGNN_TRY(launch_expand_dz(rows, N, gidx, scale, Gm, w.Bb, s));
      a.Bz = w.Bb;
      st = launch_gemm_dw_tc(Kd, N, a, s);
      if (st != RGNN_OK && st != RGNN_E_UNSUPPORTED) return st;
    }
    if (st != RGNN_OK) {
      a.Bz = nullptr; a.Bg = Gm; a.bgather = gidx; a.bscale = scale;
      RGNN_TRY(gemm_dw_f32(xprec, Kd, N, a, s));
    }
    return launch_dw_reduce(xprec, Kd, N, nseg, nch, cseg, w.dwpart, nullptr, nullptr, nullptr, nullptr, out,
                            nullptr, nullptr, s);
  };
  {
    // relation gradients over the run pieces: the piece sums collapse each piece's positions
    // (same relation and destination) into one GEMM row
    Phase ph("hgt_bwd_dw_rel", s);
    HgtPieceArgs pa{};
    pa.num_pieces = g->num_pieces; pa.piece_ptr = g->piece_ptr; pa.vrow = w.vrow; pa.alpha = w.alpha; pa.da = w.da;
    pa.Vn = sv.Vn; pa.Kn = sv.Kf;
    if (bf && getenv("RGNN_HGT_PIECE_BF16")) {  // bf16 copies of v and k: half the gathered bytes
      RGNN_TRY(launch_f32_to_bf16((int64_t)V * N, sv.Vn, w.Bb, s));
      RGNN_TRY(launch_f32_to_bf16((int64_t)V * N, sv.Kf, static_cast<char*>(w.Bb) + (size_t)V * N * 2, s));
      pa.Vn = w.Bb; pa.Kn = static_cast<char*>(w.Bb) + (size_t)V * N * 2; pa.in_bf16 = 1;
    }
    pa.dst_s = g->dst_s; pa.ninv = g->ninv; pa.v0 = g->v0; pa.vagg = w.vagg;
    pa.kagg = w.kagg; pa.pdst = w.pdst; pa.pq = w.pq;
    RGNN_TRY(launch_hgt_piece_agg(prec, N, pa, s));
    const int64_t NP = g->num_pieces;
    RGNN_TRY(dw(prec, N, w.vagg, nullptr, std::max<int64_t>(NP, 1), g->pchunks, g->num_pchunks, g->pchunk_seg, g->R, NP,
                dY, w.pdst, nullptr, dWm));
    RGNN_TRY(dw(prec, N, w.kagg, nullptr, std::max<int64_t>(NP, 1), g->pchunks, g->num_pchunks, g->pchunk_seg, g->R, NP,
                sv.Qf, w.pq, nullptr, dWa));
  }
  {
    Phase ph("hgt_bwd_dw_node", s);
    if (bf) {  // B rows already bf16 in node-type order (written by the walks): no expansion pass
      auto dw_b = [&](const void* Bt, float* out) -> rgnn_status {
        if (g->num_nchunks == 0) {
          RGNN_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(float) * (size_t)T * K * N, s));
          return RGNN_OK;
        }
        GemmDwArgs a{};
        a.chunks = g->nchunks; a.num_chunks = g->num_nchunks; a.rows = V; a.X = X; a.gather = g->nperm;
        a.x_rows = V; a.part = w.dwpart; a.Bz = Bt;
        rgnn_status st = launch_gemm_dw_tc(K, N, a, s);
        if (st == RGNN_E_UNSUPPORTED) st = launch_gemm_dw(prec, K, N, a, s);  // d_in = 32 / no tcgen05
        RGNN_TRY(st);
        return launch_dw_reduce(prec, K, N, (int)T, g->num_nchunks, g->nchunk_seg, w.dwpart, nullptr, nullptr,
                                nullptr, nullptr, out, nullptr, nullptr, s);
      };
      RGNN_TRY(dw_b(w.dKb, dWK));
      RGNN_TRY(dw_b(w.dVb, dWV));
      RGNN_TRY(dw_b(w.dQb, dWQ));
    } else {
      RGNN_TRY(dw(prec, K, X, g->nperm, V, g->nchunks, g->num_nchunks, g->nchunk_seg, (int)T, V, w.dK, g->nperm,
                  nullptr, dWK));
      RGNN_TRY(dw(prec, K, X, g->nperm, V, g->nchunks, g->num_nchunks, g->nchunk_seg, (int)T, V, w.dV, g->nperm,
                  nullptr, dWV));
      RGNN_TRY(dw(prec, K, X, g->nperm, V, g->nchunks, g->num_nchunks, g->nchunk_seg, (int)T, V, w.dQ, g->nperm,
                  nullptr, dWQ));
    }
  }
  if (comm) {
    float* bufs[5] = {dWK, dWQ, dWV, dWa, dWm};
    const size_t tkn = (size_t)T * K * N;
    size_t counts[5] = {tkn, tkn, tkn, rnn, rnn};
    Phase ph("comm", s);
    RGNN_TRY(comm_allreduce_sum(comm, bufs, counts, 5, s));
  }
  return RGNN_OK;
}

rgnn_status rgnn_backward(const rgnn_graph* g, rgnn_model model, int K, int N, rgnn_prec prec, const void* X,
                          const float* W, const float* W0, const float* A, float slope, const float* Y,
                          const float* dY, const void* saved, float* dW, float* dA, float* dW0, float* dX, void* ws,
                          size_t ws_bytes, rgnn_comm* comm, void* stream) {
  if (model == RGNN_HGT) return set_error(RGNN_E_UNSUPPORTED, "use hgt_backward for RGNN_HGT");
  if (model != RGNN_RGCN && model != RGNN_RGAT) return set_error(RGNN_E_INVALID_ARG, "bad model %d", (int)model);
  if (!g) return set_error(RGNN_E_INVALID_ARG, "graph is NULL");  // before any layout reads g
  const bool want_dx = dX != nullptr;
  if (want_dx && !g->has_dx)
    return set_error(RGNN_E_UNSUPPORTED, "dX needs a graph built with RGNN_GRAPH_DX");
  const WsLayout need = ws_layout(g, model, K, N, prec, nullptr, want_dx);
  RGNN_TRY(check_common(g, K, N, prec, ws, ws_bytes, need));
  if (!X || !dY || !dW) return set_error(RGNN_E_INVALID_ARG, "X, dY, dW must not be NULL");
  if (want_dx && !W) return set_error(RGNN_E_INVALID_ARG, "dX needs W");
  if (model == RGNN_RGAT && (!W || !A || !Y || !saved || !dA))
    return set_error(RGNN_E_INVALID_ARG, "RGAT backward needs W, A, Y, saved and dA");
  if (comm) RGNN_TRY(comm_check_range(comm, g->v0, g->v0 + g->V_own));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  WsLayout w = ws_layout(g, model, K, N, prec, ws, want_dx);
  SavedLayout sv = saved_layout(g, model, N, prec, const_cast<void*>(saved));

  GemmDwArgs da{};
  da.chunks = g->chunks; da.num_chunks = g->num_chunks; da.rows = g->E_own; da.X = X; da.gather = g->src_s;
  da.part = w.dwpart; da.x_rows = g->V;
  const bool tc_ok = prec == RGNN_BF16 && K >= 64;  // tcgen05 dW needs UMMA M = d_in in {64, 128}
  auto dw_gemm = [&](const GemmDwArgs& args) -> rgnn_status {
    if (tc_ok && args.Bz) {
      rgnn_status st = launch_gemm_dw_tc(K, N, args, s);
      if (st != RGNN_E_UNSUPPORTED) return st;
    }
    return gemm_dw_f32(prec, K, N, args, s);
  };
  // H_j = G_{v_j} W_{r_j}^T per (etype, dst) run j: one typed GEMM over the J runs (tf32 tensor
  // cores on the bf16 layer, W rounded as in the forward; SIMT fp32 otherwise), read by dX (NEXT-2).
  bool h_done = false;
  auto run_products = [&]() -> rgnn_status {
    { Phase ph("dx_prep", s);
      RGNN_TRY(launch_transpose_w(prec, g->R, K, N, W, w.Wt, s));
      if (model == RGNN_RGCN && W0) RGNN_TRY(launch_transpose_w(prec, 1, K, N, W0, w.Wt + (size_t)g->R * N * K, s));
      // the tf32 GEMM reads its weight transposed: (W^T)^T = W, rounded like the SIMT copy
      if (prec == RGNN_BF16) {
        RGNN_TRY(launch_round_bf16((int64_t)g->R * K * N, W, w.Wr, s));
        if (model == RGNN_RGCN && W0) RGNN_TRY(launch_round_bf16((int64_t)K * N, W0, w.Wr + (size_t)g->R * N * K, s));
      } else {
        RGNN_CUDA_TRY(cudaMemcpyAsync(w.Wr, W, sizeof(float) * g->R * K * N, cudaMemcpyDeviceToDevice, s));
        if (model == RGNN_RGCN && W0)
          RGNN_CUDA_TRY(cudaMemcpyAsync(w.Wr + (size_t)g->R * N * K, W0, sizeof(float) * K * N,
                                        cudaMemcpyDeviceToDevice, s));
      }
    }
    if (g->num_rtiles) {
      Phase ph("run_gemm", s);
      GemmFwdArgs gh{};
      gh.tiles = g->rtiles; gh.num_tiles = g->num_rtiles; gh.X = dY; gh.gather = g->run_dst; gh.W = w.Wt;
      gh.Z = w.H; gh.wt_bf16 = w.wt; gh.num_w = g->R; gh.x_rows = std::max<int64_t>(g->V_own, 1); gh.z_rows = g->J;
      RGNN_TRY(f32_gemm(prec, N, K, gh, w.Wr, s));  // GEMM K = d_out, N = d_in
    }
    h_done = true;
    return RGNN_OK;
  };
  if (model == RGNN_RGAT) {
    { Phase ph("fold_u", s); RGNN_TRY(launch_fold_u(prec, g->R, K, N, W, A, w.U, s)); }
    rgnn_status fst = RGNN_E_UNSUPPORTED;
    bool tm_done = false;
    // tensor-core backward where destination runs are long (ogbn-mag: mean run 14.5 positions); with short
    // runs (AM: 2.3) the per-run reads buy little and the fused kernel below is faster (measured r02: AM
    // 0.76 + 0.19 ms dst term vs 0.755 ms).  RGNN_BWD_TM=1 / 0 forces either.
    const int tm_env = getenv("RGNN_BWD_TM") ? atoi(getenv("RGNN_BWD_TM")) : -1;  // read per call (tests)
    const bool tm_pick = tm_env >= 0 ? tm_env != 0 : g->E_own >= 4 * std::max<int64_t>(g->J, 1);
    if (tc_ok && tm_pick && bwd_tm_enabled(K, N, prec)) {
      // tensor-core backward (bwd_tm.cu): Z tiles recomputed by tcgen05 from the staged X_src rows, the
      // destination rows read once per run, the destination term summed per run
      { Phase ph("bwd_tm", s);
        RGNN_TRY(launch_bwd_rgat_tm(K, N, g, X, W, w.wt, use_compact(g, model) ? g->crow_of_pos : nullptr, sv.s_src,
                                    w.U, sv.lse, Y, dY, slope, w.dwpart, w.dpre, want_dx ? w.ad : nullptr, s)); }
      { Phase ph("dst_term", s); RGNN_TRY(launch_dst_term(prec, K, g, w.dpre, X, w.cpart, s)); }
      Phase ph("dw_reduce", s);
      RGNN_TRY(launch_dw_reduce(prec, K, N, g->R, g->num_chunks, g->chunk_seg, w.dwpart, g->chunk_seg, w.cpart, A, W,
                                dW, dA, w.vsum, s, g->chunks, true));
      tm_done = true;
    } else if (tc_ok) {  // fused position-order backward: dZ built in smem, dW MMA + dst term in one kernel
      // (Measured r02 and rejected: dalpha_e = H_j . x_src with the run products H_j = G_v W_r^T, so the
      // kernel reads no Z rows -- ogbn-mag 3.64 -> 4.39 ms + 0.35 ms for the run GEMM, AM 0.85 -> 1.07
      // + 0.31 ms: the H row becomes one more dependent load at every destination change of the
      // compute warps, which are latency-bound there, while the Z rows it saves were prefetched by
      // the producers.)
      Phase ph("bwd_fused", s);
      fst = launch_bwd_fused_tc(K, N, g, X, sv.Z, use_compact(g, model) ? g->crow_of_pos : nullptr, sv.s_src, sv.lse,
                                Y, dY, w.U, A, slope, w.dwpart, w.cpart, want_dx ? w.ad : nullptr, s);
      if (fst != RGNN_OK && fst != RGNN_E_UNSUPPORTED) return fst;
    }
    if (tm_done) {
      // tensor-core backward above (dW, dA reduced)
    } else if (fst == RGNN_OK) {
      Phase ph("dw_reduce", s);
      RGNN_TRY(launch_dw_reduce(prec, K, N, g->R, g->num_chunks, g->chunk_seg, w.dwpart, g->chunk_seg, w.cpart, A, W,
                                dW, dA, w.vsum, s, g->chunks));
    } else {
    BwdArgs ba{};
    ba.items = g->items; ba.num_items = g->num_items; ba.pos = g->pos; ba.et_slot = g->et_slot; ba.Z = sv.Z;
    ba.s_src = sv.s_src; ba.X = X; ba.v0 = g->v0; ba.U = w.U; ba.A = A; ba.slope = slope; ba.Y = Y; ba.dY = dY;
    ba.lse = sv.lse; ba.dZ = w.dZ; ba.dpre = w.dpre; ba.zrow = use_compact(g, model) ? g->zrow_slot : nullptr;
    ba.ad = want_dx ? w.ad : nullptr;
    { Phase ph("bwd_traverse", s); RGNN_TRY(launch_bwd_traverse(prec, K, N, ba, s)); }
    { Phase ph("dst_term", s); RGNN_TRY(launch_dst_term(prec, K, g, w.dpre, X, w.cpart, s)); }
    da.Bz = w.dZ; da.dpre = w.dpre; da.dst_local = g->dst_s; da.v0 = g->v0;
    { Phase ph("gemm_dw", s); RGNN_TRY(dw_gemm(da)); }
    { Phase ph("dw_reduce", s); RGNN_TRY(launch_dw_reduce(prec, K, N, g->R, g->num_chunks, g->chunk_seg, w.dwpart, g->chunk_seg, w.cpart, A, W, dW, dA, w.vsum, s, g->chunks)); }
    }
  } else {
    rgnn_status fst = RGNN_E_UNSUPPORTED;
    if (tc_ok) {  // fused: dZ rows = G_v / c built in smem, tensor-core dW in the same kernel
      Phase ph("bwd_fused", s);
      fst = launch_bwd_fused_tc(K, N, g, X, nullptr, nullptr, nullptr, nullptr, nullptr, dY, nullptr, nullptr, 0.f, w.dwpart,
                                w.cpart, nullptr, s);
      if (fst != RGNN_OK && fst != RGNN_E_UNSUPPORTED) return fst;
    }
    if (fst != RGNN_OK) {
      if (tc_ok) {  // dZ[p] = bf16(1/c * G[dst]) materialised in position order, then the tensor-core dW
        { Phase ph("expand_dz", s); RGNN_TRY(launch_expand_dz(g->E_own, N, g->dst_s, g->inv_c, dY, w.Z, s)); }
        da.Bz = w.Z;
      } else {
        da.Bg = dY; da.bgather = g->dst_s; da.bscale = g->inv_c;
      }
      { Phase ph("gemm_dw", s); RGNN_TRY(dw_gemm(da)); }
    }
    { Phase ph("dw_reduce", s); RGNN_TRY(launch_dw_reduce(prec, K, N, g->R, g->num_chunks, g->chunk_seg, w.dwpart, nullptr, nullptr, nullptr, nullptr, dW, nullptr, nullptr, s, g->chunks)); }
    if (dW0) {
      Phase ph("gemm_dw0", s);
      GemmDwArgs d0{};
      d0.num_chunks = dw0_chunks(g); d0.rows = g->V_own; d0.chunk_rows = dw0_chunk_rows(g); d0.X = X;
      d0.gofs = g->v0; d0.part = w.dw0part; d0.x_rows = g->V;
      if (tc_ok) {
        RGNN_TRY(launch_expand_dz(g->V_own, N, nullptr, nullptr, dY, w.Z0, s));
        d0.Bz = w.Z0;
      } else {
        d0.Bg = dY;
      }
      RGNN_TRY(dw_gemm(d0));
      RGNN_TRY(launch_dw_reduce(prec, K, N, 1, d0.num_chunks, nullptr, w.dw0part, nullptr, nullptr, nullptr, nullptr, dW0, nullptr, nullptr, s));
    }
  }
  if (want_dx) {
    // dX (dx.cu): H = G_v W_r^T per (etype, dst) run by one typed GEMM, then the source walk
    // H = G_v W_r^T per run (fp32: rounding G or H to bf16 is too lossy for dX, dx.cu)
    if (!h_done) RGNN_TRY(run_products());
    if (model == RGNN_RGAT) {
      Phase ph("dx_prep", s);
      RGNN_TRY(launch_fold_u(prec, g->R, K, N, W, A, w.U0, s, 0));
    }
    const bool self = model == RGNN_RGCN && W0 && g->V_own > 0;
    if (self) {
      Phase ph("dx_gemm", s);
      GemmFwdArgs g0{};
      g0.rows = g->V_own; g0.X = dY; g0.gofs = 0; g0.W = w.Wt + (size_t)g->R * N * K; g0.Z = w.H0;
      g0.wt_bf16 = w.wt; g0.num_w = 1; g0.x_rows = g->V_own;
      RGNN_TRY(f32_gemm(prec, N, K, g0, w.Wr + (size_t)g->R * N * K, s));
    }
    {  // rows of nodes with out-edges are written by the source walk: zero only the others
      Phase ph("dx_zero", s);
      RGNN_TRY(launch_hgt_zero_rows(g->V, K, g->srow, dX, dX, 0, g->V, nullptr, 0, dX, s));
    }
    DxArgs xa{};
    xa.V = g->V; xa.V_own = g->V_own; xa.v0 = g->v0;
    xa.items = g->sitems; xa.num_items = g->num_sitems; xa.split = g->ssplit; xa.num_split = g->num_ssplit;
    xa.part = w.xpart; xa.srow = g->srow; xa.spos = g->spos; xa.srun = g->srun;
    xa.srel = g->srel; xa.sinvc = g->sinvc; xa.ad = w.ad; xa.H = w.H; xa.U0 = w.U0; xa.U1 = w.U;
    xa.ditems = g->items; xa.num_ditems = g->num_items; xa.dsplit = g->split_rows; xa.num_dsplit = g->num_split_rows;
    xa.dpart = w.dpart; xa.pos = g->pos; xa.et_slot = g->et_slot; xa.H0 = self ? w.H0 : nullptr;
    xa.dX = dX;
    RGNN_TRY(launch_dx_walk(K, model == RGNN_RGAT, xa, s));
  }
  if (comm) {
    float* bufs[3] = {dW, model == RGNN_RGAT ? dA : nullptr, model == RGNN_RGCN ? dW0 : nullptr};
    size_t counts[3] = {(size_t)g->R * K * N, (size_t)g->R * 2 * N, (size_t)K * N};
    Phase ph("comm", s);
    RGNN_TRY(comm_allreduce_sum(comm, bufs, counts, 3, s));
    if (dX) RGNN_TRY(comm_reduce_rows(comm, dX, K, s));  // dX reduce-scattered over the dst ranges
  }
  return RGNN_OK;
}

}  // extern "C"
