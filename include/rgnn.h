/*
 * rgnn.h -- C ABI of librgnn.so: one RGCN / RGAT layer over a heterogeneous
 * graph on NVIDIA B200 (sm_100a).  This is the boundary the Python binding
 * (paper_2301_06284_b200/_binding.py) and every GPU test call through.
 *
 * Paper: arXiv 2301.06284 (PAPER.md = its LaTeX source; "P:n" = line n).
 *   RGCN layer ............ Sec. 2.1 equation
 *   RGAT attention ........ Sec. 2.1, fig:rgnn_layer caption P:313,
 *                           Listing 1 P:461-478 (zi, zj, inner_prod with
 *                           concat, leakyrelu, edge_softmax)
 *   typed linear / segment MM  Sec. 2.2; P:845 ("presorted")
 *   preprocessing list .... Sec. 3.6 P:756 ("converting COO to CSR")
 *   backward .............. Sec. 3.5 P:731-742 (only the required grads)
 * Readings where the paper is silent are DESIGN.md Sec. 3 (O1..O22).
 *
 * Conventions (all entry points):
 *  - Pointers are DEVICE pointers unless marked [host].  `stream` is a
 *    cudaStream_t passed as void*; every call is asynchronous on it unless
 *    marked SYNC.  Asynchronous device faults surface at the caller's next
 *    synchronisation.
 *  - The library never allocates device memory.  Every device buffer (graph
 *    storage, scratch, workspace, saved activations, outputs) is owned by the
 *    caller (PyTorch tensors in the binding); the library carves them.
 *    Buffers must be 256-byte aligned.  The graph storage must outlive the
 *    handle; a workspace must not be shared by two concurrent calls.
 *  - Errors are status codes; nothing throws or aborts across the ABI.
 *    rgnn_last_error() (thread-local) describes the last failure.
 *  - Layouts are row major.  Ids are int32 (E < 2^31; RGNN_E_UNSUPPORTED
 *    otherwise).  Feature widths d_in, d_out must be in {32, 64, 128}.
 *  - Determinism: the forward has no atomics and is bit-reproducible; the
 *    backward reduces in a fixed order and is bit-reproducible for a fixed
 *    graph and dst range.  Row-split decisions depend only on the row, so
 *    the owned rows of a dst-range shard are bit-identical to 1-GPU rows.
 */
#ifndef RGNN_H_
#define RGNN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RGNN_OK = 0,
  RGNN_E_INVALID_ARG = 1,  /* NULL required pointer, bad size or range      */
  RGNN_E_RANGE = 2,        /* an edge id out of range (see rgnn_last_error) */
  RGNN_E_UNSUPPORTED = 3,  /* width / size / feature not supported          */
  RGNN_E_WORKSPACE = 4,    /* a caller buffer is smaller than required      */
  RGNN_E_CUDA = 5,         /* a CUDA runtime call or launch failed          */
  RGNN_E_NCCL = 6          /* an NCCL call failed                           */
} rgnn_status;

/* Operand precision of X / Z / dZ.  Accumulation is always fp32; Y, dW, dA
 * are fp32.  RGNN_BF16: X arrives as bf16, W is rounded to bf16 (RNE) inside
 * the call, the typed GEMMs run on tcgen05 tensor cores (bf16 x bf16 -> fp32
 * in TMEM) and Z / dZ are stored bf16 (RNE).  RGNN_F32: fp32 everywhere,
 * SIMT FFMA GEMMs (reading O16).                                            */
typedef enum { RGNN_F32 = 0, RGNN_BF16 = 1 } rgnn_prec;

/* RGCN normalisation 1/c_{v,r} ("a problem-specific normalization
 * factor"; reading O7): relation in-degree |N_v^r| (default), none (c = 1),
 * or a caller-supplied per-edge factor edge_norm[e].                        */
typedef enum { RGNN_NORM_REL_INDEG = 0, RGNN_NORM_NONE = 1, RGNN_NORM_EDGE = 2 } rgnn_norm;

typedef enum { RGNN_RGCN = 0, RGNN_RGAT = 1, RGNN_HGT = 2 } rgnn_model;

/* Where per-edge tensors (Z, s_src) live (Sec. 3.1.3).
 * VANILLA: one row per edge (the row number is the edge's position).
 * COMPACT: one row per unique (etype, src) pair, numbered lexicographically
 * (reading O15); the typed GEMM then runs over U_src rows instead of E.     */
/* AUTO: the compact tables are built, and each layer call picks per model:
 * RGCN compact whenever U < E_own (its backward never reads Z); RGAT compact
 * when U <= 3/4 E_own (its backward then gathers Z rows at random instead of
 * streaming them -- measured r02: ogbn-mag U/E = 0.15 and AM 0.56 win).
 * rgnn_zrows() reports the choice.                                          */
typedef enum { RGNN_MAT_VANILLA = 0, RGNN_MAT_COMPACT = 1, RGNN_MAT_AUTO = 2 } rgnn_materialization;

/* rgnn_graph_desc.flags.  RGNN_GRAPH_DX: also build the tables the input-
 * feature gradient needs (rgnn_backward with dX != NULL):
 * run of each position and its destination / relation, and a source-major
 * CSR over the positions with a split work list (≈ 7 int32 per edge + V).  */
#define RGNN_GRAPH_DX 1
/* RGNN_GRAPH_AGGFIRST: build the run-piece tables of the
 * aggregate-first RGCN forward -- Y_v = sum_r (1/c_{v,r}) (sum_{e in run(r,v)}
 * x_src) W_r: each (etype, dst) run cut into pieces of <= 64 positions,
 * A_i = sum (1/c) x_src per piece, one typed GEMM P_i = A_i W_r over the
 * pieces, and the destination walk adds each row's piece products.
 * rgcn_forward on such a graph uses that formulation (the per-edge Z is
 * never formed); the backward is unchanged.  (≈ 3 int32 per edge.)        */
#define RGNN_GRAPH_AGGFIRST 2

typedef struct rgnn_graph rgnn_graph;
typedef struct rgnn_comm rgnn_comm;

/* Graph description (heterograph; tab:ir_constructs P:498). */
typedef struct {
  int64_t num_nodes;         /* V (global)                                   */
  int64_t num_edges;         /* E = length of src / dst / etype              */
  int32_t num_etypes;        /* R (relations)                                */
  int32_t num_ntypes;        /* T; checked only if ntype != NULL             */
  const int32_t* src;        /* [E] COO source ids (or CSR column ids)       */
  const int32_t* dst;        /* [E] COO destination ids; ignored for CSR     */
  const int32_t* etype;      /* [E] relation id of each edge                 */
  const int32_t* row_ptr;    /* [V+1] CSR-by-dst input, or NULL for COO      */
  const int32_t* ntype;      /* [V] node types, or NULL (validated only)     */
  const float* edge_norm;    /* [E] required iff norm == RGNN_NORM_EDGE      */
  int32_t norm;              /* rgnn_norm                                    */
  int32_t row_split_cap;     /* max in-edges per work item; 0 = 256          */
  int64_t dst_begin;         /* owned destination range [dst_begin, dst_end) */
  int64_t dst_end;           /* (0, V) on one GPU                            */
  int32_t materialization;   /* rgnn_materialization (0 = vanilla)           */
  int32_t flags;             /* RGNN_GRAPH_* bits (0 = none)                 */
} rgnn_graph_desc;

/* What the preprocessing built (device pointers into the caller's graph
 * storage), for inspection and the bit-exact tests.  Positions p index the
 * owned edges sorted by (etype, dst), ties by ascending edge id (reading
 * O14); slots q index CSR-by-dst.                                          */
typedef struct {
  int64_t V, V_own, dst_begin, E_own, num_runs, num_tiles, num_items, num_split_rows;
  int32_t R;
  const int32_t* perm;     /* [E_own] original edge id of position p        */
  const int32_t* src_s;    /* [E_own] src of position p                     */
  const int32_t* dst_s;    /* [E_own] local dst (v - dst_begin) of p        */
  const int32_t* seg;      /* [R+1]   relation segments in position space   */
  const int32_t* row_ptr;  /* [V_own+1] CSR-by-dst over local rows          */
  const int32_t* pos;      /* [E_own] positions of each row, ascending      */
  const int32_t* et_slot;  /* [E_own] relation of slot q                    */
  const float* inv_c;      /* [E_own] RGCN factor of position p (1/c_{v,r}) */
  const int32_t* run_ptr;  /* [num_runs+1] (etype,dst) runs, position space */
  const int32_t* rseg;     /* [R+1]   runs of relation r                    */
  const int32_t* seg_host; /* [host, R+1] copy of seg                       */
  int64_t num_compact;     /* unique (etype, src) pairs U (0: not built)    */
  const int32_t* crow_of_pos; /* [E_own] compact row of position p          */
  const int32_t* csrc;     /* [num_compact] src node of compact row         */
  const int32_t* cseg;     /* [R+1] compact rows of relation r              */
  int64_t num_pieces;      /* run pieces (<= 64 positions of one run; 0: not built) */
  const int32_t* piece_ptr;  /* [num_pieces+1] first position of piece i    */
  const int32_t* slot_piece; /* [E_own] piece of slot q's position (AGGFIRST) */
  const float* slot_w;     /* [E_own] 1 for a piece's first slot in its row, else 0 (AGGFIRST) */
} rgnn_graph_view;

/* Sizes of the caller-owned graph storage (kept for the handle's life) and
 * scratch (needed only during rgnn_graph_create).  [host] desc.           */
rgnn_status rgnn_graph_bytes(const rgnn_graph_desc* desc, size_t* dev_bytes, size_t* scratch_bytes);

/* Preprocessing (Sec. 3.6; DESIGN.md Sec. 6 "a0"): validate
 * ids; keep edges whose dst is owned; stable sort by (etype, dst); relation
 * segments; CSR-by-dst; (etype,dst) runs and 1/c; GEMM tile table; degree-
 * aware work list (rows longer than row_split_cap are split into chunks).
 * SYNC: two host synchronisations -- the validation flags with the owned-
 * edge count, then the counts and relation segments (a third one when node
 * types, dX tables or run pieces are built); the 128-row tile and dW chunk
 * tables are then built on the host from the segments.
 * RGNN_E_RANGE names the SMALLEST offending edge id (atomicMin).  CSR
 * input: row_ptr is checked on the device (row_ptr[0] = 0, non-decreasing,
 * row_ptr[V] = E) before it is used; a bad one returns RGNN_E_INVALID_ARG
 * naming the first bad index (the expansion never writes outside [0, E)). */
rgnn_status rgnn_graph_create(const rgnn_graph_desc* desc, void* dev, size_t dev_bytes, void* scratch,
                              size_t scratch_bytes, void* stream, rgnn_graph** out);
rgnn_status rgnn_graph_export(const rgnn_graph* g, rgnn_graph_view* view /* [host] */);
void rgnn_graph_destroy(rgnn_graph* g); /* frees the host struct only */

/* Rows of the per-edge tensors (Z, s_src) a layer of `model` materialises on
 * this graph: U = number of unique (etype, src) pairs when compact rows are
 * used, else E_own.  [host] rows.                      */
rgnn_status rgnn_zrows(const rgnn_graph* g, rgnn_model model, int64_t* rows);

/* Workspace and saved-activation sizes for one layer call.  `saved` links a
 * forward to its backward (RGAT: Z, s_src, lse; RGCN: nothing).
 * training: 0 inference, 1 training, RGNN_WS_DX (3) training with dX -- the
 * workspace of a backward that computes dX must be sized with RGNN_WS_DX.  */
#define RGNN_WS_DX 3
rgnn_status rgnn_workspace_bytes(const rgnn_graph* g, rgnn_model model, int d_in, int d_out, rgnn_prec prec,
                                 int training, size_t* ws_bytes, size_t* saved_bytes);

/* RGCN forward: Y_v = sum_{e: dst=v} (1/c_{v,r}) X_src W_r
 * (+ X_v W0 if W0 != NULL) for owned v, pre-activation (reading O9).
 *   X  [V, d_in]  fp32 or bf16 (per prec), all V rows (replicated)
 *   W  [R, d_in, d_out] fp32, z = x W_r (reading O11); W0 [d_in, d_out] or NULL
 *   Y  [V_own, d_out] fp32 (owned rows, local order)
 * If comm != NULL and Y_full != NULL, owned rows of every rank are gathered
 * into Y_full [V, d_out] (NCCL grouped broadcasts); Y may alias
 * Y_full + dst_begin * d_out.                                              */
rgnn_status rgcn_forward(const rgnn_graph* g, int d_in, int d_out, rgnn_prec prec, const void* X, const float* W,
                         const float* W0, float* Y, void* saved, void* ws, size_t ws_bytes, rgnn_comm* comm,
                         float* Y_full, void* stream);

/* RGAT forward (Listing 1; readings O1-O6):
 *   pre_e = A[r,0].(X_src W_r) + A[r,1].(X_dst W_r),  s_e = LeakyReLU_slope(pre_e)
 *   alpha_e = softmax over ALL incoming edges of dst,  Y_v = sum alpha_e X_src W_r
 *   A [R, 2, d_out] fp32.  Zero in-degree rows give Y_v = 0.  saved must be
 *   passed unchanged to rgnn_backward.                                     */
rgnn_status rgat_forward(const rgnn_graph* g, int d_in, int d_out, rgnn_prec prec, const void* X, const float* W,
                         const float* A, float slope, float* Y, void* saved, void* ws, size_t ws_bytes,
                         rgnn_comm* comm, float* Y_full, void* stream);

/* HGT forward (reading O23):
 *   k = x_s WK[tau(s)], q = x_t WQ[tau(t)], v = x_s WV[tau(s)]   (node-typed linears)
 *   a_e = (k W_{a,r}) . q,  alpha = softmax over ALL incoming edges of t,
 *   Y_t = sum_e alpha_e (v W_{m,r})     -- one head, no extra scaling
 *   WK, WQ, WV [T, d_in, d_out] fp32; Wa, Wm [R, d_out, d_out] fp32; X as in
 *   rgat_forward.  The graph must carry node types (desc.ntype, num_ntypes
 *   = T; else RGNN_E_UNSUPPORTED).  k W_{a,r} and v W_{m,r} are formed once
 *   per (etype, src) pair when the graph has compact rows (rgnn_zrows with
 *   RGNN_HGT), else once per edge.  saved (rgnn_workspace_bytes with
 *   RGNN_HGT) receives lse [V_own] and the typed-linear outputs k, q, v,
 *   k W_{a,r}, v W_{m,r} that hgt_backward reads.                          */
rgnn_status hgt_forward(const rgnn_graph* g, int d_in, int d_out, rgnn_prec prec, const void* X, const float* WK,
                        const float* WQ, const float* WV, const float* Wa, const float* Wm, float* Y, void* saved,
                        void* ws, size_t ws_bytes, rgnn_comm* comm, float* Y_full, void* stream);

/* HGT backward (NEXT-3): gradients of L = <Y, dY> over the owned rows w.r.t.
 * the five weights, by the chain rule of hgt_forward (DESIGN.md Sec. 6 "HGT"):
 *   da_e = alpha_e (dY_t . m_e - dY_t . Y_t);  dWm[r] = sum_e v_s^T alpha_e dY_t;
 *   dWa[r] = sum_e k_s^T da_e q_t;  dq_t = sum_e da_e k_s W_{a,r};
 *   dv_s = sum_{e: src=s} alpha_e dY_t Wm_r^T;  dk_s = sum_e da_e q_t Wa_r^T;
 *   dWK / dWV / dWQ [tau] = sum over the nodes of type tau of x^T dk / dv / dq.
 *   dWK, dWQ, dWV [T, d_in, d_out], dWa, dWm [R, d_out, d_out] fp32, overwritten.
 * Y [V_own, d_out] and saved are the forward's; dY [V_own, d_out] fp32.  The
 * graph needs node types and RGNN_GRAPH_DX (source-major tables; else
 * RGNN_E_UNSUPPORTED); the workspace is sized with training = 1 (else
 * RGNN_E_WORKSPACE).  With comm != NULL the gradients are all-reduced (sum)
 * in place.  WK, WQ, WV are not read (their gradients need only X and the
 * saved activations) and may be NULL.                                      */
rgnn_status hgt_backward(const rgnn_graph* g, int d_in, int d_out, rgnn_prec prec, const void* X, const float* WK,
                         const float* WQ, const float* WV, const float* Wa, const float* Wm, const float* Y,
                         const float* dY, const void* saved, float* dWK, float* dWQ, float* dWV, float* dWa,
                         float* dWm, void* ws, size_t ws_bytes, rgnn_comm* comm, void* stream);

/* Backward of L = <Y, dY> over the owned rows (Sec. 3.5; reading O17):
 *   dW [R, d_in, d_out] fp32 (required), dA [R, 2, d_out] (RGAT, required),
 *   dW0 [d_in, d_out] (RGCN, iff W0 was used, else NULL).  Y is the forward
 *   output for the owned rows and dY [V_own, d_out] fp32.
 *   dX [V, d_in] fp32 or NULL: input-feature gradient (the
 *   chain rule of the forward through X_src and, for RGAT, X_dst; DESIGN.md
 *   Sec. 6 "dX") over ALL V rows -- a shard's contribution from its owned
 *   edges.  Needs a graph built with RGNN_GRAPH_DX and a workspace sized
 *   with RGNN_WS_DX (else RGNN_E_UNSUPPORTED / RGNN_E_WORKSPACE); RGCN with a
 *   self loop also needs W0 [d_in, d_out] (NULL: no self-loop term).
 *   With comm != NULL, dW / dA / dW0 are all-reduced (sum) in place across
 *   ranks, and dX is reduce-scattered over the dst partition: rows
 *   [bounds[k], bounds[k+1]) of rank k's dX hold the full sum (the rows the
 *   previous layer's rank k owns); its other rows keep rank k's partial
 *   sums.  Outputs are overwritten.                                        */
rgnn_status rgnn_backward(const rgnn_graph* g, rgnn_model model, int d_in, int d_out, rgnn_prec prec,
                          const void* X, const float* W, const float* W0, const float* A, float slope,
                          const float* Y, const float* dY, const void* saved, float* dW, float* dA, float* dW0,
                          float* dX, void* ws, size_t ws_bytes, rgnn_comm* comm, void* stream);

/* Multi-GPU (one process per GPU; dst-range partition).
 * rgnn_comm_unique_id writes a 128-byte NCCL id to `id` [host]; rank 0
 * creates it and the caller broadcasts it (torch.distributed).  `bounds`
 * (identical on every rank) gives rank k the rows [bounds[k], bounds[k+1]);
 * each rank's graph must be created with exactly its range.  SYNC.        */
rgnn_status rgnn_comm_unique_id(void* id /* [host] 128 B */);
rgnn_status rgnn_comm_create(const void* id /* [host] 128 B */, int nranks, int rank,
                             const int64_t* bounds /* [host] nranks+1 dst-range cut */, rgnn_comm** out);
void rgnn_comm_destroy(rgnn_comm* c);

/* Gather options (SURVEY.md Sec. 8(e) mitigations; default 0 = synchronous fp32 gather):
 *   RGNN_COMM_GATHER_ASYNC  the forward's Y gather runs on the communicator's
 *     own stream (a second NCCL communicator split from the first) after an
 *     event on the caller's stream, which continues at once -- e.g. with the
 *     backward, which reads only owned rows.  rgnn_comm_join(c, stream) makes
 *     `stream` wait for the pending gather: call it before Y_full is read
 *     (and before the end of a CUDA-graph capture that issued the gather).
 *   RGNN_COMM_GATHER_BF16   Y_full is bf16 [V, d_out]: the owned rows are
 *     rounded (RNE) into Y_full's own slice and broadcast from there (half
 *     the NVLink volume); Y stays the fp32 owned rows.                      */
#define RGNN_COMM_GATHER_ASYNC 1
#define RGNN_COMM_GATHER_BF16 2
rgnn_status rgnn_comm_set_options(rgnn_comm* c, int flags);
rgnn_status rgnn_comm_join(rgnn_comm* c, void* stream);

/* Peer-memory communicator ("P2P stores fused into the N-K2 epilogue"; no
 * NCCL).  One process per GPU; the buffers of every rank are mapped into every process with CUDA
 * IPC, so a forward's walk kernels store each finished Y row straight into every rank's Y_full (the
 * transfer overlaps the rest of the walk; NVLink stores on a multi-GPU box) and a device-side
 * barrier (signal words, release / acquire at system scope) ends the call: Y_full is complete on
 * every rank in stream order, with no host synchronisation (CUDA-graph capturable).  An entry
 * barrier before the first peer store orders it after everything each rank did with its Y_full
 * earlier in its stream.  dW / dA / dW0
 * are all-reduced through the staging buffers (each rank sums all ranks' partials in rank order:
 * bit-identical on every rank).  Y_full is fp32 (the gather options above do not apply); dX is not
 * supported (RGNN_E_UNSUPPORTED; use NCCL).  Ranks may share one GPU (tests).
 *   rgnn_comm_create_local: the communicator without transport (nranks <= 8).  [host]
 *   rgnn_ipc_export: the IPC handle [host, 64 B] of the allocation holding `ptr` and ptr's offset in it.
 *   rgnn_comm_attach_peers: `handles` [host, nranks x 3 x 64 B] and `offsets` [host, nranks x 3]
 *     are every rank's exports of (Y_full, sig, stage) in rank order (exchanged by the caller, e.g.
 *     torch.distributed); Y_full [V, d_out] fp32, sig >= 9 uint32 zeroed before first use, stage
 *     >= the gradient floats of one backward (R*d_in*d_out + R*2*d_out + d_in*d_out) -- all
 *     caller-owned, alive for the communicator's life.  SYNC (opens the mappings).              */
rgnn_status rgnn_comm_create_local(int nranks, int rank, const int64_t* bounds /* [host] nranks+1 */,
                                   rgnn_comm** out);
rgnn_status rgnn_ipc_export(const void* ptr, void* handle /* [host] 64 B */, int64_t* offset /* [host] */);
rgnn_status rgnn_comm_attach_peers(rgnn_comm* c, const void* handles, const int64_t* offsets, float* Y_full,
                                   uint32_t* sig, float* stage, size_t stage_floats);

/* Balanced dst-range cut from the global in-degree prefix (host helper):
 * bounds[k] = the v whose indeg_prefix[v] is closest to k*E/P (ties -> the
 * smaller v), nondecreasing, bounds[0] = 0, bounds[P] = V.  Deterministic.
 * indeg_prefix [host, V+1], bounds [host, P+1].                            */
rgnn_status rgnn_partition_dst(int64_t V, const int64_t* indeg_prefix, int nparts, int64_t* bounds);

/* Phase profiler (tracing).  When enabled, every layer call records CUDA
 * events on the caller's stream around each kernel phase ("gemm_fwd",
 * "aggregate", "merge", "bwd_traverse", "gemm_dw", "dw_reduce", "fold_u",
 * "comm").  rgnn_profile_read (SYNC: waits for the events) returns up to
 * `max` phases -- name (32 chars each, NUL padded), total ms and number of
 * launches since the last read -- and resets the accumulators.             */
void rgnn_profile_enable(int on);
int rgnn_profile_read(char* names /* [host] max*32 */, double* ms /* [host] */, int64_t* count /* [host] */,
                      int max);

/* Kernel-launch counter (every kernel the library launches increments it). */
uint64_t rgnn_launch_count(void);

const char* rgnn_last_error(void);
const char* rgnn_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RGNN_H_ */
