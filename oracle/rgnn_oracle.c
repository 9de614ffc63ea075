/*
 * rgnn_oracle.c -- plain, slow, fp64 CPU oracle for one RGCN / RGAT layer.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2301_06284_b200/csrc); it never includes include/rgnn.h.
 *
 * What it computes (PAPER.md = the paper's LaTeX source, "P:n" = line n):
 *   RGCN  (Sec. 2.1 equation)
 *     Y_v = sum_r sum_{u in N_v^r} (1/c_{v,r}) h_u W_r  (+ h_v W_0)
 *   RGAT  (Sec. 2.1, fig:rgnn_layer caption P:313, Listing 1)
 *     zi_e = h_src W_{r}, zj_e = h_dst W_{r}            (Listing 1)
 *     a_e  = leakyrelu(<attn_vec[r], [zi_e ; zj_e]>)    (Listing 1)
 *     alpha_e = exp(a_e) / sum_{e' -> dst} exp(a_e')    (edge softmax)
 *     Y_v  = sum_{e -> v} alpha_e zi_e                  (reading O1: message = zi)
 *   Backward: dW (and dA for RGAT, dW0 for RGCN) of L = <Y, G>; derived by the
 *   chain rule from the forward definition above (SURVEY.md Sec. 8 "Backward";
 *   DESIGN.md Sec. 3 readings).  No rank-1 shortcut, no fused U vector: zd
 *   is recomputed explicitly per edge.
 *   Preprocessing (Sec. 3.6 P:756 "converting COO to CSR"; P:845 presort for
 *   segment MM): the definitions of DESIGN.md reading O14, written out with a
 *   total-order qsort and counting passes.
 *
 * Readings of the paper used here (DESIGN.md Sec. 3 lists them all): O1 message
 * = zi; O2 A[r,0] pairs with zi, A[r,1] with zj; O3 softmax over ALL incoming
 * edges; O4 leaky slope is a parameter; O5 max-subtraction (flag to disable);
 * O6 zero in-degree -> 0 and lse = -inf; O7 c_{v,r} modes; O8 optional W0;
 * O11 z = x W_r with W[R,K,N] row major; O13 multi/self edges distinct.
 *
 * Arrays: row-major, int32 ids, fp64 values.  OpenMP parallelises over
 * destination rows only; reductions over threads are done in thread-index
 * order (deterministic for a fixed thread count).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#else
static int omp_get_max_threads(void) { return 1; }
static int omp_get_thread_num(void) { return 0; }
#endif

/* ------------------------------------------------------------------ */
/* Preprocessing (bit-exact contract, reading O14)           */
/* ------------------------------------------------------------------ */

typedef struct { int32_t et, dst, eid; } okey;

static int okey_cmp(const void* a, const void* b) {
  const okey* x = (const okey*)a;
  const okey* y = (const okey*)b;
  if (x->et != y->et) return x->et < y->et ? -1 : 1;
  if (x->dst != y->dst) return x->dst < y->dst ? -1 : 1;
  if (x->eid != y->eid) return x->eid < y->eid ? -1 : 1;
  return 0;
}

/* Returns E_own (edges whose dst is in [v0, v1)), or -1 on an id out of range.
 * Outputs (all sized by the caller for E_own / R+1 / V_own+1):
 *   perm[p]    original edge id at position p; positions = own edges sorted by
 *              (etype, dst), ties by ascending edge id (a stable sort)
 *   src_s[p]   src[perm[p]]
 *   seg[r]     number of own edges with etype < r  (seg[R] = E_own)
 *   row_ptr[i] CSR-by-dst over local rows i = v - v0
 *   pos[q]     positions p of row i listed in ascending p
 *   et_slot[q] etype of slot q
 *   cnt[p]     c_{v,r} = |N_v^r| counting multi-edges (reading O7)
 * bad_edge (may be NULL) receives the smallest offending edge id.            */
int64_t oracle_preprocess(int64_t V, int64_t E, int32_t R, const int32_t* src, const int32_t* dst,
                          const int32_t* et, int64_t v0, int64_t v1, int32_t* perm, int32_t* src_s,
                          int32_t* seg, int32_t* row_ptr, int32_t* pos, int32_t* et_slot, int32_t* cnt,
                          int64_t* bad_edge) {
  for (int64_t e = 0; e < E; ++e) {
    if (src[e] < 0 || src[e] >= V || dst[e] < 0 || dst[e] >= V || et[e] < 0 || et[e] >= R) {
      if (bad_edge) *bad_edge = e;
      return -1;
    }
  }
  int64_t Vown = v1 - v0;
  int64_t Eown = 0;
  for (int64_t e = 0; e < E; ++e) Eown += (dst[e] >= v0 && dst[e] < v1);
  okey* keys = (okey*)malloc(sizeof(okey) * (size_t)(Eown > 0 ? Eown : 1));
  int64_t n = 0;
  for (int64_t e = 0; e < E; ++e)
    if (dst[e] >= v0 && dst[e] < v1) { keys[n].et = et[e]; keys[n].dst = dst[e]; keys[n].eid = (int32_t)e; ++n; }
  qsort(keys, (size_t)Eown, sizeof(okey), okey_cmp);
  for (int64_t p = 0; p < Eown; ++p) { perm[p] = keys[p].eid; src_s[p] = src[keys[p].eid]; }
  /* seg: count per etype then prefix */
  for (int32_t r = 0; r <= R; ++r) seg[r] = 0;
  for (int64_t p = 0; p < Eown; ++p) seg[keys[p].et + 1]++;
  for (int32_t r = 0; r < R; ++r) seg[r + 1] += seg[r];
  /* row_ptr: count per dst then prefix */
  for (int64_t i = 0; i <= Vown; ++i) row_ptr[i] = 0;
  for (int64_t p = 0; p < Eown; ++p) row_ptr[keys[p].dst - v0 + 1]++;
  for (int64_t i = 0; i < Vown; ++i) row_ptr[i + 1] += row_ptr[i];
  /* pos: stable counting sort of positions by dst (ascending p within a row) */
  int32_t* fill = (int32_t*)malloc(sizeof(int32_t) * (size_t)(Vown > 0 ? Vown : 1));
  for (int64_t i = 0; i < Vown; ++i) fill[i] = row_ptr[i];
  for (int64_t p = 0; p < Eown; ++p) {
    int64_t i = keys[p].dst - v0;
    pos[fill[i]++] = (int32_t)p;
  }
  for (int64_t q = 0; q < Eown; ++q) et_slot[q] = keys[pos[q]].et;
  /* cnt: length of the run of equal (etype, dst) keys containing p */
  int64_t p = 0;
  while (p < Eown) {
    int64_t s = p;
    while (p < Eown && keys[p].et == keys[s].et && keys[p].dst == keys[s].dst) ++p;
    for (int64_t t = s; t < p; ++t) cnt[t] = (int32_t)(p - s);
  }
  free(fill);
  free(keys);
  return Eown;
}

/* ------------------------------------------------------------------ */
/* Shared forward helpers (oracle-private)                             */
/* ------------------------------------------------------------------ */

/* In-edge lists for every node: in_ptr[V+1], in_eid[E] (ascending edge id). */
static void build_in_lists(int64_t V, int64_t E, const int32_t* dst, int64_t** in_ptr_out, int32_t** in_eid_out) {
  int64_t* ptr = (int64_t*)calloc((size_t)V + 1, sizeof(int64_t));
  int32_t* eid = (int32_t*)malloc(sizeof(int32_t) * (size_t)(E > 0 ? E : 1));
  for (int64_t e = 0; e < E; ++e) ptr[dst[e] + 1]++;
  for (int64_t v = 0; v < V; ++v) ptr[v + 1] += ptr[v];
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(V > 0 ? V : 1));
  for (int64_t v = 0; v < V; ++v) fill[v] = ptr[v];
  for (int64_t e = 0; e < E; ++e) eid[fill[dst[e]]++] = (int32_t)e;
  free(fill);
  *in_ptr_out = ptr;
  *in_eid_out = eid;
}

/* z = x W_r : x [K], W_r [K,N] row major (reading O11) */
static void vecmat(int K, int N, const double* x, const double* Wr, double* z) {
  for (int n = 0; n < N; ++n) z[n] = 0.0;
  for (int k = 0; k < K; ++k) {
    double xk = x[k];
    const double* w = Wr + (size_t)k * N;
    for (int n = 0; n < N; ++n) z[n] += xk * w[n];
  }
}

static double dot(int N, const double* a, const double* b) {
  double s = 0.0;
  for (int n = 0; n < N; ++n) s += a[n] * b[n];
  return s;
}

static double leaky(double x, double slope) { return x > 0.0 ? x : slope * x; }   /* O4: f(0)=0 */
static double leaky_grad(double x, double slope) { return x > 0.0 ? 1.0 : slope; } /* O4 */

/* c_{v,r} counts for one row (reading O7, mode 0): cnt[r] = |N_v^r| over ALL of
 * v's incoming edges (multi-edges counted).  Caller clears with row_count_clear. */
static void row_count(int64_t lo, int64_t hi, const int32_t* in_eid, const int32_t* et, int64_t* cnt) {
  for (int64_t q = lo; q < hi; ++q) cnt[et[in_eid[q]]]++;
}
static void row_count_clear(int64_t lo, int64_t hi, const int32_t* in_eid, const int32_t* et, int64_t* cnt) {
  for (int64_t q = lo; q < hi; ++q) cnt[et[in_eid[q]]] = 0;
}
/* 1/c factor of edge e under norm mode (O7): 0 = 1/|N_v^r|, 1 = none, 2 = caller per-edge norm. */
static double rgcn_factor(int norm, const double* edge_norm, const int64_t* cnt, const int32_t* et, int32_t e) {
  if (norm == 1) return 1.0;
  if (norm == 2) return edge_norm[e];
  return 1.0 / (double)cnt[et[e]];
}

/* ------------------------------------------------------------------ */
/* RGCN forward                                            */
/* ------------------------------------------------------------------ */
/* Y[i,:] for v = rows[i].  W0 may be NULL (reading O8).                */
void oracle_rgcn_forward(int64_t V, int64_t E, int32_t R, int32_t K, int32_t N, const int32_t* src,
                         const int32_t* dst, const int32_t* et, const double* X, const double* W,
                         const double* W0, int32_t norm, const double* edge_norm, int64_t n_rows,
                         const int64_t* rows, double* Y) {
  int64_t* in_ptr;
  int32_t* in_eid;
  build_in_lists(V, E, dst, &in_ptr, &in_eid);
#pragma omp parallel
  {
    double* z = (double*)malloc(sizeof(double) * (size_t)N);
    int64_t* cnt = (int64_t*)calloc((size_t)R, sizeof(int64_t));
#pragma omp for schedule(dynamic, 64)
    for (int64_t i = 0; i < n_rows; ++i) {
      int64_t v = rows[i];
      double* acc = Y + (size_t)i * N;
      if (W0) vecmat(K, N, X + (size_t)v * K, W0, acc);
      else for (int n = 0; n < N; ++n) acc[n] = 0.0;
      row_count(in_ptr[v], in_ptr[v + 1], in_eid, et, cnt);
      for (int64_t q = in_ptr[v]; q < in_ptr[v + 1]; ++q) {
        int32_t e = in_eid[q];
        int32_t r = et[e];
        vecmat(K, N, X + (size_t)src[e] * K, W + (size_t)r * K * N, z);
        double f = rgcn_factor(norm, edge_norm, cnt, et, e);
        for (int n = 0; n < N; ++n) acc[n] += z[n] * f;
      }
      row_count_clear(in_ptr[v], in_ptr[v + 1], in_eid, et, cnt);
    }
    free(z);
    free(cnt);
  }
  free(in_ptr);
  free(in_eid);
}

/* ------------------------------------------------------------------ */
/* RGAT forward (Listing 1)               */
/* ------------------------------------------------------------------ */
/* Outputs Y[i,:], lse[i] = m + ln(l) (-inf at zero in-degree, O6) and, if
 * alpha != NULL, alpha[e] for every incoming edge e of the listed rows.
 * stabilize = 1 subtracts the per-destination max (O5); 0 evaluates the
 * paper's plain exp/sum exp.                                               */
void oracle_rgat_forward(int64_t V, int64_t E, int32_t R, int32_t K, int32_t N, const int32_t* src,
                         const int32_t* dst, const int32_t* et, const double* X, const double* W,
                         const double* A, double slope, int32_t stabilize, int64_t n_rows, const int64_t* rows,
                         double* Y, double* lse, double* alpha) {
  (void)R;
  int64_t* in_ptr;
  int32_t* in_eid;
  build_in_lists(V, E, dst, &in_ptr, &in_eid);
#pragma omp parallel
  {
    double* zi = (double*)malloc(sizeof(double) * (size_t)N);
    double* zj = (double*)malloc(sizeof(double) * (size_t)N);
    int64_t cap = 0;
    double* s = NULL;
#pragma omp for schedule(dynamic, 16)
    for (int64_t i = 0; i < n_rows; ++i) {
      int64_t v = rows[i];
      int64_t lo = in_ptr[v], hi = in_ptr[v + 1], deg = hi - lo;
      double* acc = Y + (size_t)i * N;
      for (int n = 0; n < N; ++n) acc[n] = 0.0;
      if (deg == 0) { lse[i] = -INFINITY; continue; }
      if (deg > cap) { cap = deg; s = (double*)realloc(s, sizeof(double) * (size_t)cap); }
      /* pass 1: scores a_e = leakyrelu(A[r,0].zi + A[r,1].zj) */
      double m = -INFINITY;
      for (int64_t q = lo; q < hi; ++q) {
        int32_t e = in_eid[q], r = et[e];
        const double* Wr = W + (size_t)r * K * N;
        vecmat(K, N, X + (size_t)src[e] * K, Wr, zi);
        vecmat(K, N, X + (size_t)v * K, Wr, zj);
        double pre = dot(N, A + (size_t)r * 2 * N, zi) + dot(N, A + (size_t)r * 2 * N + N, zj);
        s[q - lo] = leaky(pre, slope);
        if (s[q - lo] > m) m = s[q - lo];
      }
      if (!stabilize) m = 0.0;
      /* pass 2: l = sum exp(s - m); Y_v = sum alpha_e zi_e (zi recomputed) */
      double l = 0.0;
      for (int64_t q = lo; q < hi; ++q) l += exp(s[q - lo] - m);
      for (int64_t q = lo; q < hi; ++q) {
        int32_t e = in_eid[q], r = et[e];
        double a = exp(s[q - lo] - m) / l;
        if (alpha) alpha[e] = a;
        vecmat(K, N, X + (size_t)src[e] * K, W + (size_t)r * K * N, zi);
        for (int n = 0; n < N; ++n) acc[n] += a * zi[n];
      }
      lse[i] = m + log(l);
    }
    free(zi);
    free(zj);
    free(s);
  }
  free(in_ptr);
  free(in_eid);
}

/* ------------------------------------------------------------------ */
/* Backward of L = <Y, G> (gradients of the forward definitions above) */
/* ------------------------------------------------------------------ */
/* Only destinations v in [v0, v1) contribute (a dst-range shard; summing the
 * shards over a partition of [0,V) gives the full gradient).  G is indexed by
 * node id [V, N].  rel_mask (R bytes, may be NULL) restricts the OUTPUT to the
 * selected relations; every softmax still runs over all incoming edges (O3).
 *
 * RGAT per edge e = (u -> v, r), recomputing everything:
 *   zi = x_u W_r, zj = x_v W_r, pre = A[r,0].zi + A[r,1].zj, s = leaky(pre)
 *   alpha = softmax_v(s);  dalpha_e = G_v . zi;  S_v = sum_e alpha_e dalpha_e
 *   ds_e = alpha_e (dalpha_e - S_v);  dpre_e = ds_e * leaky'(pre)
 *   dzi = alpha_e G_v + dpre_e A[r,0];  dzj = dpre_e A[r,1]
 *   dW_r += x_u^T dzi + x_v^T dzj;  dA[r,0] += dpre_e zi;  dA[r,1] += dpre_e zj   */
void oracle_rgat_backward(int64_t V, int64_t E, int32_t R, int32_t K, int32_t N, const int32_t* src,
                          const int32_t* dst, const int32_t* et, const double* X, const double* W,
                          const double* A, double slope, const double* G, int64_t v0, int64_t v1,
                          const uint8_t* rel_mask, double* dW, double* dA) {
  int64_t* in_ptr;
  int32_t* in_eid;
  build_in_lists(V, E, dst, &in_ptr, &in_eid);
  int nt = omp_get_max_threads();
  size_t wsz = (size_t)R * K * N, asz = (size_t)R * 2 * N;
  double* tdW = (double*)calloc((size_t)nt * wsz, sizeof(double));
  double* tdA = (double*)calloc((size_t)nt * asz, sizeof(double));
#pragma omp parallel
  {
    int tid = omp_get_thread_num();
    double* mydW = tdW + (size_t)tid * wsz;
    double* mydA = tdA + (size_t)tid * asz;
    double* zi = (double*)malloc(sizeof(double) * (size_t)N);
    double* zj = (double*)malloc(sizeof(double) * (size_t)N);
    double* dzi = (double*)malloc(sizeof(double) * (size_t)N);
    int64_t cap = 0;
    double *pre = NULL, *al = NULL, *da = NULL;
#pragma omp for schedule(dynamic, 16)
    for (int64_t v = v0; v < v1; ++v) {
      int64_t lo = in_ptr[v], hi = in_ptr[v + 1], deg = hi - lo;
      if (deg == 0) continue;
      int any = (rel_mask == NULL);
      for (int64_t q = lo; q < hi && !any; ++q) any = rel_mask[et[in_eid[q]]] != 0;
      if (!any) continue;
      if (deg > cap) {
        cap = deg;
        pre = (double*)realloc(pre, sizeof(double) * (size_t)cap);
        al = (double*)realloc(al, sizeof(double) * (size_t)cap);
        da = (double*)realloc(da, sizeof(double) * (size_t)cap);
      }
      const double* Gv = G + (size_t)v * N;
      double m = -INFINITY;
      for (int64_t q = lo; q < hi; ++q) {
        int32_t e = in_eid[q], r = et[e];
        const double* Wr = W + (size_t)r * K * N;
        vecmat(K, N, X + (size_t)src[e] * K, Wr, zi);
        vecmat(K, N, X + (size_t)v * K, Wr, zj);
        pre[q - lo] = dot(N, A + (size_t)r * 2 * N, zi) + dot(N, A + (size_t)r * 2 * N + N, zj);
        double s = leaky(pre[q - lo], slope);
        if (s > m) m = s;
        da[q - lo] = dot(N, Gv, zi);
      }
      double l = 0.0;
      for (int64_t q = lo; q < hi; ++q) { al[q - lo] = exp(leaky(pre[q - lo], slope) - m); l += al[q - lo]; }
      double S = 0.0;
      for (int64_t q = lo; q < hi; ++q) { al[q - lo] /= l; S += al[q - lo] * da[q - lo]; }
      for (int64_t q = lo; q < hi; ++q) {
        int32_t e = in_eid[q], r = et[e];
        if (rel_mask && !rel_mask[r]) continue;
        const double* Wr = W + (size_t)r * K * N;
        const double* xu = X + (size_t)src[e] * K;
        const double* xv = X + (size_t)v * K;
        const double* A0 = A + (size_t)r * 2 * N;
        const double* A1 = A0 + N;
        double a = al[q - lo];
        double dpre = a * (da[q - lo] - S) * leaky_grad(pre[q - lo], slope);
        vecmat(K, N, xu, Wr, zi);
        vecmat(K, N, xv, Wr, zj);
        for (int n = 0; n < N; ++n) dzi[n] = a * Gv[n] + dpre * A0[n];
        double* dWr = mydW + (size_t)r * K * N;
        for (int k = 0; k < K; ++k) {
          double xuk = xu[k], xvk = xv[k];
          double* row = dWr + (size_t)k * N;
          for (int n = 0; n < N; ++n) row[n] += xuk * dzi[n] + xvk * (dpre * A1[n]);
        }
        double* dAr = mydA + (size_t)r * 2 * N;
        for (int n = 0; n < N; ++n) { dAr[n] += dpre * zi[n]; dAr[N + n] += dpre * zj[n]; }
      }
    }
    free(zi); free(zj); free(dzi); free(pre); free(al); free(da);
  }
  memset(dW, 0, sizeof(double) * wsz);
  memset(dA, 0, sizeof(double) * asz);
  for (int t = 0; t < nt; ++t) {
    for (size_t i = 0; i < wsz; ++i) dW[i] += tdW[(size_t)t * wsz + i];
    for (size_t i = 0; i < asz; ++i) dA[i] += tdA[(size_t)t * asz + i];
  }
  free(tdW);
  free(tdA);
  free(in_ptr);
  free(in_eid);
}

/* RGCN: dW_r = sum_{e in r, dst in [v0,v1)} x_u^T G_v / c_{v,r};
 *       dW0  = sum_{v in [v0,v1)} x_v^T G_v   (if dW0 != NULL).           */
void oracle_rgcn_backward(int64_t V, int64_t E, int32_t R, int32_t K, int32_t N, const int32_t* src,
                          const int32_t* dst, const int32_t* et, const double* X, int32_t norm,
                          const double* edge_norm, const double* G, int64_t v0, int64_t v1,
                          const uint8_t* rel_mask, double* dW, double* dW0) {
  int64_t* in_ptr;
  int32_t* in_eid;
  build_in_lists(V, E, dst, &in_ptr, &in_eid);
  int nt = omp_get_max_threads();
  size_t wsz = (size_t)R * K * N, w0sz = (size_t)K * N;
  double* tdW = (double*)calloc((size_t)nt * wsz, sizeof(double));
  double* tdW0 = (double*)calloc((size_t)nt * w0sz, sizeof(double));
#pragma omp parallel
  {
    int tid = omp_get_thread_num();
    double* mydW = tdW + (size_t)tid * wsz;
    double* mydW0 = tdW0 + (size_t)tid * w0sz;
    int64_t* cnt = (int64_t*)calloc((size_t)R, sizeof(int64_t));
#pragma omp for schedule(dynamic, 64)
    for (int64_t v = v0; v < v1; ++v) {
      const double* Gv = G + (size_t)v * N;
      if (dW0) {
        const double* xv = X + (size_t)v * K;
        for (int k = 0; k < K; ++k)
          for (int n = 0; n < N; ++n) mydW0[(size_t)k * N + n] += xv[k] * Gv[n];
      }
      row_count(in_ptr[v], in_ptr[v + 1], in_eid, et, cnt);
      for (int64_t q = in_ptr[v]; q < in_ptr[v + 1]; ++q) {
        int32_t e = in_eid[q], r = et[e];
        if (rel_mask && !rel_mask[r]) continue;
        double f = rgcn_factor(norm, edge_norm, cnt, et, e);
        const double* xu = X + (size_t)src[e] * K;
        double* dWr = mydW + (size_t)r * K * N;
        for (int k = 0; k < K; ++k) {
          double c = xu[k] * f;
          for (int n = 0; n < N; ++n) dWr[(size_t)k * N + n] += c * Gv[n];
        }
      }
      row_count_clear(in_ptr[v], in_ptr[v + 1], in_eid, et, cnt);
    }
    free(cnt);
  }
  memset(dW, 0, sizeof(double) * wsz);
  for (int t = 0; t < nt; ++t)
    for (size_t i = 0; i < wsz; ++i) dW[i] += tdW[(size_t)t * wsz + i];
  if (dW0) {
    memset(dW0, 0, sizeof(double) * w0sz);
    for (int t = 0; t < nt; ++t)
      for (size_t i = 0; i < w0sz; ++i) dW0[i] += tdW0[(size_t)t * w0sz + i];
  }
  free(tdW);
  free(tdW0);
  free(in_ptr);
  free(in_eid);
}

/* ------------------------------------------------------------------ */
/* Input-feature gradient dX ("required       */
/* gradients"), written out by the chain rule from the forward above.  */
/* ------------------------------------------------------------------ */

/* y += W_r d : W_r [K,N] row major, d [N] -> y [K]  (d z W_r^T for z = x W_r) */
static void matvec_t(int K, int N, const double* Wr, const double* d, double* y) {
  for (int k = 0; k < K; ++k) {
    double acc = 0.0;
    for (int n = 0; n < N; ++n) acc += Wr[(size_t)k * N + n] * d[n];
    y[k] += acc;
  }
}

/* RGAT dX [V, K] of L = <Y, G> restricted to dst in [v0, v1):
 *   zi_e = x_src W_r, zj_e = x_dst W_r, pre_e = A[r,0].zi + A[r,1].zj (Listing 1)
 *   dzi_e = alpha_e G_v + dpre_e A[r,0]   ->  dX[src] += dzi_e W_r^T
 *   dzj_e = dpre_e A[r,1]                 ->  dX[dst] += dzj_e W_r^T
 * with alpha, dpre exactly as in oracle_rgat_backward.  Thread partials of dX
 * are summed in thread order.                                              */
void oracle_rgat_dx(int64_t V, int64_t E, int32_t R, int32_t K, int32_t N, const int32_t* src, const int32_t* dst,
                    const int32_t* et, const double* X, const double* W, const double* A, double slope,
                    const double* G, int64_t v0, int64_t v1, double* dX) {
  int64_t* in_ptr;
  int32_t* in_eid;
  build_in_lists(V, E, dst, &in_ptr, &in_eid);
  int nt = omp_get_max_threads();
  size_t xsz = (size_t)V * K;
  double* tdX = (double*)calloc((size_t)nt * xsz + 1, sizeof(double));
#pragma omp parallel
  {
    double* mydX = tdX + (size_t)omp_get_thread_num() * xsz;
    double* zi = (double*)malloc(sizeof(double) * (size_t)N);
    double* zj = (double*)malloc(sizeof(double) * (size_t)N);
    double* dz = (double*)malloc(sizeof(double) * (size_t)N);
    int64_t cap = 0;
    double *pre = NULL, *al = NULL, *da = NULL;
#pragma omp for schedule(dynamic, 16)
    for (int64_t v = v0; v < v1; ++v) {
      int64_t lo = in_ptr[v], hi = in_ptr[v + 1], deg = hi - lo;
      if (deg == 0) continue;
      if (deg > cap) {
        cap = deg;
        pre = (double*)realloc(pre, sizeof(double) * (size_t)cap);
        al = (double*)realloc(al, sizeof(double) * (size_t)cap);
        da = (double*)realloc(da, sizeof(double) * (size_t)cap);
      }
      const double* Gv = G + (size_t)v * N;
      double m = -INFINITY;
      for (int64_t q = lo; q < hi; ++q) {
        int32_t e = in_eid[q], r = et[e];
        const double* Wr = W + (size_t)r * K * N;
        vecmat(K, N, X + (size_t)src[e] * K, Wr, zi);
        vecmat(K, N, X + (size_t)v * K, Wr, zj);
        pre[q - lo] = dot(N, A + (size_t)r * 2 * N, zi) + dot(N, A + (size_t)r * 2 * N + N, zj);
        double s = leaky(pre[q - lo], slope);
        if (s > m) m = s;
        da[q - lo] = dot(N, Gv, zi);
      }
      double l = 0.0;
      for (int64_t q = lo; q < hi; ++q) { al[q - lo] = exp(leaky(pre[q - lo], slope) - m); l += al[q - lo]; }
      double S = 0.0;
      for (int64_t q = lo; q < hi; ++q) { al[q - lo] /= l; S += al[q - lo] * da[q - lo]; }
      for (int64_t q = lo; q < hi; ++q) {
        int32_t e = in_eid[q], r = et[e];
        const double* Wr = W + (size_t)r * K * N;
        const double* A0 = A + (size_t)r * 2 * N;
        const double* A1 = A0 + N;
        double a = al[q - lo];
        double dpre = a * (da[q - lo] - S) * leaky_grad(pre[q - lo], slope);
        for (int n = 0; n < N; ++n) dz[n] = a * Gv[n] + dpre * A0[n];
        matvec_t(K, N, Wr, dz, mydX + (size_t)src[e] * K);
        for (int n = 0; n < N; ++n) dz[n] = dpre * A1[n];
        matvec_t(K, N, Wr, dz, mydX + (size_t)v * K);
      }
    }
    free(zi); free(zj); free(dz); free(pre); free(al); free(da);
  }
  memset(dX, 0, sizeof(double) * xsz);
  for (int t = 0; t < nt; ++t)
    for (size_t i = 0; i < xsz; ++i) dX[i] += tdX[(size_t)t * xsz + i];
  free(tdX);
  free(in_ptr);
  free(in_eid);
}

/* RGCN dX [V, K] of L = <Y, G> restricted to dst in [v0, v1):
 *   dX[src] += (1/c_{v,r}) G_v W_r^T  for every edge (src -> v, r),
 *   dX[v]   += G_v W0^T               (self loop, if W0 != NULL).          */
void oracle_rgcn_dx(int64_t V, int64_t E, int32_t R, int32_t K, int32_t N, const int32_t* src, const int32_t* dst,
                    const int32_t* et, const double* W, const double* W0, int32_t norm, const double* edge_norm,
                    const double* G, int64_t v0, int64_t v1, double* dX) {
  int64_t* in_ptr;
  int32_t* in_eid;
  build_in_lists(V, E, dst, &in_ptr, &in_eid);
  int nt = omp_get_max_threads();
  size_t xsz = (size_t)V * K;
  double* tdX = (double*)calloc((size_t)nt * xsz + 1, sizeof(double));
#pragma omp parallel
  {
    double* mydX = tdX + (size_t)omp_get_thread_num() * xsz;
    double* dz = (double*)malloc(sizeof(double) * (size_t)N);
    int64_t* cnt = (int64_t*)calloc((size_t)R, sizeof(int64_t));
#pragma omp for schedule(dynamic, 64)
    for (int64_t v = v0; v < v1; ++v) {
      const double* Gv = G + (size_t)v * N;
      if (W0) matvec_t(K, N, W0, Gv, mydX + (size_t)v * K);
      row_count(in_ptr[v], in_ptr[v + 1], in_eid, et, cnt);
      for (int64_t q = in_ptr[v]; q < in_ptr[v + 1]; ++q) {
        int32_t e = in_eid[q], r = et[e];
        double f = rgcn_factor(norm, edge_norm, cnt, et, e);
        for (int n = 0; n < N; ++n) dz[n] = f * Gv[n];
        matvec_t(K, N, W + (size_t)r * K * N, dz, mydX + (size_t)src[e] * K);
      }
      row_count_clear(in_ptr[v], in_ptr[v + 1], in_eid, et, cnt);
    }
    free(dz);
    free(cnt);
  }
  memset(dX, 0, sizeof(double) * xsz);
  for (int t = 0; t < nt; ++t)
    for (size_t i = 0; i < xsz; ++i) dX[i] += tdX[(size_t)t * xsz + i];
  free(tdX);
  free(in_ptr);
  free(in_eid);
}

/* ------------------------------------------------------------------ */
/* HGT layer         */
/* ------------------------------------------------------------------ */
/* Forward, for each destination t and incoming edge e = (s -> t, r):
 *   k_e = x_s WK[tau(s)],  q_t = x_t WQ[tau(t)],  v_e = x_s WV[tau(s)]   (typed linear W_tau(n))
 *   a_e = k_e^T W_{a,r} q_t = sum_{m,n} k_e[m] Wa[r][m][n] q_t[n]
 *   alpha_e = softmax over all incoming edges of t
 *   m_e = v_e W_{m,r}  ("determined by source node features and edge types")
 *   Y_t = sum_e alpha_e m_e                                                (reading O23)
 * WK/WQ/WV [T, K, N]; Wa/Wm [R, N, N] row major.  Zero in-degree: Y = 0, lse = -inf. */
void oracle_hgt_forward(int64_t V, int64_t E, int32_t R, int32_t T, int32_t K, int32_t N, const int32_t* src,
                        const int32_t* dst, const int32_t* et, const int32_t* ntype, const double* X,
                        const double* WK, const double* WQ, const double* WV, const double* Wa, const double* Wm,
                        int64_t n_rows, const int64_t* rows, double* Y, double* lse) {
  (void)R; (void)T;
  int64_t* in_ptr;
  int32_t* in_eid;
  build_in_lists(V, E, dst, &in_ptr, &in_eid);
#pragma omp parallel
  {
    double* q = (double*)malloc(sizeof(double) * (size_t)N);
    double* k = (double*)malloc(sizeof(double) * (size_t)N);
    double* kw = (double*)malloc(sizeof(double) * (size_t)N);
    double* vv = (double*)malloc(sizeof(double) * (size_t)N);
    double* mm = (double*)malloc(sizeof(double) * (size_t)N);
    int64_t cap = 0;
    double* s = NULL;
#pragma omp for schedule(dynamic, 16)
    for (int64_t i = 0; i < n_rows; ++i) {
      int64_t t = rows[i];
      int64_t lo = in_ptr[t], hi = in_ptr[t + 1], deg = hi - lo;
      double* acc = Y + (size_t)i * N;
      for (int n = 0; n < N; ++n) acc[n] = 0.0;
      if (deg == 0) { lse[i] = -INFINITY; continue; }
      if (deg > cap) { cap = deg; s = (double*)realloc(s, sizeof(double) * (size_t)cap); }
      vecmat(K, N, X + (size_t)t * K, WQ + (size_t)ntype[t] * K * N, q);
      double m = -INFINITY;
      for (int64_t e_ = lo; e_ < hi; ++e_) {
        int32_t e = in_eid[e_], r = et[e], u = src[e];
        vecmat(K, N, X + (size_t)u * K, WK + (size_t)ntype[u] * K * N, k);
        vecmat(N, N, k, Wa + (size_t)r * N * N, kw);
        s[e_ - lo] = dot(N, kw, q);
        if (s[e_ - lo] > m) m = s[e_ - lo];
      }
      double l = 0.0;
      for (int64_t e_ = lo; e_ < hi; ++e_) l += exp(s[e_ - lo] - m);
      for (int64_t e_ = lo; e_ < hi; ++e_) {
        int32_t e = in_eid[e_], r = et[e], u = src[e];
        double a = exp(s[e_ - lo] - m) / l;
        vecmat(K, N, X + (size_t)u * K, WV + (size_t)ntype[u] * K * N, vv);
        vecmat(N, N, vv, Wm + (size_t)r * N * N, mm);
        for (int n = 0; n < N; ++n) acc[n] += a * mm[n];
      }
      lse[i] = m + log(l);
    }
    free(q); free(k); free(kw); free(vv); free(mm); free(s);
  }
  free(in_ptr);
  free(in_eid);
}

/* HGT backward (NEXT-3): gradients of L = <Y, G> restricted to dst in [v0, v1) w.r.t.
 * WK, WQ, WV [T, K, N] and Wa, Wm [R, N, N], by the chain rule of oracle_hgt_forward:
 *   dm_e = alpha_e G_t,  dalpha_e = G_t . m_e,  S_t = sum_e alpha_e dalpha_e,
 *   da_e = alpha_e (dalpha_e - S_t),
 *   dWm[r] += v_e^T dm_e,  dv_e = dm_e Wm[r]^T,  dWV[tau(s)] += x_s^T dv_e
 *   dkw_e = da_e q_t,  dWa[r] += k_e^T dkw_e,  dk_e = dkw_e Wa[r]^T,  dWK[tau(s)] += x_s^T dk_e
 *   dq_t = sum_e da_e kw_e,  dWQ[tau(t)] += x_t^T dq_t
 * Thread partials summed in thread order.                                      */
void oracle_hgt_backward(int64_t V, int64_t E, int32_t R, int32_t T, int32_t K, int32_t N, const int32_t* src,
                         const int32_t* dst, const int32_t* et, const int32_t* ntype, const double* X,
                         const double* WK, const double* WQ, const double* WV, const double* Wa, const double* Wm,
                         const double* G, int64_t v0, int64_t v1, double* dWK, double* dWQ, double* dWV, double* dWa,
                         double* dWm) {
  int64_t* in_ptr;
  int32_t* in_eid;
  build_in_lists(V, E, dst, &in_ptr, &in_eid);
  int nt = omp_get_max_threads();
  size_t tsz = (size_t)T * K * N, rsz = (size_t)R * N * N, tot = 3 * tsz + 2 * rsz;
  double* part = (double*)calloc((size_t)nt * tot + 1, sizeof(double));
#pragma omp parallel
  {
    double* my = part + (size_t)omp_get_thread_num() * tot;
    double *mWK = my, *mWQ = my + tsz, *mWV = my + 2 * tsz, *mWa = my + 3 * tsz, *mWm = my + 3 * tsz + rsz;
    double* q = (double*)malloc(sizeof(double) * (size_t)N);
    double* k = (double*)malloc(sizeof(double) * (size_t)N);
    double* kw = (double*)malloc(sizeof(double) * (size_t)N);
    double* vv = (double*)malloc(sizeof(double) * (size_t)N);
    double* mm = (double*)malloc(sizeof(double) * (size_t)N);
    double* dq = (double*)malloc(sizeof(double) * (size_t)N);
    double* d1 = (double*)malloc(sizeof(double) * (size_t)N);
    double* d2 = (double*)malloc(sizeof(double) * (size_t)N);
    int64_t cap = 0;
    double *a = NULL, *al = NULL, *da = NULL;
#pragma omp for schedule(dynamic, 16)
    for (int64_t t = v0; t < v1; ++t) {
      int64_t lo = in_ptr[t], hi = in_ptr[t + 1], deg = hi - lo;
      if (deg == 0) continue;
      if (deg > cap) {
        cap = deg;
        a = (double*)realloc(a, sizeof(double) * (size_t)cap);
        al = (double*)realloc(al, sizeof(double) * (size_t)cap);
        da = (double*)realloc(da, sizeof(double) * (size_t)cap);
      }
      const double* Gt = G + (size_t)t * N;
      const double* xt = X + (size_t)t * K;
      vecmat(K, N, xt, WQ + (size_t)ntype[t] * K * N, q);
      double m = -INFINITY;
      for (int64_t e_ = lo; e_ < hi; ++e_) {
        int32_t e = in_eid[e_], r = et[e], u = src[e];
        vecmat(K, N, X + (size_t)u * K, WK + (size_t)ntype[u] * K * N, k);
        vecmat(N, N, k, Wa + (size_t)r * N * N, kw);
        a[e_ - lo] = dot(N, kw, q);
        if (a[e_ - lo] > m) m = a[e_ - lo];
        vecmat(K, N, X + (size_t)u * K, WV + (size_t)ntype[u] * K * N, vv);
        vecmat(N, N, vv, Wm + (size_t)r * N * N, mm);
        da[e_ - lo] = dot(N, Gt, mm); /* dalpha_e */
      }
      double l = 0.0;
      for (int64_t e_ = lo; e_ < hi; ++e_) { al[e_ - lo] = exp(a[e_ - lo] - m); l += al[e_ - lo]; }
      double S = 0.0;
      for (int64_t e_ = lo; e_ < hi; ++e_) { al[e_ - lo] /= l; S += al[e_ - lo] * da[e_ - lo]; }
      for (int n = 0; n < N; ++n) dq[n] = 0.0;
      for (int64_t e_ = lo; e_ < hi; ++e_) {
        int32_t e = in_eid[e_], r = et[e], u = src[e];
        const double* xu = X + (size_t)u * K;
        double aa = al[e_ - lo], dae = aa * (da[e_ - lo] - S);
        vecmat(K, N, xu, WK + (size_t)ntype[u] * K * N, k);
        vecmat(N, N, k, Wa + (size_t)r * N * N, kw);
        vecmat(K, N, xu, WV + (size_t)ntype[u] * K * N, vv);
        /* message path: dm = alpha G; dWm[r] += v^T dm; dv = dm Wm^T; dWV[tau(u)] += x_u^T dv */
        double* gWm = mWm + (size_t)r * N * N;
        for (int i = 0; i < N; ++i)
          for (int j = 0; j < N; ++j) gWm[(size_t)i * N + j] += vv[i] * aa * Gt[j];
        for (int i = 0; i < N; ++i) d1[i] = 0.0;
        for (int j = 0; j < N; ++j) d2[j] = aa * Gt[j];
        matvec_t(N, N, Wm + (size_t)r * N * N, d2, d1);
        double* gWV = mWV + (size_t)ntype[u] * K * N;
        for (int i = 0; i < K; ++i)
          for (int j = 0; j < N; ++j) gWV[(size_t)i * N + j] += xu[i] * d1[j];
        /* score path: dkw = da q; dWa[r] += k^T dkw; dk = dkw Wa^T; dWK[tau(u)] += x_u^T dk; dq += da kw */
        double* gWa = mWa + (size_t)r * N * N;
        for (int i = 0; i < N; ++i)
          for (int j = 0; j < N; ++j) gWa[(size_t)i * N + j] += k[i] * dae * q[j];
        for (int i = 0; i < N; ++i) d1[i] = 0.0;
        for (int j = 0; j < N; ++j) d2[j] = dae * q[j];
        matvec_t(N, N, Wa + (size_t)r * N * N, d2, d1);
        double* gWK = mWK + (size_t)ntype[u] * K * N;
        for (int i = 0; i < K; ++i)
          for (int j = 0; j < N; ++j) gWK[(size_t)i * N + j] += xu[i] * d1[j];
        for (int n = 0; n < N; ++n) dq[n] += dae * kw[n];
      }
      double* gWQ = mWQ + (size_t)ntype[t] * K * N;
      for (int i = 0; i < K; ++i)
        for (int j = 0; j < N; ++j) gWQ[(size_t)i * N + j] += xt[i] * dq[j];
    }
    free(q); free(k); free(kw); free(vv); free(mm); free(dq); free(d1); free(d2); free(a); free(al); free(da);
  }
  double* outs[5] = {dWK, dWQ, dWV, dWa, dWm};
  size_t offs[5] = {0, tsz, 2 * tsz, 3 * tsz, 3 * tsz + rsz};
  size_t lens[5] = {tsz, tsz, tsz, rsz, rsz};
  for (int o = 0; o < 5; ++o) {
    memset(outs[o], 0, sizeof(double) * lens[o]);
    for (int th = 0; th < nt; ++th)
      for (size_t i = 0; i < lens[o]; ++i) outs[o][i] += part[(size_t)th * tot + offs[o] + i];
  }
  free(part);
  free(in_ptr);
  free(in_eid);
}

int oracle_num_threads(void) { return omp_get_max_threads(); }
