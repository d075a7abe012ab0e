/*
 * oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for one SAGA-NN
 * GNN layer at inference (Zhang et al., "Architectural Implications of Graph
 * Neural Networks", IEEE CAL 2020, arXiv 2009.00804).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.  It
 * shares no code, header, table or helper with the CUDA path
 * (paper_2009_00804_b200/csrc); neither includes the other.
 *
 * Every function computes the plain definition in SAGA order (PAPER.md
 * Section 2 "Model Decomposition", lines 135-147: Scatter -> ApplyEdge ->
 * Gather -> ApplyVertex; Table 1 `tbl:benchmark`, lines 176-180), in double
 * precision, one destination vertex at a time, with no blocking, fusion or
 * algebraic reordering.  Inputs are the exact stored values (bf16 and fp32
 * inputs are upcast exactly to double).  The readings A1..A23 referenced
 * below are listed in DESIGN.md section "Readings of the paper".
 *
 * Pins (tests/test_oracle_*.py, `-m "not gpu"`): dense-adjacency brute force
 * (NumPy, torch fp64), d-regular GCN closed form, hand-computed path graph,
 * softmax sums, GRU closed forms and torch.nn.GRUCell(fp64), relabelling
 * invariance, SPEC examples for CSR.  No function here is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_X_F32 0
#define ORACLE_X_BF16 1
#define ORACLE_X_F64 2

/* Read element (row, col) of a row-major feature matrix of width `cols`
 * stored as fp32, bf16 (raw uint16 bits) or fp64; exact upcast to double. */
static double load_x(const void *x, int dtype, int64_t row, int64_t cols, int64_t col) {
    int64_t i = row * cols + col;
    if (dtype == ORACLE_X_F32) return (double)((const float *)x)[i];
    if (dtype == ORACLE_X_F64) return ((const double *)x)[i];
    uint32_t bits = ((uint32_t)((const uint16_t *)x)[i]) << 16;
    float f;
    memcpy(&f, &bits, sizeof f);
    return (double)f;
}

/* ------------------------------------------------------------------------
 * CSR build (S0).  PAPER.md line 130 ("the graph structure in the form of
 * adjacency matrix"), lines 351-354 (row = destination vertex, column = its
 * in-edge); reading A7: rows sorted by destination, ties kept in ascending
 * COO index (a stable counting sort), row_ptr int64, the rest int32.
 * Returns -1 on success, else the LOWEST COO index whose src/dst (or etype)
 * is out of range (nothing is written in that case).
 * ---------------------------------------------------------------------- */
int64_t oracle_csr_build(int32_t n, int64_t e, const int32_t *src, const int32_t *dst,
                         const int32_t *etype, int32_t num_etypes,
                         int64_t *row_ptr, int32_t *col_src, int32_t *edge_id,
                         int32_t *etype_csr, int32_t *in_deg, int32_t *out_deg) {
    for (int64_t i = 0; i < e; ++i) {
        if (src[i] < 0 || src[i] >= n || dst[i] < 0 || dst[i] >= n) return i;
        if (etype && (etype[i] < 0 || etype[i] >= num_etypes)) return i;
    }
    for (int32_t v = 0; v < n; ++v) { in_deg[v] = 0; out_deg[v] = 0; }
    for (int64_t i = 0; i < e; ++i) { in_deg[dst[i]] += 1; out_deg[src[i]] += 1; }
    row_ptr[0] = 0;
    for (int32_t v = 0; v < n; ++v) row_ptr[v + 1] = row_ptr[v] + in_deg[v];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    for (int32_t v = 0; v < n; ++v) fill[v] = row_ptr[v];
    for (int64_t i = 0; i < e; ++i) {          /* ascending COO index => stable */
        int64_t p = fill[dst[i]]++;
        edge_id[p] = (int32_t)i;
        col_src[p] = src[i];
        etype_csr[p] = etype ? etype[i] : 0;
    }
    free(fill);
    return -1;
}

/* Rows to evaluate: rows[0..nrows) or, if rows == NULL, all n rows. */
static int64_t row_at(const int64_t *rows, int64_t i) { return rows ? rows[i] : i; }

/* ------------------------------------------------------------------------
 * GCN layer (configs C1, C5).  Table 1: Scatter -, ApplyEdge -,
 * Gather sum(in_edges), ApplyVertex MLP.  Symmetric normalisation
 * D^-1/2 (A+I) D^-1/2 (BASELINE.json configs C1/C5) with A[v][u] = number
 * of edges u->v (reading A1: D = in-degree of A+I; the self-loops are
 * already edges of the COO, reading A2).  Per in-edge weight
 * w(u->v) = deg(u)^-1/2 deg(v)^-1/2 (0 for degree 0, reading A12).
 *   gather[v] = sum_{e=(u->v)} w(u->v) X[u]            (Gather, fp64)
 *   out[v]    = act(gather[v] . W + b)                  (ApplyVertex)
 * W is [f_in][f_out] row-major (reading A8); act: 0 none, 1 ReLU.
 * out is [nrows][f_out] in the order of `rows`.
 * ---------------------------------------------------------------------- */
void oracle_gcn(int32_t n, const int64_t *row_ptr, const int32_t *col_src, const int32_t *in_deg,
                const void *x, int x_dtype, int32_t f_in, const double *W, int32_t f_out,
                const double *b, int act, const int64_t *rows, int64_t nrows, double *out) {
    if (!rows) nrows = n;
#pragma omp parallel
    {
        double *g = (double *)malloc(sizeof(double) * (size_t)f_in);
#pragma omp for schedule(dynamic, 64)
        for (int64_t i = 0; i < nrows; ++i) {
            int64_t v = row_at(rows, i);
            for (int32_t k = 0; k < f_in; ++k) g[k] = 0.0;
            double dv = in_deg[v] > 0 ? 1.0 / sqrt((double)in_deg[v]) : 0.0;
            for (int64_t p = row_ptr[v]; p < row_ptr[v + 1]; ++p) {
                int32_t u = col_src[p];
                double du = in_deg[u] > 0 ? 1.0 / sqrt((double)in_deg[u]) : 0.0;
                double w = du * dv;
                for (int32_t k = 0; k < f_in; ++k) g[k] += w * load_x(x, x_dtype, u, f_in, k);
            }
            double *o = out + i * (int64_t)f_out;
            for (int32_t j = 0; j < f_out; ++j) o[j] = b ? b[j] : 0.0;
            for (int32_t k = 0; k < f_in; ++k)
                for (int32_t j = 0; j < f_out; ++j) o[j] += g[k] * W[(int64_t)k * f_out + j];
            if (act == 1)
                for (int32_t j = 0; j < f_out; ++j) o[j] = o[j] > 0.0 ? o[j] : 0.0;
        }
        free(g);
    }
}

/* ------------------------------------------------------------------------
 * GraphSAGE-mean layer (config C2).  Table 1 line 180 gives GraphSAGE's
 * stage shape (Gather over in_edges plus the vertex itself, ApplyVertex MLP);
 * BASELINE.json config C2 fixes the mean aggregator and
 * concat(self, neighbour-mean) then GEMM (reading A11):
 *   M[v]   = (1/deg(v)) sum_{e=(u->v)} X[u]   (0 if deg(v) = 0, A12)
 *   out[v] = act([X[v] || M[v]] . W + b)      W is [2 f_in][f_out]
 * ---------------------------------------------------------------------- */
void oracle_sage_mean(int32_t n, const int64_t *row_ptr, const int32_t *col_src, const int32_t *in_deg,
                      const void *x, int x_dtype, int32_t f_in, const double *W, int32_t f_out,
                      const double *b, int act, const int64_t *rows, int64_t nrows, double *out) {
    if (!rows) nrows = n;
#pragma omp parallel
    {
        double *cat = (double *)malloc(sizeof(double) * 2 * (size_t)f_in);
#pragma omp for schedule(dynamic, 64)
        for (int64_t i = 0; i < nrows; ++i) {
            int64_t v = row_at(rows, i);
            for (int32_t k = 0; k < f_in; ++k) {
                cat[k] = load_x(x, x_dtype, v, f_in, k);
                cat[f_in + k] = 0.0;
            }
            for (int64_t p = row_ptr[v]; p < row_ptr[v + 1]; ++p)
                for (int32_t k = 0; k < f_in; ++k) cat[f_in + k] += load_x(x, x_dtype, col_src[p], f_in, k);
            if (in_deg[v] > 0)
                for (int32_t k = 0; k < f_in; ++k) cat[f_in + k] /= (double)in_deg[v];
            double *o = out + i * (int64_t)f_out;
            for (int32_t j = 0; j < f_out; ++j) o[j] = b ? b[j] : 0.0;
            for (int32_t k = 0; k < 2 * f_in; ++k)
                for (int32_t j = 0; j < f_out; ++j) o[j] += cat[k] * W[(int64_t)k * f_out + j];
            if (act == 1)
                for (int32_t j = 0; j < f_out; ++j) o[j] = o[j] > 0.0 ? o[j] : 0.0;
        }
        free(cat);
    }
}

/* ------------------------------------------------------------------------
 * GAT layer (config C3).  Table 1: Scatter src&dst, ApplyEdge MLP
 * producing an edge embedding of size 1 (the attention score, lines
 * 324-325), Gather attention(in_edges), ApplyVertex MLP.  With heads H and
 * head width D (reading A13: heads concatenated, a_src applied to the source
 * and a_dst to the destination, every edge incl. self-loop and parallel
 * edges its own softmax term, ELU after aggregation):
 *   z[u]      = X[u] . W                            (W: [f_in][H*D])
 *   s(e,h)    = LeakyReLU_slope( z[u,h,:].a_src[h,:] + z[v,h,:].a_dst[h,:] )
 *               (= a_h^T [z_u,h || z_v,h], the ApplyEdge "MLP" of size 1, A14)
 *   alpha(e,h)= exp(s(e,h) - max_e' s(e',h)) / sum_e' exp(s(e',h) - max)
 *   out[v,h,:]= ELU( sum_e alpha(e,h) z[u,h,:] ),   ELU(x) = x>0 ? x : e^x - 1
 * z is computed for all n vertices first (ApplyEdge needs z of every source).
 * alpha_out (nullable): [E][H] in CSR position order, only for rows == NULL.
 * ---------------------------------------------------------------------- */
void oracle_gat(int32_t n, const int64_t *row_ptr, const int32_t *col_src,
                const void *x, int x_dtype, int32_t f_in, const double *W, int32_t heads, int32_t hd,
                const double *a_src, const double *a_dst, double slope,
                const int64_t *rows, int64_t nrows, double *out, double *alpha_out) {
    int32_t f_out = heads * hd;
    double *z = (double *)malloc(sizeof(double) * (size_t)n * (size_t)f_out);
#pragma omp parallel for schedule(static)
    for (int64_t u = 0; u < n; ++u) {
        double *zu = z + u * f_out;
        for (int32_t j = 0; j < f_out; ++j) zu[j] = 0.0;
        for (int32_t k = 0; k < f_in; ++k) {
            double xk = load_x(x, x_dtype, u, f_in, k);
            for (int32_t j = 0; j < f_out; ++j) zu[j] += xk * W[(int64_t)k * f_out + j];
        }
    }
    if (!rows) nrows = n;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < nrows; ++i) {
        int64_t v = row_at(rows, i);
        double *o = out + i * (int64_t)f_out;
        for (int32_t h = 0; h < heads; ++h) {
            double er = 0.0;
            for (int32_t k = 0; k < hd; ++k) er += z[v * f_out + h * hd + k] * a_dst[h * hd + k];
            double smax = -INFINITY;
            for (int64_t p = row_ptr[v]; p < row_ptr[v + 1]; ++p) {
                int64_t u = col_src[p];
                double el = 0.0;
                for (int32_t k = 0; k < hd; ++k) el += z[u * f_out + h * hd + k] * a_src[h * hd + k];
                double s = el + er;
                s = s > 0.0 ? s : slope * s;
                if (s > smax) smax = s;
            }
            double denom = 0.0;
            for (int64_t p = row_ptr[v]; p < row_ptr[v + 1]; ++p) {
                int64_t u = col_src[p];
                double el = 0.0;
                for (int32_t k = 0; k < hd; ++k) el += z[u * f_out + h * hd + k] * a_src[h * hd + k];
                double s = el + er;
                s = s > 0.0 ? s : slope * s;
                denom += exp(s - smax);
            }
            for (int32_t k = 0; k < hd; ++k) o[h * hd + k] = 0.0;
            for (int64_t p = row_ptr[v]; p < row_ptr[v + 1]; ++p) {
                int64_t u = col_src[p];
                double el = 0.0;
                for (int32_t k = 0; k < hd; ++k) el += z[u * f_out + h * hd + k] * a_src[h * hd + k];
                double s = el + er;
                s = s > 0.0 ? s : slope * s;
                double alpha = exp(s - smax) / denom;
                if (alpha_out && !rows) alpha_out[p * heads + h] = alpha;
                for (int32_t k = 0; k < hd; ++k) o[h * hd + k] += alpha * z[u * f_out + h * hd + k];
            }
            for (int32_t k = 0; k < hd; ++k) {
                double a = o[h * hd + k];
                o[h * hd + k] = a > 0.0 ? a : expm1(a);
            }
        }
    }
    free(z);
}

/* sigma(x) = 1 / (1 + e^-x) */
static double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }

/* ------------------------------------------------------------------------
 * Gated graph layer (config C4).  PAPER.md lines 142-147 (GGNN walkthrough:
 * Gather sums the in-edge messages, ApplyVertex is a GRU) and Table 1 line
 * 178; BASELINE.json config C4 fixes a per-edge-type message weight W_t and
 * the GRU shapes (readings A6, A15, A16):
 *   msg_e  = H[u] . W_{type(e)}   for e = (u -> v)     (ApplyEdge, per edge; W_t: [f][f])
 *   m[v]   = sum_{e=(u->v)} msg_e                      (Gather, sum)
 *   r  = sigma(m W_ir + b_ir + h W_hr + b_hr)
 *   zg = sigma(m W_iz + b_iz + h W_hz + b_hz)
 *   ng = tanh (m W_in + b_in + r * (h W_hn + b_hn))
 *   h' = (1 - zg) * ng + zg * h                        (h = H[v])
 * W_type [T][f][f], W_ih [3][f][hid], W_hh [3][hid][hid], b_* [3][hid],
 * gate order r, z, n (PyTorch GRUCell form, reading A15).  f == hid.
 * ---------------------------------------------------------------------- */
void oracle_gated(int32_t n, const int64_t *row_ptr, const int32_t *col_src, const int32_t *etype_csr,
                  int32_t num_etypes, const void *x, int x_dtype, int32_t f,
                  const double *W_type, const double *W_ih, const double *W_hh,
                  const double *b_ih, const double *b_hh,
                  const int64_t *rows, int64_t nrows, double *out) {
    int32_t hid = f;
    if (!rows) nrows = n;
#pragma omp parallel
    {
        double *xu = (double *)malloc(sizeof(double) * (size_t)f);
        double *m = (double *)malloc(sizeof(double) * (size_t)f);
        double *h = (double *)malloc(sizeof(double) * (size_t)f);
        double *gi = (double *)malloc(sizeof(double) * 3 * (size_t)hid);
        double *gh = (double *)malloc(sizeof(double) * 3 * (size_t)hid);
#pragma omp for schedule(dynamic, 64)
        for (int64_t i = 0; i < nrows; ++i) {
            int64_t v = row_at(rows, i);
            for (int32_t j = 0; j < f; ++j) m[j] = 0.0;
            for (int64_t p = row_ptr[v]; p < row_ptr[v + 1]; ++p) {   /* in-edges in CSR order */
                int32_t t = etype_csr ? etype_csr[p] : 0;
                for (int32_t k = 0; k < f; ++k) xu[k] = load_x(x, x_dtype, col_src[p], f, k);   /* Scatter */
                for (int32_t j = 0; j < f; ++j) {                                              /* ApplyEdge */
                    double msg = 0.0;
                    for (int32_t k = 0; k < f; ++k) msg += xu[k] * W_type[((int64_t)t * f + k) * f + j];
                    m[j] += msg;                                                               /* Gather */
                }
            }
            for (int32_t k = 0; k < f; ++k) h[k] = load_x(x, x_dtype, v, f, k);
            for (int32_t g = 0; g < 3; ++g)
                for (int32_t j = 0; j < hid; ++j) {
                    gi[g * hid + j] = b_ih[g * hid + j];
                    gh[g * hid + j] = b_hh[g * hid + j];
                }
            for (int32_t g = 0; g < 3; ++g)
                for (int32_t k = 0; k < f; ++k)
                    for (int32_t j = 0; j < hid; ++j) {
                        gi[g * hid + j] += m[k] * W_ih[((int64_t)g * f + k) * hid + j];
                        gh[g * hid + j] += h[k] * W_hh[((int64_t)g * hid + k) * hid + j];
                    }
            double *o = out + i * (int64_t)hid;
            for (int32_t j = 0; j < hid; ++j) {
                double r = sigmoid(gi[j] + gh[j]);
                double zg = sigmoid(gi[hid + j] + gh[hid + j]);
                double ng = tanh(gi[2 * hid + j] + r * gh[2 * hid + j]);
                o[j] = (1.0 - zg) * ng + zg * h[j];
            }
        }
        free(xu); free(m); free(h); free(gi); free(gh);
    }
}

/* ------------------------------------------------------------------------
 * R-GCN layer.  Table 1: Scatter edge+src
 * (the edge's relation type and the source embedding), ApplyEdge MLP (a
 * per-type transform: "RGCN assigns another edge type attribute to
 * different edges ... first needs to select edges with the same type and then
 * batches them to GEMM", lines 327-328), Gather sum(in_edges) + vertex,
 * ApplyVertex sum.  Reading A24: the relational GCN of the
 * cited R-GCN paper with per-(destination, type) mean normalisation
 * c_{v,t} = |N_t(v)| and a self connection W_self:
 *   out[v] = act( sum_t (1/c_{v,t}) sum_{e=(u->v), type(e)=t} H[u] . W_t
 *                 + H[v] . W_self + b )
 * (a type with no in-edges of v contributes 0).  W_type [T][f][f_out],
 * W_self [f][f_out], act 0 none / 1 ReLU.
 * ---------------------------------------------------------------------- */
void oracle_rgcn(int32_t n, const int64_t *row_ptr, const int32_t *col_src, const int32_t *etype_csr,
                 int32_t num_etypes, const void *x, int x_dtype, int32_t f, const double *W_type,
                 const double *W_self, int32_t f_out, const double *b, int act,
                 const int64_t *rows, int64_t nrows, double *out) {
    if (!rows) nrows = n;
#pragma omp parallel
    {
        double *xu = (double *)malloc(sizeof(double) * (size_t)f);
        int64_t *cnt = (int64_t *)malloc(sizeof(int64_t) * (size_t)num_etypes);
#pragma omp for schedule(dynamic, 64)
        for (int64_t i = 0; i < nrows; ++i) {
            int64_t v = row_at(rows, i);
            for (int32_t t = 0; t < num_etypes; ++t) cnt[t] = 0;
            for (int64_t p = row_ptr[v]; p < row_ptr[v + 1]; ++p) cnt[etype_csr ? etype_csr[p] : 0] += 1;  /* c_{v,t} */
            double *o = out + i * (int64_t)f_out;
            for (int32_t j = 0; j < f_out; ++j) o[j] = b ? b[j] : 0.0;
            for (int64_t p = row_ptr[v]; p < row_ptr[v + 1]; ++p) {   /* per in-edge, CSR order */
                int32_t t = etype_csr ? etype_csr[p] : 0;
                for (int32_t k = 0; k < f; ++k) xu[k] = load_x(x, x_dtype, col_src[p], f, k);   /* Scatter */
                for (int32_t j = 0; j < f_out; ++j) {                                          /* ApplyEdge */
                    double msg = 0.0;
                    for (int32_t k = 0; k < f; ++k) msg += xu[k] * W_type[((int64_t)t * f + k) * f_out + j];
                    o[j] += msg / (double)cnt[t];                                              /* Gather, mean */
                }
            }
            for (int32_t k = 0; k < f; ++k) {                                 /* the vertex's own term */
                double hk = load_x(x, x_dtype, v, f, k);
                for (int32_t j = 0; j < f_out; ++j) o[j] += hk * W_self[(int64_t)k * f_out + j];
            }
            if (act == 1)
                for (int32_t j = 0; j < f_out; ++j) o[j] = o[j] > 0.0 ? o[j] : 0.0;
        }
        free(xu);
        free(cnt);
    }
}

/* ------------------------------------------------------------------------
 * GraphSAGE-LSTM layer.  Table 1: Gather
 * LSTM(in_edges) + vertex, ApplyVertex MLP; lines 357-360: the LSTM "treats
 * the inedges of a vertex as a sequence and outputs a new vector".
 * Reading A25: the sequence is v's in-edges in CSR order
 * (ascending COO index, reading A7), the cell is the
 * PyTorch LSTMCell (gates i, f, g, o; zero initial h, c), the gathered
 * vector is the final h (0 for a vertex without in-edges), and ApplyVertex
 * is the GraphSAGE concat-GEMM of reading A11:
 *   for the in-edges u_1..u_d of v:  z = x[u_s] . W_ih + b_ih + h . W_hh + b_hh
 *     i = s(z_i), f = s(z_f), g = tanh(z_g), o = s(z_o)
 *     c = f * c + i * g,  h = o * tanh(c)
 *   out[v] = act([x[v] || h] . W + b)
 * W_ih [4][f][f], W_hh [4][f][f], b_ih/b_hh [4][f] (gate order i, f, g, o),
 * W [2f][f_out]; act 0 none / 1 ReLU.
 * ---------------------------------------------------------------------- */
void oracle_sage_lstm(int32_t n, const int64_t *row_ptr, const int32_t *col_src, const void *x, int x_dtype,
                      int32_t f, const double *W_ih, const double *W_hh, const double *b_ih, const double *b_hh,
                      const double *W, int32_t f_out, const double *b, int act,
                      const int64_t *rows, int64_t nrows, double *out) {
    if (!rows) nrows = n;
#pragma omp parallel
    {
        double *h = (double *)malloc(sizeof(double) * (size_t)f);
        double *c = (double *)malloc(sizeof(double) * (size_t)f);
        double *z = (double *)malloc(sizeof(double) * 4 * (size_t)f);
        double *hn = (double *)malloc(sizeof(double) * (size_t)f);
#pragma omp for schedule(dynamic, 16)
        for (int64_t i = 0; i < nrows; ++i) {
            int64_t v = row_at(rows, i);
            for (int32_t k = 0; k < f; ++k) { h[k] = 0.0; c[k] = 0.0; }
            for (int64_t p = row_ptr[v]; p < row_ptr[v + 1]; ++p) {          /* the in-edge sequence */
                int32_t u = col_src[p];
                for (int32_t g = 0; g < 4; ++g)
                    for (int32_t j = 0; j < f; ++j) z[g * f + j] = b_ih[g * f + j] + b_hh[g * f + j];
                for (int32_t g = 0; g < 4; ++g)
                    for (int32_t k = 0; k < f; ++k) {
                        double xk = load_x(x, x_dtype, u, f, k), hk = h[k];
                        for (int32_t j = 0; j < f; ++j)
                            z[g * f + j] += xk * W_ih[((int64_t)g * f + k) * f + j] + hk * W_hh[((int64_t)g * f + k) * f + j];
                    }
                for (int32_t j = 0; j < f; ++j) {
                    double ig = sigmoid(z[j]), fg = sigmoid(z[f + j]), gg = tanh(z[2 * f + j]),
                           og = sigmoid(z[3 * f + j]);
                    c[j] = fg * c[j] + ig * gg;
                    hn[j] = og * tanh(c[j]);
                }
                for (int32_t j = 0; j < f; ++j) h[j] = hn[j];
            }
            double *o = out + i * (int64_t)f_out;                              /* ApplyVertex: [x || h] . W */
            for (int32_t j = 0; j < f_out; ++j) o[j] = b ? b[j] : 0.0;
            for (int32_t k = 0; k < f; ++k) {
                double xk = load_x(x, x_dtype, v, f, k);
                for (int32_t j = 0; j < f_out; ++j)
                    o[j] += xk * W[(int64_t)k * f_out + j] + h[k] * W[(int64_t)(f + k) * f_out + j];
            }
            if (act == 1)
                for (int32_t j = 0; j < f_out; ++j) o[j] = o[j] > 0.0 ? o[j] : 0.0;
        }
        free(h); free(c); free(z); free(hn);
    }
}

/* ------------------------------------------------------------------------
 * Paper-form GGNN layer.
 * (the GGNN walkthrough) and Table 1, taken literally (reading A26):
 *   Scatter:     x_e = [H[u] || H[v]]                 (e = u -> v, 2f wide)
 *   ApplyEdge:   y_e = act(x_e . W_e + b_e)           (a one-layer MLP, W_e [2f][f])
 *   Gather:      m[v] = sum_{e into v} y_e            ("sums the edge^{l+1} of all
 *                its inedges"; agg = 1 takes the elementwise max instead,
 *                the max of line 218); 0 for a vertex without in-edges
 *   ApplyVertex: h' = GRUCell(m[v], H[v])             (gate order r, z, n, reading A15)
 * act 0 none / 1 ReLU.  W_ih [3][f][f], W_hh [3][f][f], b_* [3][f].
 * ---------------------------------------------------------------------- */
void oracle_ggnn(int32_t n, const int64_t *row_ptr, const int32_t *col_src, const void *x, int x_dtype,
                 int32_t f, const double *W_e, const double *b_e, int act, int agg,
                 const double *W_ih, const double *W_hh, const double *b_ih, const double *b_hh,
                 const int64_t *rows, int64_t nrows, double *out) {
    if (!rows) nrows = n;
#pragma omp parallel
    {
        double *xe = (double *)malloc(sizeof(double) * 2 * (size_t)f);
        double *y = (double *)malloc(sizeof(double) * (size_t)f);
        double *m = (double *)malloc(sizeof(double) * (size_t)f);
        double *h = (double *)malloc(sizeof(double) * (size_t)f);
        double *gi = (double *)malloc(sizeof(double) * 3 * (size_t)f);
        double *gh = (double *)malloc(sizeof(double) * 3 * (size_t)f);
#pragma omp for schedule(dynamic, 16)
        for (int64_t i = 0; i < nrows; ++i) {
            int64_t v = row_at(rows, i);
            int64_t p0 = row_ptr[v], p1 = row_ptr[v + 1];
            for (int32_t j = 0; j < f; ++j) m[j] = 0.0;
            for (int64_t p = p0; p < p1; ++p) {
                int32_t u = col_src[p];
                for (int32_t k = 0; k < f; ++k) {                                   /* Scatter */
                    xe[k] = load_x(x, x_dtype, u, f, k);
                    xe[f + k] = load_x(x, x_dtype, v, f, k);
                }
                for (int32_t j = 0; j < f; ++j) y[j] = b_e ? b_e[j] : 0.0;          /* ApplyEdge */
                for (int32_t k = 0; k < 2 * f; ++k)
                    for (int32_t j = 0; j < f; ++j) y[j] += xe[k] * W_e[(int64_t)k * f + j];
                if (act == 1)
                    for (int32_t j = 0; j < f; ++j) y[j] = y[j] > 0.0 ? y[j] : 0.0;
                for (int32_t j = 0; j < f; ++j)                                     /* Gather */
                    m[j] = (agg == 1 && p > p0) ? (y[j] > m[j] ? y[j] : m[j]) : (agg == 1 ? y[j] : m[j] + y[j]);
            }
            for (int32_t k = 0; k < f; ++k) h[k] = load_x(x, x_dtype, v, f, k);    /* ApplyVertex */
            for (int32_t g = 0; g < 3; ++g)
                for (int32_t j = 0; j < f; ++j) {
                    gi[g * f + j] = b_ih[g * f + j];
                    gh[g * f + j] = b_hh[g * f + j];
                }
            for (int32_t g = 0; g < 3; ++g)
                for (int32_t k = 0; k < f; ++k)
                    for (int32_t j = 0; j < f; ++j) {
                        gi[g * f + j] += m[k] * W_ih[((int64_t)g * f + k) * f + j];
                        gh[g * f + j] += h[k] * W_hh[((int64_t)g * f + k) * f + j];
                    }
            double *o = out + i * (int64_t)f;
            for (int32_t j = 0; j < f; ++j) {
                double r = sigmoid(gi[j] + gh[j]);
                double zg = sigmoid(gi[f + j] + gh[f + j]);
                double ng = tanh(gi[2 * f + j] + r * gh[2 * f + j]);
                o[j] = (1.0 - zg) * ng + zg * h[j];
            }
        }
        free(xe); free(y); free(m); free(h); free(gi); free(gh);
    }
}
