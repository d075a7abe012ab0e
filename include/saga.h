/*
 * saga.h -- C ABI of the B200-native SAGA-NN layer library (libsaga.so).
 *
 * One GNN layer at inference in the SAGA-NN decomposition of Zhang et al.,
 * "Architectural Implications of Graph Neural Networks" (IEEE CAL 2020,
 * arXiv 2009.00804): Scatter -> ApplyEdge -> Gather -> ApplyVertex
 * (Section 2; Table 1 `tbl:benchmark`, lines
 * 176-180).  The operations and their exact definitions are the ones the
 * fp64 oracle (oracle/oracle.c) writes out; DESIGN.md lists every reading of
 * the paper they rest on (A1..A26).
 *
 * Conventions shared by every entry point
 *  - All array arguments are DEVICE pointers (CUDA global memory on the
 *    current device) unless marked "host".  Matrices are row-major and
 *    contiguous; every feature/weight/output/workspace pointer must be
 *    16-byte aligned (SAGA_EINVAL otherwise).
 *  - Work is enqueued on `cuda_stream` (a cudaStream_t; NULL = legacy default
 *    stream) and is asynchronous: buffers must stay alive until the stream
 *    reaches that point.  The caller owns every buffer it passes; the library
 *    never frees them.  The only host<->device synchronisation in the library
 *    is the range check inside saga_graph_build.
 *  - Every function returns a saga_status; no C++ exception crosses the ABI.
 *    On failure, saga_last_error() returns a thread-local message valid until
 *    the next call on the same thread.  Nothing is enqueued when a call fails
 *    its argument checks.
 */
#ifndef SAGA_H_
#define SAGA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SAGA_ABI_VERSION 4  /* 2: SAGA_GGNN, saga_layer_opts.aggregator; 3: .fused; 4: .workspace_zeroed */

#if defined(__GNUC__)
#define SAGA_API __attribute__((visibility("default")))
#else
#define SAGA_API
#endif

typedef enum {
    SAGA_OK = 0,
    SAGA_EINVAL = 1,       /* bad pointer / alignment / size / workspace too small   */
    SAGA_ERANGE = 2,       /* a COO entry is out of range (see saga_graph_build)      */
    SAGA_ESHAPE = 3,       /* tensor shape does not match graph or options            */
    SAGA_EDTYPE = 4,       /* dtype combination not allowed for the model             */
    SAGA_ENOMEM = 5,       /* device allocation failed                                */
    SAGA_ECUDA = 6,        /* CUDA runtime / launch error (message has details)       */
    SAGA_EUNSUPPORTED = 7, /* valid request this build does not implement             */
    SAGA_EINTERNAL = 8
} saga_status;

typedef enum { SAGA_F32 = 0, SAGA_BF16 = 1 } saga_dtype;

/* Table 1 rows this library implements. */
typedef enum {
    SAGA_GCN = 0,   /* Gather sum(in_edges) with D^-1/2 (A+I) D^-1/2 weights, ApplyVertex MLP  */
    SAGA_SAGE = 1,  /* Gather mean(in_edges) + vertex, ApplyVertex MLP on [x || mean]          */
    SAGA_GAT = 2,   /* ApplyEdge attention score, Gather attention(in_edges), ELU              */
    SAGA_GATED = 3, /* per-edge-type message W_t, Gather sum(in_edges), ApplyVertex GRU        */
    SAGA_RGCN = 4,  /* per-type mean messages W_t + self term, ApplyVertex sum */
    SAGA_SAGE_LSTM = 5, /* Gather LSTM(in_edges) + vertex, ApplyVertex MLP    */
    SAGA_GGNN = 6   /* Scatter src&dst, ApplyEdge MLP, Gather sum|max, ApplyVertex GRU (NEXT-4) */
} saga_model;

/* Gather reduction of SAGA_GGNN (line 218: "sum/mean/max"). */
typedef enum { SAGA_AGG_SUM = 0, SAGA_AGG_MAX = 1 } saga_aggregator;

typedef enum { SAGA_ACT_NONE = 0, SAGA_ACT_RELU = 1, SAGA_ACT_ELU = 2 } saga_act;

/* Opaque, immutable after saga_graph_build; safe to share between streams. */
typedef struct saga_graph saga_graph;

/* A dense row-major device matrix [rows][cols]. */
typedef struct {
    void *data;
    int32_t dtype;  /* saga_dtype */
    int64_t rows, cols;
} saga_tensor;

typedef struct {
    int32_t in_dim, out_dim;  /* feature widths (GAT: out_dim = heads * head_dim)         */
    int32_t heads, head_dim;  /* GAT only (else ignored)                                  */
    int32_t act;              /* saga_act applied by ApplyVertex: GCN/SAGE (RELU or NONE); */
                              /* GAT must be ELU; GATED ignores it (GRU)                   */
    float leaky_slope;        /* GAT LeakyReLU negative slope in [0, 1] (0.2 in config C3) */
    int32_t aggregator;       /* saga_aggregator, GGNN only (else ignored)                 */
    int32_t fused;            /* SAGE, BF16 GCN: 1 = Gather and the ApplyVertex GEMM as ONE */
                              /* kernel.       */
                              /* SAGE: in_dim 128, out_dim 64 or 128.  GCN: in_dim 256,     */
                              /* out_dim 64, 128 or 256, E < 2^31 - 64, aggregate first     */
                              /* (SAGA order): deg(u)^-1/2 and the aggregated row are       */
                              /* rounded to BF16 (the default rounds Y = XW instead).  0 =  */
                              /* the multi-kernel path (default).  Other kinds ignore it.   */
    int32_t workspace_zeroed; /* 1 = the caller guarantees the workspace's ticket-counter   */
                              /* region is zero: the memory was zero-filled before its     */
                              /* first saga_layer call, and since then only completed      */
                              /* saga_layer calls (which leave it zero) have used it; the  */
                              /* call then skips zeroing it (one memset node per call).    */
                              /* 0 = the library zeroes it (contents ignored on entry)     */
} saga_layer_opts;

/* Weights (device, row-major, [in][out] orientation = x . W, reading A8).
 * Unused members may be NULL.                                               */
typedef struct {
    const void *W;         /* GCN [in][out]; SAGE [2*in][out] (self rows first); GAT [in][heads*hd];
                              RGCN: W_self [in][out] fp32; GGNN: edge MLP W_e [2*in][in] fp32
                              (source rows first); dtype = features dtype                         */
    const float *bias;     /* [out] fp32, nullable (= 0); GGNN: the edge MLP bias b_e [in]          */
    const float *attn_src; /* GAT [heads][hd] fp32 (applied to the source z)                      */
    const float *attn_dst; /* GAT [heads][hd] fp32 (applied to the destination z)                 */
    const float *W_type;   /* GATED, RGCN [T][f][f] fp32                                           */
    const void *W_ih;      /* GATED, GGNN [3][f][f] fp32, gate order r, z, n (PyTorch GRUCell form);
                              SAGE_LSTM [4][f][f] bf16, gate order i, f, g, o (LSTMCell form)    */
    const void *W_hh;      /* GATED, GGNN [3][f][f] fp32; SAGE_LSTM [4][f][f] bf16               */
    const float *b_ih;     /* GATED, GGNN [3][f], SAGE_LSTM [4][f] fp32                            */
    const float *b_hh;     /* GATED, GGNN [3][f], SAGE_LSTM [4][f] fp32                            */
} saga_weights;

/* Returns SAGA_ABI_VERSION. */
SAGA_API int saga_abi_version(void);

/*
 * saga_graph_build -- COO edge list -> destination-sorted CSR (S0).
 *
 * Definition: PAPER.md line 130 (a layer's input is the graph "in the form
 * of adjacency matrix") and lines 351-354 (adjacency row = destination
 * vertex, nonzero = one of its in-edges).  Reading A7: row v holds v's
 * in-edges in ascending COO index (a stable sort by dst); multiplicity and
 * self-loops are kept exactly as given (no implicit self-loops, A2).
 *
 *  num_vertices  N >= 0;  num_edges E >= 0 (E < 2^31)
 *  src, dst      int32[E] device, COO edge u -> v = (src[i], dst[i])
 *  etype         int32[E] device or NULL (then all types are 0 and T = 1);
 *                must lie in [0, num_etypes)
 *  cuda_stream   stream all device work is ordered on
 *  out           host: receives the new graph handle (NULL on failure)
 *  first_bad_edge host, nullable: on SAGA_ERANGE receives the LOWEST COO
 *                index whose src, dst or etype is out of range; -1 otherwise
 *
 * The handle owns device arrays (row_ptr int64[N+1], col_src/edge_id/etype
 * int32[E], in/out degree int32[N], per-vertex norms, the load-balance
 * schedule), allocated stream-ordered; release it with saga_free.  This call
 * synchronises `cuda_stream` once (to read the range-check result).
 */
SAGA_API saga_status saga_graph_build(int32_t num_vertices, int64_t num_edges, const int32_t *src,
                             const int32_t *dst, const int32_t *etype, int32_t num_etypes,
                             void *cuda_stream, saga_graph **out, int64_t *first_bad_edge);

/* Sizes of a built graph (host outputs, each nullable). */
SAGA_API saga_status saga_graph_info(const saga_graph *g, int32_t *num_vertices, int64_t *num_edges,
                            int32_t *num_etypes);

/*
 * Copy the CSR arrays into caller-provided DEVICE buffers (each nullable):
 * row_ptr int64[N+1], col_src int32[E] (= src[edge_id[p]]), edge_id int32[E]
 * (CSR position -> COO index), etype int32[E] (in CSR order), in_deg int32[N],
 * out_deg int32[N].  Asynchronous on cuda_stream.
 */
SAGA_API saga_status saga_graph_copy_csr(const saga_graph *g, int64_t *row_ptr, int32_t *col_src,
                                int32_t *edge_id, int32_t *etype, int32_t *in_deg,
                                int32_t *out_deg, void *cuda_stream);

/* Workspace bytes saga_layer needs for (kind, g, opts); host output. */
SAGA_API saga_status saga_layer_workspace_bytes(saga_model kind, const saga_graph *g,
                                       const saga_layer_opts *opts, size_t *bytes);

/*
 * saga_layer -- one SAGA-NN layer (Scatter, ApplyEdge, Gather, ApplyVertex).
 *
 * Definitions (in SAGA order; the GPU may reorder by linearity, fold the
 * normalisation and split reductions, which changes only rounding):
 *  GCN   (Table 1; BASELINE.json C1/C5; A1, A2, A12):
 *        out[v] = act( sum_{u->v} deg(u)^-1/2 deg(v)^-1/2 x[u] . W + bias )
 *        features F32 (fused aggregate + SIMT GEMV, in_dim in {16, 32, 64, 128},
 *        1 <= out_dim <= 64) or BF16 (tcgen05 GEMM first, then aggregation;
 *        in_dim in {64,128,192,256}, out_dim in {64,128,256}; opts.fused: one
 *        kernel, aggregation first, in_dim 256).
 *  SAGE  (Table 1; BASELINE.json C2; A11, A12):
 *        out[v] = act( [x[v] || mean_{u->v} x[u]] . W + bias ), W [2*in][out]
 *        BF16, in_dim in {64, 128}, out_dim in {64, 128, 256}.
 *  GAT   (Table 1; BASELINE.json C3; A13, A14):
 *        z = x . W; s(u->v,h) = LeakyReLU(z[u,h].a_src[h] + z[v,h].a_dst[h]);
 *        out[v,h] = ELU( sum softmax_{in-edges of v}(s) z[u,h] )
 *        BF16, in_dim in {64..256 step 64}, heads * head_dim = out_dim = 64,
 *        head_dim = 8.
 *  GATED (lines 142-147, Table 1; BASELINE.json C4; A6, A15, A16):
 *        m[v] = sum_{u->v} x[u] . W_type[t(u->v)]; out[v] = GRUCell(m[v], x[v])
 *        F32, in_dim = out_dim = 128, num_etypes <= 4.
 *        Precision (GATED and GGNN): the message / GRU GEMMs run as split-TF32
 *        (22-bit operands, fp32 tensor-core accumulation) for rows with
 *        in-degree < 256; rows with in-degree >= 256, whose summed message
 *        grows with the in-degree, are recomputed with fp64 products, sums and
 *        nonlinearities from the fp32-stored S / m ("Precision").
 *  SAGE_LSTM (Table 1; A25):
 *        h[v] = final state of LSTMCell(W_ih, W_hh, b_ih, b_hh) run over x[u]
 *        for v's in-edges u -> v in CSR order from a zero state (0 without
 *        in-edges); out[v] = act([x[v] || h[v]] . W + bias), W [2*in][out]
 *        BF16, in_dim = 128, out_dim in {64, 128, 256}, act NONE or RELU.
 *  RGCN  (Table 1; A24):
 *        out[v] = act( sum_t mean_{u->v, type t} x[u] . W_type[t] + x[v] . W + bias )
 *        (a type with no in-edges of v contributes 0); F32, in_dim = out_dim
 *        = 128, num_etypes <= 4, act NONE or RELU.
 *  GGNN  (lines 142-147, Table 1; A26):
 *        y(u->v) = act([x[u] || x[v]] . W_e + b_e)   (act = opts.act, NONE or RELU)
 *        m[v] = sum (or elementwise max, opts.aggregator) of y over v's in-edges,
 *        0 without in-edges; out[v] = GRUCell(m[v], x[v]) (weights as GATED)
 *        F32, in_dim = out_dim = 128; edge types are ignored.
 *  features  [N][in_dim];  out  [N][out_dim] with the features' dtype
 *  workspace device scratch of at least saga_layer_workspace_bytes() bytes;
 *            contents on entry are ignored unless opts->workspace_zeroed = 1
 *            (then its first bytes -- the split-row ticket counters -- must be
 *            zero, which every completed call leaves them); it must not be
 *            shared by calls in flight on other streams.
 * Never allocates, never synchronises.  Deterministic: identical inputs give
 * bit-identical outputs (no floating-point atomics).
 */
SAGA_API saga_status saga_layer(saga_model kind, const saga_graph *g, const saga_tensor *features,
                       const saga_weights *w, saga_tensor *out, const saga_layer_opts *opts,
                       void *workspace, size_t workspace_bytes, void *cuda_stream);

/* Release a graph.  NULL-safe.  The device arrays are freed stream-ordered
 * on the stream the graph was BUILT on (cudaFreeAsync); the caller must make
 * sure that work on any OTHER stream that reads the graph has completed (or
 * is ordered before that stream, e.g. by an event) -- the Python Graph.close()
 * synchronises the device first.  The build stream must still exist. */
SAGA_API void saga_free(saga_graph *g);

/*
 * Optional per-kernel timing (tracing).  When enabled (process-wide), every
 * kernel saga_layer launches is bracketed by a CUDA event pair recorded on
 * the caller's stream; saga_profile_get synchronises those events and
 * returns, per kernel name, the launch count and the summed device time in
 * milliseconds since the last saga_profile_enable call (which resets).
 * Costs two event records per launch; disabled by default.
 */
SAGA_API saga_status saga_profile_enable(int enable);
/* Restrict the brackets to the launches with this label (NULL or "" = all).
 * With a filter, the unbracketed kernels keep their programmatic dependent
 * launches, so the bracketed kernel is timed inside an otherwise unchanged
 * step (its own launch is serialised by the event records). */
SAGA_API saga_status saga_profile_filter(const char *label);
SAGA_API int32_t saga_profile_count(void);
SAGA_API saga_status saga_profile_get(int32_t index, const char **name, int64_t *launches, double *total_ms);
/* Stage timeline (the B200 analogue of the paper's per-stage breakdown,
 * PAPER.md Fig. 5 / lines 289, 309-310): every bracketed launch since the
 * last saga_profile_enable, in launch order, as [start_ms, end_ms) measured
 * by the same event pairs from the first bracket's start event.  `name` is the
 * library's label (owned by the library, valid until unload).  Synchronises
 * the pending events; SAGA_EINVAL for an index outside [0, count). */
SAGA_API int32_t saga_profile_trace_count(void);
SAGA_API saga_status saga_profile_trace_get(int32_t index, const char **name, double *start_ms, double *end_ms);

/* Thread-local message of the last failing call on this thread ("" if none). */
SAGA_API const char *saga_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* SAGA_H_ */
