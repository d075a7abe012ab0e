// internal.cuh -- shared declarations of the CUDA path (not part of the ABI).
#pragma once
#include <cstddef>
#include <cstdint>
#include <utility>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../../include/saga.h"

namespace saga {

constexpr int kNumSMs = 148;
// Rows whose in-degree reaches this run the gated / GGNN ApplyVertex in fp64
// (gru_f64.cu): their summed message outgrows the tensor core's fp32 accumulator.
constexpr int32_t kHeavyInDeg = 256;
// Graphs whose in-degrees are all <= this get the ELL view (graph_build.cu)
// and the row-wise fused fp32 GCN (aggregate.cu)
constexpr int32_t kEllMaxDeg = 64;

// ---- Programmatic dependent launch (PDL) ----------------------------------
// Inside one saga_layer call every kernel after the first is launched with
// programmatic stream serialisation: it may be scheduled while its
// predecessor drains (its launch latency and prologue -- barrier init, TMEM
// allocation, weight staging -- overlap the predecessor's tail).  Contract
// for every kernel launched through saga::launch: (1) it calls griddep_wait()
// before touching memory an earlier kernel of the call writes (and before any
// global write), so the grid cannot complete before its predecessor (the
// chain stays transitive); (2) it may call griddep_launch() to let its own
// dependent be scheduled early.  Both are no-ops for a normal launch.  The
// first kernel of a call is a normal launch, so it is ordered after all
// earlier work of the stream (the caller's writes to x and the weights).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Host side: g_pdl_call is set by saga_layer for the duration of a call
// (never while per-kernel profiling records events between the kernels);
// g_pdl_armed becomes true after the call's first launch.
extern thread_local bool g_pdl_call, g_pdl_armed;

// kPdl = false: always a normal launch (kernels measured slower as PDL
// secondaries: the split-TF32 GEMMs and their weight-split kernels).
template <bool kPdl = true, typename... KArgs, typename... Args>
cudaError_t launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args &&...args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = kPdl && g_pdl_armed ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
    if (g_pdl_call) g_pdl_armed = true;
    return e;
}

// Device arrays owned by a built graph (saga_graph_build, S0).
struct GraphDev {
    int32_t n = 0;
    int64_t e = 0;
    int32_t num_etypes = 1;
    int64_t *row_ptr = nullptr;   // [n+1]
    int32_t *col_src = nullptr;   // [e]
    int32_t *edge_id = nullptr;   // [e]
    int32_t *etype = nullptr;     // [e] (nullptr when no types were given)
    int32_t *in_deg = nullptr;    // [n]
    int32_t *out_deg = nullptr;   // [n]
    float *dinv = nullptr;        // [n]  in_deg^-1/2 (0 if 0)  -- S1, GCN
    float *inv_deg = nullptr;     // [n]  1/in_deg (0 if 0)     -- S1, SAGE
    int32_t *deg_order = nullptr; // [n]  vertices by in-degree, descending, ties by id (LSTM work queue)
    int32_t max_in_deg = 0;       // host copy (read back with the range check)
    int32_t n_heavy = 0;          // host: #vertices with in-degree >= kHeavyInDeg (= the head of deg_order)
    int32_t *heavy_slot = nullptr; // [n]  v's position in deg_order if v is heavy, else -1
    // Merge-path load-balance schedule (S6): items = E edges + N row ends,
    // task k covers items [k*T, min((k+1)T, E+N)); its start coordinate is
    // (task_v[k], task_p[k]).  Arrays have ntasks+1 entries.
    // ~1 task per resident warp (32 per SM): the sum/mean/typed gathers.
    int64_t task_items = 0;       // T
    int64_t ntasks = 0;
    int32_t *task_v = nullptr;
    int64_t *task_p = nullptr;
    // A 4x finer schedule of the same CSR for the GAT edge softmax, whose
    // per-item cost varies more (its tail balances better over 4 tasks/warp).
    int64_t ftask_items = 0, fntasks = 0;
    int32_t *ftask_v = nullptr;
    int64_t *ftask_p = nullptr;
    // Typed view (built when edge types are given): an internal CSR whose
    // rows are (destination, type) pairs r = v * num_etypes + t, edges in
    // (dst, type, COO index) order; the typed gathers (gated, R-GCN) are plain
    // segment sums over it.  Same merge-path schedule layout as above.
    int64_t *trow_ptr = nullptr;  // [n * T + 1]
    int32_t *tcol_src = nullptr;  // [e]
    float *tinv_deg = nullptr;    // [n * T]  1 / |row| (0 if empty)
    int64_t ttask_items = 0, tntasks = 0;
    int32_t *ttask_v = nullptr;
    int64_t *ttask_p = nullptr;
    // Aggregation view (built when some rows' in-edges are nothing but one
    // self-loop, or none): those rows' GAT output (ELU(z[v]), or 0) is written
    // by the GEMM epilogue, their GCN output act(dinv[v] Y[v] + b) by a
    // streaming pass over erow, and the gathers run over a compacted CSR of
    // the other rows only (row i = vertex arow[i]).
    int32_t an = 0;               // host: aggregation rows
    int64_t ae = 0;               // host: their in-edges
    int32_t *arow = nullptr;      // [an]  vertex of compact row i
    int64_t *arow_ptr = nullptr;  // [an+1]
    int32_t *acol_src = nullptr;  // [ae]
    float *adinv = nullptr;       // [an]  dinv[arow[i]]
    int64_t aftask_items = 0, afntasks = 0;  // its merge-path schedule (the 4x finer one, GAT)
    int32_t *aftask_v = nullptr;
    int64_t *aftask_p = nullptr;
    int64_t atask_items = 0, antasks = 0;    // its one-task-per-warp schedule (GCN)
    int32_t *atask_v = nullptr;
    int64_t *atask_p = nullptr;
    int32_t ne = 0;               // host: the other rows (self-loop only, or no in-edge): n - an
    int32_t *erow = nullptr;      // [ne]  their vertices, ascending
    // ELL view (built when every in-degree is <= kEllMaxDeg and the padded
    // array holds at most max(4 E, 1M) cells): row v's sources
    // at ell[v * ell_w ..], CSR order, padded with -1 -- the row-wise kernels
    // find a row's edges without the row_ptr round trip
    int32_t ell_w = 0;            // host: width (max in-degree rounded up to 4; 0: no view)
    int32_t *ell = nullptr;       // [n][ell_w]
    cudaStream_t stream = nullptr;  // stream the graph was built on (for saga_free)
};

// Graph build (graph_build.cu). Returns cudaError / ERANGE via first_bad.
saga_status build_graph(int32_t n, int64_t e, const int32_t *src, const int32_t *dst, const int32_t *etype,
                        int32_t num_etypes, cudaStream_t st, GraphDev *g, int64_t *first_bad, const char **why);
void free_graph(GraphDev *g);

// ---------------------------------------------------------- aggregation ----
// Merge-path segment-reduce family (aggregate.cu).  Partials/counters live in
// the caller's workspace; counters must be zero on entry (host memsets).
struct AggWorkspace {
    int32_t *counters = nullptr;  // [ntasks]
    float *partials = nullptr;    // [2*ntasks][partial_floats]
};
size_t agg_partial_floats(saga_model kind, int32_t width, int32_t heads);

// C5 / bf16 GCN: out[v] = act(dinv[v] * sum Y[u] + bias), Y already scaled by dinv[u].
cudaError_t launch_agg_gcn_bf16(const GraphDev &g, const __nv_bfloat16 *Y, int32_t f, const float *bias, int act,
                                __nv_bfloat16 *out, AggWorkspace ws, cudaStream_t st);
// C1 / fp32 GCN fused: out[v] = act((dinv[v] * sum dinv[u] x[u]) . W + bias).
// True when launch_gcn_f32_fused runs one warp per row (no split-row tickets,
// so saga_layer skips zeroing the ticket counters).
bool gcn_f32_rowwise(const GraphDev &g);
cudaError_t launch_gcn_f32_fused(const GraphDev &g, const float *X, int32_t f_in, const float *W, int32_t f_out,
                                 const float *bias, int act, float *out, AggWorkspace ws, cudaStream_t st);
// SAGE: M[v] = inv_deg[v] * sum x[u]  (bf16 out)
cudaError_t launch_agg_mean_bf16(const GraphDev &g, const __nv_bfloat16 *X, int32_t f, __nv_bfloat16 *M,
                                 AggWorkspace ws, cudaStream_t st);
// GAT fused edge kernel: online softmax + aggregate + ELU.
// GAT softmax shift (reading A29): the GEMM's per-CTA maxima of el and their
// maximum per head, M_h (k_gat_maxel).
struct GatSoftmaxWs {
    float *parts = nullptr;  // [nparts][8], written by the GAT GEMM (GemmArgs::elmax)
    int nparts = 0;
    float *Mh = nullptr;     // [8]
};
cudaError_t launch_gat_edge(const GraphDev &g, const __nv_bfloat16 *z, const float *el, const float *er,
                            const GatSoftmaxWs &sw, float slope, __nv_bfloat16 *out, AggWorkspace ws,
                            cudaStream_t st);
// GATED typed sums: S[v][t][:] = sum_{type t} H[u]  (fp32)
// GATED / RGCN typed sums over the typed view (mean = per-type means, R-GCN):
// S[v][t][:] for t < T (layout [n][T][f], fp32 out, fp64 accumulation); without
// edge types T = 1 and the plain CSR is used.
// Sx (nullable): the heavy rows' sums also in fp64, [n_heavy][T][f] (gated layer).
cudaError_t launch_agg_typed_f32(const GraphDev &g, const float *H, int32_t f, float *S, bool mean, double *Sx,
                                 AggWorkspace ws, cudaStream_t st);

// ----------------------------------------------------------------- GEMM ----
enum GemmEpi { EPI_ROWSCALE = 0, EPI_BIAS_ACT = 1, EPI_GAT = 2 };
struct GemmArgs {
    int64_t M = 0;
    int32_t K0 = 0, K1 = 0;          // K split over two A sources (K1 = 0: one source)
    int32_t N = 0;
    const __nv_bfloat16 *A0 = nullptr, *A1 = nullptr;  // [M][K0], [M][K1]
    const __nv_bfloat16 *W = nullptr;                  // [K0+K1][N] row-major
    __nv_bfloat16 *out = nullptr;                      // [M][N]
    GemmEpi epi = EPI_ROWSCALE;
    const float *row_scale = nullptr;                  // EPI_ROWSCALE
    // EPI_GAT, optional with the aggregation view: for every row out2[v] =
    // ELU(z[v]) if row_scale[v] > 0 (one in-edge, the self-loop: a single
    // softmax term), else 0 (bf16 z, [M][64]); the view's rows overwrite theirs
    __nv_bfloat16 *out2 = nullptr;
    const float *bias = nullptr;                       // EPI_BIAS_ACT
    int act = 0;
    const float *a_src = nullptr, *a_dst = nullptr;    // EPI_GAT [heads][8]
    float *el = nullptr, *er = nullptr;                // EPI_GAT [M][heads]
    float *elmax = nullptr;  // EPI_GAT: per-CTA maxima of el per head [gemm_bf16_tc_grid(M)][heads]
};
cudaError_t launch_gemm_bf16_tc(const GemmArgs &a, cudaStream_t st, const char **why);
int gemm_bf16_tc_grid(int64_t M);  // CTAs of launch_gemm_bf16_tc for M rows

// Heavy rows deg_order[0 .. n_heavy) of the gated / GGNN layers (gru_f64.cu):
// fp64 ApplyVertex -- the message GEMM from Sx [n_heavy][T][f] (gated) or m
// from mx [n_heavy][f] (GGNN), then the GRU -- and, for GGNN, the heavy rows'
// B = H W_b + b_e in fp64 for the edge-MLP gather.  Workspace: HeavyWs.
struct HeavyWs {
    double *Sx = nullptr, *Bx = nullptr, *mx = nullptr, *W64 = nullptr;
    int T = 0;
};
size_t heavy_workspace_bytes(const GraphDev &g, saga_model kind, int32_t f);
HeavyWs heavy_ws(const GraphDev &g, saga_model kind, void *base);
// Element i of the heavy kernels' fp64 weights [W_type (nt f f) | W_ih (3 f f) |
// W_hh | W_b (f f, if given)], every [K][f] matrix in the fp64 MMA's B-fragment
// order [k/4][n/8][n%8][k%4] (f = 128).  Written by the call's split-weights
// kernel (gemm_tf32split.cu) in the same pass as the tf32 hi/lo split; the
// count is heavy_weights_f64_count.
__device__ __forceinline__ void heavy_weights_f64_item(int64_t i, int32_t nt, const float *__restrict__ W_type,
                                                       const float *__restrict__ W_ih, const float *__restrict__ W_hh,
                                                       const float *__restrict__ W_b, double *__restrict__ out) {
    constexpr int f = 128;
    const int64_t a = (int64_t)nt * f * f, g = (int64_t)3 * f * f;
    const float x = i < a ? W_type[i] : i < a + g ? W_ih[i - a] : i < a + 2 * g ? W_hh[i - a - g] : W_b[i - a - 2 * g];
    // every matrix starts at a multiple of f f, so permuting the whole buffer
    // as [rows][f] permutes each matrix in place
    const int64_t k = i / f;
    const int n = (int)(i % f);
    out[((k >> 2) * (f / 8) + (n >> 3)) * 32 + (n & 7) * 4 + (k & 3)] = (double)x;
}
__host__ __device__ inline int64_t heavy_weights_f64_count(int32_t nt, bool with_b) { return (int64_t)(nt + 6 + (with_b ? 1 : 0)) * 128 * 128; }
cudaError_t launch_ggnn_heavy_b(const GraphDev &g, const HeavyWs &w, const float *H, const float *b_e,
                                cudaStream_t st);
cudaError_t launch_gru_heavy_f64(const GraphDev &g, const HeavyWs &w, const float *H, const float *b_ih,
                                 const float *b_hh, float *out, cudaStream_t st);

// split-TF32 (3 MMAs per product) tcgen05 GEMMs (gemm_tf32split.cu), config C4.
// GGNN (NEXT-4): AB = H . [W_a | W_b] + [0 | b_e] (split-TF32, also splits the
// GRU weights into wsplit), the edge-MLP gather m = sum|max act(A[u] + B[v]),
// and the GRU GEMM over [m || h].
// 2-D bf16 row-major [rows][cols] tensor map, {64 col, box_rows row} box, 128B swizzle (gemm_tc.cu).
bool make_map_bf16(CUtensorMap *m, const void *base, int64_t rows, int64_t cols, int box_rows = 128);

// NEXT-1 (GCN, C5): the aggregation fused with its tcgen05 GEMM in SAGA order
// (gcn_fused.cu); ws = workspace for the staged W^T image and the tile counter.
bool gcn_fused_supported(int32_t in_dim, int32_t out_dim);
size_t gcn_fused_workspace_bytes(int32_t out_dim);
cudaError_t launch_gcn_fused(const GraphDev &g, const __nv_bfloat16 *X, int32_t in_dim, const __nv_bfloat16 *W,
                             int32_t out_dim, const float *bias, int act, __nv_bfloat16 *out, void *ws,
                             cudaStream_t st, const char **why);

// NEXT-1: GraphSAGE-mean aggregation fused with its tcgen05 concat-GEMM
// (sage_fused.cu); img = workspace for the staged W^T image.
bool sage_fused_supported(int32_t in_dim, int32_t out_dim);
size_t sage_fused_workspace_bytes(int32_t out_dim);
cudaError_t launch_sage_fused(const GraphDev &g, const __nv_bfloat16 *X, int32_t in_dim, const __nv_bfloat16 *W,
                              int32_t out_dim, const float *bias, int act, __nv_bfloat16 *out, void *img,
                              cudaStream_t st, const char **why);

size_t ggnn_tc_workspace_floats(int32_t f);
// w64 (nullable): also the heavy kernels' fp64 weights (heavy_weights_f64_item)
cudaError_t launch_ggnn_split_weights(int32_t f, const float *W_e, const float *b_e, const float *W_ih,
                                      const float *W_hh, float *wsplit, double *w64, cudaStream_t st);
// GGNN edge-MLP projection AB = H . [W_a | W_b] + [0 | b_e] on the int8 tensor
// cores with exact accumulation (gemm_i8x.cu); ws: ggnn_i8_workspace_bytes(M).
size_t ggnn_i8_workspace_bytes(int64_t M);
cudaError_t launch_ggnn_edge_i8x(int64_t M, int32_t f, const float *H, const float *W_e, const float *b_e, void *ws,
                                 float *AB, cudaStream_t st, const char **why);
// Bx: the heavy rows' B = H W_b + b_e in fp64 [n_heavy][f]; mx: their m in fp64 (out).
cudaError_t launch_agg_edge_mlp_f32(const GraphDev &g, const float *AB, int32_t f, bool relu, bool max, float *m,
                                    const double *Bx, double *mx, AggWorkspace ws, cudaStream_t st);
cudaError_t launch_ggnn_gru_tc(int64_t M, int32_t f, const float *m, const float *H, const float *b_ih,
                               const float *b_hh, const float *wsplit, float *out, cudaStream_t st, const char **why);
size_t gated_tc_workspace_floats(int32_t f, int32_t T);
cudaError_t launch_gated_apply_tc(int64_t M, int32_t f, int32_t T, const float *S, const float *H,
                                  const float *W_type, const float *W_ih, const float *W_hh, const float *b_ih,
                                  const float *b_hh, float *m_ws, float *wsplit, double *w64, float *out,
                                  cudaStream_t st, const char **why);

// GraphSAGE-LSTM Gather (lstm_gather.cu, NEXT-2): h_out[v] = final LSTM state over v's in-edges.
size_t lstm_workspace_bytes();  // staged W_hh^T + the work-queue head
cudaError_t launch_lstm_gather(const GraphDev &g, const __nv_bfloat16 *P, const __nv_bfloat16 *W_hh,
                               const float *b_ih, const float *b_hh, __nv_bfloat16 *h_out, void *wt_ws,
                               cudaStream_t st);

// R-GCN ApplyVertex (NEXT-3): out = act([S_0..S_{T-1} || H] . [W_0; ..; W_{T-1}; W_self] + b), 3xTF32.
size_t rgcn_tc_workspace_floats(int32_t f, int32_t T);
cudaError_t launch_rgcn_apply_tc(int64_t M, int32_t f, int32_t T, const float *S, const float *H, const float *W_type,
                                 const float *W_self, const float *bias, int act, float *wsplit, float *out,
                                 cudaStream_t st, const char **why);

}  // namespace saga
