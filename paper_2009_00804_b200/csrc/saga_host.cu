// saga_host.cu -- the C ABI (include/saga.h): argument validation, workspace
// planning and kernel sequencing for one SAGA-NN layer.  No allocation and no
// synchronisation on the layer path; every launch goes on the caller's stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <mutex>
#include <string>
#include <vector>

#include "internal.cuh"

struct saga_graph {
    saga::GraphDev d;
};

namespace saga {
thread_local bool g_pdl_call = false, g_pdl_armed = false;
}

namespace {

thread_local std::string g_last_error;

saga_status fail(saga_status s, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
saga_status fail(saga_status s, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return s;
}

saga_status cuda_fail(cudaError_t e, const char *what) {
    return fail(e == cudaErrorMemoryAllocation ? SAGA_ENOMEM : SAGA_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// ------------------------------------------------------------ profiling ----
struct ProfRec {
    int name;
    cudaEvent_t a, b;
};
struct Prof {
    std::mutex mu;
    bool on = false;
    std::string only;  // non-empty: bracket only the launches with this label (PDL stays on for the rest)
    std::vector<std::string> names;
    std::vector<int64_t> launches;
    std::vector<double> ms;
    std::vector<ProfRec> pending;
    std::vector<cudaEvent_t> pool;
    // timeline: every bracketed launch in launch order, start and end in ms
    // from the first bracket opened since saga_profile_enable (origin)
    cudaEvent_t origin = nullptr;
    struct Span { int name; double t0, t1; };
    std::vector<Span> trace;
    cudaEvent_t get() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
    int id(const char *n) {
        for (size_t i = 0; i < names.size(); ++i)
            if (names[i] == n) return (int)i;
        names.emplace_back(n);
        launches.push_back(0);
        ms.push_back(0.0);
        return (int)names.size() - 1;
    }
    void drain() {
        for (auto &r : pending) {
            cudaEventSynchronize(r.b);
            float t = 0.f;
            cudaEventElapsedTime(&t, r.a, r.b);
            ms[r.name] += t;
            launches[r.name] += 1;
            float t0 = 0.f;
            cudaEventElapsedTime(&t0, origin, r.a);
            trace.push_back(Span{r.name, (double)t0, (double)t0 + t});
            if (r.a != origin) pool.push_back(r.a);
            pool.push_back(r.b);
        }
        pending.clear();
    }
};
Prof g_prof;

// RAII bracket around one kernel launch (no-op unless profiling is on).
struct ProfScope {
    bool on;
    unsigned flags = cudaEventRecordDefault;
    ProfRec r{};
    cudaStream_t st;
    ProfScope(const char *name, cudaStream_t s) : on(false), st(s) {
        std::lock_guard<std::mutex> lk(g_prof.mu);
        if (!g_prof.on || (!g_prof.only.empty() && g_prof.only != name)) return;
        on = true;
        r.name = g_prof.id(name);
        r.a = g_prof.get();
        r.b = g_prof.get();
        if (!g_prof.origin) g_prof.origin = r.a;
        // under stream capture the pair must be event-record NODES of the graph
        // (external); outside capture the flag is an error
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive)
            flags = cudaEventRecordExternal;
        cudaEventRecordWithFlags(r.a, st, flags);
    }
    ~ProfScope() {
        if (!on) return;
        cudaEventRecordWithFlags(r.b, st, flags);
        std::lock_guard<std::mutex> lk(g_prof.mu);
        g_prof.pending.push_back(r);
    }
};

// Scope of one saga_layer call for programmatic dependent launch
// (internal.cuh); SAGA_NO_PDL=1 in the environment turns it off.
struct PdlCall {
    PdlCall() {
        static const bool off = [] {
            const char *v = getenv("SAGA_NO_PDL");
            return v && *v && *v != '0';
        }();
        bool prof;
        {
            std::lock_guard<std::mutex> lk(g_prof.mu);
            prof = g_prof.on && g_prof.only.empty();  // a filtered profile keeps PDL for the other kernels
        }
        saga::g_pdl_call = !off && !prof;
        saga::g_pdl_armed = false;
    }
    ~PdlCall() { saga::g_pdl_call = saga::g_pdl_armed = false; }
};

// The graph arrays and the build's scratch come from the device's default
// stream-ordered pool.  With the pool's default release threshold (0) every
// synchronisation -- the build's range check -- hands the memory back to the
// driver and the next build maps it again; keep up to 4 GiB cached instead
// (raised once per device, never lowered below a caller's setting).
void keep_pool_memory() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return;
    uint64_t cur = 0;
    if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &cur) != cudaSuccess) return;
    uint64_t want = uint64_t(4) << 30;
    if (cur < want) cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &want);
}

constexpr size_t kAlign = 256;
constexpr int kGatMaxParts = 1024;  // GAT: per-CTA maxima slots (the GEMM runs one CTA per SM)
size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

// Workspace plan: [counters | partials | model intermediates].
struct Plan {
    size_t counters = 0, partials = 0, inter0 = 0, inter1 = 0, inter2 = 0, inter3 = 0, total = 0;
};

Plan plan_for(saga_model kind, const saga::GraphDev &g, const saga_layer_opts &o) {
    Plan p;
    // the typed gathers run over the typed view's own schedule
    const size_t nt = (size_t)std::max({g.ntasks, g.tntasks, g.fntasks, g.afntasks, g.antasks});
    const size_t n = (size_t)g.n;
    size_t width = 0;
    switch (kind) {
        case SAGA_GCN: width = (size_t)(o.in_dim <= 0 ? 0 : (o.out_dim > 0 ? o.out_dim : 0)); break;
        case SAGA_SAGE: width = (size_t)o.in_dim; break;
        case SAGA_GAT: width = (size_t)o.out_dim; break;
        case SAGA_GATED: width = (size_t)o.in_dim; break;
        case SAGA_RGCN: width = (size_t)o.in_dim; break;
        case SAGA_SAGE_LSTM: width = (size_t)o.in_dim; break;
        case SAGA_GGNN: width = (size_t)o.in_dim; break;
    }
    size_t pf = saga::agg_partial_floats(kind, (int32_t)width, 8);
    if (kind == SAGA_GCN) pf = (size_t)2 * std::max({o.in_dim, o.out_dim, 32});  // fp64 partials on the fp32 path
    pf = std::max<size_t>(pf, 32);                                                  // >= one fp32 per lane
    p.counters = align_up(sizeof(int32_t) * (nt + 1));
    p.partials = align_up(sizeof(float) * pf * 2 * (nt + 1));
    switch (kind) {
        case SAGA_GCN:
            p.inter0 = align_up((size_t)2 * n * (size_t)std::max(o.out_dim, 0));                // Y bf16 (two-kernel path)
            if (o.fused) p.inter1 = align_up(saga::gcn_fused_workspace_bytes(std::max(o.out_dim, 0)));  // W^T image, tile counter
            break;
        case SAGA_SAGE:
            p.inter0 = align_up((size_t)2 * n * (size_t)std::max(o.in_dim, 0));                // M bf16 (two-kernel path)
            p.inter1 = align_up(saga::sage_fused_workspace_bytes(std::max(o.out_dim, 0)));     // W^T image (fused)
            break;
        case SAGA_GAT:
            p.inter0 = align_up((size_t)2 * n * (size_t)std::max(o.out_dim, 0));               // z bf16
            p.inter1 = align_up(sizeof(float) * n * 8);                                         // el
            // er, then the GEMM's per-CTA maxima of el and their maximum M_h
            p.inter2 = align_up(sizeof(float) * (n * 8 + (size_t)kGatMaxParts * 8 + 8));
            break;
        case SAGA_GATED:
            p.inter0 = align_up(sizeof(float) * n * (size_t)g.num_etypes * (size_t)std::max(o.in_dim, 0));  // S [n][T][f]
            p.inter1 = align_up(sizeof(float) * n * (size_t)std::max(o.in_dim, 0));            // m
            p.inter2 = align_up(sizeof(float) * saga::gated_tc_workspace_floats(128, 4));       // split W
            break;
        case SAGA_SAGE_LSTM:
            p.inter0 = align_up((size_t)2 * 4 * n * (size_t)std::max(o.in_dim, 0));             // P = X W_ih, bf16
            p.inter1 = align_up((size_t)2 * n * (size_t)std::max(o.in_dim, 0));                 // h (LSTM out), bf16
            p.inter2 = align_up(saga::lstm_workspace_bytes());                                  // staged W_hh^T
            break;
        case SAGA_GGNN:
            p.inter0 = align_up(sizeof(float) * n * 2 * (size_t)std::max(o.in_dim, 0));        // AB = [A | B]
            p.inter1 = align_up(sizeof(float) * n * (size_t)std::max(o.in_dim, 0));            // m
            p.inter2 = align_up(sizeof(float) * saga::ggnn_tc_workspace_floats(128)) +         // split GRU weights
                       align_up(saga::ggnn_i8_workspace_bytes((int64_t)n));                    // int8 digit planes
            break;
        case SAGA_RGCN:
            p.inter0 = align_up(sizeof(float) * n * (size_t)g.num_etypes * (size_t)std::max(o.in_dim, 0));  // S (type means)
            p.inter2 = align_up(sizeof(float) * saga::rgcn_tc_workspace_floats(128, 4));        // split W
            break;
    }
    // gated / GGNN heavy rows: the fp64 sums (Sx) or B and m (Bx, mx), gru_f64.cu
    p.inter3 = align_up(saga::heavy_workspace_bytes(g, kind, std::max(o.in_dim, 0)));
    p.total = p.counters + p.partials + p.inter0 + p.inter1 + p.inter2 + p.inter3;
    return p;
}

// Every argument check of saga_layer, before anything is enqueued (saga.h).
saga_status validate(saga_model kind, const saga::GraphDev &d, const saga_tensor *x, const saga_weights *w,
                     const saga_layer_opts &o) {
    switch (kind) {
        case SAGA_GCN:
            if (!w->W) return fail(SAGA_EINVAL, "GCN needs W");
            if (o.act != SAGA_ACT_NONE && o.act != SAGA_ACT_RELU) return fail(SAGA_EUNSUPPORTED, "GCN act must be NONE/RELU");
            if (x->dtype == SAGA_F32) {
                if (!(o.in_dim == 16 || o.in_dim == 32 || o.in_dim == 64 || o.in_dim == 128) || o.out_dim < 1 ||
                    o.out_dim > 64)
                    return fail(SAGA_EUNSUPPORTED, "fp32 GCN supports in_dim in {16,32,64,128}, out_dim <= 64");
                return SAGA_OK;
            }
            if (x->dtype != SAGA_BF16) return fail(SAGA_EDTYPE, "GCN features must be F32 or BF16");
            if (o.in_dim % 64 || o.in_dim > 256 || o.in_dim == 0 ||
                !(o.out_dim == 64 || o.out_dim == 128 || o.out_dim == 256))
                return fail(SAGA_EUNSUPPORTED, "bf16 GCN supports in_dim in {64..256 step 64}, out_dim in {64,128,256}");
            if (o.fused && !saga::gcn_fused_supported(o.in_dim, o.out_dim))
                return fail(SAGA_EUNSUPPORTED, "fused GCN supports in_dim 256, out_dim 64, 128 or 256");
            return SAGA_OK;
        case SAGA_SAGE:
            if (x->dtype != SAGA_BF16) return fail(SAGA_EDTYPE, "SAGE supports BF16 features");
            if (!w->W) return fail(SAGA_EINVAL, "SAGE needs W");
            if (!(o.in_dim == 64 || o.in_dim == 128) || !(o.out_dim == 64 || o.out_dim == 128 || o.out_dim == 256))
                return fail(SAGA_EUNSUPPORTED, "SAGE supports in_dim in {64,128}, out_dim in {64,128,256}");
            if (o.act != SAGA_ACT_NONE && o.act != SAGA_ACT_RELU) return fail(SAGA_EUNSUPPORTED, "SAGE act must be NONE/RELU");
            if (o.fused && !saga::sage_fused_supported(o.in_dim, o.out_dim))
                return fail(SAGA_EUNSUPPORTED, "fused SAGE supports in_dim 128, out_dim 64 or 128");
            return SAGA_OK;
        case SAGA_GAT:
            if (x->dtype != SAGA_BF16) return fail(SAGA_EDTYPE, "GAT supports BF16 features");
            if (!w->W || !w->attn_src || !w->attn_dst) return fail(SAGA_EINVAL, "GAT needs W, attn_src, attn_dst");
            if (o.heads != 8 || o.head_dim != 8 || o.out_dim != 64 || o.in_dim % 64 || o.in_dim > 256 || !o.in_dim)
                return fail(SAGA_EUNSUPPORTED, "GAT supports heads=8, head_dim=8, in_dim in {64..256 step 64}");
            if (o.act != SAGA_ACT_ELU) return fail(SAGA_EUNSUPPORTED, "GAT act must be ELU");
            if (!(o.leaky_slope >= 0.0f && o.leaky_slope <= 1.0f))
                return fail(SAGA_EUNSUPPORTED, "GAT leaky_slope must lie in [0, 1]");
            if (saga::gemm_bf16_tc_grid(d.n) > kGatMaxParts)  // the GEMM's per-CTA maxima slots (one CTA per SM)
                return fail(SAGA_EUNSUPPORTED, "GAT: more than %d SMs", kGatMaxParts);
            return SAGA_OK;
        case SAGA_GATED:
            if (x->dtype != SAGA_F32) return fail(SAGA_EDTYPE, "GATED supports F32 features");
            if (o.in_dim != 128 || o.out_dim != 128) return fail(SAGA_EUNSUPPORTED, "GATED supports in=out=128");
            if (d.num_etypes > 4) return fail(SAGA_EUNSUPPORTED, "GATED supports <= 4 edge types");
            if (!w->W_type || !w->W_ih || !w->W_hh || !w->b_ih || !w->b_hh)
                return fail(SAGA_EINVAL, "GATED needs W_type, W_ih, W_hh, b_ih, b_hh");
            return SAGA_OK;
        case SAGA_SAGE_LSTM:
            if (x->dtype != SAGA_BF16) return fail(SAGA_EDTYPE, "SAGE_LSTM supports BF16 features");
            if (o.in_dim != 128 || !(o.out_dim == 64 || o.out_dim == 128 || o.out_dim == 256))
                return fail(SAGA_EUNSUPPORTED, "SAGE_LSTM supports in_dim 128, out_dim in {64,128,256}");
            if (o.act != SAGA_ACT_NONE && o.act != SAGA_ACT_RELU) return fail(SAGA_EUNSUPPORTED, "SAGE_LSTM act must be NONE/RELU");
            if (!w->W || !w->W_ih || !w->W_hh || !w->b_ih || !w->b_hh)
                return fail(SAGA_EINVAL, "SAGE_LSTM needs W, W_ih, W_hh, b_ih, b_hh");
            return SAGA_OK;
        case SAGA_GGNN:
            if (x->dtype != SAGA_F32) return fail(SAGA_EDTYPE, "GGNN supports F32 features");
            if (o.in_dim != 128 || o.out_dim != 128) return fail(SAGA_EUNSUPPORTED, "GGNN supports in=out=128");
            if (o.act != SAGA_ACT_NONE && o.act != SAGA_ACT_RELU) return fail(SAGA_EUNSUPPORTED, "GGNN act must be NONE/RELU");
            if (o.aggregator != SAGA_AGG_SUM && o.aggregator != SAGA_AGG_MAX)
                return fail(SAGA_EUNSUPPORTED, "GGNN aggregator must be SUM or MAX");
            if (!w->W || !w->W_ih || !w->W_hh || !w->b_ih || !w->b_hh)
                return fail(SAGA_EINVAL, "GGNN needs W (edge MLP), W_ih, W_hh, b_ih, b_hh");
            return SAGA_OK;
        case SAGA_RGCN:
            if (x->dtype != SAGA_F32) return fail(SAGA_EDTYPE, "RGCN supports F32 features");
            if (o.in_dim != 128 || o.out_dim != 128) return fail(SAGA_EUNSUPPORTED, "RGCN supports in=out=128");
            if (d.num_etypes > 4) return fail(SAGA_EUNSUPPORTED, "RGCN supports <= 4 edge types");
            if (o.act != SAGA_ACT_NONE && o.act != SAGA_ACT_RELU) return fail(SAGA_EUNSUPPORTED, "RGCN act must be NONE/RELU");
            if (!w->W_type || !w->W) return fail(SAGA_EINVAL, "RGCN needs W_type and W (self)");
            return SAGA_OK;
    }
    return fail(SAGA_EINVAL, "unknown model kind %d", (int)kind);
}

}  // namespace

extern "C" {

int saga_abi_version(void) { return SAGA_ABI_VERSION; }

const char *saga_last_error(void) { return g_last_error.c_str(); }

saga_status saga_graph_build(int32_t num_vertices, int64_t num_edges, const int32_t *src, const int32_t *dst,
                             const int32_t *etype, int32_t num_etypes, void *cuda_stream, saga_graph **out,
                             int64_t *first_bad_edge) {
    g_last_error.clear();
    if (first_bad_edge) *first_bad_edge = -1;
    if (!out) return fail(SAGA_EINVAL, "out is NULL");
    *out = nullptr;
    if (num_vertices < 0 || num_edges < 0 || num_edges >= (int64_t(1) << 31))
        return fail(SAGA_EINVAL, "invalid sizes N=%d E=%lld", num_vertices, (long long)num_edges);
    if (num_edges > 0 && (!src || !dst)) return fail(SAGA_EINVAL, "src/dst is NULL");
    if (etype && num_etypes < 1) return fail(SAGA_EINVAL, "num_etypes must be >= 1 with etype");
    if (num_vertices == 0 && num_edges > 0) {
        if (first_bad_edge) *first_bad_edge = 0;
        return fail(SAGA_ERANGE, "COO entry 0 out of range (N = 0)");
    }
    saga_graph *g = new (std::nothrow) saga_graph();
    if (!g) return fail(SAGA_ENOMEM, "host allocation failed");
    keep_pool_memory();
    int64_t bad = -1;
    const char *why = "";
    saga_status s = saga::build_graph(num_vertices, num_edges, src, dst, etype, num_etypes,
                                      static_cast<cudaStream_t>(cuda_stream), &g->d, &bad, &why);
    if (s != SAGA_OK) {
        if (first_bad_edge) *first_bad_edge = bad;
        saga::free_graph(&g->d);
        delete g;
        if (s == SAGA_ERANGE) return fail(s, "COO entry %lld out of range", (long long)bad);
        return fail(s, "graph build failed: %s", why);
    }
    *out = g;
    return SAGA_OK;
}

saga_status saga_graph_info(const saga_graph *g, int32_t *n, int64_t *e, int32_t *t) {
    if (!g) return fail(SAGA_EINVAL, "graph is NULL");
    if (n) *n = g->d.n;
    if (e) *e = g->d.e;
    if (t) *t = g->d.num_etypes;
    return SAGA_OK;
}

saga_status saga_graph_copy_csr(const saga_graph *g, int64_t *row_ptr, int32_t *col_src, int32_t *edge_id,
                                int32_t *etype, int32_t *in_deg, int32_t *out_deg, void *cuda_stream) {
    if (!g) return fail(SAGA_EINVAL, "graph is NULL");
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    const saga::GraphDev &d = g->d;
    cudaError_t e = cudaSuccess;
    auto cp = [&](void *dst, const void *srcp, size_t bytes) {
        if (dst && bytes && e == cudaSuccess) e = cudaMemcpyAsync(dst, srcp, bytes, cudaMemcpyDeviceToDevice, st);
    };
    cp(row_ptr, d.row_ptr, sizeof(int64_t) * ((size_t)d.n + 1));
    cp(col_src, d.col_src, sizeof(int32_t) * (size_t)d.e);
    cp(edge_id, d.edge_id, sizeof(int32_t) * (size_t)d.e);
    if (etype) {
        if (d.etype)
            cp(etype, d.etype, sizeof(int32_t) * (size_t)d.e);
        else if (d.e && e == cudaSuccess)
            e = cudaMemsetAsync(etype, 0, sizeof(int32_t) * (size_t)d.e, st);
    }
    cp(in_deg, d.in_deg, sizeof(int32_t) * (size_t)d.n);
    cp(out_deg, d.out_deg, sizeof(int32_t) * (size_t)d.n);
    return e ? cuda_fail(e, "copy_csr") : SAGA_OK;
}

saga_status saga_layer_workspace_bytes(saga_model kind, const saga_graph *g, const saga_layer_opts *opts,
                                       size_t *bytes) {
    if (!g || !opts || !bytes) return fail(SAGA_EINVAL, "NULL argument");
    if (kind < SAGA_GCN || kind > SAGA_GGNN) return fail(SAGA_EINVAL, "unknown model kind %d", (int)kind);
    *bytes = plan_for(kind, g->d, *opts).total;
    return SAGA_OK;
}

saga_status saga_profile_enable(int enable) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    g_prof.drain();
    g_prof.on = enable != 0;
    if (g_prof.origin) g_prof.pool.push_back(g_prof.origin);
    g_prof.origin = nullptr;
    g_prof.trace.clear();
    std::fill(g_prof.launches.begin(), g_prof.launches.end(), 0);
    std::fill(g_prof.ms.begin(), g_prof.ms.end(), 0.0);
    return SAGA_OK;
}

saga_status saga_profile_filter(const char *label) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    g_prof.only = label ? label : "";
    return SAGA_OK;
}

int32_t saga_profile_count(void) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    return (int32_t)g_prof.names.size();
}

saga_status saga_profile_get(int32_t index, const char **name, int64_t *launches, double *total_ms) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    g_prof.drain();
    if (index < 0 || index >= (int32_t)g_prof.names.size()) return fail(SAGA_EINVAL, "profile index out of range");
    if (name) *name = g_prof.names[index].c_str();
    if (launches) *launches = g_prof.launches[index];
    if (total_ms) *total_ms = g_prof.ms[index];
    return SAGA_OK;
}

int32_t saga_profile_trace_count(void) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    g_prof.drain();
    return (int32_t)g_prof.trace.size();
}

saga_status saga_profile_trace_get(int32_t index, const char **name, double *start_ms, double *end_ms) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    g_prof.drain();
    if (index < 0 || index >= (int32_t)g_prof.trace.size()) return fail(SAGA_EINVAL, "trace index out of range");
    const Prof::Span &sp = g_prof.trace[index];
    if (name) *name = g_prof.names[sp.name].c_str();
    if (start_ms) *start_ms = sp.t0;
    if (end_ms) *end_ms = sp.t1;
    return SAGA_OK;
}

void saga_free(saga_graph *g) {
    if (!g) return;
    saga::free_graph(&g->d);
    delete g;
}



saga_status saga_layer(saga_model kind, const saga_graph *g, const saga_tensor *x, const saga_weights *w,
                       saga_tensor *out, const saga_layer_opts *opts, void *workspace, size_t workspace_bytes,
                       void *cuda_stream) {
    using namespace saga;
    g_last_error.clear();
    if (!g || !x || !w || !out || !opts) return fail(SAGA_EINVAL, "NULL argument");
    const GraphDev &d = g->d;
    const saga_layer_opts &o = *opts;
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    if (kind < SAGA_GCN || kind > SAGA_GGNN) return fail(SAGA_EINVAL, "unknown model kind %d", (int)kind);
    if (x->rows != d.n) return fail(SAGA_ESHAPE, "features.rows=%lld != N=%d", (long long)x->rows, d.n);
    if (x->cols != o.in_dim) return fail(SAGA_ESHAPE, "features.cols=%lld != in_dim=%d", (long long)x->cols, o.in_dim);
    if (out->rows != d.n || out->cols != o.out_dim)
        return fail(SAGA_ESHAPE, "out shape [%lld][%lld] != [%d][%d]", (long long)out->rows, (long long)out->cols, d.n,
                    o.out_dim);
    if (out->dtype != x->dtype) return fail(SAGA_EDTYPE, "out dtype must equal features dtype");
    if (d.n > 0 && (!x->data || !out->data)) return fail(SAGA_EINVAL, "features/out data is NULL");
    if (!aligned16(x->data) || !aligned16(out->data) || !aligned16(workspace))
        return fail(SAGA_EINVAL, "features/out/workspace must be 16-byte aligned");
    const Plan plan = plan_for(kind, d, o);
    if (workspace_bytes < plan.total || (plan.total && !workspace))
        return fail(SAGA_EINVAL, "workspace too small: %zu < %zu", workspace_bytes, plan.total);
    const saga_status vs = validate(kind, d, x, w, o);
    if (vs != SAGA_OK) return vs;
    if (d.n == 0) return SAGA_OK;

    uint8_t *ws = static_cast<uint8_t *>(workspace);
    AggWorkspace aw;
    aw.counters = reinterpret_cast<int32_t *>(ws);
    aw.partials = reinterpret_cast<float *>(ws + plan.counters);
    uint8_t *i0 = ws + plan.counters + plan.partials;
    uint8_t *i1 = i0 + plan.inter0;
    uint8_t *i2 = i1 + plan.inter1;
    uint8_t *i3 = i2 + plan.inter2;
    cudaError_t e = cudaSuccess;
    PdlCall pdl_call;
    // split-row tickets start at 0; every ticket's winner resets its counter,
    // so a completed call leaves them zero (opts.workspace_zeroed skips this)
    if (!o.workspace_zeroed && !(kind == SAGA_GCN && x->dtype == SAGA_F32 && gcn_f32_rowwise(d))) {
        e = cudaMemsetAsync(aw.counters, 0, sizeof(int32_t) * (size_t)std::max({d.ntasks, d.tntasks, d.fntasks, d.afntasks, d.antasks}),
                            st);
        if (e) return cuda_fail(e, "memset counters");
    }
    const char *why = "";

    switch (kind) {
        case SAGA_GCN: {
            if (x->dtype == SAGA_F32) {
                {
                    ProfScope ps_("gcn_f32_fused", st);
                    e = launch_gcn_f32_fused(d, static_cast<const float *>(x->data), o.in_dim,
                                             static_cast<const float *>(w->W), o.out_dim, w->bias, o.act,
                                             static_cast<float *>(out->data), aw, st);
                }
                if (e) return cuda_fail(e, "gcn_f32_fused");
                return SAGA_OK;
            }
            if (o.fused) {
                // NEXT-1: SAGA order, the aggregation and the ApplyVertex GEMM in one kernel
                {
                    ProfScope ps_("gcn_fused_tc", st);
                    e = launch_gcn_fused(d, static_cast<const __nv_bfloat16 *>(x->data), o.in_dim,
                                         static_cast<const __nv_bfloat16 *>(w->W), o.out_dim, w->bias, o.act,
                                         static_cast<__nv_bfloat16 *>(out->data), i1, st, &why);
                }
                if (e) return fail(SAGA_ECUDA, "gcn fused: %s (%s)", cudaGetErrorString(e), why);
                return SAGA_OK;
            }
            // S2: Y = diag(dinv) . X . W  (tcgen05), then S3-S5 aggregation
            __nv_bfloat16 *Y = reinterpret_cast<__nv_bfloat16 *>(i0);
            GemmArgs a;
            a.M = d.n; a.K0 = o.in_dim; a.K1 = 0; a.N = o.out_dim;
            a.A0 = static_cast<const __nv_bfloat16 *>(x->data);
            a.W = static_cast<const __nv_bfloat16 *>(w->W);
            a.out = Y;
            a.epi = EPI_ROWSCALE;
            a.row_scale = d.dinv;
            {
                ProfScope ps_("gemm_bf16_tc", st);
                e = launch_gemm_bf16_tc(a, st, &why);
            }
            if (e) return fail(SAGA_ECUDA, "gcn gemm: %s (%s)", cudaGetErrorString(e), why);
            {
                ProfScope ps_("agg_gcn_bf16", st);
                e = launch_agg_gcn_bf16(d, Y, o.out_dim, w->bias, o.act, static_cast<__nv_bfloat16 *>(out->data), aw, st);
            }
            if (e) return cuda_fail(e, "gcn aggregate");
            return SAGA_OK;
        }
        case SAGA_SAGE: {
            if (o.fused) {
                // NEXT-1: mean aggregation and the concat-GEMM in one kernel
                {
                    ProfScope ps_("sage_fused_tc", st);
                    e = launch_sage_fused(d, static_cast<const __nv_bfloat16 *>(x->data), o.in_dim,
                                          static_cast<const __nv_bfloat16 *>(w->W), o.out_dim, w->bias, o.act,
                                          static_cast<__nv_bfloat16 *>(out->data), i1, st, &why);
                }
                if (e) return fail(SAGA_ECUDA, "sage fused: %s (%s)", cudaGetErrorString(e), why);
                return SAGA_OK;
            }
            __nv_bfloat16 *M = reinterpret_cast<__nv_bfloat16 *>(i0);
            {
                ProfScope ps_("agg_mean_bf16", st);
                e = launch_agg_mean_bf16(d, static_cast<const __nv_bfloat16 *>(x->data), o.in_dim, M, aw, st);
            }
            if (e) return cuda_fail(e, "sage aggregate");
            GemmArgs a;
            a.M = d.n; a.K0 = o.in_dim; a.K1 = o.in_dim; a.N = o.out_dim;
            a.A0 = static_cast<const __nv_bfloat16 *>(x->data);
            a.A1 = M;
            a.W = static_cast<const __nv_bfloat16 *>(w->W);
            a.out = static_cast<__nv_bfloat16 *>(out->data);
            a.epi = EPI_BIAS_ACT;
            a.bias = w->bias;
            a.act = o.act;
            {
                ProfScope ps_("gemm_bf16_tc", st);
                e = launch_gemm_bf16_tc(a, st, &why);
            }
            if (e) return fail(SAGA_ECUDA, "sage gemm: %s (%s)", cudaGetErrorString(e), why);
            return SAGA_OK;
        }
        case SAGA_GAT: {
            __nv_bfloat16 *z = reinterpret_cast<__nv_bfloat16 *>(i0);
            float *el = reinterpret_cast<float *>(i1), *er = reinterpret_cast<float *>(i2);
            GatSoftmaxWs sw;
            sw.parts = er + (size_t)d.n * 8;
            sw.Mh = sw.parts + (size_t)kGatMaxParts * 8;
            sw.nparts = gemm_bf16_tc_grid(d.n);  // <= kGatMaxParts (validate)
            GemmArgs a;
            a.M = d.n; a.K0 = o.in_dim; a.K1 = 0; a.N = 64;
            a.A0 = static_cast<const __nv_bfloat16 *>(x->data);
            a.W = static_cast<const __nv_bfloat16 *>(w->W);
            a.out = z;
            a.epi = EPI_GAT;
            a.a_src = w->attn_src; a.a_dst = w->attn_dst; a.el = el; a.er = er; a.elmax = sw.parts;
            if (d.arow) {  // the epilogue writes ELU(z) of the self-loop-only rows (aggregation view)
                a.row_scale = d.dinv;
                a.out2 = static_cast<__nv_bfloat16 *>(out->data);
            }
            {
                ProfScope ps_("gemm_bf16_tc_gat", st);
                e = launch_gemm_bf16_tc(a, st, &why);
            }
            if (e) return fail(SAGA_ECUDA, "gat gemm: %s (%s)", cudaGetErrorString(e), why);
            {
                ProfScope ps_("gat_edge", st);
                e = launch_gat_edge(d, z, el, er, sw, o.leaky_slope, static_cast<__nv_bfloat16 *>(out->data), aw, st);
            }
            if (e) return cuda_fail(e, "gat edge");
            return SAGA_OK;
        }
        case SAGA_GATED: {
            float *S = reinterpret_cast<float *>(i0), *m = reinterpret_cast<float *>(i1);
            const float *H = static_cast<const float *>(x->data);
            const HeavyWs hw = heavy_ws(d, SAGA_GATED, i3);
            {
                ProfScope ps_("agg_typed_f32", st);
                e = launch_agg_typed_f32(d, H, o.in_dim, S, false, hw.Sx, aw, st);
            }
            if (e) return cuda_fail(e, "typed aggregate");
            {
                ProfScope ps_("gated_apply_tf32x3", st);
                e = launch_gated_apply_tc(d.n, o.in_dim, d.num_etypes, S, H, w->W_type,
                                          static_cast<const float *>(w->W_ih), static_cast<const float *>(w->W_hh),
                                          w->b_ih, w->b_hh, m, reinterpret_cast<float *>(i2),
                                          d.n_heavy ? hw.W64 : nullptr, static_cast<float *>(out->data), st, &why);
            }
            if (e) return fail(SAGA_ECUDA, "gated apply: %s (%s)", cudaGetErrorString(e), why);
            if (d.n_heavy) {
                ProfScope ps_("gru_heavy_f64", st);  // (fp64 weights: written by the gated apply's split kernel)
                e = launch_gru_heavy_f64(d, hw, H, w->b_ih, w->b_hh, static_cast<float *>(out->data), st);
            }
            if (e) return cuda_fail(e, "gated heavy rows");
            return SAGA_OK;
        }
        case SAGA_SAGE_LSTM: {
            const int F = o.in_dim;
            __nv_bfloat16 *P = reinterpret_cast<__nv_bfloat16 *>(i0);
            __nv_bfloat16 *hagg = reinterpret_cast<__nv_bfloat16 *>(i1);
            const __nv_bfloat16 *Wih = static_cast<const __nv_bfloat16 *>(w->W_ih);
            for (int gt = 0; gt < 4 && !e; ++gt) {  // P_g = X . W_ih[g] (tensor cores)
                GemmArgs a;
                a.M = d.n; a.K0 = F; a.K1 = 0; a.N = F;
                a.A0 = static_cast<const __nv_bfloat16 *>(x->data);
                a.W = Wih + (size_t)gt * F * F;
                a.out = P + (size_t)gt * d.n * F;
                a.epi = EPI_BIAS_ACT;
                a.bias = nullptr;
                a.act = SAGA_ACT_NONE;
                ProfScope ps_("lstm_input_gemm", st);
                e = launch_gemm_bf16_tc(a, st, &why);
            }
            if (e) return fail(SAGA_ECUDA, "lstm input gemm: %s (%s)", cudaGetErrorString(e), why);
            {
                ProfScope ps_("lstm_gather", st);
                e = launch_lstm_gather(d, P, static_cast<const __nv_bfloat16 *>(w->W_hh), w->b_ih, w->b_hh, hagg, i2,
                                       st);
            }
            if (e) return cuda_fail(e, "lstm gather");
            GemmArgs a;
            a.M = d.n; a.K0 = F; a.K1 = F; a.N = o.out_dim;
            a.A0 = static_cast<const __nv_bfloat16 *>(x->data);
            a.A1 = hagg;
            a.W = static_cast<const __nv_bfloat16 *>(w->W);
            a.out = static_cast<__nv_bfloat16 *>(out->data);
            a.epi = EPI_BIAS_ACT;
            a.bias = w->bias;
            a.act = o.act;
            {
                ProfScope ps_("gemm_bf16_tc", st);
                e = launch_gemm_bf16_tc(a, st, &why);
            }
            if (e) return fail(SAGA_ECUDA, "sage_lstm gemm: %s (%s)", cudaGetErrorString(e), why);
            return SAGA_OK;
        }
        case SAGA_GGNN: {
            const float *H = static_cast<const float *>(x->data);
            float *AB = reinterpret_cast<float *>(i0), *m = reinterpret_cast<float *>(i1);
            float *wsplit = reinterpret_cast<float *>(i2);
            const HeavyWs hw = heavy_ws(d, SAGA_GGNN, i3);
            {
                ProfScope ps_("ggnn_split_weights", st);  // (and the heavy rows' fp64 weights)
                e = launch_ggnn_split_weights(o.in_dim, static_cast<const float *>(w->W), w->bias,
                                              static_cast<const float *>(w->W_ih), static_cast<const float *>(w->W_hh),
                                              wsplit, d.n_heavy ? hw.W64 : nullptr, st);
            }
            if (e) return cuda_fail(e, "ggnn split weights");
            {
                // edge-MLP projection on the int8 tensor cores, exact accumulation (unbiased A, B)
                ProfScope ps_("ggnn_edge_i8x", st);
                e = launch_ggnn_edge_i8x(d.n, o.in_dim, H, static_cast<const float *>(w->W), w->bias,
                                         reinterpret_cast<uint8_t *>(wsplit) +
                                             align_up(sizeof(float) * ggnn_tc_workspace_floats(128)),
                                         AB, st, &why);
            }
            if (e) return fail(SAGA_ECUDA, "ggnn edge gemm: %s (%s)", cudaGetErrorString(e), why);
            if (d.n_heavy) {
                ProfScope ps_("ggnn_heavy_b_f64", st);
                e = launch_ggnn_heavy_b(d, hw, H, w->bias, st);
            }
            if (e) return cuda_fail(e, "ggnn heavy B");
            {
                ProfScope ps_("agg_edge_mlp_f32", st);
                e = launch_agg_edge_mlp_f32(d, AB, o.in_dim, o.act == SAGA_ACT_RELU, o.aggregator == SAGA_AGG_MAX, m,
                                            hw.Bx, hw.mx, aw, st);
            }
            if (e) return cuda_fail(e, "ggnn edge-mlp gather");
            {
                ProfScope ps_("ggnn_gru_tf32x3", st);
                e = launch_ggnn_gru_tc(d.n, o.in_dim, m, H, w->b_ih, w->b_hh, wsplit, static_cast<float *>(out->data),
                                       st, &why);
            }
            if (e) return fail(SAGA_ECUDA, "ggnn gru: %s (%s)", cudaGetErrorString(e), why);
            if (d.n_heavy) {
                ProfScope ps_("gru_heavy_f64", st);
                e = launch_gru_heavy_f64(d, hw, H, w->b_ih, w->b_hh, static_cast<float *>(out->data), st);
            }
            if (e) return cuda_fail(e, "ggnn heavy rows");
            return SAGA_OK;
        }
        case SAGA_RGCN: {
            float *S = reinterpret_cast<float *>(i0);
            {
                ProfScope ps_("agg_typed_mean_f32", st);
                e = launch_agg_typed_f32(d, static_cast<const float *>(x->data), o.in_dim, S, true, nullptr, aw, st);
            }
            if (e) return cuda_fail(e, "rgcn typed aggregate");
            {
                ProfScope ps_("rgcn_apply_tf32x3", st);
                e = launch_rgcn_apply_tc(d.n, o.in_dim, d.num_etypes, S, static_cast<const float *>(x->data), w->W_type,
                                         static_cast<const float *>(w->W), w->bias, o.act,
                                         reinterpret_cast<float *>(i2), static_cast<float *>(out->data), st, &why);
            }
            if (e) return fail(SAGA_ECUDA, "rgcn apply: %s (%s)", cudaGetErrorString(e), why);
            return SAGA_OK;
        }
    }
    return fail(SAGA_EINTERNAL, "unreachable model kind %d", (int)kind);
}

}  // extern "C"
