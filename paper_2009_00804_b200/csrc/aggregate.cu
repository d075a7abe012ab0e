// aggregate.cu -- Scatter + ApplyEdge + Gather (S3, S4) and the vertex-side
// epilogues (S5) as one merge-path segment-reduce engine.
//
// Paper: the Gather stage reduces each vertex's in-edges (PAPER.md lines
// 343-355); fused with Scatter it is "the multiplication between the
// adjacency matrix and the embedding matrix" (line 354) -- the SpMM shape,
// which is HBM-bound on B200 (~0 FLOP/byte).  Power-law in-degrees (lines
// 359-365) make per-vertex scheduling unbalanced, so work is cut by
// merge-path: the item sequence is, for every row v in order, its deg(v)
// edges followed by one row-end marker; task k owns items [kT, (k+1)T).
// A group of G lanes (16 bytes of the row per lane) streams its task's
// col_src in coalesced chunks, keeps U independent 16-byte row gathers in
// flight, and flushes a row (epilogue + coalesced store) at each row end.
// Rows split across tasks (hubs, and rows straddling a task boundary) write
// fp32 partials; the last contributor (atomic ticket) merges all partials in
// task order, so results are deterministic and no float atomics are used.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "internal.cuh"
#include "ptx.cuh"

namespace saga {
namespace {

constexpr int kBlock = 256;

struct GraphView {
    const int64_t *row_ptr;
    const int32_t *col_src;
    const int32_t *etype;
    const int32_t *task_v;
    const int64_t *task_p;
    int64_t T, ntasks;
    int32_t n;
};

GraphView view(const GraphDev &g) {
    return GraphView{g.row_ptr, g.col_src, g.etype, g.task_v, g.task_p, g.task_items, g.ntasks, g.n};
}

template <int G>
struct Group {
    int lane;       // lane within the group
    uint32_t mask;  // warp mask of the group
    __device__ Group() {
        const int wl = threadIdx.x & 31;
        lane = wl & (G - 1);
        mask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (wl & ~(G - 1)));
    }
    template <typename V>
    __device__ __forceinline__ V shfl(V v, int src) const {
        return __shfl_sync(mask, v, src, G);
    }
    __device__ __forceinline__ void sync() const { __syncwarp(mask); }
};

__device__ __forceinline__ void add_bf16x8(float (&a)[8], const uint4 &u, float w = 1.0f) {
    const uint32_t q[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float2 f = ptx::unpack_bf16x2(q[i]);
        a[2 * i] = fmaf(w, f.x, a[2 * i]);
        a[2 * i + 1] = fmaf(w, f.y, a[2 * i + 1]);
    }
}

__device__ __forceinline__ uint4 pack8(const float (&o)[8]) {
    return make_uint4(ptx::pack_bf16x2(o[0], o[1]), ptx::pack_bf16x2(o[2], o[3]), ptx::pack_bf16x2(o[4], o[5]),
                      ptx::pack_bf16x2(o[6], o[7]));
}

__device__ __forceinline__ float act_fn(float x, int act) {
    if (act == SAGA_ACT_RELU) return fmaxf(x, 0.0f);
    if (act == SAGA_ACT_ELU) return x > 0.0f ? x : expm1f(x);
    return x;
}

// ===================================================================== ops ==
// Sum of bf16 rows (8 per lane) -> act(scale[v] * acc + bias) in bf16.
// GCN (Y pre-scaled by dinv[u], scale = dinv[v]) and SAGE-mean (scale = 1/deg).
struct SumBf16Op {
    __device__ void set_smem(const float *) {}
    static constexpr int kAccF = 8;
    struct Acc { float a[8]; };
    struct Val { uint4 x; };
    const __nv_bfloat16 *X;
    int32_t f;
    const float *scale;
    const float *bias;
    int act;
    __nv_bfloat16 *out;
    __device__ void setup(int) {}
    __device__ __forceinline__ void zero(Acc &c) const {
#pragma unroll
        for (int i = 0; i < 8; ++i) c.a[i] = 0.0f;
    }
    __device__ __forceinline__ void begin_row(int32_t, int) {}
    __device__ __forceinline__ Val load(int32_t u, int lane) const {
        return Val{ptx::ldg_nc_v4(X + (int64_t)u * f + lane * 8)};
    }
    __device__ __forceinline__ void add(Acc &c, const Val &v, int32_t) const { add_bf16x8(c.a, v.x); }
    __device__ __forceinline__ void finish(int32_t v, const Acc &c, int lane) const {
        const float s = scale[v];
        float b[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (bias) {
            const float4 *bp = reinterpret_cast<const float4 *>(bias + lane * 8);
            float4 b0 = __ldg(bp), b1 = __ldg(bp + 1);
            b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
            b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
        }
        float o[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = act_fn(fmaf(s, c.a[i], b[i]), act);
        *reinterpret_cast<uint4 *>(out + (int64_t)v * f + lane * 8) = pack8(o);
    }
    __device__ __forceinline__ void save(float *slot, const Acc &c, int lane) const {
        float4 *p = reinterpret_cast<float4 *>(slot + lane * 8);
        p[0] = make_float4(c.a[0], c.a[1], c.a[2], c.a[3]);
        p[1] = make_float4(c.a[4], c.a[5], c.a[6], c.a[7]);
    }
    __device__ __forceinline__ void merge(Acc &c, const float *slot, int lane) const {
        const float4 *p = reinterpret_cast<const float4 *>(slot + lane * 8);
        float4 x = __ldcg(p), y = __ldcg(p + 1);
        c.a[0] += x.x; c.a[1] += x.y; c.a[2] += x.z; c.a[3] += x.w;
        c.a[4] += y.x; c.a[5] += y.y; c.a[6] += y.z; c.a[7] += y.w;
    }
};

// C1: fp32 rows (4 per lane), weight dinv[u] per edge, then the ApplyVertex
// GEMV (W staged in shared memory) fused into the row flush.
struct GcnF32FusedOp {
    static constexpr int kAccF = 4;
    struct Acc { float a[4]; };
    struct Val { float4 x; float w; };
    const float *X;
    int32_t f_in, f_out;
    const float *dinv;
    const float *W;  // global [f_in][f_out]
    const float *bias;
    int act;
    float *out;
    const float *Ws;  // shared copy (set by the engine)
    __device__ void setup(int) {}
    __device__ void set_smem(const float *p) { Ws = p; }
    __device__ __forceinline__ void zero(Acc &c) const { c.a[0] = c.a[1] = c.a[2] = c.a[3] = 0.0f; }
    __device__ __forceinline__ void begin_row(int32_t, int) {}
    __device__ __forceinline__ Val load(int32_t u, int lane) const {
        Val v;
        v.x = __ldg(reinterpret_cast<const float4 *>(X + (int64_t)u * f_in) + lane);
        v.w = __ldg(dinv + u);
        return v;
    }
    __device__ __forceinline__ void add(Acc &c, const Val &v, int32_t) const {
        c.a[0] = fmaf(v.w, v.x.x, c.a[0]);
        c.a[1] = fmaf(v.w, v.x.y, c.a[1]);
        c.a[2] = fmaf(v.w, v.x.z, c.a[2]);
        c.a[3] = fmaf(v.w, v.x.w, c.a[3]);
    }
    template <int G>
    __device__ __forceinline__ void finish_g(int32_t v, const Acc &c, const Group<G> &grp) const {
        const float s = dinv[v];
        float h[4] = {s * c.a[0], s * c.a[1], s * c.a[2], s * c.a[3]};
        // lane j computes outputs j, j+G, ...: out_j = sum_k h_k W[k][j]
        constexpr int kMaxOut = 64 / G > 0 ? (64 + G - 1) / G : 1;
        float o[kMaxOut];
#pragma unroll
        for (int t = 0; t < kMaxOut; ++t) o[t] = 0.0f;
        for (int k4 = 0; k4 < f_in / 4; ++k4) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                float hk = grp.shfl(h[i], k4);
                const float *wr = Ws + (k4 * 4 + i) * f_out;
#pragma unroll
                for (int t = 0; t < kMaxOut; ++t) {
                    int j = grp.lane + t * G;
                    if (j < f_out) o[t] = fmaf(hk, wr[j], o[t]);
                }
            }
        }
#pragma unroll
        for (int t = 0; t < kMaxOut; ++t) {
            int j = grp.lane + t * G;
            if (j < f_out) out[(int64_t)v * f_out + j] = act_fn(o[t] + (bias ? bias[j] : 0.0f), act);
        }
    }
    __device__ __forceinline__ void save(float *slot, const Acc &c, int lane) const {
        reinterpret_cast<float4 *>(slot)[lane] = make_float4(c.a[0], c.a[1], c.a[2], c.a[3]);
    }
    __device__ __forceinline__ void merge(Acc &c, const float *slot, int lane) const {
        float4 x = __ldcg(reinterpret_cast<const float4 *>(slot) + lane);
        c.a[0] += x.x; c.a[1] += x.y; c.a[2] += x.z; c.a[3] += x.w;
    }
};

// C3: GAT.  Lane = head (8 bf16 = head_dim 8 = 16 bytes of z).  Per edge:
// s = LeakyReLU(el[u,h] + er[v,h]) (additive form of a^T[z_u||z_v], A14);
// online softmax state (m, l, acc[8]) per head; flush ELU(acc / l).
struct GatOp {
    __device__ void set_smem(const float *) {}
    static constexpr int kAccF = 10;
    struct Acc { float m, l, a[8]; };
    struct Val { uint4 z; float el; };
    const __nv_bfloat16 *z;
    const float *el, *er;
    float slope;
    __nv_bfloat16 *out;
    float er_h;
    __device__ void setup(int) {}
    __device__ __forceinline__ void zero(Acc &c) const {
        c.m = -INFINITY;
        c.l = 0.0f;
#pragma unroll
        for (int i = 0; i < 8; ++i) c.a[i] = 0.0f;
    }
    __device__ __forceinline__ void begin_row(int32_t v, int lane) { er_h = __ldg(er + (int64_t)v * 8 + lane); }
    __device__ __forceinline__ Val load(int32_t u, int lane) const {
        Val v;
        v.z = ptx::ldg_nc_v4(z + (int64_t)u * 64 + lane * 8);
        v.el = __ldg(el + (int64_t)u * 8 + lane);
        return v;
    }
    __device__ __forceinline__ void add(Acc &c, const Val &v, int32_t) const {
        float s = v.el + er_h;
        s = s > 0.0f ? s : slope * s;
        float mn = fmaxf(c.m, s);
        float co = __expf(c.m - mn);  // 0 when c.m = -inf
        float cn = __expf(s - mn);
        c.l = fmaf(c.l, co, cn);
        const uint32_t q[4] = {v.z.x, v.z.y, v.z.z, v.z.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            float2 f = ptx::unpack_bf16x2(q[i]);
            c.a[2 * i] = fmaf(c.a[2 * i], co, cn * f.x);
            c.a[2 * i + 1] = fmaf(c.a[2 * i + 1], co, cn * f.y);
        }
        c.m = mn;
    }
    __device__ __forceinline__ void finish(int32_t v, const Acc &c, int lane) const {
        float inv = c.l > 0.0f ? 1.0f / c.l : 0.0f;
        float o[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float x = c.a[i] * inv;
            o[i] = x > 0.0f ? x : expm1f(x);
        }
        *reinterpret_cast<uint4 *>(out + (int64_t)v * 64 + lane * 8) = pack8(o);
    }
    __device__ __forceinline__ void save(float *slot, const Acc &c, int lane) const {
        float *p = slot + lane * 12;
        reinterpret_cast<float4 *>(p)[0] = make_float4(c.m, c.l, c.a[0], c.a[1]);
        reinterpret_cast<float4 *>(p)[1] = make_float4(c.a[2], c.a[3], c.a[4], c.a[5]);
        reinterpret_cast<float2 *>(p)[4] = make_float2(c.a[6], c.a[7]);
    }
    __device__ __forceinline__ void merge(Acc &c, const float *slot, int lane) const {
        const float *p = slot + lane * 12;
        float4 x = __ldcg(reinterpret_cast<const float4 *>(p));
        float4 y = __ldcg(reinterpret_cast<const float4 *>(p) + 1);
        float2 w = __ldcg(reinterpret_cast<const float2 *>(p) + 4);
        float pm = x.x, pl = x.y;
        float pa[8] = {x.z, x.w, y.x, y.y, y.z, y.w, w.x, w.y};
        float mn = fmaxf(c.m, pm);
        if (mn == -INFINITY) return;  // both empty
        float co = __expf(c.m - mn), cp = __expf(pm - mn);
        c.l = c.l * co + pl * cp;
#pragma unroll
        for (int i = 0; i < 8; ++i) c.a[i] = c.a[i] * co + pa[i] * cp;
        c.m = mn;
    }
};

// C4: per-edge-type sums of fp32 rows (4 floats per lane, 4 type slots).
struct TypedF32Op {
    __device__ void set_smem(const float *) {}
    static constexpr int kAccF = 16;
    struct Acc { float a[4][4]; };
    struct Val { float4 x; };
    const float *H;
    int32_t f;
    float *S;  // [n][4][f]
    __device__ void setup(int) {}
    __device__ __forceinline__ void zero(Acc &c) const {
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int i = 0; i < 4; ++i) c.a[t][i] = 0.0f;
    }
    __device__ __forceinline__ void begin_row(int32_t, int) {}
    __device__ __forceinline__ Val load(int32_t u, int lane) const {
        return Val{__ldg(reinterpret_cast<const float4 *>(H + (int64_t)u * f) + lane)};
    }
    __device__ __forceinline__ void add(Acc &c, const Val &v, int32_t t) const {
#pragma unroll
        for (int tt = 0; tt < 4; ++tt)
            if (t == tt) {
                c.a[tt][0] += v.x.x;
                c.a[tt][1] += v.x.y;
                c.a[tt][2] += v.x.z;
                c.a[tt][3] += v.x.w;
            }
    }
    __device__ __forceinline__ void finish(int32_t v, const Acc &c, int lane) const {
#pragma unroll
        for (int t = 0; t < 4; ++t)
            reinterpret_cast<float4 *>(S + ((int64_t)v * 4 + t) * f)[lane] =
                make_float4(c.a[t][0], c.a[t][1], c.a[t][2], c.a[t][3]);
    }
    __device__ __forceinline__ void save(float *slot, const Acc &c, int lane) const {
#pragma unroll
        for (int t = 0; t < 4; ++t)
            reinterpret_cast<float4 *>(slot + t * 128)[lane] = make_float4(c.a[t][0], c.a[t][1], c.a[t][2], c.a[t][3]);
    }
    __device__ __forceinline__ void merge(Acc &c, const float *slot, int lane) const {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            float4 x = __ldcg(reinterpret_cast<const float4 *>(slot + t * 128) + lane);
            c.a[t][0] += x.x; c.a[t][1] += x.y; c.a[t][2] += x.z; c.a[t][3] += x.w;
        }
    }
};

// Ops whose flush needs the whole group (the fused GEMV) implement finish_g.
template <typename Op, int G>
__device__ __forceinline__ auto do_finish(Op &op, int32_t v, const typename Op::Acc &c, const Group<G> &grp, int)
    -> decltype(op.template finish_g<G>(v, c, grp), void()) {
    op.template finish_g<G>(v, c, grp);
}
template <typename Op, int G>
__device__ __forceinline__ void do_finish(Op &op, int32_t v, const typename Op::Acc &c, const Group<G> &grp, long) {
    op.finish(v, c, grp.lane);
}

// Contribute the partial `acc` of split row r (edges [rb, re)) to `slot`; the
// last of its parts (atomic ticket on the task that holds r's end item)
// merges all parts in task order and writes the row.  Rare path: outlined.
template <int G, typename Op>
__device__ __noinline__ void contribute(Op &op, const typename Op::Acc &acc, const Group<G> &grp, AggWorkspace ws,
                                        int32_t slot_floats, int64_t T, int32_t r, int64_t rb, int64_t re,
                                        int64_t slot) {
    const int64_t k1 = (rb + r) / T, k2 = (re + r) / T;
    op.save(ws.partials + slot * slot_floats, acc, grp.lane);
    __threadfence();
    grp.sync();
    int old = 0;
    if (grp.lane == 0) old = atomicAdd(ws.counters + k2, 1);
    old = grp.shfl(old, 0);
    if (old == (int)(k2 - k1)) {
        __threadfence();
        typename Op::Acc m;
        op.zero(m);
        op.begin_row(r, grp.lane);
        op.merge(m, ws.partials + (2 * k1 + 1) * slot_floats, grp.lane);
        for (int64_t kk = k1 + 1; kk <= k2; ++kk) op.merge(m, ws.partials + (2 * kk) * slot_floats, grp.lane);
        do_finish(op, r, m, grp, 0);
    }
}

// ================================================================== engine ==
template <int G, int U, bool kTyped, typename Op>
__global__ void __launch_bounds__(kBlock, 2) k_segreduce(GraphView g, Op op, AggWorkspace ws, int32_t slot_floats,
                                                      const float *Wg, int32_t w_elems) {
    extern __shared__ float smem_w[];
    if (Wg) {  // stage the ApplyVertex weight (fused-GEMV ops)
        for (int i = threadIdx.x; i < w_elems; i += blockDim.x) smem_w[i] = Wg[i];
        __syncthreads();
    }
    op.set_smem(smem_w);
    const Group<G> grp;
    const int64_t k = (int64_t)blockIdx.x * (kBlock / G) + threadIdx.x / G;
    if (k >= g.ntasks) return;
    op.setup(grp.lane);

    const int64_t T = g.T;
    int32_t v = g.task_v[k];
    int64_t p = g.task_p[k];
    const int32_t v1 = g.task_v[k + 1];
    const int64_t p1 = g.task_p[k + 1];
    const int32_t v0 = v;
    int64_t row_beg = g.row_ptr[v];
    int64_t row_end = g.row_ptr[v + 1];
    const bool head = row_beg < p;  // first row began in an earlier task

    typename Op::Acc acc;
    op.zero(acc);
    op.begin_row(v, grp.lane);

    auto flush = [&]() {
        if (head && v == v0)
            contribute<G>(op, acc, grp, ws, slot_floats, T, v, row_beg, row_end, 2 * k);
        else
            do_finish(op, v, acc, grp, 0);
        ++v;
        row_beg = row_end;
        if (v < g.n) row_end = g.row_ptr[v + 1];
        op.zero(acc);
        if (v < g.n) op.begin_row(v, grp.lane);
    };

    for (int64_t q0 = p; q0 < p1; q0 += G) {
        const int cnt = (int)(p1 - q0 < (int64_t)G ? p1 - q0 : (int64_t)G);
        const int32_t cs = grp.lane < cnt ? __ldg(g.col_src + q0 + grp.lane) : 0;
        int32_t ct = 0;
        if (kTyped) ct = grp.lane < cnt ? __ldg(g.etype + q0 + grp.lane) : 0;
        for (int j0 = 0; j0 < cnt; j0 += U) {
            // issue U independent row gathers, then consume them row segment by
            // row segment (one copy of the flush code per batch)
            typename Op::Val vals[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int32_t src = grp.shfl(cs, (j0 + u) & (G - 1));
                if (j0 + u < cnt) vals[u] = op.load(src, grp.lane);
            }
            const int nb = cnt - j0 < U ? cnt - j0 : U;
            const int64_t qb = q0 + j0;
            int u0 = 0;
            while (true) {
                const int64_t lim64 = row_end - qb;
                const int lim = lim64 < (int64_t)nb ? (int)lim64 : nb;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    int32_t t = 0;
                    if (kTyped) t = grp.shfl(ct, (j0 + u) & (G - 1));
                    if (u >= u0 && u < lim) op.add(acc, vals[u], t);
                }
                if (lim >= nb) break;
                u0 = lim;
                do flush(); while (qb + u0 >= row_end);
            }
        }
    }
    while (v < v1) flush();
    if (v < g.n && p1 > row_beg) {  // tail: row v continues into the next task
        const int64_t slot = (head && v == v0) ? 2 * k : 2 * k + 1;
        contribute<G>(op, acc, grp, ws, slot_floats, T, v, row_beg, row_end, slot);
    }
}

template <int G, int U, bool kTyped, typename Op>
cudaError_t run(const GraphDev &g, const Op &op, AggWorkspace ws, int32_t slot_floats, cudaStream_t st,
                const float *Wg = nullptr, int32_t w_elems = 0) {
    if (g.ntasks == 0) return cudaSuccess;
    const int64_t groups_per_block = kBlock / G;
    const unsigned blocks = (unsigned)((g.ntasks + groups_per_block - 1) / groups_per_block);
    const size_t smem = Wg ? sizeof(float) * w_elems : 0;
    k_segreduce<G, U, kTyped, Op><<<blocks, kBlock, smem, st>>>(view(g), op, ws, slot_floats, Wg, w_elems);
    return cudaGetLastError();
}

}  // namespace

size_t agg_partial_floats(saga_model kind, int32_t width, int32_t heads) {
    switch (kind) {
        case SAGA_GCN: return (size_t)width;        // one fp32 per feature (f_out bf16 or f_in fp32)
        case SAGA_SAGE: return (size_t)width;
        case SAGA_GAT: return (size_t)heads * 12;   // (m, l, acc[8]) padded to 12
        case SAGA_GATED: return (size_t)4 * width;  // 4 type slots
    }
    return 0;
}

cudaError_t launch_agg_gcn_bf16(const GraphDev &g, const __nv_bfloat16 *Y, int32_t f, const float *bias, int act,
                                __nv_bfloat16 *out, AggWorkspace ws, cudaStream_t st) {
    SumBf16Op op{};
    op.X = Y; op.f = f; op.scale = g.dinv; op.bias = bias; op.act = act; op.out = out;
    switch (f) {
        case 256: return run<32, 8, false>(g, op, ws, f, st);
        case 128: return run<16, 8, false>(g, op, ws, f, st);
        case 64: return run<8, 8, false>(g, op, ws, f, st);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_agg_mean_bf16(const GraphDev &g, const __nv_bfloat16 *X, int32_t f, __nv_bfloat16 *M,
                                 AggWorkspace ws, cudaStream_t st) {
    SumBf16Op op{};
    op.X = X; op.f = f; op.scale = g.inv_deg; op.bias = nullptr; op.act = SAGA_ACT_NONE; op.out = M;
    switch (f) {
        case 256: return run<32, 8, false>(g, op, ws, f, st);
        case 128: return run<16, 8, false>(g, op, ws, f, st);
        case 64: return run<8, 8, false>(g, op, ws, f, st);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_gcn_f32_fused(const GraphDev &g, const float *X, int32_t f_in, const float *W, int32_t f_out,
                                 const float *bias, int act, float *out, AggWorkspace ws, cudaStream_t st) {
    GcnF32FusedOp op{};
    op.X = X; op.f_in = f_in; op.f_out = f_out; op.dinv = g.dinv; op.W = W; op.bias = bias; op.act = act;
    op.out = out;
    op.Ws = nullptr;  // set on device to the dynamic shared array
    const int32_t welems = f_in * f_out;
    switch (f_in) {
        case 128: return run<32, 4, false>(g, op, ws, f_in, st, W, welems);
        case 64: return run<16, 4, false>(g, op, ws, f_in, st, W, welems);
        case 32: return run<8, 4, false>(g, op, ws, f_in, st, W, welems);
        case 16: return run<4, 4, false>(g, op, ws, f_in, st, W, welems);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_gat_edge(const GraphDev &g, const __nv_bfloat16 *z, const float *el, const float *er,
                            float slope, __nv_bfloat16 *out, AggWorkspace ws, cudaStream_t st) {
    GatOp op{};
    op.z = z; op.el = el; op.er = er; op.slope = slope; op.out = out;
    return run<8, 8, false>(g, op, ws, 8 * 12, st);
}

cudaError_t launch_agg_typed_f32(const GraphDev &g, const float *H, int32_t f, float *S, AggWorkspace ws,
                                 cudaStream_t st) {
    TypedF32Op op{};
    op.H = H; op.f = f; op.S = S;
    if (f != 128) return cudaErrorInvalidValue;
    if (g.etype) return run<32, 8, true>(g, op, ws, 4 * f, st);
    return run<32, 8, false>(g, op, ws, 4 * f, st);
}

}  // namespace saga
