// aggregate.cu -- Scatter + ApplyEdge + Gather (S3, S4) and the vertex-side
// epilogues (S5) as one merge-path segment-reduce engine.
//
// Paper: the Gather stage reduces each vertex's in-edges (PAPER.md lines
// 343-355); fused with Scatter it is "the multiplication between the
// adjacency matrix and the embedding matrix" (line 354) -- the SpMM shape,
// which is HBM/L2-bound on B200 (~0 FLOP/byte).  Power-law in-degrees (lines
// 359-365) make per-vertex scheduling unbalanced, so work is cut by
// merge-path: the item sequence is, for every row v in order, its deg(v)
// edges followed by one row-end marker; task k owns items [kT, (k+1)T).
//
// One WARP owns one task, so every branch below is warp-uniform:
//  * G lanes cover one feature row (16 bytes per lane); the warp's S = 32/G
//    sub-groups take S different in-edges of the same row per step, and a
//    batch is U steps = U*S edges of ONE row (a batch never crosses a row
//    end, so the reduction needs no per-edge row test); the U*S 16-byte row
//    gathers of a batch are all issued before any is consumed;
//  * col_src (and etype) arrive in coalesced 32-edge chunks, one ahead;
//  * row_end and per-row epilogue data (dinv[v], GAT er[v,:]) come from
//    32-lane register windows refilled once per 32 rows;
//  * at a row end the S sub-group partials are combined with xor-shuffles
//    and sub-group 0 runs the fused epilogue and the coalesced store.
// Feature rows are read with plain ld.global.nc (L2 evict-normal): the hot
// (high out-degree) rows then stay in the 126 MB L2 -- an L1::no_allocate
// load is treated as evict-first by L2 and cost ~45% in a probe
// (scripts/gather_probe.cu).  bf16 rows are accumulated with sm_100's
// mixed-precision add (add.f32.bf16: one FHADD per element, no unpacking).
// Rows split across tasks (hubs, and rows straddling a task boundary) write
// fp32 partials; the last contributor (integer ticket) merges all partials in
// task order, so results are deterministic and no float atomics are used.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>
#include <cstdlib>

#include "internal.cuh"
#include "ptx.cuh"

namespace saga {
namespace {

constexpr int kBlock = 256;
constexpr int kWarpsPerBlock = kBlock / 32;
constexpr uint32_t kFull = 0xffffffffu;

struct GraphView {
    const int64_t *row_ptr;
    const int32_t *col_src;
    const int32_t *etype;
    const int32_t *task_v;
    const int64_t *task_p;
    int64_t T, ntasks;
    int32_t n;
    int32_t e;
};

GraphView view(const GraphDev &g) {
    return GraphView{g.row_ptr, g.col_src, g.etype, g.task_v, g.task_p, g.task_items, g.ntasks, g.n, (int32_t)g.e};
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
// Op interface (all const; per-row state is the float `rs` the engine fetches
// from its window: kWin values per row, lane gl % kWin's one):
//   Acc, Val; kWin; row_value(v, j)
//   zero(acc); load(u, gl); add(acc, val, rs, t); reduce_xor(acc, offset)
//   finish(v, acc, rs, gl, store)  [or finish_w: warp-wide epilogue]
//   save(slot, acc, gl); merge(acc, slot, gl)

// Sum of bf16 rows (8 per lane) -> act(scale[v] * acc + bias) in bf16.
// GCN (Y pre-scaled by dinv[u], scale = dinv[v]) and SAGE-mean (scale = 1/deg).
template <int kAct>
struct SumBf16Op {
    static constexpr int kWin = 1;
    __device__ static int win_col(int) { return 0; }
    struct Acc { float a[8]; };
    struct Val { uint4 x; };
    const __nv_bfloat16 *X;
    int32_t f;
    const float *scale;
    const float *bias;
    __nv_bfloat16 *out;
    __device__ __forceinline__ float row_value(int32_t v, int) const { return __ldg(scale + v); }
    __device__ __forceinline__ void zero(Acc &c) const {
#pragma unroll
        for (int i = 0; i < 8; ++i) c.a[i] = 0.0f;
    }
    // row u, lane gl: one IMAD.WIDE.U32 per address (row byte offsets < 2^32
    // is guaranteed by saga_layer's size checks)
    __device__ __forceinline__ Val load(int32_t u, int gl) const {
        const char *base = reinterpret_cast<const char *>(X) + gl * 16;
        return Val{__ldg(reinterpret_cast<const uint4 *>(base + (uint64_t)(uint32_t)u * (uint32_t)(f * 2)))};
    }
    int unpack;
    __device__ __forceinline__ void add(Acc &c, const Val &v, float, int32_t) const {
        if (unpack) {
            const uint32_t q[4] = {v.x.x, v.x.y, v.x.z, v.x.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                c.a[2 * i] += __uint_as_float(q[i] << 16);
                c.a[2 * i + 1] += __uint_as_float(q[i] & 0xffff0000u);
            }
            return;
        }
        ptx::add_bf16x2_f32(c.a[0], c.a[1], v.x.x);
        ptx::add_bf16x2_f32(c.a[2], c.a[3], v.x.y);
        ptx::add_bf16x2_f32(c.a[4], c.a[5], v.x.z);
        ptx::add_bf16x2_f32(c.a[6], c.a[7], v.x.w);
    }
    __device__ __forceinline__ void reduce_xor(Acc &c, int o) const {
#pragma unroll
        for (int i = 0; i < 8; ++i) c.a[i] += __shfl_xor_sync(kFull, c.a[i], o);
    }
    // epilogue in two 4-wide halves (keeps the flush's register peak low)
    __device__ __forceinline__ void finish(int32_t v, const Acc &c, float rs, int gl, bool store) const {
        uint32_t pk[4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
            if (bias) b = __ldg(reinterpret_cast<const float4 *>(bias + gl * 8) + h);
            pk[2 * h] = ptx::pack_bf16x2(act_fn(fmaf(rs, c.a[4 * h + 0], b.x), kAct),
                                         act_fn(fmaf(rs, c.a[4 * h + 1], b.y), kAct));
            pk[2 * h + 1] = ptx::pack_bf16x2(act_fn(fmaf(rs, c.a[4 * h + 2], b.z), kAct),
                                             act_fn(fmaf(rs, c.a[4 * h + 3], b.w), kAct));
        }
        if (store) *reinterpret_cast<uint4 *>(out + (int64_t)v * f + gl * 8) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
    __device__ __forceinline__ void save(float *slot, const Acc &c, int gl) const {
        float4 *p = reinterpret_cast<float4 *>(slot + gl * 8);
        p[0] = make_float4(c.a[0], c.a[1], c.a[2], c.a[3]);
        p[1] = make_float4(c.a[4], c.a[5], c.a[6], c.a[7]);
    }
    __device__ __forceinline__ void merge(Acc &c, const float *slot, int gl) const {
        const float4 *p = reinterpret_cast<const float4 *>(slot + gl * 8);
        const float4 x = __ldcg(p), y = __ldcg(p + 1);
        c.a[0] += x.x; c.a[1] += x.y; c.a[2] += x.z; c.a[3] += x.w;
        c.a[4] += y.x; c.a[5] += y.y; c.a[6] += y.z; c.a[7] += y.w;
    }
};

// C1: fp32 rows (4 per lane), weight dinv[u] per edge, then the ApplyVertex
// GEMV (W staged in shared memory) fused into the row flush, spread over all
// 32 lanes (lane L computes outputs L and L + 32).
struct GcnF32FusedOp {
    static constexpr int kWin = 1;
    struct Acc { float a[4]; };
    struct Val { float4 x; float w; };
    const float *X;
    int32_t f_in, f_out;
    const float *dinv;
    const float *bias;
    int act;
    float *out;
    __device__ __forceinline__ float row_value(int32_t v, int) const { return __ldg(dinv + v); }
    __device__ __forceinline__ void zero(Acc &c) const { c.a[0] = c.a[1] = c.a[2] = c.a[3] = 0.0f; }
    __device__ __forceinline__ Val load(int32_t u, int gl) const {
        Val v;
        v.x = __ldg(reinterpret_cast<const float4 *>(X + (int64_t)u * f_in) + gl);
        v.w = __ldg(dinv + u);
        return v;
    }
    __device__ __forceinline__ void add(Acc &c, const Val &v, float, int32_t) const {
        c.a[0] = fmaf(v.w, v.x.x, c.a[0]);
        c.a[1] = fmaf(v.w, v.x.y, c.a[1]);
        c.a[2] = fmaf(v.w, v.x.z, c.a[2]);
        c.a[3] = fmaf(v.w, v.x.w, c.a[3]);
    }
    __device__ __forceinline__ void reduce_xor(Acc &c, int o) const {
#pragma unroll
        for (int i = 0; i < 4; ++i) c.a[i] += __shfl_xor_sync(kFull, c.a[i], o);
    }
    // h = rs * acc lives in lanes 0..f_in/4-1 (4 values each, sub-group 0)
    __device__ __forceinline__ void finish_w(int32_t v, const Acc &c, float rs, const float *Ws, int lane) const {
        const float h[4] = {rs * c.a[0], rs * c.a[1], rs * c.a[2], rs * c.a[3]};
        float o0 = 0.0f, o1 = 0.0f;
        const int j0 = lane, j1 = lane + 32;
        for (int k4 = 0; k4 < f_in / 4; ++k4) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float hk = __shfl_sync(kFull, h[i], k4);
                const float *wr = Ws + (k4 * 4 + i) * f_out;
                if (j0 < f_out) o0 = fmaf(hk, wr[j0], o0);
                if (j1 < f_out) o1 = fmaf(hk, wr[j1], o1);
            }
        }
        if (j0 < f_out) out[(int64_t)v * f_out + j0] = act_fn(o0 + (bias ? __ldg(bias + j0) : 0.0f), act);
        if (j1 < f_out) out[(int64_t)v * f_out + j1] = act_fn(o1 + (bias ? __ldg(bias + j1) : 0.0f), act);
    }
    __device__ __forceinline__ void save(float *slot, const Acc &c, int gl) const {
        reinterpret_cast<float4 *>(slot)[gl] = make_float4(c.a[0], c.a[1], c.a[2], c.a[3]);
    }
    __device__ __forceinline__ void merge(Acc &c, const float *slot, int gl) const {
        const float4 x = __ldcg(reinterpret_cast<const float4 *>(slot) + gl);
        c.a[0] += x.x; c.a[1] += x.y; c.a[2] += x.z; c.a[3] += x.w;
    }
};

// C3: GAT.  Lane gl = head (8 bf16 = head_dim 8 = 16 bytes of z).  Per edge:
// s = LeakyReLU(el[u,h] + er[v,h]) (additive form of a^T[z_u||z_v], A14);
// online softmax state (m, l, acc[8]) per head; flush ELU(acc / l).
// Row value: er[v, gl] (kWin = 8 heads).
struct GatOp {
    static constexpr int kWin = 8;
    struct Acc { float m, l, a[8]; };
    struct Val { uint4 z; float el; };
    const __nv_bfloat16 *z;
    const float *el, *er;
    float slope;
    __nv_bfloat16 *out;
    __device__ __forceinline__ float row_value(int32_t v, int j) const { return __ldg(er + (int64_t)v * 8 + j); }
    __device__ __forceinline__ void zero(Acc &c) const {
        c.m = -INFINITY;
        c.l = 0.0f;
#pragma unroll
        for (int i = 0; i < 8; ++i) c.a[i] = 0.0f;
    }
    __device__ __forceinline__ Val load(int32_t u, int gl) const {
        Val v;
        v.z = __ldg(reinterpret_cast<const uint4 *>(z + (int64_t)u * 64) + gl);
        v.el = __ldg(el + (int64_t)u * 8 + gl);
        return v;
    }
    __device__ __forceinline__ void add(Acc &c, const Val &v, float er_h, int32_t) const {
        float s = v.el + er_h;
        s = s > 0.0f ? s : slope * s;
        const float mn = fmaxf(c.m, s);
        const float co = __expf(c.m - mn);  // 0 when c.m = -inf
        const float cn = __expf(s - mn);
        c.l = fmaf(c.l, co, cn);
        const uint32_t q[4] = {v.z.x, v.z.y, v.z.z, v.z.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = ptx::unpack_bf16x2(q[i]);
            c.a[2 * i] = fmaf(c.a[2 * i], co, cn * f.x);
            c.a[2 * i + 1] = fmaf(c.a[2 * i + 1], co, cn * f.y);
        }
        c.m = mn;
    }
    // merge another partial (pm, pl, pa) into c (flash-decoding merge)
    __device__ __forceinline__ static void merge_parts(Acc &c, float pm, float pl, const float (&pa)[8]) {
        const float mn = fmaxf(c.m, pm);
        if (mn == -INFINITY) return;  // both empty
        const float co = __expf(c.m - mn), cp = __expf(pm - mn);
        c.l = c.l * co + pl * cp;
#pragma unroll
        for (int i = 0; i < 8; ++i) c.a[i] = c.a[i] * co + pa[i] * cp;
        c.m = mn;
    }
    __device__ __forceinline__ void reduce_xor(Acc &c, int o) const {
        const float pm = __shfl_xor_sync(kFull, c.m, o), pl = __shfl_xor_sync(kFull, c.l, o);
        float pa[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) pa[i] = __shfl_xor_sync(kFull, c.a[i], o);
        merge_parts(c, pm, pl, pa);
    }
    __device__ __forceinline__ void finish(int32_t v, const Acc &c, float, int gl, bool store) const {
        const float inv = c.l > 0.0f ? 1.0f / c.l : 0.0f;
        float o[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float x = c.a[i] * inv;
            o[i] = x > 0.0f ? x : expm1f(x);
        }
        if (store) *reinterpret_cast<uint4 *>(out + (int64_t)v * 64 + gl * 8) = pack8(o);
    }
    __device__ __forceinline__ void save(float *slot, const Acc &c, int gl) const {
        float *p = slot + gl * 12;
        reinterpret_cast<float4 *>(p)[0] = make_float4(c.m, c.l, c.a[0], c.a[1]);
        reinterpret_cast<float4 *>(p)[1] = make_float4(c.a[2], c.a[3], c.a[4], c.a[5]);
        reinterpret_cast<float2 *>(p)[4] = make_float2(c.a[6], c.a[7]);
    }
    __device__ __forceinline__ void merge(Acc &c, const float *slot, int gl) const {
        const float *p = slot + gl * 12;
        const float4 x = __ldcg(reinterpret_cast<const float4 *>(p));
        const float4 y = __ldcg(reinterpret_cast<const float4 *>(p) + 1);
        const float2 w = __ldcg(reinterpret_cast<const float2 *>(p) + 4);
        const float pa[8] = {x.z, x.w, y.x, y.y, y.z, y.w, w.x, w.y};
        merge_parts(c, x.x, x.y, pa);
    }
};

// C3 on the dense engine: all 32 lanes work on ONE edge; lane L owns head
// h = L / 4 and output columns 2L, 2L+1 (a 4-byte slice of the 128-byte z
// row).  Per edge s = LeakyReLU(el[u,h] + er[v,h]) (A14) and a single-exp
// online-softmax update: with d = s - m, e = exp(-|d|); if d > 0 the state is
// rescaled by e and the new term weighs 1, else the new term weighs e.
struct GatDenseOp {
    static constexpr int kWin = 8;
    __device__ static int win_col(int lane) { return lane >> 2; }
    struct Acc { float m, l, a0, a1; };
    struct Val { uint32_t z2; float el; };
    const __nv_bfloat16 *z;
    const float *el, *er;
    float slope;
    __nv_bfloat16 *out;
    __device__ __forceinline__ float row_value(int32_t v, int j) const { return __ldg(er + (int64_t)v * 8 + j); }
    __device__ __forceinline__ void zero(Acc &c) const { c.m = -INFINITY; c.l = 0.f; c.a0 = 0.f; c.a1 = 0.f; }
    __device__ __forceinline__ Val load(int32_t u, int lane) const {
        Val v;
        v.z2 = __ldg(reinterpret_cast<const uint32_t *>(z + (int64_t)u * 64) + lane);
        v.el = __ldg(el + (int64_t)u * 8 + (lane >> 2));
        return v;
    }
    __device__ __forceinline__ void add(Acc &c, const Val &v, float er_h, int32_t) const {
        float s = v.el + er_h;
        s = s > 0.0f ? s : slope * s;
        const float d = s - c.m;                 // +inf for the first term
        const float e = __expf(-fabsf(d));       // 0 for the first term
        const bool up = d > 0.0f;
        const float co = up ? e : 1.0f, cn = up ? 1.0f : e;
        const float2 f = ptx::unpack_bf16x2(v.z2);
        c.l = fmaf(c.l, co, cn);
        c.a0 = fmaf(c.a0, co, cn * f.x);
        c.a1 = fmaf(c.a1, co, cn * f.y);
        c.m = up ? s : c.m;
    }
    __device__ __forceinline__ void finish(int32_t v, const Acc &c, float, int lane, bool store) const {
        const float inv = c.l > 0.0f ? 1.0f / c.l : 0.0f;
        float x0 = c.a0 * inv, x1 = c.a1 * inv;
        x0 = x0 > 0.0f ? x0 : expm1f(x0);
        x1 = x1 > 0.0f ? x1 : expm1f(x1);
        if (store) reinterpret_cast<uint32_t *>(out + (int64_t)v * 64)[lane] = ptx::pack_bf16x2(x0, x1);
    }
    __device__ __forceinline__ void save(float *slot, const Acc &c, int lane) const {
        reinterpret_cast<float4 *>(slot)[lane] = make_float4(c.m, c.l, c.a0, c.a1);
    }
    __device__ __forceinline__ void merge(Acc &c, const float *slot, int lane) const {
        const float4 x = __ldcg(reinterpret_cast<const float4 *>(slot) + lane);
        const float mn = fmaxf(c.m, x.x);
        if (mn == -INFINITY) return;
        const float co = __expf(c.m - mn), cp = __expf(x.x - mn);
        c.l = c.l * co + x.y * cp;
        c.a0 = c.a0 * co + x.z * cp;
        c.a1 = c.a1 * co + x.w * cp;
        c.m = mn;
    }
};

// C4: per-edge-type sums of fp32 rows (4 floats per lane, 4 type slots).
struct TypedF32Op {
    static constexpr int kWin = 0;
    __device__ static int win_col(int) { return 0; }
    struct Acc { float a[4][4]; };
    struct Val { float4 x; };
    const float *H;
    int32_t f;
    float *S;  // [n][4][f]
    __device__ __forceinline__ float row_value(int32_t, int) const { return 0.0f; }
    __device__ __forceinline__ void zero(Acc &c) const {
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int i = 0; i < 4; ++i) c.a[t][i] = 0.0f;
    }
    __device__ __forceinline__ Val load(int32_t u, int gl) const {
        const char *base = reinterpret_cast<const char *>(H) + gl * 16;
        return Val{__ldg(reinterpret_cast<const float4 *>(base + (uint64_t)(uint32_t)u * (uint32_t)(f * 4)))};
    }
    __device__ __forceinline__ void add(Acc &c, const Val &v, float, int32_t t) const {
#pragma unroll
        for (int tt = 0; tt < 4; ++tt)
            if (t == tt) {
                c.a[tt][0] += v.x.x;
                c.a[tt][1] += v.x.y;
                c.a[tt][2] += v.x.z;
                c.a[tt][3] += v.x.w;
            }
    }
    __device__ __forceinline__ void reduce_xor(Acc &c, int o) const {
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int i = 0; i < 4; ++i) c.a[t][i] += __shfl_xor_sync(kFull, c.a[t][i], o);
    }
    __device__ __forceinline__ void finish(int32_t v, const Acc &c, float, int gl, bool store) const {
        if (!store) return;
#pragma unroll
        for (int t = 0; t < 4; ++t)
            reinterpret_cast<float4 *>(S + ((int64_t)v * 4 + t) * f)[gl] =
                make_float4(c.a[t][0], c.a[t][1], c.a[t][2], c.a[t][3]);
    }
    __device__ __forceinline__ void save(float *slot, const Acc &c, int gl) const {
#pragma unroll
        for (int t = 0; t < 4; ++t)
            reinterpret_cast<float4 *>(slot + t * 128)[gl] = make_float4(c.a[t][0], c.a[t][1], c.a[t][2], c.a[t][3]);
    }
    __device__ __forceinline__ void merge(Acc &c, const float *slot, int gl) const {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const float4 x = __ldcg(reinterpret_cast<const float4 *>(slot + t * 128) + gl);
            c.a[t][0] += x.x; c.a[t][1] += x.y; c.a[t][2] += x.z; c.a[t][3] += x.w;
        }
    }
};

// Ops whose epilogue needs the whole warp (the fused GEMV) implement finish_w.
template <typename Op>
__device__ __forceinline__ auto do_finish(const Op &op, int32_t v, const typename Op::Acc &c, float rs, int gl,
                                          int lane, bool store, const float *Ws, int)
    -> decltype(op.finish_w(v, c, rs, Ws, lane), void()) {
    op.finish_w(v, c, rs, Ws, lane);
}
template <typename Op>
__device__ __forceinline__ void do_finish(const Op &op, int32_t v, const typename Op::Acc &c, float rs, int gl, int,
                                          bool store, const float *, long) {
    op.finish(v, c, rs, gl, store);
}

template <typename Op>
__device__ __forceinline__ float row_rs(const Op &op, int32_t v, int gl) {
    return Op::kWin ? op.row_value(v, Op::kWin == 1 ? 0 : gl % (Op::kWin ? Op::kWin : 1)) : 0.0f;
}
// (GatDenseOp's epilogue does not use the row value, so row_rs's column
// choice is irrelevant for it.)

// Split rows (hubs, rows straddling a task boundary): every task holding part
// of row r saves its fp32 partial (combined over sub-groups) to its slot, then
// takes an integer ticket on the task k2 that holds r's end item; the last
// arrival merges all parts in task order and runs the epilogue.  The ticket is
// taken after the task's main loop (never inside it), so the hot loop carries
// no call.
template <typename Op>
__device__ __forceinline__ void save_partial(const Op &op, const typename Op::Acc &acc, AggWorkspace ws,
                                             int32_t slot_floats, int64_t slot, int gl, int sub) {
    if (sub == 0) op.save(ws.partials + slot * slot_floats, acc, gl);
}
template <typename Op>
__device__ __noinline__ void ticket_merge(const Op &op, AggWorkspace ws, int32_t slot_floats, int64_t T, int32_t r,
                                          int64_t rb, int64_t re, int gl, int sub, const float *Ws) {
    const int lane = threadIdx.x & 31;
    const int64_t k1 = (rb + r) / T, k2 = (re + r) / T;
    __threadfence();
    __syncwarp();
    int old = 0;
    if (lane == 0) old = atomicAdd(ws.counters + k2, 1);
    old = __shfl_sync(kFull, old, 0);
    if (old == (int)(k2 - k1)) {
        __threadfence();
        typename Op::Acc m;
        op.zero(m);
        op.merge(m, ws.partials + (2 * k1 + 1) * slot_floats, gl);
        for (int64_t kk = k1 + 1; kk <= k2; ++kk) op.merge(m, ws.partials + (2 * kk) * slot_floats, gl);
        do_finish(op, r, m, row_rs(op, r, gl), gl, lane, sub == 0, Ws, 0);
    }
}

// ================================================================== engine ==
template <int G, int U, int kMinB, bool kTyped, typename Op>
__global__ void __launch_bounds__(kBlock, kMinB) k_segreduce(const GraphView g, const Op op, const AggWorkspace ws,
                                                          const int32_t slot_floats, const float *Wg,
                                                          const int32_t w_elems) {
    constexpr int S = 32 / G;  // sub-groups (edges per step)
    constexpr int B = U * S;   // edges per batch
    static_assert(B <= 32, "a batch must fit in one col_src chunk");
    constexpr int kWin = Op::kWin;
    constexpr int kWinD = kWin ? kWin : 1;
    constexpr int kWinRows = 32 / kWinD;

    extern __shared__ float smem_w[];
    if (Wg) {  // stage the ApplyVertex weight (fused-GEMV ops)
        for (int i = threadIdx.x; i < w_elems; i += blockDim.x) smem_w[i] = Wg[i];
        __syncthreads();
    }
    const int lane = threadIdx.x & 31;
    const int sub = lane / G, gl = lane & (G - 1);
    const int64_t k = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    if (k >= g.ntasks) return;

    const int64_t T = g.T;
    const int32_t n = g.n;
    int32_t v = g.task_v[k];
    const int32_t p = (int32_t)g.task_p[k];
    const int32_t v1 = g.task_v[k + 1];
    const int32_t p1 = (int32_t)g.task_p[k + 1];
    const int32_t v0 = v;
    int32_t row_beg = (int32_t)g.row_ptr[v];
    const bool head = row_beg < p;  // first row began in an earlier task
    const int32_t head_beg = row_beg;
    int32_t head_end = -1;          // set when the head row's partial is saved

    // row windows: lane i holds row_end(wr + i); lane i holds value i % kWin
    // of row wv + i / kWin
    auto load_re = [&](int32_t wbase) -> int32_t {
        const int32_t r = wbase + lane;
        return r < n ? (int32_t)__ldg(g.row_ptr + r + 1) : g.e;
    };
    auto load_rv = [&](int32_t wbase) -> float {
        if (!kWin) return 0.0f;
        const int32_t r = wbase + lane / kWinD;
        return r < n ? op.row_value(r, lane % kWinD) : 0.0f;
    };
    int32_t wr = v, wv = v;
    int32_t w_re = load_re(wr);
    float w_rv = load_rv(wv);
    int32_t row_end = __shfl_sync(kFull, w_re, 0);
    float rs = kWin ? __shfl_sync(kFull, w_rv, kWin == 1 ? 0 : gl % kWinD) : 0.0f;

    typename Op::Acc acc;
    op.zero(acc);

    auto flush = [&]() {
#pragma unroll
        for (int o = G; o < 32; o <<= 1) op.reduce_xor(acc, o);
        if (head && v == v0) {
            save_partial(op, acc, ws, slot_floats, 2 * k, gl, sub);
            head_end = row_end;
        } else {
            do_finish(op, v, acc, rs, gl, lane, sub == 0, smem_w, 0);
        }
        ++v;
        row_beg = row_end;
        if (v - wr == 32) {
            wr += 32;
            w_re = load_re(wr);
        }
        row_end = __shfl_sync(kFull, w_re, v - wr);
        if (kWin) {
            if (v - wv == kWinRows) {
                wv += kWinRows;
                w_rv = load_rv(wv);
            }
            rs = __shfl_sync(kFull, w_rv, (v - wv) * kWinD + (kWin == 1 ? 0 : gl % kWinD));
        }
        op.zero(acc);
    };

    // col_src / etype in 32-edge chunks, one chunk ahead
    auto load_cs = [&](int32_t base) -> int32_t {
        const int32_t q = base + lane;
        return q < p1 ? __ldcs(g.col_src + q) : 0;
    };
    auto load_ct = [&](int32_t base) -> int32_t {
        const int32_t q = base + lane;
        return (kTyped && q < p1) ? __ldcs(g.etype + q) : 0;
    };
    int32_t cb = p;
    int32_t cs_a = load_cs(cb), cs_b = load_cs(cb + 32);
    int32_t ct_a = load_ct(cb), ct_b = load_ct(cb + 32);

    int32_t q = p;
    while (true) {
        while (v < v1 && row_end <= q) flush();  // rows whose edges are all consumed
        if (q >= p1) break;
        const int32_t lim = row_end < p1 ? row_end : p1;
        const int c = lim - q < B ? (int)(lim - q) : B;
        if (q - cb >= 32) {
            cb += 32;
            cs_a = cs_b;
            ct_a = ct_b;
            cs_b = load_cs(cb + 32);
            ct_b = load_ct(cb + 32);
        }
        const int base = q - cb;
        typename Op::Val val[U];
        int32_t ty[U];
#pragma unroll
        for (int t = 0; t < U; ++t) {
            const int e = t * S + sub;
            const int idx = base + e;
            const int32_t sa = __shfl_sync(kFull, cs_a, idx & 31);
            const int32_t sb = __shfl_sync(kFull, cs_b, idx & 31);
            if (kTyped) {
                const int32_t ta = __shfl_sync(kFull, ct_a, idx & 31);
                const int32_t tb = __shfl_sync(kFull, ct_b, idx & 31);
                ty[t] = idx < 32 ? ta : tb;
            } else {
                ty[t] = 0;
            }
            if (e < c) val[t] = op.load(idx < 32 ? sa : sb, gl);
        }
#pragma unroll
        for (int t = 0; t < U; ++t)
            if (t * S + sub < c) op.add(acc, val[t], rs, ty[t]);
        q += c;
    }
    if (v < n && p1 > row_beg) {  // tail: row v continues into the next task
#pragma unroll
        for (int o = G; o < 32; o <<= 1) op.reduce_xor(acc, o);
        const int64_t slot = (head && v == v0) ? 2 * k : 2 * k + 1;
        save_partial(op, acc, ws, slot_floats, slot, gl, sub);
        ticket_merge(op, ws, slot_floats, T, v, row_beg, row_end, gl, sub, smem_w);
    }
    if (head_end >= 0 && !(v == v0))  // head row ended inside this task
        ticket_merge(op, ws, slot_floats, T, v0, head_beg, head_end, gl, sub, smem_w);
}

// Dense variant for full-warp rows (G = 32: one edge per step): batches are
// U CONSECUTIVE edges of the task regardless of row ends, so every batch
// keeps U row gathers in flight and the adds are unpredicated.  A batch in
// which a row ends takes the slow path: its U rows are parked in a per-warp
// shared-memory slot (each lane re-reads only what it wrote) and reduced edge
// by edge with a row-end test after each.  Everything the fast path does not
// touch (row windows, head bookkeeping) lives in a per-warp shared record, so
// the registers go to in-flight rows: U = 8 fits 64 registers without spills
// (32 warps per SM, 256 rows of 512 B in flight per SM).
template <int U, typename Val, int kWinD>
struct DenseWarp {
    Val park[U][32];
    int32_t re[32];        // row_end of rows wr .. wr+31
    float rv[32 * kWinD];  // per-row values of the same rows (kWinD per row)
    int32_t wr, v0, row_beg, head_beg, head_end, head;
};

template <int U, int kMinB, bool kTyped, typename Op>
__global__ void __launch_bounds__(kBlock, kMinB) k_segreduce_dense(const GraphView g, const Op op,
                                                                const AggWorkspace ws, const int32_t slot_floats,
                                                                const int dbg) {
    constexpr int kWin = Op::kWin;
    constexpr int kWinD = kWin ? kWin : 1;
    static_assert(32 % U == 0, "U must divide the 32-edge chunk");
    using DW = DenseWarp<U, typename Op::Val, kWinD>;
    __shared__ DW warps[kWarpsPerBlock];
    DW &W = warps[threadIdx.x >> 5];
    volatile DW &VW = W;
    const int lane = threadIdx.x & 31;
    const int64_t k = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    if (k >= g.ntasks) return;

    int32_t v = g.task_v[k];
    const int32_t p = (int32_t)g.task_p[k];
    const int32_t v1 = g.task_v[k + 1];
    const int32_t p1 = (int32_t)g.task_p[k + 1];

    auto fill_window = [&](int32_t wbase) {
        const int32_t r = wbase + lane;
        const bool in = r < g.n;
        VW.re[lane] = in ? (int32_t)__ldg(g.row_ptr + r + 1) : g.e;
        if (kWin) {
#pragma unroll
            for (int j = 0; j < kWinD; ++j) {  // value (i % kWinD) of row wbase + i / kWinD
                const int i = j * 32 + lane;
                const int32_t rr = wbase + i / kWinD;
                VW.rv[i] = rr < g.n ? op.row_value(rr, i % kWinD) : 0.0f;
            }
        }
        if (lane == 0) VW.wr = wbase;
        __syncwarp();
    };
    if (lane == 0) {
        const int32_t rb = (int32_t)g.row_ptr[v];
        VW.v0 = v;
        VW.row_beg = rb;
        VW.head_beg = rb;
        VW.head_end = -1;
        VW.head = rb < p;
    }
    fill_window(v);
    int32_t row_end = VW.re[0];
    // this lane's per-row value (e.g. GAT er[v, head]): column Op::win_col(lane)
    float rs = kWin ? VW.rv[Op::win_col(lane)] : 0.0f;

    typename Op::Acc acc;
    op.zero(acc);

    // finish row v (or save its partial if it is the head row), advance to v+1
    auto flush = [&]() {
        const int32_t wr = VW.wr;
        if (VW.head && v == VW.v0) {
            save_partial(op, acc, ws, slot_floats, 2 * k, lane, 0);
            if (lane == 0) VW.head_end = row_end;
        } else {
            op.finish(v, acc, rs, lane, !(dbg & 1));
        }
        ++v;
        __syncwarp();
        if (lane == 0) VW.row_beg = row_end;
        if (v - wr == 32) fill_window(wr + 32);
        row_end = VW.re[v - VW.wr];
        if (kWin) rs = VW.rv[(v - VW.wr) * kWinD + Op::win_col(lane)];
        op.zero(acc);
    };

    auto load_cs = [&](int32_t base) -> int32_t {
        const int32_t q = base + lane;
        return q < p1 ? __ldcs(g.col_src + q) : 0;
    };
    auto load_ct = [&](int32_t base) -> int32_t {
        const int32_t q = base + lane;
        return (kTyped && q < p1) ? __ldcs(g.etype + q) : 0;
    };
    int32_t cb = p;
    int32_t cs_a = load_cs(cb), cs_b = load_cs(cb + 32);
    int32_t ct_a = load_ct(cb), ct_b = load_ct(cb + 32);
    // keeps q - cb < 32; batches start at p + multiple of U and U | 32, so a
    // batch never straddles a chunk
    auto slide = [&](int32_t q) {
        if (q - cb >= 32) {
            cb += 32;
            cs_a = cs_b;
            ct_a = ct_b;
            cs_b = load_cs(cb + 32);
            ct_b = load_ct(cb + 32);
        }
    };

    while (v < v1 && row_end <= p) flush();  // rows that end before the first edge
    int32_t q = p;
    for (; q + U <= p1; q += U) {
        slide(q);
        const int base = q - cb;
        typename Op::Val val[U];
#pragma unroll
        for (int u = 0; u < U; ++u) val[u] = op.load(__shfl_sync(kFull, cs_a, base + u), lane);
        if ((dbg & 2) || row_end > q + U) {
            // fast path: no row ends inside the batch
#pragma unroll
            for (int u = 0; u < U; ++u) op.add(acc, val[u], rs, kTyped ? __shfl_sync(kFull, ct_a, base + u) : 0);
        } else {
            // slow path: park the batch, reduce edge by edge
#pragma unroll
            for (int u = 0; u < U; ++u) W.park[u][lane] = val[u];
#pragma unroll 1
            for (int u = 0; u < U; ++u) {
                const int32_t t = kTyped ? __shfl_sync(kFull, ct_a, base + u) : 0;
                const typename Op::Val x = W.park[u][lane];
                op.add(acc, x, rs, t);
                while (v < v1 && row_end == q + u + 1) flush();
            }
        }
    }
    for (; q < p1; ++q) {  // remainder, one edge at a time
        slide(q);
        const int idx = q - cb;
        const int32_t t = kTyped ? __shfl_sync(kFull, ct_a, idx) : 0;
        op.add(acc, op.load(__shfl_sync(kFull, cs_a, idx), lane), rs, t);
        while (v < v1 && row_end == q + 1) flush();
    }
    if (dbg & 2) return;
    while (v < v1) flush();
    const int32_t v0 = VW.v0, row_beg = VW.row_beg;
    const bool head = VW.head;
    if (v < g.n && p1 > row_beg) {  // tail: row v continues into the next task
        const int64_t sl = (head && v == v0) ? 2 * k : 2 * k + 1;
        save_partial(op, acc, ws, slot_floats, sl, lane, 0);
        ticket_merge(op, ws, slot_floats, g.T, v, row_beg, row_end, lane, 0, nullptr);
    }
    const int32_t head_end = VW.head_end;
    if (head_end >= 0 && v != v0)  // the head row ended inside this task
        ticket_merge(op, ws, slot_floats, g.T, v0, VW.head_beg, head_end, lane, 0, nullptr);
}

int agg_dbg() {
    static int v = [] {
        const char *s = getenv("SAGA_AGG_DBG");
        return s ? atoi(s) : 0;
    }();
    return v;
}
template <int U, bool kTyped, int kMinB, typename Op>
cudaError_t run_dense(const GraphDev &g, const Op &op, AggWorkspace ws, int32_t slot_floats, cudaStream_t st) {
    if (g.ntasks == 0) return cudaSuccess;
    const unsigned blocks = (unsigned)((g.ntasks + kWarpsPerBlock - 1) / kWarpsPerBlock);
    k_segreduce_dense<U, kMinB, kTyped, Op><<<blocks, kBlock, 0, st>>>(view(g), op, ws, slot_floats, agg_dbg());
    return cudaGetLastError();
}

template <int G, int U, bool kTyped, int kMinB, typename Op>
cudaError_t run(const GraphDev &g, const Op &op, AggWorkspace ws, int32_t slot_floats, cudaStream_t st,
                const float *Wg = nullptr, int32_t w_elems = 0) {
    if (g.ntasks == 0) return cudaSuccess;
    const unsigned blocks = (unsigned)((g.ntasks + kWarpsPerBlock - 1) / kWarpsPerBlock);
    const size_t smem = Wg ? sizeof(float) * w_elems : 0;
    k_segreduce<G, U, kMinB, kTyped, Op><<<blocks, kBlock, smem, st>>>(view(g), op, ws, slot_floats, Wg, w_elems);
    return cudaGetLastError();
}

// Development knob: SAGA_AGG_VARIANT selects the (U, blocks/SM) instance of
// the G = 32 bf16 sum kernel, for measuring the register / in-flight trade-off.
int agg_variant() {
    static int v = [] {
        const char *s = getenv("SAGA_AGG_VARIANT");
        return s ? atoi(s) : 0;
    }();
    return v;
}

}  // namespace

size_t agg_partial_floats(saga_model kind, int32_t width, int32_t heads) {
    switch (kind) {
        case SAGA_GCN: return (size_t)width;        // one fp32 per feature (f_out bf16 or f_in fp32)
        case SAGA_SAGE: return (size_t)width;
        case SAGA_GAT: return (size_t)(heads * 12 > 128 ? heads * 12 : 128);  // 32 lanes x (m, l, a0, a1)
        case SAGA_GATED: return (size_t)4 * width;  // 4 type slots
    }
    return 0;
}

template <int kAct>
cudaError_t agg_sum_bf16(const GraphDev &g, const __nv_bfloat16 *X, int32_t f, const float *scale,
                         const float *bias, __nv_bfloat16 *out, AggWorkspace ws, cudaStream_t st) {
    SumBf16Op<kAct> op{};
    op.X = X; op.f = f; op.scale = scale; op.bias = bias; op.out = out; op.unpack = (agg_dbg() & 4) != 0;
    switch (f) {
        case 256:
            switch (agg_variant()) {
                case 1: return run_dense<8, false, 3>(g, op, ws, f, st);
                case 2: return run_dense<4, false, 4>(g, op, ws, f, st);
                case 3: return run_dense<8, false, 2>(g, op, ws, f, st);
            }
            return run_dense<8, false, 4>(g, op, ws, f, st);
        case 128: return run<16, 8, false, 3>(g, op, ws, f, st);
        case 64: return run<8, 4, false, 3>(g, op, ws, f, st);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_agg_gcn_bf16(const GraphDev &g, const __nv_bfloat16 *Y, int32_t f, const float *bias, int act,
                                __nv_bfloat16 *out, AggWorkspace ws, cudaStream_t st) {
    if (act == SAGA_ACT_RELU) return agg_sum_bf16<SAGA_ACT_RELU>(g, Y, f, g.dinv, bias, out, ws, st);
    return agg_sum_bf16<SAGA_ACT_NONE>(g, Y, f, g.dinv, bias, out, ws, st);
}

cudaError_t launch_agg_mean_bf16(const GraphDev &g, const __nv_bfloat16 *X, int32_t f, __nv_bfloat16 *M,
                                 AggWorkspace ws, cudaStream_t st) {
    return agg_sum_bf16<SAGA_ACT_NONE>(g, X, f, g.inv_deg, nullptr, M, ws, st);
}

cudaError_t launch_gcn_f32_fused(const GraphDev &g, const float *X, int32_t f_in, const float *W, int32_t f_out,
                                 const float *bias, int act, float *out, AggWorkspace ws, cudaStream_t st) {
    GcnF32FusedOp op{};
    op.X = X; op.f_in = f_in; op.f_out = f_out; op.dinv = g.dinv; op.bias = bias; op.act = act; op.out = out;
    const int32_t welems = f_in * f_out;
    switch (f_in) {
        case 128: return run<32, 4, false, 2>(g, op, ws, f_in, st, W, welems);
        case 64: return run<16, 4, false, 2>(g, op, ws, f_in, st, W, welems);
        case 32: return run<8, 4, false, 2>(g, op, ws, f_in, st, W, welems);
        case 16: return run<4, 4, false, 2>(g, op, ws, f_in, st, W, welems);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_gat_edge(const GraphDev &g, const __nv_bfloat16 *z, const float *el, const float *er,
                            float slope, __nv_bfloat16 *out, AggWorkspace ws, cudaStream_t st) {
    if (agg_variant() == 9) {
        GatOp op{};
        op.z = z; op.el = el; op.er = er; op.slope = slope; op.out = out;
        return run<8, 4, false, 3>(g, op, ws, 8 * 12, st);
    }
    GatDenseOp op{};
    op.z = z; op.el = el; op.er = er; op.slope = slope; op.out = out;
    switch (agg_variant()) {
        case 10: return run_dense<16, false, 3>(g, op, ws, 32 * 4, st);
        case 11: return run_dense<8, false, 3>(g, op, ws, 32 * 4, st);
    }
    return run_dense<8, false, 4>(g, op, ws, 32 * 4, st);
}

cudaError_t launch_agg_typed_f32(const GraphDev &g, const float *H, int32_t f, float *S, AggWorkspace ws,
                                 cudaStream_t st) {
    TypedF32Op op{};
    op.H = H; op.f = f; op.S = S;
    if (f != 128) return cudaErrorInvalidValue;
    if (g.etype) {
        switch (agg_variant()) {
            case 13: return run_dense<4, true, 4>(g, op, ws, 4 * f, st);
            case 14: return run_dense<8, true, 2>(g, op, ws, 4 * f, st);
        }
        return run_dense<8, true, 3>(g, op, ws, 4 * f, st);
    }
    return run_dense<8, false, 3>(g, op, ws, 4 * f, st);
}

}  // namespace saga
