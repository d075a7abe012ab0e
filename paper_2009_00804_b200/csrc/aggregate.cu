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
// One WARP owns one task and all 32 lanes work on ONE edge at a time (each
// lane a 4..16-byte slice of the source row), so every branch is
// warp-uniform:
//  * batches are U CONSECUTIVE edges of the task regardless of row ends, so
//    every batch keeps U row gathers in flight; col_src arrives in
//    coalesced 32-edge chunks, one chunk ahead, and a batch never straddles
//    a chunk (U | 32);
//  * when no row ends inside the batch (the common case) the U rows are
//    reduced with unpredicated adds; otherwise the batch is parked in a
//    per-warp shared-memory slot (each lane re-reads only what it wrote) and
//    reduced edge by edge with a row-end test after each, so no register holds
//    a batch across a row flush;
//  * row_end and the per-row epilogue data (dinv[v], GAT er[v,:]) live in a
//    32-row shared-memory window, refilled once per 32 rows, with the rest of
//    the cold bookkeeping -- registers go to rows in flight (U = 8 at 64
//    registers: 32 warps and 256 rows of 512 B in flight per SM).
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
#include <algorithm>
#include <cstdint>
#include <type_traits>

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
    const int32_t *task_v;
    const int64_t *task_p;
    int64_t T, ntasks;
    int32_t n;
    int32_t e;
    const int32_t *rmap;  // view row -> output row (nullptr: identity)
};

GraphView view(const GraphDev &g) {
    return GraphView{g.row_ptr, g.col_src, g.task_v, g.task_p, g.task_items, g.ntasks, g.n, (int32_t)g.e, nullptr};
}
// the same CSR with the 4x finer schedule (GAT)
GraphView view_fine(const GraphDev &g) {
    return GraphView{g.row_ptr, g.col_src, g.ftask_v, g.ftask_p, g.ftask_items, g.fntasks, g.n, (int32_t)g.e,
                     nullptr};
}
// rows (v, t) -> r = v * num_etypes + t (built when the graph has edge types)
GraphView view_typed(const GraphDev &g) {
    return GraphView{g.trow_ptr, g.tcol_src, g.ttask_v, g.ttask_p, g.ttask_items, g.tntasks,
                     g.n * g.num_etypes, (int32_t)g.e, nullptr};
}
// the aggregation rows only (graph_build.cu step 8; GAT): rows whose in-edges
// are nothing but one self-loop, or none, are finished by the GEMM epilogue
GraphView view_agg_fine(const GraphDev &g) {
    return GraphView{g.arow_ptr, g.acol_src, g.aftask_v, g.aftask_p, g.aftask_items, g.afntasks, g.an, (int32_t)g.ae,
                     g.arow};
}

// the aggregation rows only, one task per resident warp (GCN)
GraphView view_agg(const GraphDev &g) {
    return GraphView{g.arow_ptr, g.acol_src, g.atask_v, g.atask_p, g.atask_items, g.antasks, g.an, (int32_t)g.ae,
                     g.arow};
}

__device__ __forceinline__ float act_fn(float x, int act) {
    if (act == SAGA_ACT_RELU) return fmaxf(x, 0.0f);
    if (act == SAGA_ACT_ELU) return x > 0.0f ? x : expm1f(x);
    return x;
}

// ===================================================================== ops ==
// Op interface (all const; the engine passes `rs`, this lane's per-row value,
// column win_col(lane) of the kWin values each row carries):
//   Acc, Val; kWin, win_col(lane), row_value(v, j)
//   zero(acc); load(u, lane); add(acc, val, rs)
//   finish(v, acc, rs, lane)  [or finish_w(v, acc, rs, Ws, lane): warp GEMV]
//   save(slot, acc, lane); merge(acc, slot, lane); kSlot = floats per partial

// Sum of bf16 rows (NB = 2, 4, 8 elements per lane: row width 32 NB) ->
// act(scale[v] * acc + bias) in bf16.  GCN (Y pre-scaled by dinv[u], scale =
// dinv[v]) and SAGE-mean (scale = 1/deg).
template <int kAct, int NB>
struct SumBf16Op {
    static_assert(NB == 2 || NB == 4 || NB == 8, "2, 4 or 8 bf16 per lane");
    static constexpr int kWin = 1;
    static constexpr int kSlot = 32 * NB;
    // C2's 128-wide rows: -3.5%; C5's 256-wide rows: +40% (registers)
    static constexpr bool kSplitBatch = NB <= 4;
    __device__ static int win_col(int) { return 0; }
    struct Acc { float a[NB]; };
    struct alignas(2 * NB) Val { uint32_t w[NB / 2]; };  // parks as one vector access
    const __nv_bfloat16 *X;
    const float *scale;
    const float *bias;
    __nv_bfloat16 *out;
    __device__ __forceinline__ float row_value(int32_t v, int) const { return __ldg(scale + v); }
    __device__ __forceinline__ void zero(Acc &c) const {
#pragma unroll
        for (int i = 0; i < NB; ++i) c.a[i] = 0.0f;
    }
    // row u, lane slice: one IMAD.WIDE.U32 per address
    __device__ __forceinline__ Val load(int32_t u, int lane) const {
        const char *p = ptx::mad_wide((uint32_t)u, 64u * NB, reinterpret_cast<const char *>(X) + lane * (2 * NB));
        Val v;
        if constexpr (NB == 8) {
            const uint4 x = __ldg(reinterpret_cast<const uint4 *>(p));
            v.w[0] = x.x; v.w[1] = x.y; v.w[2] = x.z; v.w[3] = x.w;
        } else if constexpr (NB == 4) {
            const uint2 x = __ldg(reinterpret_cast<const uint2 *>(p));
            v.w[0] = x.x; v.w[1] = x.y;
        } else {
            v.w[0] = __ldg(reinterpret_cast<const uint32_t *>(p));
        }
        return v;
    }
    __device__ __forceinline__ void add(Acc &c, const Val &v, float) const {
#pragma unroll
        for (int i = 0; i < NB / 2; ++i) ptx::add_bf16x2_f32(c.a[2 * i], c.a[2 * i + 1], v.w[i]);
    }
    // Ws: the bias staged in shared memory by the engine (nullptr: no bias)
    __device__ __forceinline__ void finish(int32_t v, const Acc &c, float rs, int lane, const float *Ws) const {
        uint32_t pk[NB / 2];
#pragma unroll
        for (int h = 0; h < NB / 2; ++h) {
            float2 b = make_float2(0.f, 0.f);
            if (bias) b = reinterpret_cast<const float2 *>(Ws + lane * NB)[h];
            pk[h] = ptx::pack_bf16x2(act_fn(fmaf(rs, c.a[2 * h], b.x), kAct),
                                     act_fn(fmaf(rs, c.a[2 * h + 1], b.y), kAct));
        }
        char *p = reinterpret_cast<char *>(out + (int64_t)v * (32 * NB)) + lane * (2 * NB);
        if constexpr (NB == 8)
            *reinterpret_cast<uint4 *>(p) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        else if constexpr (NB == 4)
            *reinterpret_cast<uint2 *>(p) = make_uint2(pk[0], pk[1]);
        else
            *reinterpret_cast<uint32_t *>(p) = pk[0];
    }
    __device__ __forceinline__ void save(float *slot, const Acc &c, int lane) const {
#pragma unroll
        for (int i = 0; i < NB; ++i) slot[lane * NB + i] = c.a[i];
    }
    __device__ __forceinline__ void merge(Acc &c, const float *slot, int lane) const {
#pragma unroll
        for (int i = 0; i < NB; ++i) c.a[i] += __ldcg(slot + lane * NB + i);
    }
};

// C1: fp32 rows (NPL = 1, 2 or 4 per lane; f_in = 16 uses half the warp),
// weight dinv[u] per edge, then the ApplyVertex GEMV (W staged in shared
// memory) fused into the row flush, spread over the warp (lane L computes
// outputs L and L + 32).
// kRowwise (graphs whose in-degrees are all <= kEllMaxDeg, one warp per
// row): fp32 accumulation -- a sum of <= 64 terms is within ~4e-6 of fp64,
// and the fp32 -> fp64 conversions (XU pipe) were 12% of C1's stalls.
template <int NPL, bool kRowwise = false>
struct GcnF32FusedOp {
    static constexpr int kWin = 1;
    static constexpr int kSlot = 2 * 32 * NPL;  // doubles as float pairs
    __device__ static int win_col(int) { return 0; }
    using AccT = typename std::conditional<kRowwise, float, double>::type;
    struct Acc { AccT a[NPL]; };  // merge-path: fp64 accumulation (see SumF32Op)
    // W [f_in][f_out] elements per thread of a 256-thread block (f_in <= 32 NPL, f_out <= 64)
    static constexpr int kWPerThread = 8 * NPL;
    struct Val { float x[NPL]; float w; };
    const float *X;
    int32_t f_in, f_out;
    const float *dinv;
    const float *bias;
    int act;
    float *out;
    __device__ __forceinline__ float row_value(int32_t v, int) const { return __ldg(dinv + v); }
    __device__ __forceinline__ void zero(Acc &c) const {
#pragma unroll
        for (int i = 0; i < NPL; ++i) c.a[i] = 0.0f;
    }
    __device__ __forceinline__ Val load(int32_t u, int lane) const {
        Val v;
        v.w = __ldg(dinv + u);
        const float *p = reinterpret_cast<const float *>(
            ptx::mad_wide((uint32_t)u, 4u * (uint32_t)f_in, reinterpret_cast<const char *>(X + lane * NPL)));
        const bool on = lane * NPL < f_in;
        if constexpr (NPL == 4) {
            const float4 x = on ? __ldg(reinterpret_cast<const float4 *>(p)) : make_float4(0.f, 0.f, 0.f, 0.f);
            v.x[0] = x.x; v.x[1] = x.y; v.x[2] = x.z; v.x[3] = x.w;
        } else if constexpr (NPL == 2) {
            const float2 x = on ? __ldg(reinterpret_cast<const float2 *>(p)) : make_float2(0.f, 0.f);
            v.x[0] = x.x; v.x[1] = x.y;
        } else {
            v.x[0] = on ? __ldg(p) : 0.0f;
        }
        return v;
    }
    __device__ __forceinline__ void add(Acc &c, const Val &v, float) const {
#pragma unroll
        for (int i = 0; i < NPL; ++i) c.a[i] = fma((AccT)v.w, (AccT)v.x[i], c.a[i]);
    }
    __device__ __forceinline__ void finish_w(int32_t v, const Acc &c, float rs, const float *Ws, int lane) const {
        float h[NPL];
#pragma unroll
        for (int i = 0; i < NPL; ++i) h[i] = (float)((AccT)rs * c.a[i]);
        if (f_out <= 16) {
            // narrow outputs (C1: 64 -> 16): lane = (k half, column); each half
            // runs its own dependent FMA chains over half the inputs (one per
            // NPL slot), folded by one shuffle -- a quarter of the chain length.
            // The halves' W rows are f_in f_out / 2 floats apart (0 mod 32 at
            // f_out = 16): the upper half walks its NPL slots in reverse, so
            // the two addresses of one load differ by an odd multiple of 16
            // floats and fall in disjoint banks (NPL >= 2).
            const int j = lane & 15, kh = lane >> 4, nk = f_in / NPL;
            float o[NPL];
#pragma unroll
            for (int i = 0; i < NPL; ++i) o[i] = 0.0f;
            for (int kl = kh * (nk / 2); kl < (kh + 1) * (nk / 2); ++kl) {
#pragma unroll
                for (int i = 0; i < NPL; ++i) {
                    const int ii = kh ? NPL - 1 - i : i;
                    // (lane kl serves the half that reads kl: lanes >= nk / 2 the upper one)
                    const float hk = __shfl_sync(kFull, lane >= nk / 2 ? h[NPL - 1 - i] : h[i], kl);
                    if (j < f_out) o[i] = fmaf(hk, Ws[(kl * NPL + ii) * f_out + j], o[i]);
                }
            }
            float acc = 0.0f;
#pragma unroll
            for (int i = 0; i < NPL; ++i) acc += o[i];
            acc += __shfl_xor_sync(kFull, acc, 16);
            if (kh == 0 && j < f_out) out[(int64_t)v * f_out + j] = act_fn(acc + (bias ? __ldg(bias + j) : 0.0f), act);
            return;
        }
        float o0 = 0.0f, o1 = 0.0f;
        const int j0 = lane, j1 = lane + 32;
        for (int kl = 0; kl < f_in / NPL; ++kl) {  // lane kl holds inputs kl*NPL ..
#pragma unroll
            for (int i = 0; i < NPL; ++i) {
                const float hk = __shfl_sync(kFull, h[i], kl);
                const float *wr = Ws + (kl * NPL + i) * f_out;
                if (j0 < f_out) o0 = fmaf(hk, wr[j0], o0);
                if (j1 < f_out) o1 = fmaf(hk, wr[j1], o1);
            }
        }
        if (j0 < f_out) out[(int64_t)v * f_out + j0] = act_fn(o0 + (bias ? __ldg(bias + j0) : 0.0f), act);
        if (j1 < f_out) out[(int64_t)v * f_out + j1] = act_fn(o1 + (bias ? __ldg(bias + j1) : 0.0f), act);
    }
    __device__ __forceinline__ void save(float *slot, const Acc &c, int lane) const {
#pragma unroll
        for (int i = 0; i < NPL; ++i) reinterpret_cast<double *>(slot)[lane * NPL + i] = (double)c.a[i];
    }
    __device__ __forceinline__ void merge(Acc &c, const float *slot, int lane) const {
#pragma unroll
        for (int i = 0; i < NPL; ++i) c.a[i] += (AccT)__ldcg(reinterpret_cast<const double *>(slot) + lane * NPL + i);
    }
};

// C3: GAT with the softmax shift fixed per row (reading A29).  The
// edge softmax is invariant under a per-row shift of the scores; with M_h =
// max_u el[u,h] (the GEMM's per-CTA maxima, reduced by k_gat_maxel) every
// score of row v is at most S_v = LeakyReLU(M_h + er[v,h]), so the weight of
// edge u -> v is exp(LeakyReLU(el[u] + er[v]) - S_v) <= 1: no running maximum,
// no rescaling, and a partial row state (l, a0, a1) merges by plain addition.
// A row whose weights all underflow (sum < kGatTiny: every score of the row
// ~69 or more below its bound) is recomputed with the online softmax by
// gat_row_online.  Lane L owns head h = L / 4 and output columns 2L, 2L+1 (a
// 4-byte slice of the 128-byte z row); row value: er[v, h].
constexpr float kGatTiny = 1e-30f;

// the underflow fallback: row v's in-edges from the full CSR (the aggregation
// view's rows keep every in-edge), single-pass online softmax, ELU(acc / l)
__device__ __forceinline__ void gat_row_online(int32_t v, int lane, const int64_t *row_ptr, const int32_t *col_src,
                                               const __nv_bfloat16 *z, const float *el, const float *er, float slope,
                                               __nv_bfloat16 *out) {
    const int h = lane >> 2;
    const float erv = __ldg(er + (int64_t)v * 8 + h);
    float m = -INFINITY, l = 0.0f, a0 = 0.0f, a1 = 0.0f;
    for (int64_t q = __ldg(row_ptr + v), q1 = __ldg(row_ptr + v + 1); q < q1; ++q) {
        const int32_t u = __ldg(col_src + q);
        float x = __ldg(el + (int64_t)u * 8 + h) + erv;
        x = fmaxf(x, slope * x);
        const float mn = fmaxf(m, x);
        const float co = __expf(m - mn), pe = __expf(x - mn);
        const float2 f = ptx::unpack_bf16x2(__ldg(reinterpret_cast<const uint32_t *>(z + (int64_t)u * 64) + lane));
        l = l * co + pe;
        a0 = a0 * co + pe * f.x;
        a1 = a1 * co + pe * f.y;
        m = mn;
    }
    const float inv = l > 0.0f ? 1.0f / l : 0.0f;
    float x0 = a0 * inv, x1 = a1 * inv;
    x0 = x0 > 0.0f ? x0 : __expf(x0) - 1.0f;
    x1 = x1 > 0.0f ? x1 : __expf(x1) - 1.0f;
    reinterpret_cast<uint32_t *>(out + (int64_t)v * 64)[lane] = ptx::pack_bf16x2(x0, x1);
}

template <bool kMap>
struct GatShiftOp {
    static constexpr int kWin = 8;
    static constexpr int kSlot = 128;
    __device__ static int win_col(int lane) { return lane >> 2; }
    // l is lane-partial: the head's 4 lanes each sum part of the weights
    // (finish adds them up; save / merge keep the lane partials)
    struct Acc { float l, a0, a1, S; };
    struct alignas(8) Val { uint32_t z2; float el; };
    const __nv_bfloat16 *z;
    const float *el, *er;
    const float *Mh;   // [8] max_u el[u, h]
    float slope;
    __nv_bfloat16 *out;
    const int32_t *rmap;  // kMap: the aggregation view's row -> vertex
    const int64_t *row_ptr;  // the fallback's full CSR
    const int32_t *col_src;
    __device__ __forceinline__ float row_value(int32_t v, int j) const {
        const int32_t u = kMap ? __ldg(rmap + v) : v;
        return __ldg(er + (int64_t)u * 8 + j);
    }
    __device__ __forceinline__ void zero(Acc &c) const { c.l = 0.f; c.a0 = 0.f; c.a1 = 0.f; }
    // the row's shift S_v (times log2 e)
    __device__ __forceinline__ void begin_row(Acc &c, int32_t, int lane, float er_h) const {
        const float x = __ldg(Mh + (lane >> 2)) + er_h;
        c.S = fmaxf(x, slope * x) * 1.4426950408889634f;
    }
    __device__ __forceinline__ float weight(float el_u, float er_h, float S) const {
        const float x = el_u + er_h;
        return ptx::exp2_ftz(fmaf(fmaxf(x, slope * x), 1.4426950408889634f, -S));  // LeakyReLU, 0 <= slope <= 1
    }
    __device__ __forceinline__ Val load(int32_t u, int lane) const {
        Val v;
        v.z2 = __ldg(reinterpret_cast<const uint32_t *>(
            ptx::mad_wide((uint32_t)u, 128u, reinterpret_cast<const char *>(z) + lane * 4)));
        v.el = __ldg(reinterpret_cast<const float *>(
            ptx::mad_wide((uint32_t)u, 32u, reinterpret_cast<const char *>(el) + (lane >> 2) * 4)));
        return v;
    }
    // one edge (the parked path): lane 4h of each head adds the weight to l
    __device__ __forceinline__ void add(Acc &c, const Val &v, float er_h) const {
        const float pe = weight(v.el, er_h, c.S);
        const float2 f = ptx::unpack_bf16x2(v.z2);
        if ((threadIdx.x & 3) == 0) c.l += pe;
        c.a0 = fmaf(pe, f.x, c.a0);
        c.a1 = fmaf(pe, f.y, c.a1);
    }
    // Grouped weights (the engine's batch hooks, U = 8): lane 4h + i loads el
    // of edges i and i + 4 and forms their two weights; each weight is
    // broadcast to the head's 4 lanes by a shuffle.
    static constexpr bool kGroupScores = true;
    struct Batch { float el1, el2; };
    template <int U>
    __device__ __forceinline__ void load_batch(Val (&v)[U], Batch &b, int32_t cs, int base, int lane) const {
        static_assert(U == 8, "two edges per lane of a head's 4 lanes");
        // el first: the weights are formed while the z rows are in flight
        const int e1 = lane & 3;
        const int32_t s1 = __shfl_sync(0xffffffffu, cs, base + e1);
        const int32_t s2 = __shfl_sync(0xffffffffu, cs, base + e1 + 4);
        const char *elh = reinterpret_cast<const char *>(el) + (lane >> 2) * 4;
        b.el1 = __ldg(reinterpret_cast<const float *>(ptx::mad_wide((uint32_t)s1, 32u, elh)));
        b.el2 = __ldg(reinterpret_cast<const float *>(ptx::mad_wide((uint32_t)s2, 32u, elh)));
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t src = __shfl_sync(0xffffffffu, cs, base + u);
            v[u].z2 = __ldg(reinterpret_cast<const uint32_t *>(
                ptx::mad_wide((uint32_t)src, 128u, reinterpret_cast<const char *>(z) + lane * 4)));
        }
    }
    template <int U>
    __device__ __forceinline__ void add_batch_grouped(Acc &c, const Val (&v)[U], const Batch &b, float er_h,
                                                      int lane) const {
        const float p1 = weight(b.el1, er_h, c.S), p2 = weight(b.el2, er_h, c.S);
        c.l += p1 + p2;
        const int gb = lane & ~3;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const float pe = __shfl_sync(0xffffffffu, u < 4 ? p1 : p2, gb | (u & 3));
            const float2 f = ptx::unpack_bf16x2(v[u].z2);
            c.a0 = fmaf(pe, f.x, c.a0);
            c.a1 = fmaf(pe, f.y, c.a1);
        }
    }
    // a batch leaving the fast path: every lane takes its head's el of each edge
    template <int U>
    __device__ __forceinline__ void unpack_batch(Val (&v)[U], const Batch &b, int lane) const {
        const int gb = lane & ~3;
#pragma unroll
        for (int u = 0; u < U; ++u) v[u].el = __shfl_sync(0xffffffffu, u < 4 ? b.el1 : b.el2, gb | (u & 3));
    }
    __device__ __forceinline__ void finish(int32_t v, const Acc &c, float, int lane, const float *) const {
        float l = c.l + __shfl_xor_sync(kFull, c.l, 1);
        l += __shfl_xor_sync(kFull, l, 2);
        if (__any_sync(kFull, l < kGatTiny)) {  // (warp-uniform: every caller runs the whole warp)
            gat_row_online(v, lane, row_ptr, col_src, z, el, er, slope, out);
            return;
        }
        const float inv = 1.0f / l;
        float x0 = c.a0 * inv, x1 = c.a1 * inv;
        x0 = x0 > 0.0f ? x0 : __expf(x0) - 1.0f;  // ELU; within 1e-7 absolute of expm1 (output is bf16)
        x1 = x1 > 0.0f ? x1 : __expf(x1) - 1.0f;
        reinterpret_cast<uint32_t *>(out + (int64_t)v * 64)[lane] = ptx::pack_bf16x2(x0, x1);
    }
    __device__ __forceinline__ void save(float *slot, const Acc &c, int lane) const {
        reinterpret_cast<float4 *>(slot)[lane] = make_float4(c.l, c.a0, c.a1, 0.0f);
    }
    __device__ __forceinline__ void merge(Acc &c, const float *slot, int lane) const {
        const float4 x = __ldcg(reinterpret_cast<const float4 *>(slot) + lane);
        c.l += x.x;
        c.a0 += x.y;
        c.a1 += x.z;
    }
};

// M_h = max over the GAT GEMM's per-CTA maxima of el (one warp)
__global__ void __launch_bounds__(32) k_gat_maxel(const float *__restrict__ parts, int nparts, float *__restrict__ Mh) {
    griddep_wait();  // the maxima come from the GEMM
    const int lane = threadIdx.x;
    float m = -INFINITY;
    for (int i = lane >> 3; i < nparts; i += 4) m = fmaxf(m, __ldcg(parts + i * 8 + (lane & 7)));
    m = fmaxf(m, __shfl_xor_sync(kFull, m, 8));
    m = fmaxf(m, __shfl_xor_sync(kFull, m, 16));
    if (lane < 8) Mh[lane] = m;
    griddep_launch();
}

// C4 / R-GCN: sums (or means) of fp32 rows of 128 over the graph's typed view,
// whose rows are (destination, type) pairs r = v * T + t (graph_build.cu step
// 7), so S[r] lands at S[v][t][:] -- one accumulator per lane, no per-edge
// type select.  Accumulated in fp64: a 70K-edge hub summed in fp32 loses
// ~1e-4 of the normwise output accuracy through the GRU (the fp32 configs'
// tolerance), while FP64 adds cost nothing on this memory-bound loop; a
// fast-path batch is pre-summed in fp32 (U = 8 terms).  Row value: 1/|row|
// (R-GCN per-type mean, reading A24; 0 for a type with no in-edges) or none.
template <bool kHeavy>
struct SumF32Op {
    static constexpr int kWin = 1;
    static constexpr int kSlot = 2 * 32 * 4;  // doubles as float pairs
    static constexpr bool kSplitBatch = true;  // C4 -3.3%, C6 -4.2%
    __device__ static int win_col(int) { return 0; }
    struct Acc { double a[4]; };
    struct Val { float4 x; };
    const float *H;
    const float *scale;  // nullptr: plain sum
    float *S;
    // gated layer: the heavy rows' sums (in-degree >= kHeavyInDeg) also in fp64,
    // Sx[slot][t][128], for the fp64 ApplyVertex (gru_f64.cu); nullptr: none
    const int32_t *hslot;
    double *Sx;
    int32_t T;
    // Row value (read through the engine's 32-row window, never a dependent
    // load in the row flush): the mean's 1/|row|, or for the plain sum 1, or
    // -(slot + 1) for a heavy row (its fp64 copy goes to Sx[slot]).
    __device__ __forceinline__ float row_value(int32_t r, int) const {
        if constexpr (kHeavy) {  // (the gated layer's plain sums: no scale)
            const int32_t hs = __ldg(hslot + r / T);
            return hs >= 0 ? -(float)(hs + 1) : 1.0f;
        }
        return scale ? __ldg(scale + r) : 1.0f;
    }
    __device__ __forceinline__ void zero(Acc &c) const {
#pragma unroll
        for (int i = 0; i < 4; ++i) c.a[i] = 0.0;
    }
    __device__ __forceinline__ Val load(int32_t u, int lane) const {
        const char *p = ptx::mad_wide((uint32_t)u, 512u, reinterpret_cast<const char *>(H) + lane * 16);
        return Val{__ldg(reinterpret_cast<const float4 *>(p))};
    }
    static constexpr bool kBatchAdd = true;
    template <int U>
    __device__ __forceinline__ void add_batch(Acc &c, const Val (&v)[U], float) const {
        float4 s = v[0].x;
#pragma unroll
        for (int u = 1; u < U; ++u) {
            s.x += v[u].x.x;
            s.y += v[u].x.y;
            s.z += v[u].x.z;
            s.w += v[u].x.w;
        }
        c.a[0] += (double)s.x;
        c.a[1] += (double)s.y;
        c.a[2] += (double)s.z;
        c.a[3] += (double)s.w;
    }
    __device__ __forceinline__ void add(Acc &c, const Val &v, float) const {
        c.a[0] += (double)v.x.x;
        c.a[1] += (double)v.x.y;
        c.a[2] += (double)v.x.z;
        c.a[3] += (double)v.x.w;
    }
    __device__ __forceinline__ void finish(int32_t r, const Acc &c, float rs, int lane, const float *) const {
        const double d = (kHeavy && rs < 0.0f) ? 1.0 : (double)rs;
        reinterpret_cast<float4 *>(S + (int64_t)r * 128)[lane] =
            make_float4((float)(c.a[0] * d), (float)(c.a[1] * d), (float)(c.a[2] * d), (float)(c.a[3] * d));
        if (kHeavy && rs < 0.0f) {  // heavy row: also the fp64 sums
            const int64_t hs = (int64_t)(-rs) - 1;
            double2 *x = reinterpret_cast<double2 *>(Sx + (hs * T + r % T) * 128) + lane * 2;
            x[0] = make_double2(c.a[0], c.a[1]);
            x[1] = make_double2(c.a[2], c.a[3]);
        }
    }
    __device__ __forceinline__ void save(float *slot, const Acc &c, int lane) const {
        double2 *d = reinterpret_cast<double2 *>(slot) + lane * 2;
        d[0] = make_double2(c.a[0], c.a[1]);
        d[1] = make_double2(c.a[2], c.a[3]);
    }
    __device__ __forceinline__ void merge(Acc &c, const float *slot, int lane) const {
        const double2 *d = reinterpret_cast<const double2 *>(slot) + lane * 2;
        const double2 x = __ldcg(d), y = __ldcg(d + 1);
        c.a[0] += x.x;
        c.a[1] += x.y;
        c.a[2] += y.x;
        c.a[3] += y.y;
    }
};

// NEXT-4 paper-form GGNN (reading A26): per in-edge u -> v the message
// act([H[u] || H[v]] . W_e + b_e) = act(A[u] + B[v]) by linearity, with A =
// H W_a and B = H W_b + b_e from one node-level GEMM (AB [n][2f], f = 128);
// the lane's 4-column slice of B[v] is loaded once per row (begin_row).
// Sum (fp64 accumulation, as SumF32Op) or elementwise max (exact; -inf
// marks "no edge yet", 0 for a vertex without in-edges).
template <bool kMax, bool kRelu>
struct EdgeMlpOp {
    static constexpr int kWin = 0;
    static constexpr int kSlot = 2 * 32 * 4;  // doubles as float pairs
    __device__ static int win_col(int) { return 0; }
    // hs: the row's heavy slot (>= 0: in-degree >= kHeavyInDeg) -- warp-uniform
    struct Acc { double a[4]; float4 b; int32_t hs; };
    struct Val { float4 x; };
    const float *AB;       // [n][256]
    float *m;              // [n][128]
    const int32_t *hslot;  // [n] heavy slot or -1 (GraphDev::heavy_slot)
    const double *Bx;      // [n_heavy][128] B of the heavy rows in fp64 (gru_f64.cu)
    double *mx;            // [n_heavy][128] m of the heavy rows, never rounded to fp32
    __device__ __forceinline__ float row_value(int32_t, int) const { return 0.0f; }
    __device__ __forceinline__ void zero(Acc &c) const {
#pragma unroll
        for (int i = 0; i < 4; ++i) c.a[i] = kMax ? -INFINITY : 0.0;
    }
    __device__ __forceinline__ void begin_row(Acc &c, int32_t v, int lane, float) const {
        c.hs = __ldg(hslot + v);
        c.b = __ldg(reinterpret_cast<const float4 *>(
            ptx::mad_wide((uint32_t)v, 1024u, reinterpret_cast<const char *>(AB) + 512 + lane * 16)));
    }
    __device__ __forceinline__ Val load(int32_t u, int lane) const {
        return Val{__ldg(reinterpret_cast<const float4 *>(
            ptx::mad_wide((uint32_t)u, 1024u, reinterpret_cast<const char *>(AB) + lane * 16)))};
    }
    // Heavy rows (in-degree >= kHeavyInDeg) add their fp64 B[v] to every
    // in-edge's A[u] in fp64: B[v] enters the sum deg(v) times, so the tensor
    // GEMM's fp32 B (error ~1e-7) would be amplified by the in-degree into m.
    __device__ __forceinline__ void add_heavy(Acc &c, const float4 &x, const double (&bd)[4]) const {
        const double y[4] = {(double)x.x + bd[0], (double)x.y + bd[1], (double)x.z + bd[2], (double)x.w + bd[3]};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const double t = kRelu ? fmax(y[i], 0.0) : y[i];
            c.a[i] = kMax ? fmax(c.a[i], t) : c.a[i] + t;
        }
    }
    __device__ __forceinline__ void load_bd(double (&bd)[4], int32_t hs, int lane) const {
        const double2 *bp = reinterpret_cast<const double2 *>(Bx + (int64_t)hs * 128) + lane * 2;
        const double2 b0 = __ldg(bp), b1 = __ldg(bp + 1);
        bd[0] = b0.x; bd[1] = b0.y; bd[2] = b1.x; bd[3] = b1.y;
    }
    // fast path: the batch's messages reduced in fp32 (sum of U terms, or the
    // exact max), then one fp64 update per element -- as SumF32Op
    static constexpr bool kBatchAdd = true;
    template <int U>
    __device__ __forceinline__ void add_batch(Acc &c, const Val (&v)[U], float) const {
        if (c.hs >= 0) {
            double bd[4];
            load_bd(bd, c.hs, threadIdx.x & 31);
#pragma unroll
            for (int u = 0; u < U; ++u) add_heavy(c, v[u].x, bd);
            return;
        }
        float s[4];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            float y[4] = {v[u].x.x + c.b.x, v[u].x.y + c.b.y, v[u].x.z + c.b.z, v[u].x.w + c.b.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                if (kRelu) y[i] = fmaxf(y[i], 0.0f);
                s[i] = u == 0 ? y[i] : (kMax ? fmaxf(s[i], y[i]) : s[i] + y[i]);
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) c.a[i] = kMax ? fmax(c.a[i], (double)s[i]) : c.a[i] + (double)s[i];
    }
    __device__ __forceinline__ void add(Acc &c, const Val &v, float) const {
        if (c.hs >= 0) {
            double bd[4];
            load_bd(bd, c.hs, threadIdx.x & 31);
            add_heavy(c, v.x, bd);
            return;
        }
        float y[4] = {v.x.x + c.b.x, v.x.y + c.b.y, v.x.z + c.b.z, v.x.w + c.b.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (kRelu) y[i] = fmaxf(y[i], 0.0f);
            if (kMax)
                c.a[i] = fmax(c.a[i], (double)y[i]);
            else
                c.a[i] += (double)y[i];
        }
    }
    __device__ __forceinline__ void finish(int32_t v, const Acc &c, float, int lane, const float *) const {
        double o[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) o[i] = (kMax && c.a[i] == -INFINITY) ? 0.0 : c.a[i];
        reinterpret_cast<float4 *>(m + (int64_t)v * 128)[lane] =
            make_float4((float)o[0], (float)o[1], (float)o[2], (float)o[3]);
        if (c.hs >= 0) {  // (a merged split row gets begin_row in ticket_merge too)
            double2 *d = reinterpret_cast<double2 *>(mx + (int64_t)c.hs * 128) + lane * 2;
            d[0] = make_double2(o[0], o[1]);
            d[1] = make_double2(o[2], o[3]);
        }
    }
    __device__ __forceinline__ void save(float *slot, const Acc &c, int lane) const {
        double2 *d = reinterpret_cast<double2 *>(slot) + lane * 2;
        d[0] = make_double2(c.a[0], c.a[1]);
        d[1] = make_double2(c.a[2], c.a[3]);
    }
    __device__ __forceinline__ void merge(Acc &c, const float *slot, int lane) const {
        const double2 *d = reinterpret_cast<const double2 *>(slot) + lane * 2;
        const double2 x = __ldcg(d), y = __ldcg(d + 1);
        const double p[4] = {x.x, x.y, y.x, y.y};
#pragma unroll
        for (int i = 0; i < 4; ++i) c.a[i] = kMax ? fmax(c.a[i], p[i]) : c.a[i] + p[i];
    }
};

// Ops whose epilogue needs the whole warp (the fused GEMV) implement finish_w.
template <typename Op>
__device__ __forceinline__ auto do_finish(const Op &op, int32_t v, const typename Op::Acc &c, float rs, int lane,
                                          const float *Ws, int) -> decltype(op.finish_w(v, c, rs, Ws, lane), void()) {
    op.finish_w(v, c, rs, Ws, lane);
}
template <typename Op>
__device__ __forceinline__ void do_finish(const Op &op, int32_t v, const typename Op::Acc &c, float rs, int lane,
                                          const float *Ws, long) {
    op.finish(v, c, rs, lane, Ws);
}

// Ops that carry per-row state loaded at the row's start implement begin_row.
template <typename Op, typename = void>
struct has_begin_row { static constexpr bool value = false; };
template <typename Op>
struct has_begin_row<Op, decltype(void(&Op::begin_row))> { static constexpr bool value = true; };
template <typename Op>
__device__ __forceinline__ void begin_row_of(const Op &op, typename Op::Acc &c, int32_t v, int32_t n, int lane,
                                             float rs) {
    if constexpr (has_begin_row<Op>::value) {
        if (v < n) op.begin_row(c, v, lane, rs);
    }
}

// Split rows (hubs, rows straddling a task boundary): every task holding part
// of row r saves its fp32 partial to its slot, then takes an integer ticket on
// the task k2 that holds r's end item; the last arrival merges all parts in
// task order and runs the epilogue.  The ticket is taken after the task's
// main loop (never inside it), so the hot loop carries no call.
template <typename Op>
__device__ __noinline__ void ticket_merge(const Op &op, AggWorkspace ws, int64_t T, int32_t r, int64_t rb,
                                          int64_t re, const float *Ws, const int32_t *rmap) {
    const int lane = threadIdx.x & 31;
    const int64_t k1 = (rb + r) / T, k2 = (re + r) / T;
    // release the partial stores before the ticket; acquire the others'
    // after winning (acq_rel, not the sequentially consistent __threadfence:
    // MEMBAR.SC.GPU stalled the task tails, 10% of C2's warp samples)
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    __syncwarp();
    int old = 0;
    if (lane == 0) old = atomicAdd(ws.counters + k2, 1);
    old = __shfl_sync(kFull, old, 0);
    if (old == (int)(k2 - k1)) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        if (lane == 0) ws.counters[k2] = 0;  // every contributor has taken its ticket: leave it zero
        const float rs = Op::kWin ? op.row_value(r, Op::win_col(lane)) : 0.0f;
        typename Op::Acc m;
        op.zero(m);
        begin_row_of(op, m, r, r + 1, lane, rs);  // per-row state the epilogue may read
        op.merge(m, ws.partials + (2 * k1 + 1) * Op::kSlot, lane);
        for (int64_t kk = k1 + 1; kk <= k2; ++kk) op.merge(m, ws.partials + (2 * kk) * Op::kSlot, lane);
        do_finish(op, rmap ? __ldg(rmap + r) : r, m, rs, lane, Ws, 0);
    }
}

// Ops with a batch-level fast-path update declare kBatchAdd.
template <typename Op, typename = void>
struct has_batch_add { static constexpr bool value = false; };
template <typename Op>
struct has_batch_add<Op, decltype(void(Op::kBatchAdd))> { static constexpr bool value = Op::kBatchAdd; };

// Ops whose batch loads and scores are shared across lanes declare kGroupScores
// (GatShiftOp: load_batch / add_batch_grouped / unpack_batch and a Batch type).
template <typename Op, typename = void>
struct has_group_scores { static constexpr bool value = false; };
template <typename Op>
struct has_group_scores<Op, decltype(void(Op::kGroupScores))> { static constexpr bool value = Op::kGroupScores; };
struct NoBatch {};
template <typename Op, bool = has_group_scores<Op>::value>
struct BatchOf { using type = NoBatch; };
template <typename Op>
struct BatchOf<Op, true> { using type = typename Op::Batch; };

// Ops that keep a batch split by one row end in registers declare kSplitBatch.
template <typename Op, typename = void>
struct has_split_batch { static constexpr bool value = false; };
template <typename Op>
struct has_split_batch<Op, decltype(void(Op::kSplitBatch))> { static constexpr bool value = Op::kSplitBatch; };

// ================================================================== engine ==
template <int U, typename Val, int kWinD, bool kRmap>
struct DenseWarp {
    Val park[U][32];
    int32_t re[32];                 // row_end of rows wr .. wr+31
    int32_t rid[kRmap ? 32 : 1];    // their output rows (the view's rmap)
    float rv[32 * kWinD];           // per-row values of the same rows (kWinD per row)
    int32_t wr, head_end;
};

// kRmap: the view maps its rows to output rows (the aggregation view); a
// compile-time switch -- as a runtime one it cost the GAT kernel 25%.
template <int U, int kMinB, typename Op, bool kRmap>
__global__ void __launch_bounds__(kBlock, kMinB) k_segreduce(const GraphView g, const __grid_constant__ Op op, const AggWorkspace ws,
                                                          const float *Wg, const int32_t w_elems) {
    constexpr int kWin = Op::kWin;
    constexpr int kWinD = kWin ? kWin : 1;
    static_assert(32 % U == 0, "U must divide the 32-edge chunk");
    // Ops that declare kSplitBatch keep a batch with one row end in registers
    // across the flush; the others park it (measured per op: GAT +2.5%, C5's
    // 256-wide bf16 rows +40% from the registers held across the flush)
    constexpr bool kSplitBatch = has_split_batch<Op>::value;
    constexpr bool kGroup = has_group_scores<Op>::value;
    static_assert(!(kSplitBatch && kGroup), "grouped-score ops park split batches");
    using DW = DenseWarp<U, typename Op::Val, kWinD, kRmap>;
    __shared__ DW warps[kWarpsPerBlock];
    extern __shared__ float Ws[];  // epilogue operand staged per block: fused-GEMV weight, or bias
    if (Wg) {
        for (int i = threadIdx.x; i < w_elems; i += blockDim.x) Ws[i] = Wg[i];
        __syncthreads();
    }
    griddep_wait();  // features / messages come from the call's previous kernel
    // the dependent may be scheduled from here on: every earlier kernel of the
    // call has completed (k_gcn_epi_rows relies on this to read Y unwaited)
    griddep_launch();
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
        VW.re[lane] = r < g.n ? (int32_t)__ldg(g.row_ptr + r + 1) : g.e;
        if constexpr (kRmap) VW.rid[lane] = r < g.n ? __ldg(g.rmap + r) : 0;
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
    // col_src in 32-edge chunks, two chunks ahead of the one in use (one
    // chunk -- 4 batches -- left 10% of the C5 stalls on the col_src load);
    // the first three are issued before the row window is filled, so the two
    // prologue round trips overlap
    auto load_cs = [&](int32_t base) -> int32_t {
        const int32_t q = base + lane;
        return q < p1 ? __ldcs(g.col_src + q) : 0;
    };
    int32_t cb = p;
    int32_t cs_a = load_cs(cb), cs_b = load_cs(cb + 32), cs_c = load_cs(cb + 64);
    const int32_t v0 = v;
    const int32_t head_beg = (int32_t)g.row_ptr[v];
    bool head_open = head_beg < p;  // the first row began in an earlier task (its partial is pending)
    const bool head = head_open;
    if (lane == 0) VW.head_end = -1;
    fill_window(v);
    int32_t row_end = VW.re[0];
    float rs = kWin ? VW.rv[Op::win_col(lane)] : 0.0f;

    typename Op::Acc acc;
    op.zero(acc);
    begin_row_of(op, acc, v, g.n, lane, rs);

    // finish row v (or save its partial if it is the head row), advance to v+1
    auto flush = [&]() {
        if (head_open) {
            op.save(ws.partials + 2 * k * Op::kSlot, acc, lane);
            if (lane == 0) VW.head_end = row_end;
            head_open = false;
        } else {
            if constexpr (kRmap)
                do_finish(op, VW.rid[v - VW.wr], acc, rs, lane, Ws, 0);
            else
                do_finish(op, v, acc, rs, lane, Ws, 0);
        }
        ++v;
        if (v - VW.wr == 32) {
            __syncwarp();
            fill_window(v);
        }
        const int32_t wr = VW.wr;
        row_end = VW.re[v - wr];
        if (kWin) rs = VW.rv[(v - wr) * kWinD + Op::win_col(lane)];
        op.zero(acc);
        begin_row_of(op, acc, v, g.n, lane, rs);
    };

    // keeps q - cb < 32; batches start at p + multiple of U and U | 32, so a
    // batch never straddles a chunk
    auto slide = [&](int32_t q) {
        if (q - cb >= 32) {
            cb += 32;
            cs_a = cs_b;
            cs_b = cs_c;
            cs_c = load_cs(cb + 64);
        }
    };

    while (v < v1 && row_end <= p) flush();  // rows that end before the first edge
    // cs_a is kept rotated so that lane 0 holds edge q's source: every
    // shuffle of a batch takes an immediate lane, and one shfl.down per batch
    // replaces the U per-edge lane-index adds
    int32_t q = p;
    for (; q + U <= p1; q += U) {
        slide(q);
        constexpr int base = 0;
        typename Op::Val val[U];
        [[maybe_unused]] typename BatchOf<Op>::type bt;
        if constexpr (kGroup) {
            op.template load_batch<U>(val, bt, cs_a, base, lane);
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u) val[u] = op.load(__shfl_sync(kFull, cs_a, base + u), lane);
        }
        if (row_end > q + U) {
            // fast path: no row ends inside the batch
            if constexpr (kGroup) {
                op.template add_batch_grouped<U>(acc, val, bt, rs, lane);
            } else if constexpr (has_batch_add<Op>::value) {
                op.template add_batch<U>(acc, val, rs);
            } else {
#pragma unroll
                for (int u = 0; u < U; ++u) op.add(acc, val[u], rs);
            }
        } else if (kSplitBatch && v < v1) {
            // one row ends inside the batch (the common case for rows longer
            // than U): its part, the flush, the rest -- in registers, the
            // adds predicated on the (warp-uniform) split point j
            const int j = row_end - q;  // 1 .. U
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (u < j) op.add(acc, val[u], rs);
            flush();
            while (v < v1 && row_end == q + j) flush();  // empty rows
            if (row_end >= q + U) {
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (u >= j) op.add(acc, val[u], rs);
                while (v < v1 && row_end == q + U) flush();
            } else {
                // more row ends: park the rest, reduce edge by edge
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (u >= j) W.park[u][lane] = val[u];
#pragma unroll 1
                for (int u = j; u < U; ++u) {
                    const typename Op::Val x = W.park[u][lane];
                    op.add(acc, x, rs);
                    while (v < v1 && row_end == q + u + 1) flush();
                }
            }
        } else {
            // slow path: park the batch, reduce edge by edge
            if constexpr (kGroup) op.template unpack_batch<U>(val, bt, lane);
#pragma unroll
            for (int u = 0; u < U; ++u) W.park[u][lane] = val[u];
#pragma unroll 1
            for (int u = 0; u < U; ++u) {
                const typename Op::Val x = W.park[u][lane];
                op.add(acc, x, rs);
                while (v < v1 && row_end == q + u + 1) flush();
            }
        }
        cs_a = __shfl_down_sync(kFull, cs_a, U);
    }
    for (; q < p1; ++q) {  // remainder, one edge at a time
        slide(q);
        op.add(acc, op.load(__shfl_sync(kFull, cs_a, 0), lane), rs);
        while (v < v1 && row_end == q + 1) flush();
        cs_a = __shfl_down_sync(kFull, cs_a, 1);
    }
    while (v < v1) flush();
    const int32_t row_beg = (v == v0) ? head_beg : (v < g.n ? (int32_t)__ldg(g.row_ptr + v) : g.e);
    if (v < g.n && p1 > row_beg) {  // tail: row v continues into the next task
        const int64_t slot = (head && v == v0) ? 2 * k : 2 * k + 1;
        op.save(ws.partials + slot * Op::kSlot, acc, lane);
        ticket_merge(op, ws, g.T, v, row_beg, row_end, Ws, kRmap ? g.rmap : nullptr);
    }
    const int32_t head_end = VW.head_end;
    if (head_end >= 0 && v != v0)  // the head row ended inside this task
        ticket_merge(op, ws, g.T, v0, head_beg, head_end, Ws, kRmap ? g.rmap : nullptr);
}

template <int U, int kMinB, typename Op>
cudaError_t run(const GraphView &g, const Op &op, AggWorkspace ws, cudaStream_t st, const float *Wg = nullptr,
                int32_t w_elems = 0) {
    if (g.ntasks == 0) return cudaSuccess;
    const unsigned blocks = (unsigned)((g.ntasks + kWarpsPerBlock - 1) / kWarpsPerBlock);
    const size_t smem = Wg ? sizeof(float) * w_elems : 0;
    if (g.rmap) return launch(k_segreduce<U, kMinB, Op, true>, blocks, kBlock, smem, st, g, op, ws, Wg, w_elems);
    return launch(k_segreduce<U, kMinB, Op, false>, blocks, kBlock, smem, st, g, op, ws, Wg, w_elems);
}

// Small-degree graphs (every in-degree <= kEllMaxDeg): one warp per row,
// no merge-path tasks and no split rows, edges from the graph's ELL view (a
// row's sources at a fixed offset: one dependent load fewer than row_ptr ->
// col_src on a cold step).  Used for C1's fused GCN layer, where the
// merge-path engine's per-task prologue and split-row tickets dominated a
// 12K-edge graph.
template <int U, int kMinB, typename Op>
__global__ void __launch_bounds__(kBlock, kMinB) k_rowwise(const int32_t *__restrict__ ell, int32_t ell_w,
                                                         int32_t n, const Op op, const float *Wg,
                                                         const int32_t w_elems) {
    extern __shared__ float Ws[];
    constexpr int kWReg = Op::kWPerThread;  // W elements per thread in flight (w_elems <= kWReg * kBlock)
    const int lane = threadIdx.x & 31;
    int32_t r = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    const bool first = r < n;
    griddep_launch();
    // the block's W loads are issued first and stay in flight (registers)
    // while the first row is gathered: W is only needed by the epilogue GEMV.
    // (Staging W before the gather put its DRAM round trip in series with the
    // row's three: 23% of C1's stall samples waited on it.)
    float wreg[kWReg];
#pragma unroll
    for (int k = 0; k < kWReg; ++k) {
        const int i = threadIdx.x + k * kBlock;
        wreg[k] = i < w_elems ? __ldg(Wg + i) : 0.0f;
    }
    griddep_wait();
    auto gather = [&](int32_t row, typename Op::Acc &acc, float &rs) {
        rs = op.row_value(row, 0);
        op.zero(acc);
        for (int32_t q0 = 0; q0 < ell_w; q0 += 32) {
            const int32_t c = q0 + lane < ell_w ? __ldg(ell + (int64_t)row * ell_w + q0 + lane) : -1;
            const int32_t cnt = __popc(__ballot_sync(kFull, c >= 0));  // the row's sources come first
            const int32_t cs = c >= 0 ? c : 0;
            if (cnt == 0) break;
            for (int j = 0; j < cnt; j += U) {
                typename Op::Val val[U];
#pragma unroll
                for (int u = 0; u < U; ++u) val[u] = op.load(__shfl_sync(kFull, cs, (j + u) & 31), lane);
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (j + u < cnt) op.add(acc, val[u], rs);
            }
        }
    };
    typename Op::Acc acc;
    float rs = 0.0f;
    if (first) gather(r, acc, rs);
#pragma unroll
    for (int k = 0; k < kWReg; ++k) {
        const int i = threadIdx.x + k * kBlock;
        if (i < w_elems) Ws[i] = wreg[k];
    }
    __syncthreads();
    if (first) do_finish(op, r, acc, rs, lane, Ws, 0);
    for (r += gridDim.x * kWarpsPerBlock; r < n; r += gridDim.x * kWarpsPerBlock) {
        gather(r, acc, rs);
        do_finish(op, r, acc, rs, lane, Ws, 0);
    }
}

// GCN rows outside the aggregation view (graph_build.cu step 8): the sum over
// the in-edges is the self-loop's Y[v] alone, or empty, so out[v] =
// act(dinv[v] Y[v] + b) -- a streaming pass over the listed rows (512-B row
// slices, 16 B per lane, kU rows in flight per warp) instead of a one-edge
// row flush each in the merge-path engine.
//
// Launched after the view's gather (unwaited = 1): the gather triggers its
// dependents only after its own griddepcontrol.wait, i.e. once the GEMM has
// completed, so this pass reads Y without waiting for the gather and its
// blocks fill the SMs the gather's tail leaves idle (the two write disjoint
// output rows).  unwaited = 0: the predecessor is the GEMM itself.
template <int kAct, int NB>
__global__ void __launch_bounds__(256) k_gcn_epi_rows(int32_t ne, const int32_t *__restrict__ erow,
                                                      const __nv_bfloat16 *__restrict__ Y,
                                                      const float *__restrict__ dinv, const float *__restrict__ bias,
                                                      __nv_bfloat16 *__restrict__ out, int unwaited) {
    constexpr int kU = 8;
    griddep_launch();
    const int lane = threadIdx.x & 31;
    float b[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) b[i] = bias ? __ldg(bias + lane * NB + i) : 0.0f;
    if (!unwaited) griddep_wait();  // Y comes from the call's GEMM
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * kU; i0 < ne; i0 += nw * kU) {
        const int64_t my = i0 + lane;
        const int32_t vl = (lane < kU && my < ne) ? __ldg(erow + my) : -1;
        const float sl = vl >= 0 ? __ldg(dinv + vl) : 0.0f;
        typename SumBf16Op<kAct, NB>::Val x[kU];
        int32_t v[kU];
        float sc[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            v[u] = __shfl_sync(kFull, vl, u);
            sc[u] = __shfl_sync(kFull, sl, u);
            if (v[u] >= 0 && sc[u] != 0.0f) {
                const char *p = reinterpret_cast<const char *>(Y) + (int64_t)v[u] * (64 * NB) + lane * (2 * NB);
                if constexpr (NB == 8) {
                    const uint4 q = __ldg(reinterpret_cast<const uint4 *>(p));
                    x[u].w[0] = q.x; x[u].w[1] = q.y; x[u].w[2] = q.z; x[u].w[3] = q.w;
                } else if constexpr (NB == 4) {
                    const uint2 q = __ldg(reinterpret_cast<const uint2 *>(p));
                    x[u].w[0] = q.x; x[u].w[1] = q.y;
                } else {
                    x[u].w[0] = __ldg(reinterpret_cast<const uint32_t *>(p));
                }
            } else {
#pragma unroll
                for (int i = 0; i < NB / 2; ++i) x[u].w[i] = 0u;
            }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            if (v[u] < 0) break;
            uint32_t pk[NB / 2];
#pragma unroll
            for (int h = 0; h < NB / 2; ++h) {
                const float2 y = ptx::unpack_bf16x2(x[u].w[h]);
                pk[h] = ptx::pack_bf16x2(act_fn(fmaf(sc[u], y.x, b[2 * h]), kAct),
                                         act_fn(fmaf(sc[u], y.y, b[2 * h + 1]), kAct));
            }
            char *o = reinterpret_cast<char *>(out + (int64_t)v[u] * (32 * NB)) + lane * (2 * NB);
            if constexpr (NB == 8)
                *reinterpret_cast<uint4 *>(o) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            else if constexpr (NB == 4)
                *reinterpret_cast<uint2 *>(o) = make_uint2(pk[0], pk[1]);
            else
                *reinterpret_cast<uint32_t *>(o) = pk[0];
        }
    }
}

template <int kAct, int NB>
cudaError_t gcn_epi_rows(const GraphDev &g, const __nv_bfloat16 *Y, const float *bias, __nv_bfloat16 *out,
                         cudaStream_t st, int unwaited) {
    if (g.ne == 0) return cudaSuccess;
    const int64_t warps = ((int64_t)g.ne + 7) / 8;
    const unsigned blocks = (unsigned)std::min<int64_t>((warps + 7) / 8, (int64_t)kNumSMs * 8);
    return launch(k_gcn_epi_rows<kAct, NB>, blocks, 256, 0, st, g.ne, (const int32_t *)g.erow, Y,
                  (const float *)g.dinv, bias, out, unwaited);
}

template <int kAct>
cudaError_t agg_sum_bf16(const GraphView &gv, const __nv_bfloat16 *X, int32_t f, const float *scale,
                         const float *bias, __nv_bfloat16 *out, AggWorkspace ws, cudaStream_t st) {
    switch (f) {
        case 256: {
            SumBf16Op<kAct, 8> op{X, scale, bias, out};
            return run<8, 4>(gv, op, ws, st, bias, bias ? f : 0);
        }
        case 128: {
            SumBf16Op<kAct, 4> op{X, scale, bias, out};
            return run<8, 4>(gv, op, ws, st, bias, bias ? f : 0);
        }
        case 64: {
            SumBf16Op<kAct, 2> op{X, scale, bias, out};
            return run<8, 4>(gv, op, ws, st, bias, bias ? f : 0);
        }
    }
    return cudaErrorInvalidValue;
}

template <int NPL>
cudaError_t gcn_f32(const GraphDev &g, const float *X, int32_t f_in, const float *W, int32_t f_out,
                    const float *bias, int act, float *out, AggWorkspace ws, cudaStream_t st) {
    if (gcn_f32_rowwise(g)) {
        if (g.n == 0) return cudaSuccess;
        GcnF32FusedOp<NPL, true> op{X, f_in, f_out, g.dinv, bias, act, out};
        const unsigned blocks = (unsigned)((g.n + kWarpsPerBlock - 1) / kWarpsPerBlock);
        return launch(k_rowwise<8, NPL == 4 ? 2 : 3, GcnF32FusedOp<NPL, true>>, blocks, kBlock,
                      sizeof(float) * f_in * f_out, st, (const int32_t *)g.ell, g.ell_w, g.n, op, W, f_in * f_out);
    }
    GcnF32FusedOp<NPL> op{X, f_in, f_out, g.dinv, bias, act, out};
    return run<8, NPL == 4 ? 2 : 3>(view(g), op, ws, st, W, f_in * f_out);
}

}  // namespace

size_t agg_partial_floats(saga_model kind, int32_t width, int32_t heads) {
    (void)heads;
    switch (kind) {
        case SAGA_GCN: return (size_t)2 * (width > 32 ? width : 32);  // 32 lanes x (1..8) fp32, or fp64 (fp32 path)
        case SAGA_SAGE: return (size_t)(width > 32 ? width : 32);
        case SAGA_GAT: return 128;                                // 32 lanes x (m, l, a0, a1)
        case SAGA_GATED:
        case SAGA_RGCN:
        case SAGA_GGNN: return (size_t)2 * 128;                   // 32 lanes x 4 fp64
    }
    return 0;
}

cudaError_t launch_agg_gcn_bf16(const GraphDev &g, const __nv_bfloat16 *Y, int32_t f, const float *bias, int act,
                                __nv_bfloat16 *out, AggWorkspace ws, cudaStream_t st) {
    // Rows whose only in-edge is the self-loop (52% of C5's) go through a
    // streaming pass; the engine runs over the aggregation view of the rest.
    // C5, ncu: 0.36 ms (2.2 GB at 6.1 TB/s) + 2.65 ms, against 3.09 ms for the
    // engine over every row; in-step 3.80 -> 3.70 ms.  The pass runs after
    // the gather and fills its tail (3.73-3.75 -> 3.61 ms with the pass
    // first).  (Finishing those rows in the GEMM epilogue instead cost the
    // GEMM 0.45-0.5 ms: TMA tile stores write every row.)
    if (g.arow) {
        cudaError_t e = act == SAGA_ACT_RELU
                            ? agg_sum_bf16<SAGA_ACT_RELU>(view_agg(g), Y, f, g.adinv, bias, out, ws, st)
                            : agg_sum_bf16<SAGA_ACT_NONE>(view_agg(g), Y, f, g.adinv, bias, out, ws, st);
        if (e) return e;
        const int unwaited = g.antasks > 0;
        if (f == 256)
            e = act == SAGA_ACT_RELU ? gcn_epi_rows<SAGA_ACT_RELU, 8>(g, Y, bias, out, st, unwaited)
                                     : gcn_epi_rows<SAGA_ACT_NONE, 8>(g, Y, bias, out, st, unwaited);
        else if (f == 128)
            e = act == SAGA_ACT_RELU ? gcn_epi_rows<SAGA_ACT_RELU, 4>(g, Y, bias, out, st, unwaited)
                                     : gcn_epi_rows<SAGA_ACT_NONE, 4>(g, Y, bias, out, st, unwaited);
        else
            e = act == SAGA_ACT_RELU ? gcn_epi_rows<SAGA_ACT_RELU, 2>(g, Y, bias, out, st, unwaited)
                                     : gcn_epi_rows<SAGA_ACT_NONE, 2>(g, Y, bias, out, st, unwaited);
        return e;
    }
    if (act == SAGA_ACT_RELU) return agg_sum_bf16<SAGA_ACT_RELU>(view(g), Y, f, g.dinv, bias, out, ws, st);
    return agg_sum_bf16<SAGA_ACT_NONE>(view(g), Y, f, g.dinv, bias, out, ws, st);
}

cudaError_t launch_agg_mean_bf16(const GraphDev &g, const __nv_bfloat16 *X, int32_t f, __nv_bfloat16 *M,
                                 AggWorkspace ws, cudaStream_t st) {
    return agg_sum_bf16<SAGA_ACT_NONE>(view(g), X, f, g.inv_deg, nullptr, M, ws, st);
}

cudaError_t launch_gcn_f32_fused(const GraphDev &g, const float *X, int32_t f_in, const float *W, int32_t f_out,
                                 const float *bias, int act, float *out, AggWorkspace ws, cudaStream_t st) {
    switch (f_in) {
        case 128: return gcn_f32<4>(g, X, f_in, W, f_out, bias, act, out, ws, st);
        case 64: return gcn_f32<2>(g, X, f_in, W, f_out, bias, act, out, ws, st);
        case 32:
        case 16: return gcn_f32<1>(g, X, f_in, W, f_out, bias, act, out, ws, st);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_gat_edge(const GraphDev &g, const __nv_bfloat16 *z, const float *el, const float *er,
                            const GatSoftmaxWs &sw, float slope, __nv_bfloat16 *out, AggWorkspace ws,
                            cudaStream_t st) {
    // With the aggregation view (the GEMM epilogue has written ELU(z) of the
    // rows whose only in-edge is the self-loop, and 0 for rows without one) the
    // kernel runs over the other rows only: C3 gat_edge 205 -> 183 us for +9 us
    // of GEMM output stores (round 1 kernel, online softmax).
    if (g.n == 0) return cudaSuccess;
    cudaError_t e = launch(k_gat_maxel, 1, 32, 0, st, (const float *)sw.parts, sw.nparts, sw.Mh);
    if (e) return e;
    if (g.arow)
        return run<8, 5>(view_agg_fine(g),
                         GatShiftOp<true>{z, el, er, sw.Mh, slope, out, g.arow, g.row_ptr, g.col_src}, ws, st);
    return run<8, 5>(view_fine(g), GatShiftOp<false>{z, el, er, sw.Mh, slope, out, nullptr, g.row_ptr, g.col_src},
                     ws, st);
}

cudaError_t launch_agg_typed_f32(const GraphDev &g, const float *H, int32_t f, float *S, bool mean, double *Sx,
                                 AggWorkspace ws, cudaStream_t st) {
    if (f != 128) return cudaErrorInvalidValue;
    const GraphView gv = g.trow_ptr ? view_typed(g) : view(g);  // no edge types: T = 1
    // U = 4 at 64 registers: measured 3-4% faster than U = 8 (C4, C6), and
    // U = 8 needs more registers (spills at 64, 15% slower at 3 blocks/SM)
    const float *scale = mean ? (g.trow_ptr ? g.tinv_deg : g.inv_deg) : nullptr;
    const int32_t T = g.trow_ptr ? g.num_etypes : 1;
    if (Sx) return run<4, 4>(gv, SumF32Op<true>{H, scale, S, g.heavy_slot, Sx, T}, ws, st);
    return run<4, 4>(gv, SumF32Op<false>{H, scale, S, nullptr, nullptr, T}, ws, st);
}

cudaError_t launch_agg_edge_mlp_f32(const GraphDev &g, const float *AB, int32_t f, bool relu, bool max, float *m,
                                    const double *Bx, double *mx, AggWorkspace ws, cudaStream_t st) {
    if (f != 128) return cudaErrorInvalidValue;
    const int32_t *hs = g.heavy_slot;
    if (max) {
        if (relu) return run<4, 4>(view(g), EdgeMlpOp<true, true>{AB, m, hs, Bx, mx}, ws, st);
        return run<4, 4>(view(g), EdgeMlpOp<true, false>{AB, m, hs, Bx, mx}, ws, st);
    }
    if (relu) return run<4, 4>(view(g), EdgeMlpOp<false, true>{AB, m, hs, Bx, mx}, ws, st);
    return run<4, 4>(view(g), EdgeMlpOp<false, false>{AB, m, hs, Bx, mx}, ws, st);
}

bool gcn_f32_rowwise(const GraphDev &g) { return g.ell != nullptr; }

}  // namespace saga
