// gcn_fused.cu -- SURVEY.md 8(f) NEXT-1 for the GCN layer at scale (config C5):
// the aggregation fused with its tcgen05 GEMM in SAGA order (aggregate first),
//   out[v] = act((dinv[v] * sum_{u->v} dinv[u] x[u]) . W + b)      (reading A1)
// in ONE kernel: no pre-projected Y = X W (2 GiB at C5) is written to HBM and
// read back, and the layer is one launch instead of three.
//
// Paper: "fine-grained pipelining the different stages" between Gather and the
// ApplyVertex GEMM; Table 1 line 177 fixes the GCN
// stages (Scatter: source features, ApplyEdge: the normalisation weight,
// Gather: sum, ApplyVertex: GEMM + ReLU).
//
// Persistent, one CTA (32 warps, 64 registers per thread) per SM; 128-row
// tiles of destinations are dealt dynamically (an atomic tile counter, fetched
// two tiles ahead), because a tile's work varies by 10^2x on a power-law
// graph.  The dependent cold loads at a tile's start (row_ptr -> col_src ->
// rows) are taken off the critical path: the next tile's row tables travel in
// registers during this tile's gather, and each warp plans its share of the
// next tile and issues its first col_src chunks before the barrier that
// precedes this tile's MMA.
//   * W^T (pre-staged once per call as the exact shared-memory image, K-major,
//     128-byte swizzle, 128 KB at out = 256) arrives once per CTA by one bulk
//     copy and stays resident;
//   * the 32 warps split the tile's items (edges + row ends) by merge-path,
//     gather 512-byte bf16 rows (one 16-byte load per lane, batches of U = 4
//     rows, each batch prefetched into L2 two batches ahead of its loads) and
//     accumulate dinv[u] * x[u] in fp32 on the mixed-precision FMA (dinv[u]
//     as a bf16 pair); a finished row is scaled by dinv[v], rounded to bf16
//     and written straight into the A operand (64 KB, four 64-column K
//     chunks, swizzled); a row split between warps is merged after a barrier
//     in warp order (deterministic): the warp holding the row's start keeps
//     its part in registers, the others leave theirs in shared memory;
//   * one thread issues the 16 tcgen05.mma (M = 128, N = out, K = 16) into
//     TMEM and the CTA moves on: the next tile's gather waits for the MMA only
//     at its first write into A, and the accumulator is drained (TMEM -> bias,
//     act, bf16 -> out) after that gather, before the next MMA is issued.
// Measured (C5): 7.23 ms against 3.63 ms for the two-kernel path -- the kernel
// is bound by its instruction count ("NEXT-1 for C5"), so
// it is opt-in (opts.fused).
// Supported: in = 256, out in {64, 128, 256}; other shapes use the two-kernel
// path (gemm_tc.cu + aggregate.cu).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "internal.cuh"
#include "ptx.cuh"

#ifndef GF_PROBE
#define GF_PROBE 0  // development timing probes (1: no MMA / epilogue, 2: no row loads); 0 in every build
#endif

namespace saga {
namespace {

constexpr int kWarps = 32;            // 64 registers per thread
constexpr int kThreads = 32 * kWarps;
constexpr int kRows = 128;           // tile rows = UMMA M
constexpr int kF = 256;              // input width (8 bf16 per lane)
constexpr int kU = 4;                // rows per batch
constexpr int kAhead = 2;            // batches prefetched into L2 ahead of the loads
constexpr int kChunk = kRows * 128;  // one 64-column K chunk of A (16 KB)
constexpr uint32_t kFull = 0xffffffffu;

template <int FO>
struct Smem {
    static constexpr int kA = 0;                                 // A: 4 K chunks
    static constexpr int kB = kA + 4 * kChunk;                   // W^T image: 4 K chunks of FO rows
    static constexpr int kBBytes = 4 * FO * 128;
    static constexpr int kPart = kB + kBBytes;                   // [warp][2][lane] float4: the warp's head partial
    static constexpr int kRendStride = kRows + 4;                // int32 per table buffer (129 used)
    static constexpr int kRend = kPart + kWarps * 2 * 32 * 16;  // 2 x row_ptr[r0 .. r0 + 128] (int32)
    static constexpr int kRinv = kRend + 2 * kRendStride * 4;    // 2 x dinv[r0 ..]
    static constexpr int kMisc = kRinv + 2 * kRows * 4;          // head_row [warp], barriers, tmem, tile
    static constexpr int kBytes = kMisc + kWarps * 4 + 64;   // the dynamic window is 1024-byte aligned (checked)
    static_assert(kBytes <= 232448, "shared memory");
};

// 16 bytes (8 bf16 of row r, columns 8 lane .. 8 lane + 7) into the A operand:
// K chunk lane / 8, 16-byte unit (lane % 8) XOR (r % 8).
__device__ __forceinline__ void put_row(uint8_t *A, int r, int lane, const float (&m)[8]) {
    uint8_t *p = A + (lane >> 3) * kChunk + r * 128 + (((lane & 7) ^ (r & 7)) << 4);
    *reinterpret_cast<uint4 *>(p) = make_uint4(ptx::pack_bf16x2(m[0], m[1]), ptx::pack_bf16x2(m[2], m[3]),
                                               ptx::pack_bf16x2(m[4], m[5]), ptx::pack_bf16x2(m[6], m[7]));
}

// lo += w.lo * x.lo, hi += w.hi * x.hi: bf16 x bf16 products accumulated in
// fp32 (sm_100 mixed-precision FMA, one FHFMA.BF16 each, no unpacking).
__device__ __forceinline__ void fma_pair(float &lo, float &hi, uint32_t w, uint32_t x) {
    asm("{\n.reg .b16 wl, wh, xl, xh;\nmov.b32 {wl, wh}, %2;\nmov.b32 {xl, xh}, %3;\n"
        "fma.rn.f32.bf16 %0, wl, xl, %0;\nfma.rn.f32.bf16 %1, wh, xh, %1;\n}"
        : "+f"(lo), "+f"(hi)
        : "r"(w), "r"(x));
}

template <int FO>
__global__ void __launch_bounds__(kThreads, 1)
    k_gcn_fused(int32_t n, const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col_src,
                const float *__restrict__ dinv, const __nv_bfloat16 *__restrict__ X,
                const uint8_t *__restrict__ wt_image, const float *__restrict__ bias, int act,
                __nv_bfloat16 *__restrict__ out, int32_t *tile_ctr) {
    using S = Smem<FO>;
    extern __shared__ __align__(1024) uint8_t sm[];
    if ((ptx::smem_u32(sm) & 1023u) != 0) __trap();  // the swizzled operands need 1024-byte alignment
    griddep_wait();  // the W^T image and the zeroed tile counter come from k_stage_gcn
    uint8_t *A = sm + S::kA;
    uint8_t *B = sm + S::kB;
    float4 *part = reinterpret_cast<float4 *>(sm + S::kPart);
    int32_t *rend2 = reinterpret_cast<int32_t *>(sm + S::kRend);
    float *rinv2 = reinterpret_cast<float *>(sm + S::kRinv);
    int32_t *head_row = reinterpret_cast<int32_t *>(sm + S::kMisc);
    uint64_t *bar_w = reinterpret_cast<uint64_t *>(head_row + kWarps);
    uint64_t *bar_mma = bar_w + 1;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar_w + 2);
    int32_t *tile_slot = reinterpret_cast<int32_t *>(tmem_slot + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int32_t ntiles = (n + kRows - 1) / kRows;

    if (threadIdx.x == 0) {
        ptx::mbar_init(bar_w, 1);
        ptx::mbar_init(bar_mma, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0) ptx::tmem_alloc<FO>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) {  // W^T image: once per CTA
        ptx::mbar_arrive_expect_tx(bar_w, S::kBBytes);
        ptx::bulk_g2s(B, wt_image, (uint32_t)S::kBBytes, bar_w);
    }
    const char *xl = reinterpret_cast<const char *>(X) + lane * 16;
    auto load = [&](int32_t u) -> uint4 {
        return __ldg(reinterpret_cast<const uint4 *>(ptx::mad_wide((uint32_t)u, 2u * kF, xl)));
    };

    // TMEM -> out for the tile whose MMA was committed last: warp -> TMEM lane
    // quarter warp % 4, columns (warp / 4) * FO / (kWarps / 4) ...
    auto epilogue = [&](int32_t r0, int nrows) {
        constexpr int kWq = kWarps / 4 >= 8 ? 8 : (kWarps / 4 >= 4 ? 4 : 2);  // column groups: a power of two
        constexpr int kEpiWarps = 4 * (kWq < FO / 16 ? kWq : FO / 16);
        constexpr int kCols = FO / (kEpiWarps / 4);
        if (warp >= kEpiWarps) return;
        const int qd = warp & 3, cbk = warp >> 2;
        const int r = qd * 32 + lane;
#pragma unroll
        for (int piece = 0; piece < kCols / 16; ++piece) {
            const int c0 = cbk * kCols + piece * 16;
            uint32_t vv[16];
            ptx::tmem_ld16(tmem + ((uint32_t)(qd * 32) << 16) + c0, vv);
            ptx::tmem_ld_wait();
            if (r < nrows) {
                uint32_t pk[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    float a = __uint_as_float(vv[2 * i]) + (bias ? __ldg(bias + c0 + 2 * i) : 0.0f);
                    float b = __uint_as_float(vv[2 * i + 1]) + (bias ? __ldg(bias + c0 + 2 * i + 1) : 0.0f);
                    if (act == SAGA_ACT_RELU) {
                        a = fmaxf(a, 0.0f);
                        b = fmaxf(b, 0.0f);
                    }
                    pk[i] = ptx::pack_bf16x2(a, b);
                }
                uint4 *o = reinterpret_cast<uint4 *>(out + (int64_t)(r0 + r) * FO + c0);
                o[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                o[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
            }
        }
    };

    // A tile's row tables (row_ptr as int32, dinv): thread t holds entry t in
    // registers from the global load until the store into a table buffer.
    auto table_load = [&](int32_t t, int32_t &e_reg, float &d_reg) {
        const int32_t tr0 = t * kRows;
        const int tn = min(kRows, n - tr0);
        const int i = threadIdx.x;
        if (i <= kRows) e_reg = (int32_t)__ldg(row_ptr + tr0 + min(i, tn));
        if (i < kRows) d_reg = i < tn ? __ldg(dinv + tr0 + i) : 0.0f;
    };
    auto table_store = [&](int buf, int32_t e_reg, float d_reg) {
        const int i = threadIdx.x;
        if (i <= kRows) rend2[buf * S::kRendStride + i] = e_reg;
        if (i < kRows) rinv2[buf * kRows + i] = d_reg;
    };
    // A warp's share of a tile's items (edges + row ends, merge-path) and the
    // first three 32-edge chunks of its sources, loaded coalesced.
    auto plan = [&](const int32_t *re, int nr, int32_t &v, int32_t &p, int32_t &v1, int32_t &p1, int32_t &ca,
                    int32_t &cb2, int32_t &cc) {
        const int32_t E0 = re[0];
        const int32_t items = (re[nr] - E0) + nr;
        const int32_t T = (items + kWarps - 1) / kWarps;
        auto coord = [&](int32_t d, int32_t &row, int32_t &edge) {  // row = #rows whose end item < d
            int32_t lo = 0, hi = nr;
            while (lo < hi) {
                const int32_t mid = (lo + hi) >> 1;
                if ((re[mid + 1] - E0) + mid >= d)
                    hi = mid;
                else
                    lo = mid + 1;
            }
            row = lo;
            edge = E0 + d - lo;
        };
        coord(min(warp * T, items), v, p);
        coord(min((warp + 1) * T, items), v1, p1);
        ca = p + lane < p1 ? __ldg(col_src + p + lane) : 0;
        cb2 = p + 32 + lane < p1 ? __ldg(col_src + p + 32 + lane) : 0;
        cc = p + 64 + lane < p1 ? __ldg(col_src + p + 64 + lane) : 0;
    };

    // Tiles: blockIdx.x and blockIdx.x + gridDim.x are this CTA's first two;
    // the rest are dealt from the counter, fetched two tiles ahead.
    int32_t tile = blockIdx.x, tile_next = blockIdx.x + gridDim.x;
    int32_t e_reg = 0;
    float d_reg = 0.0f;
    table_load(tile, e_reg, d_reg);
    table_store(0, e_reg, d_reg);
    if (lane == 0) head_row[warp] = -1;
    __syncthreads();
    int32_t v, p, v1, p1, cs_a, cs_b, cs_c;
    plan(rend2, min(kRows, n - tile * kRows), v, p, v1, p1, cs_a, cs_b, cs_c);
    if (tile_next < ntiles) table_load(tile_next, e_reg, d_reg);

    int32_t prev_r0 = -1;
    int prev_nrows = 0;
    for (uint32_t it = 0;; ++it) {
        const int32_t r0 = tile * kRows;
        const int nrows = min(kRows, n - r0);
        const int32_t *rend = rend2 + (it & 1) * S::kRendStride;
        const float *rinv = rinv2 + (it & 1) * kRows;
        const bool has_next = tile_next < ntiles;
        int32_t nn = 0;
        if (threadIdx.x == 0) nn = 2 * (int32_t)gridDim.x + atomicAdd(tile_ctr, 1);  // used at the tile's end

        // The previous tile's MMA still reads A and its accumulator still sits
        // in TMEM.  Neither is waited for here: the wait moves to this tile's
        // first write into A (a_free), and the accumulator is drained after
        // this tile's gather, when the MMA has long retired (probe: waiting
        // and draining at the tile's top cost 1.5 of 7.25 ms).
        bool a_free = prev_r0 < 0 || GF_PROBE == 1;
        auto wait_a = [&]() {
            if (!a_free) {
                ptx::mbar_wait(bar_mma, (it - 1) & 1);
                ptx::tc_fence_after();
                a_free = true;
            }
        };

        // -------------------------------------------- gather: merge-path --
        // sources (and their dinv) in coalesced 32-edge chunks, two chunks ahead;
        // batches start at p + multiple of kU and kU | 32, so a batch never
        // straddles a chunk
        const int32_t E1 = rend[nrows];
        const int32_t v0 = v;
        int32_t cb = p;
        auto load_cs = [&](int32_t base) -> int32_t { return base + lane < p1 ? __ldg(col_src + base + lane) : 0; };
        // a source's weight dinv[u] as a bf16 pair {w, w}: the products run on the
        // mixed-precision FMA (bf16 x bf16 in fp32, no unpacking).  Rounding
        // the weight to bf16 is the aggregate-first counterpart of the default
        // path's bf16 rounding of Y[u] = dinv[u] (x[u] . W) (reading A17).
        auto wpair = [&](int32_t cs) -> uint32_t {
            const float w = __ldg(dinv + cs);
            return ptx::pack_bf16x2(w, w);
        };
        uint32_t dw_a = wpair(cs_a), dw_b = wpair(cs_b);
        auto slide = [&](int32_t qq) {
            if (qq - cb >= 32) {
                cb += 32;
                cs_a = cs_b;
                dw_a = dw_b;
                cs_b = cs_c;
                dw_b = wpair(cs_b);
                cs_c = load_cs(cb + 64);
            }
        };
        bool head_open = v < nrows && rend[v] < p;
        const bool head = head_open;
        float acc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = 0.f;
        int32_t row_end = v < nrows ? rend[v + 1] : E1;

        auto flush = [&]() {
            if (head_open) {
                float4 *ps = part + warp * 64 + lane;
                ps[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
                ps[32] = make_float4(acc[4], acc[5], acc[6], acc[7]);
                if (lane == 0) head_row[warp] = v;
                head_open = false;
            } else {
                const float sc = rinv[v];
                float m[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) m[i] = acc[i] * sc;
                wait_a();
                put_row(A, v, lane, m);
            }
            ++v;
            row_end = v < nrows ? rend[v + 1] : E1;
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = 0.f;
        };
        auto addw = [&](const uint4 &x, uint32_t w) {
            fma_pair(acc[0], acc[1], w, x.x);
            fma_pair(acc[2], acc[3], w, x.y);
            fma_pair(acc[4], acc[5], w, x.z);
            fma_pair(acc[6], acc[7], w, x.w);
        };
        // A batch of kU edges from qq.  Registers hold one batch (two batches
        // per warp at 16 warps left the compiler moving freshly loaded rows
        // between registers, which waits for each load where it is issued);
        // the DRAM latency is taken by an L2 prefetch of the batch kAhead
        // ahead instead -- one instruction per row, lane i touching bytes
        // 16 i .. 16 i + 15, no register held -- so the loads that fill the
        // registers find their rows in L2.  Every load is unconditional:
        // positions past the range re-read the range's last source with
        // weight zero (a row the accumulator they reach already holds, or an
        // accumulator that is never written).
        const char *xh = reinterpret_cast<const char *>(X) + (lane & 15) * 32;
        auto prefetch = [&](int32_t qq) {  // qq = first edge of the batch to prefetch (a multiple of kU past p)
            const int idx = qq - cb + (lane >> 4);  // < 64: the batch lies in chunk a or b (never straddles)
            const int32_t chunk = qq - cb < 32 ? cs_a : cs_b;
#pragma unroll
            for (int u = 0; u < kU; u += 2) {  // one instruction per two rows: a half-warp covers a row's 16 sectors
                const int32_t s = __shfl_sync(kFull, chunk, (idx + u) & 31);
                asm volatile("prefetch.global.L2 [%0];" ::"l"(ptx::mad_wide((uint32_t)s, 2u * kF, xh)));
            }
        };
        // kPad: the range's last, partial batch (positions past p1 clamped)
        auto batch = [&](int32_t q, auto pad) {
            constexpr bool kPad = decltype(pad)::value;
            slide(q);
            const int base = q - cb;
            const int last = p1 - 1 - cb;
            if constexpr (kAhead > 0)
                if (q + kAhead * kU < p1) prefetch(q + kAhead * kU);
            uint4 val[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u)
#if GF_PROBE == 2  // timing probe (wrong results): everything but the row loads
                val[u] = make_uint4(__shfl_sync(kFull, cs_a, base + u), 0u, 0u, 0u);
#else
                val[u] = load(__shfl_sync(kFull, cs_a, kPad ? min(base + u, last) : base + u));
#endif
            auto weight = [&](int u) -> uint32_t {
                const uint32_t w = __shfl_sync(kFull, dw_a, base + u);
                return kPad ? (q + u < p1 ? w : 0u) : w;
            };
            if (row_end > q + kU) {
#pragma unroll
                for (int u = 0; u < kU; ++u) addw(val[u], weight(u));
            } else {
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    addw(val[u], weight(u));
                    while (v < v1 && row_end == q + u + 1) flush();
                }
            }
        };
        while (v < v1 && row_end <= p) flush();
        if (p < p1) {
#pragma unroll
            for (int a = 1; a < kAhead; ++a)
                if (p + a * kU < p1) prefetch(p + a * kU);
            int32_t q = p;
            for (; q + kU <= p1; q += kU) batch(q, std::false_type{});
            if (q < p1) batch(q, std::true_type{});
        }
        while (v < v1) flush();
        // drain the previous tile's accumulator (TMEM -> out); this tile's MMA
        // is issued only after every warp has passed the two barriers below
        if (prev_r0 >= 0 && GF_PROBE != 1) {
            wait_a();
            epilogue(prev_r0, prev_nrows);
            ptx::tc_fence_before();
        }
        // row v has edges in this range and continues past it: a range wholly
        // inside a row begun earlier leaves a head partial; otherwise this
        // warp holds the row's start and keeps the partial in its registers
        int32_t tail = -1;
        if (v < nrows && p1 > rend[v]) {
            if (head && v == v0) {
                float4 *ps = part + warp * 64 + lane;
                ps[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
                ps[32] = make_float4(acc[4], acc[5], acc[6], acc[7]);
                if (lane == 0) head_row[warp] = v;
            } else {
                tail = v;
            }
        }
        // the next tile's tables (in registers since the previous tile's end)
        if (has_next) table_store((it + 1) & 1, e_reg, d_reg);
        __syncthreads();
        // rows split between warps: the warp holding the row's start merges, in warp order
        if (tail >= 0) {
            for (int w2 = warp + 1; w2 < kWarps && head_row[w2] == tail; ++w2) {
                const float4 *pb = part + w2 * 64 + lane;
                const float4 b0 = pb[0], b1 = pb[32];
                acc[0] += b0.x; acc[1] += b0.y; acc[2] += b0.z; acc[3] += b0.w;
                acc[4] += b1.x; acc[5] += b1.y; acc[6] += b1.z; acc[7] += b1.w;
            }
            const float sc = rinv[tail];
            float m[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) m[i] = acc[i] * sc;
            put_row(A, tail, lane, m);
        }
        ptx::fence_proxy_async_smem();  // generic smem writes -> visible to the tensor core
        // the next tile's share and its first source chunks: in flight across
        // the barrier, the MMA issue and the epilogue
        if (has_next)
            plan(rend2 + ((it + 1) & 1) * S::kRendStride, min(kRows, n - tile_next * kRows), v, p, v1, p1, cs_a, cs_b,
                 cs_c);
        if (threadIdx.x == 0) *tile_slot = nn;
        __syncthreads();

        // -------------------------------------------------------- MMA --
        if (threadIdx.x == 0 && GF_PROBE != 1) {  // (GF_PROBE 1, timing probe: no MMA, no epilogue)
            if (it == 0) ptx::mbar_wait(bar_w, 0);
            ptx::tc_fence_after();
            constexpr uint32_t idesc = ptx::make_idesc(1 /*BF16*/, kRows, FO);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const uint32_t a_base = ptx::smem_u32(A + c * kChunk), b_base = ptx::smem_u32(B + c * FO * 128);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    ptx::umma_f16(tmem, ptx::make_sdesc_sw128(a_base + k * 32), ptx::make_sdesc_sw128(b_base + k * 32),
                                  idesc, (c | k) != 0);
            }
            ptx::umma_commit(bar_mma);
        }
        prev_r0 = r0;
        prev_nrows = nrows;
        if (lane == 0) head_row[warp] = -1;  // every merge is past the barrier
        if (!has_next) {
            if (GF_PROBE != 1) {
                ptx::mbar_wait(bar_mma, it & 1);
                ptx::tc_fence_after();
                epilogue(prev_r0, prev_nrows);
                ptx::tc_fence_before();
            } else if (threadIdx.x == 0) {
                ptx::mbar_wait(bar_w, 0);  // the weight image's bulk copy must land before the CTA exits
            }
            break;
        }
        tile = tile_next;
        tile_next = *tile_slot;
        if (tile_next < ntiles) table_load(tile_next, e_reg, d_reg);
    }
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 0) ptx::tmem_dealloc<FO>(tmem);
}

// W [256][FO] row-major -> the shared-memory image of W^T: 4 K chunks of FO
// rows x 128 bytes, 16-byte unit u of row n at ((u ^ (n % 8)) << 4) (128-byte
// swizzle, K-major); also resets the tile counter the fused kernel deals from.
template <int FO>
__global__ void k_stage_gcn(const __nv_bfloat16 *__restrict__ W, uint8_t *img, int32_t *tile_ctr) {
    griddep_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;  // over 4 * FO * 8 units
    if (i == 0) *tile_ctr = 0;
    if (i >= 4 * FO * 8) return;
    const int u = i % 8, nn = (i / 8) % FO, c = i / (8 * FO);
    uint32_t w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int k = c * 64 + u * 8 + 2 * e;
        w[e] = (uint32_t)__bfloat16_as_ushort(W[(int64_t)k * FO + nn]) |
               ((uint32_t)__bfloat16_as_ushort(W[(int64_t)(k + 1) * FO + nn]) << 16);
    }
    *reinterpret_cast<uint4 *>(img + c * FO * 128 + nn * 128 + ((u ^ (nn & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
}

template <int FO>
cudaError_t launch_fo(const GraphDev &g, const __nv_bfloat16 *X, const __nv_bfloat16 *W, const float *bias, int act,
                      __nv_bfloat16 *out, void *ws, cudaStream_t st) {
    uint8_t *img = static_cast<uint8_t *>(ws);
    int32_t *ctr = reinterpret_cast<int32_t *>(img + (size_t)4 * FO * 128);
    cudaError_t e = launch(k_stage_gcn<FO>, (4 * FO * 8 + 255) / 256, 256, 0, st, W, img, ctr);
    if (e) return e;
    using S = Smem<FO>;
    e = cudaFuncSetAttribute(k_gcn_fused<FO>, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kBytes);
    if (e) return e;
    int dev = 0, sms = kNumSMs;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int ntiles = (g.n + kRows - 1) / kRows;
    const unsigned grid = (unsigned)(ntiles < sms ? ntiles : sms);
    return launch(k_gcn_fused<FO>, grid, kThreads, S::kBytes, st, g.n, g.row_ptr, g.col_src, g.dinv, X,
                  static_cast<const uint8_t *>(img), bias, act, out, ctr);
}

}  // namespace

bool gcn_fused_supported(int32_t in_dim, int32_t out_dim) {
    return in_dim == kF && (out_dim == 64 || out_dim == 128 || out_dim == 256);
}
// [W^T image | tile counter]
size_t gcn_fused_workspace_bytes(int32_t out_dim) { return (size_t)4 * out_dim * 128 + 16; }

cudaError_t launch_gcn_fused(const GraphDev &g, const __nv_bfloat16 *X, int32_t in_dim, const __nv_bfloat16 *W,
                             int32_t out_dim, const float *bias, int act, __nv_bfloat16 *out, void *ws,
                             cudaStream_t st, const char **why) {
    if (g.n == 0) return cudaSuccess;
    if (!gcn_fused_supported(in_dim, out_dim)) {
        *why = "fused GCN needs in_dim 256, out_dim 64, 128 or 256";
        return cudaErrorInvalidValue;
    }
    if (g.e >= (int64_t(1) << 31) - 64) {
        *why = "fused GCN indexes edges with 32 bits";
        return cudaErrorInvalidValue;
    }
    if (out_dim == 256) return launch_fo<256>(g, X, W, bias, act, out, ws, st);
    if (out_dim == 128) return launch_fo<128>(g, X, W, bias, act, out, ws, st);
    return launch_fo<64>(g, X, W, bias, act, out, ws, st);
}

}  // namespace saga
