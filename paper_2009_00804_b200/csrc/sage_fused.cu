// sage_fused.cu -- SURVEY.md 8(f) NEXT-1: the aggregation fused with its
// tcgen05 GEMM for GraphSAGE-mean (config C2):
//   out[v] = act([x[v] || mean_{u->v} x[u]] . W + b)      (reading A11)
// in ONE kernel, so the mean rows never travel through HBM/L2 and the layer
// is one launch instead of two.
//
// Paper: the paper's forward-looking design asks for "fine-grained pipelining
// of stages" between Gather and the ApplyVertex GEMM (PAPER.md lines
// 474-475); Table 1 line 180 fixes the GraphSAGE stages.
//
// Persistent, one CTA (32 warps) per SM looping over 128-row tiles of
// destinations:
//   * W^T (pre-staged once per call as the exact shared-memory image, K-major,
//     128-byte swizzle) arrives once per CTA by one bulk copy; the self half
//     of the A operand (the tile's x rows, K = 0..127) by TMA per tile;
//   * the 32 warps split the tile's items (edges + row ends) by merge-path,
//     reduce bf16 rows with FHADD.BF16 in fp32 (U = 8 rows in flight per
//     warp, the aggregate.cu engine's batch/park scheme), scale by 1/deg and
//     write each mean row as bf16 straight into the A operand's second half
//     (K = 128..255) in the swizzled layout; rows split between warps leave
//     fp32 partials in shared memory, merged after a barrier in warp order
//     (deterministic);
//   * one thread issues the 16 tcgen05.mma (M = 128, N = Fo, K = 16) into
//     TMEM; every warp then drains a 32-row x Fo/4 block: bias, act, bf16,
//     stored to out.
// Supported: in = 128, out in {64, 128} (C2's two layers); other widths use
// the two-kernel path (aggregate.cu + gemm_tc.cu).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.cuh"
#include "ptx.cuh"

namespace saga {
namespace {

constexpr int kWarps = 32;
constexpr int kThreads = 32 * kWarps;
constexpr int kRows = 128;           // tile rows = UMMA M
constexpr int kF = 128;              // input width (4 bf16 per lane)
constexpr int kU = 8;                // rows in flight per warp
constexpr int kChunk = kRows * 128;  // one 64-column K chunk of A (16 KB)
constexpr uint32_t kFull = 0xffffffffu;

template <int FO>
struct Smem {
    static constexpr int kA = 0;                                // A: 4 K chunks (x: 0, 1; mean: 2, 3)
    static constexpr int kB = kA + 4 * kChunk;                  // W^T image: 4 K chunks of FO rows
    static constexpr int kBBytes = 4 * FO * 128;
    static constexpr int kPart = kB + kBBytes;                  // [warp][head, tail][lane] float4
    static constexpr int kPark = kPart + kWarps * 2 * 32 * 16;  // [warp][u][lane] uint2
    static constexpr int kRend = kPark + kWarps * kU * 32 * 8;  // row_ptr[r0 .. r0 + 128] (int32)
    static constexpr int kRinv = kRend + (kRows + 1) * 4 + 12;  // 1/deg
    static constexpr int kMisc = kRinv + kRows * 4;             // head_row, tail_row [warp], barriers, tmem
    static constexpr int kBytes = kMisc + 2 * kWarps * 4 + 32 + 1024;  // + alignment slack
    static_assert(kBytes <= 232448, "shared memory");
};

// 8 bytes (4 bf16 of the mean row, columns 4*lane .. 4*lane+3) into the A
// operand's mean half: column k = 128 + 4 lane -> chunk 2 + lane / 16,
// 16-byte unit (lane % 16) / 2 XOR (row % 8), half (lane % 2).
__device__ __forceinline__ void put_mean(uint8_t *A, int r, int lane, const float (&m)[4]) {
    const int chunk = 2 + (lane >> 4), unit = (lane & 15) >> 1;
    uint8_t *p = A + chunk * kChunk + r * 128 + ((unit ^ (r & 7)) << 4) + (lane & 1) * 8;
    *reinterpret_cast<uint2 *>(p) = make_uint2(ptx::pack_bf16x2(m[0], m[1]), ptx::pack_bf16x2(m[2], m[3]));
}

template <int FO>
__global__ void __launch_bounds__(kThreads, 1)
    k_sage_fused(const __grid_constant__ CUtensorMap tmX, int32_t n, const int64_t *__restrict__ row_ptr,
                 const int32_t *__restrict__ col_src, const float *__restrict__ inv_deg,
                 const __nv_bfloat16 *__restrict__ X, const uint8_t *__restrict__ wt_image,
                 const float *__restrict__ bias, int act, __nv_bfloat16 *__restrict__ out) {
    using S = Smem<FO>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    griddep_wait();  // the W^T image comes from k_stage_wt
    uint8_t *A = sm + S::kA;
    uint8_t *B = sm + S::kB;
    float4 *part = reinterpret_cast<float4 *>(sm + S::kPart);
    uint2 *park = reinterpret_cast<uint2 *>(sm + S::kPark);
    int32_t *rend = reinterpret_cast<int32_t *>(sm + S::kRend);
    float *rinv = reinterpret_cast<float *>(sm + S::kRinv);
    int32_t *head_row = reinterpret_cast<int32_t *>(sm + S::kMisc);
    int32_t *tail_row = head_row + kWarps;
    uint64_t *bar_w = reinterpret_cast<uint64_t *>(tail_row + kWarps);
    uint64_t *bar_x = bar_w + 1;
    uint64_t *bar_mma = bar_w + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar_w + 3);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int32_t ntiles = (n + kRows - 1) / kRows;

    if (threadIdx.x == 0) {
        ptx::mbar_init(bar_w, 1);
        ptx::mbar_init(bar_x, 1);
        ptx::mbar_init(bar_mma, 1);
        ptx::fence_mbar_init();
        ptx::prefetch_tmap(&tmX);
    }
    if (warp == 0) ptx::tmem_alloc<FO>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) {  // W^T image: once per CTA
        ptx::mbar_arrive_expect_tx(bar_w, S::kBBytes);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                ptx::smem_u32(B)),
            "l"(wt_image), "r"((uint32_t)S::kBBytes), "r"(ptx::smem_u32(bar_w))
            : "memory");
    }
    const char *xl = reinterpret_cast<const char *>(X) + lane * 8;
    auto load = [&](int32_t u) -> uint2 {
        return __ldg(reinterpret_cast<const uint2 *>(ptx::mad_wide((uint32_t)u, 2u * kF, xl)));
    };

    uint32_t it = 0;
    for (int32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int32_t r0 = tile * kRows;
        const int nrows = min(kRows, n - r0);
        // the previous tile's MMA has retired (its epilogue waited for it) and
        // every warp is past its epilogue: A and the row tables are free
        for (int i = threadIdx.x; i <= kRows; i += kThreads) rend[i] = (int32_t)row_ptr[r0 + min(i, nrows)];
        for (int i = threadIdx.x; i < kRows; i += kThreads) rinv[i] = i < nrows ? __ldg(inv_deg + r0 + i) : 0.0f;
        if (threadIdx.x < kWarps) head_row[threadIdx.x] = tail_row[threadIdx.x] = -1;
        if (threadIdx.x == 0) {  // the tile's x rows (self half), in flight during the gather
            ptx::mbar_arrive_expect_tx(bar_x, 2 * kChunk);
            ptx::tma_load_2d(A, &tmX, bar_x, 0, r0, ptx::policy_evict_normal());
            ptx::tma_load_2d(A + kChunk, &tmX, bar_x, 64, r0, ptx::policy_evict_normal());
        }
        __syncthreads();

        // -------------------------------------------- gather: merge-path --
        const int32_t E0 = rend[0], E1 = rend[nrows];
        const int32_t items = (E1 - E0) + nrows;
        const int32_t T = (items + kWarps - 1) / kWarps;
        auto coord = [&](int32_t d, int32_t &row, int32_t &edge) {  // row = #rows whose end item < d
            int32_t lo = 0, hi = nrows;
            while (lo < hi) {
                const int32_t mid = (lo + hi) >> 1;
                if ((rend[mid + 1] - E0) + mid >= d)
                    hi = mid;
                else
                    lo = mid + 1;
            }
            row = lo;
            edge = E0 + d - lo;
        };
        int32_t v, p, v1, p1;
        coord(min(warp * T, items), v, p);
        coord(min((warp + 1) * T, items), v1, p1);
        const int32_t v0 = v;
        bool head_open = v < nrows && rend[v] < p;
        const bool head = head_open;
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        int32_t row_end = v < nrows ? rend[v + 1] : E1;

        auto flush = [&]() {
            if (head_open) {
                part[(warp * 2 + 0) * 32 + lane] = make_float4(acc[0], acc[1], acc[2], acc[3]);
                if (lane == 0) head_row[warp] = v;
                head_open = false;
            } else {
                const float sc = rinv[v];
                const float m[4] = {acc[0] * sc, acc[1] * sc, acc[2] * sc, acc[3] * sc};
                put_mean(A, v, lane, m);
            }
            ++v;
            row_end = v < nrows ? rend[v + 1] : E1;
            acc[0] = acc[1] = acc[2] = acc[3] = 0.f;
        };
        auto add = [&](const uint2 &x) {
            ptx::add_bf16x2_f32(acc[0], acc[1], x.x);
            ptx::add_bf16x2_f32(acc[2], acc[3], x.y);
        };
        // sources in coalesced 32-edge chunks, two chunks ahead; batches start
        // at p + multiple of kU and kU | 32, so a batch never straddles a chunk
        int32_t cb = p;
        auto load_cs = [&](int32_t base) -> int32_t { return base + lane < p1 ? __ldg(col_src + base + lane) : 0; };
        int32_t cs_a = load_cs(cb), cs_b = load_cs(cb + 32), cs_c = load_cs(cb + 64);
        auto slide = [&](int32_t qq) {
            if (qq - cb >= 32) {
                cb += 32;
                cs_a = cs_b;
                cs_b = cs_c;
                cs_c = load_cs(cb + 64);
            }
        };
        while (v < v1 && row_end <= p) flush();
        int32_t q = p;
        for (; q + kU <= p1; q += kU) {
            slide(q);
            const int base = q - cb;
            uint2 val[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) val[u] = load(__shfl_sync(kFull, cs_a, base + u));
            if (row_end > q + kU) {
#pragma unroll
                for (int u = 0; u < kU; ++u) add(val[u]);
            } else {
                uint2 *pk = park + warp * kU * 32;
#pragma unroll
                for (int u = 0; u < kU; ++u) pk[u * 32 + lane] = val[u];
#pragma unroll 1
                for (int u = 0; u < kU; ++u) {
                    add(pk[u * 32 + lane]);
                    while (v < v1 && row_end == q + u + 1) flush();
                }
            }
        }
        for (; q < p1; ++q) {
            slide(q);
            add(load(__shfl_sync(kFull, cs_a, q - cb)));
            while (v < v1 && row_end == q + 1) flush();
        }
        while (v < v1) flush();
        if (v < nrows && p1 > rend[v]) {  // row v has edges in this range and continues past it
            const int slot = (head && v == v0) ? 0 : 1;  // 0: the whole range inside a row begun earlier
            part[(warp * 2 + slot) * 32 + lane] = make_float4(acc[0], acc[1], acc[2], acc[3]);
            if (lane == 0) (slot ? tail_row : head_row)[warp] = v;
        }
        __syncthreads();
        // rows split between warps: the warp holding the row's start merges, in warp order
        {
            const int32_t r = tail_row[warp];
            if (r >= 0) {
                const float4 a = part[(warp * 2 + 1) * 32 + lane];
                float m[4] = {a.x, a.y, a.z, a.w};
                for (int w2 = warp + 1; w2 < kWarps && head_row[w2] == r; ++w2) {
                    const float4 b = part[(w2 * 2 + 0) * 32 + lane];
                    m[0] += b.x; m[1] += b.y; m[2] += b.z; m[3] += b.w;
                }
                const float sc = rinv[r];
                m[0] *= sc; m[1] *= sc; m[2] *= sc; m[3] *= sc;
                put_mean(A, r, lane, m);
            }
        }
        ptx::fence_proxy_async_smem();  // generic smem writes -> visible to the tensor core
        __syncthreads();

        // -------------------------------------------------------- MMA --
        if (threadIdx.x == 0) {
            if (it == 0) ptx::mbar_wait(bar_w, 0);
            ptx::mbar_wait(bar_x, it & 1);
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
        ptx::mbar_wait(bar_mma, it & 1);
        ptx::tc_fence_after();

        // --------------------------------------------------- epilogue --
        // warp -> TMEM lane quarter warp % 4, columns (warp / 4) * FO / 8 ...
        {
            constexpr int kCols = FO / 8;  // 16 (FO = 128) or 8 (FO = 64)
            const int qd = warp & 3, cbk = warp >> 2;
            const int r = qd * 32 + lane;
            const uint32_t taddr = tmem + ((uint32_t)(qd * 32) << 16) + cbk * kCols;
            uint32_t vv[16];
            if constexpr (kCols == 16) {
                ptx::tmem_ld16(taddr, vv);
            } else {
                uint32_t v8[8];
                ptx::tmem_ld8(taddr, v8);
#pragma unroll
                for (int i = 0; i < 8; ++i) vv[i] = v8[i];
            }
            ptx::tmem_ld_wait();
            if (r < nrows) {
                uint32_t pk[kCols / 2];
#pragma unroll
                for (int i = 0; i < kCols / 2; ++i) {
                    const int c0 = cbk * kCols + 2 * i;
                    float a = __uint_as_float(vv[2 * i]) + (bias ? __ldg(bias + c0) : 0.0f);
                    float b = __uint_as_float(vv[2 * i + 1]) + (bias ? __ldg(bias + c0 + 1) : 0.0f);
                    if (act == SAGA_ACT_RELU) {
                        a = fmaxf(a, 0.0f);
                        b = fmaxf(b, 0.0f);
                    }
                    pk[i] = ptx::pack_bf16x2(a, b);
                }
                uint4 *o = reinterpret_cast<uint4 *>(out + (int64_t)(r0 + r) * FO + cbk * kCols);
#pragma unroll
                for (int i = 0; i < kCols / 8; ++i)
                    o[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
            }
        }
        ptx::tc_fence_before();
        __syncthreads();  // TMEM drained, A free for the next tile
        ptx::tc_fence_after();
    }
    if (warp == 0) ptx::tmem_dealloc<FO>(tmem);
}

// W [256][FO] row-major ([x rows; mean rows] x out) -> the shared-memory image
// of W^T: 4 K chunks of FO rows x 128 bytes, 16-byte unit u of row n at
// ((u ^ (n % 8)) << 4) (128-byte swizzle, K-major).
template <int FO>
__global__ void k_stage_wt(const __nv_bfloat16 *__restrict__ W, uint8_t *img) {
    griddep_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;  // over 4 * FO * 8 units
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
                      __nv_bfloat16 *out, void *img, cudaStream_t st, const char **why) {
    cudaError_t e = launch(k_stage_wt<FO>, (4 * FO * 8 + 255) / 256, 256, 0, st, W, static_cast<uint8_t *>(img));
    if (e) return e;
    CUtensorMap tmX;
    if (!make_map_bf16(&tmX, X, g.n, kF)) {
        *why = "cuTensorMapEncodeTiled failed";
        return cudaErrorInvalidValue;
    }
    using S = Smem<FO>;
    e = cudaFuncSetAttribute(k_sage_fused<FO>, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kBytes);
    if (e) return e;
    int dev = 0, sms = kNumSMs;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int ntiles = (g.n + kRows - 1) / kRows;
    const unsigned grid = (unsigned)(ntiles < sms ? ntiles : sms);
    return launch(k_sage_fused<FO>, grid, kThreads, S::kBytes, st, tmX, g.n, g.row_ptr, g.col_src, g.inv_deg, X,
                  static_cast<const uint8_t *>(img), bias, act, out);
}

}  // namespace

bool sage_fused_supported(int32_t in_dim, int32_t out_dim) { return in_dim == kF && (out_dim == 64 || out_dim == 128); }
size_t sage_fused_workspace_bytes(int32_t out_dim) { return (size_t)4 * out_dim * 128; }

cudaError_t launch_sage_fused(const GraphDev &g, const __nv_bfloat16 *X, int32_t in_dim, const __nv_bfloat16 *W,
                              int32_t out_dim, const float *bias, int act, __nv_bfloat16 *out, void *img,
                              cudaStream_t st, const char **why) {
    if (g.n == 0) return cudaSuccess;
    if (!sage_fused_supported(in_dim, out_dim)) {
        *why = "fused SAGE needs in_dim 128, out_dim 64 or 128";
        return cudaErrorInvalidValue;
    }
    if (out_dim == 128) return launch_fo<128>(g, X, W, bias, act, out, img, st, why);
    return launch_fo<64>(g, X, W, bias, act, out, img, st, why);
}

}  // namespace saga
