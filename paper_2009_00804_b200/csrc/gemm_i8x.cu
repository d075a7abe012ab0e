// gemm_i8x.cu -- fp32 GEMM on the int8 tensor cores with EXACT accumulation
// (operands sliced into 8-bit digits, "Ozaki-scheme" style), used for the
// paper-form GGNN's node-level edge-MLP projection (config C8, NEXT-4):
//   AB[M][2f] = H[M][f] . [W_a | W_b] + [0 | b_e]      (f = 128)
// PAPER.md lines 142-147, Table 1 line 178 (ApplyEdge = an MLP on
// [h_src || h_dst]; reading A26): by linearity the per-edge message is
// act(A[u] + B[v]), so the edge MLP's dense work is this one GEMM.
//
// Why not split-TF32 here.  tcgen05's fp32 accumulator does not round to
// nearest: the accumulated result is biased toward zero (measured on B200: a
// mean signed error of -3.8e-7 * sign(A) on A = H W_a, K = 128, split-TF32 and
// cuBLAS TF32 alike: scripts/tc_accum_probe.py, DESIGN.md
// "Precision").  The Gather sums relu(A[u] + B[v]) over all in-edges of v, so
// a bias in A is multiplied by the in-degree: on a 14K-in-edge vertex the
// message m is off by ~5e-3 and the GRU output by ~6e-5 normwise.  An
// unbiased A needs either FFMA (round-to-nearest, ~2x slower here) or exact
// accumulation.  The int8 tensor cores accumulate exactly in s32, so:
//
//  * every row of A (and every column of B, i.e. row of B^T) gets a power-of-
//    two scale 2^e with max|x| < 2^e, and x 2^(22-e) is rounded to the
//    nearest integer X (|X| <= 2^22: 22 significant bits relative to the row
//    maximum, round-to-nearest, so unbiased);
//  * X = s0 2^16 + u1 2^8 + u2 with s0 = X >> 16 in [-64, 64] (signed 8-bit)
//    and u1, u2 in [0, 255] (unsigned 8-bit digits of the two's complement);
//  * sum_k X_a X_b = D0 2^32 + D1 2^24 + D2 2^16 + D3 2^8 + (u2 v2 terms),
//    D0 = sum s0 t0, D1 = sum (s0 v1 + u1 t0), D2 = sum (s0 v2 + u1 v1 + u2 t0),
//    D3 = sum (u1 v2 + u2 v1): 8 kind::i8 MMAs per 32-wide K step into 4 s32
//    TMEM accumulators (exact: |D2| <= 97665 K < 2^31 for K <= 2^14); the
//    dropped u2 v2 term is < 2^-28 of max|a| max|b| per product;
//  * the epilogue forms t = (D0 << 24) + (D1 << 16) + (D2 << 8) + D3 in int64
//    (exact), converts once with round-to-nearest and scales by
//    2^(e_a + e_b - 36): one unbiased rounding per output.
//
// Kernel (persistent, one CTA per SM, 320 threads):
//   warp 0      TMA producer: the three B^T digit planes once (resident), then
//               per 128-row tile the three A digit planes (128-byte swizzle,
//               K = 128 int8 = one swizzle row),
//   warp 1      TMEM owner + single-thread tcgen05.mma.kind::i8 issuer
//               (M = 128, N = 64, K = 32): 8 MMAs per K step,
//   warps 2..9  epilogue: 4 x tcgen05.ld per 16 columns, int64 combine,
//               cvt.rn, scale, bias; coalesced row stores.
// The four accumulators of a 64-column tile take 256 TMEM columns; two tiles
// in flight (512 columns) so the epilogue of one overlaps the MMAs of the
// next.  The digit planes come from k_slice_rows (A) and k_slice_wt (B).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <mutex>

#include "epilogue.cuh"
#include "internal.cuh"
#include "ptx.cuh"

namespace saga {
namespace {

constexpr int kK = 128;                   // K (int8 per plane row = one 128-byte swizzle row)
constexpr int kBM = 128;
constexpr int kBN = 64;                   // output columns per tile (4 accumulators x 64 = 256 TMEM columns)
constexpr int kNT = 256;                  // total output columns (B^T rows), resident
constexpr int kPlaneA = kBM * kK;         // 16 KB
constexpr int kPlaneB = kNT * kK;         // 32 KB
constexpr int kStages = 2;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kSmemBytes = 1024 + 3 * kPlaneB + kStages * 3 * kPlaneA + 4096;

struct alignas(8) Bars {
    uint64_t bfull, afull[kStages], aempty[kStages], tfull[2], tempty[2];
    uint32_t tmem_base;
    int32_t eb[kNT];
    float bias[kNT];
};

// 2^e as a float for e in [-126, 127] (clamped: operands whose scales put the
// product outside the normal range are outside this kernel's contract)
__device__ __forceinline__ float pow2f(int e) {
    e = e < -126 ? -126 : (e > 127 ? 127 : e);
    return __int_as_float((e + 127) << 23);
}

__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_i8x(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int64_t M,
               const int32_t *__restrict__ ea, const int32_t *__restrict__ eb, const float *__restrict__ bias,
               float *__restrict__ out) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *Bs = smem;                      // [3][kNT][kK]
    uint8_t *As = Bs + 3 * kPlaneB;          // [kStages][3][kBM][kK]
    Bars *bar = reinterpret_cast<Bars *>(As + kStages * 3 * kPlaneA);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t m_tiles = (M + kBM - 1) / kBM;
    constexpr int n_tiles = kNT / kBN;

    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar->bfull, 1);
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&bar->afull[s], 1);
            ptx::mbar_init(&bar->aempty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&bar->tfull[a], 1);
            ptx::mbar_init(&bar->tempty[a], 32 * kEpiWarps);
        }
        ptx::fence_mbar_init();
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
    }
    if (warp == 1) ptx::tmem_alloc<512>(&bar->tmem_base);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = bar->tmem_base;

    if (warp == 0) {
        // ============================ TMA producer ============================
        if (lane == 0) {
            griddep_wait();  // the digit planes come from the call's slicing kernels
            ptx::mbar_arrive_expect_tx(&bar->bfull, 3 * kPlaneB);
            for (int p = 0; p < 3; ++p)
                ptx::tma_load_2d(Bs + p * kPlaneB, &tmB, &bar->bfull, 0, p * kNT, ptx::policy_evict_last());
            const uint64_t pol = ptx::policy_evict_first();  // A planes are streamed once
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t t = blockIdx.x; t < m_tiles; t += gridDim.x) {
                ptx::mbar_wait(&bar->aempty[stage], phase ^ 1);
                ptx::mbar_arrive_expect_tx(&bar->afull[stage], 3 * kPlaneA);
                for (int p = 0; p < 3; ++p)
                    ptx::tma_load_2d(As + (stage * 3 + p) * kPlaneA, &tmA, &bar->afull[stage], 0,
                                     (int32_t)(p * M + t * kBM), pol);
                if (++stage == kStages) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == 1) {
        // ============================ MMA issuer ==============================
        if (lane == 0) {
            // (A digit, B digit, accumulator): s0 = digit 0 is signed, u1 / u2 unsigned
            constexpr int kPa[8] = {0, 0, 1, 0, 1, 2, 1, 2};
            constexpr int kPb[8] = {0, 1, 0, 2, 1, 0, 2, 1};
            constexpr int kD[8] = {0, 1, 1, 2, 2, 2, 3, 3};
            ptx::mbar_wait(&bar->bfull, 0);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int64_t t = blockIdx.x; t < m_tiles; t += gridDim.x) {
                ptx::mbar_wait(&bar->afull[stage], phase);
                ptx::tc_fence_after();
                const uint32_t a_base = ptx::smem_u32(As + stage * 3 * kPlaneA);
                const uint32_t b_base = ptx::smem_u32(Bs);
                for (int nt = 0; nt < n_tiles; ++nt, ++it) {
                    const int acc = it & 1;
                    const uint32_t aphase = (it >> 1) & 1;
                    ptx::mbar_wait(&bar->tempty[acc], aphase ^ 1);
                    ptx::tc_fence_after();
                    const uint32_t d = tmem + acc * (4 * kBN);
#pragma unroll
                    for (int k = 0; k < kK / 32; ++k) {
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const uint32_t idesc = ptx::make_idesc_i8(kPa[i] == 0, kPb[i] == 0, kBM, kBN);
                            const uint64_t adesc = ptx::make_sdesc_sw128(a_base + kPa[i] * kPlaneA + k * 32);
                            const uint64_t bdesc =
                                ptx::make_sdesc_sw128(b_base + kPb[i] * kPlaneB + nt * kBN * kK + k * 32);
                            // the first MMA into each accumulator at k = 0 overwrites it
                            const bool first = k == 0 && (i == 0 || i == 1 || i == 3 || i == 6);
                            ptx::umma_i8(d + kD[i] * kBN, adesc, bdesc, idesc, first ? 0u : 1u);
                        }
                    }
                    ptx::umma_commit(&bar->tfull[acc]);
                }
                ptx::umma_commit(&bar->aempty[stage]);  // the A planes are free once these MMAs retire
                if (++stage == kStages) { stage = 0; phase ^= 1; }
            }
        }
    } else {
        // ============================ epilogue ================================
        // warps 2..9: TMEM lane quarter q = warp % 4, column half of the 64-column tile
        const int q = warp & 3;
        const int half = (warp - 2) >> 2;
        const int et = threadIdx.x - 64;
        griddep_wait();  // ea, eb, bias come from the slicing kernels; before this grid's first global write
        for (int i = et; i < kNT; i += 32 * kEpiWarps) {
            bar->eb[i] = eb[i];
            bar->bias[i] = bias ? bias[i] : 0.0f;
        }
        asm volatile("bar.sync 1, %0;" ::"r"(32 * kEpiWarps));
        int it = 0;
        for (int64_t t = blockIdx.x; t < m_tiles; t += gridDim.x) {
            const int64_t row0 = t * kBM + q * 32;
            const int64_t row = row0 + lane;
            const int e_row = row < M ? __ldg(ea + row) : 0;
            for (int nt = 0; nt < n_tiles; ++nt, ++it) {
                const int acc = it & 1;
                const uint32_t aphase = (it >> 1) & 1;
                ptx::mbar_wait(&bar->tfull[acc], aphase);
                ptx::tc_fence_after();
                const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + acc * (4 * kBN);
#pragma unroll 1
                for (int c = 0; c < 2; ++c) {
                    const int cl = half * 32 + c * 16;  // column within the tile
                    uint32_t d0[16], d1[16], d2[16], d3[16];
                    ptx::tmem_ld16(tbase + cl, d0);
                    ptx::tmem_ld16(tbase + kBN + cl, d1);
                    ptx::tmem_ld16(tbase + 2 * kBN + cl, d2);
                    ptx::tmem_ld16(tbase + 3 * kBN + cl, d3);
                    ptx::tmem_ld_wait();
                    float x[16];
                    const int col0 = nt * kBN + cl;
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const long long tt = ((long long)(int32_t)d0[j] << 24) + ((long long)(int32_t)d1[j] << 16) +
                                             ((long long)(int32_t)d2[j] << 8) + (long long)(int32_t)d3[j];
                        const int s = e_row + bar->eb[col0 + j] - 36;
                        const int s1 = s / 2;  // two steps keep each factor normal
                        x[j] = __ll2float_rn(tt) * pow2f(s1) * pow2f(s - s1) + bar->bias[col0 + j];
                    }
                    epi::store_rows_coalesced<4>(x, out, kNT, row0, col0, M, lane);
                }
                ptx::tc_fence_before();
                ptx::mbar_arrive(&bar->tempty[acc]);
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem);
    }
}

// Digits of one 128-wide row (a warp; lane l holds elements 4l .. 4l+3):
// planes[p][row][k] = digit p of X = rint(x 2^(22 - e)), e = the row's scale.
__device__ __forceinline__ void slice_row(const float4 v, int lane, int8_t *p0, int8_t *p1, int8_t *p2, int32_t *e_out) {
    float mx = fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    int e = 0;
    if (mx > 0.0f) frexpf(mx, &e);  // mx = f 2^e, f in [0.5, 1): mx < 2^e
    const float sc = pow2f(22 - e);
    const float xs[4] = {v.x, v.y, v.z, v.w};
    uint32_t w0 = 0, w1 = 0, w2 = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int32_t X = __float2int_rn(xs[i] * sc);  // |X| <= 2^22
        w0 |= (uint32_t)(uint8_t)(int8_t)(X >> 16) << (8 * i);
        w1 |= (uint32_t)((X >> 8) & 255) << (8 * i);
        w2 |= (uint32_t)(X & 255) << (8 * i);
    }
    reinterpret_cast<uint32_t *>(p0)[lane] = w0;
    reinterpret_cast<uint32_t *>(p1)[lane] = w1;
    reinterpret_cast<uint32_t *>(p2)[lane] = w2;
    if (lane == 0) *e_out = e;
}

// A [M][128] fp32 -> three digit planes [3][M][128] int8 + row scales e[M]
__global__ void k_slice_rows(const float *__restrict__ A, int64_t M, int8_t *__restrict__ planes,
                             int32_t *__restrict__ e) {
    griddep_wait();  // A may come from the call's earlier kernels; planes are read by the next
    const int lane = threadIdx.x & 31;
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < M;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const float4 v = __ldg(reinterpret_cast<const float4 *>(A + r * kK) + lane);
        slice_row(v, lane, planes + r * kK, planes + (M + r) * kK, planes + (2 * M + r) * kK, e + r);
    }
}

// GGNN edge-MLP weights: B^T row n (n < f: column n of W_a = W_e[0:f]; n >= f:
// column n - f of W_b = W_e[f:2f]) -> digit planes [3][2f][f] + column scales,
// and the bias vector [0 | b_e].
__global__ void k_slice_wt_ggnn(const float *__restrict__ W_e, const float *__restrict__ b_e, int8_t *planes,
                                int32_t *e, float *bias2) {
    griddep_wait();
    const int lane = threadIdx.x & 31;
    const int n = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (n >= kNT) return;
    const int half = n / kK, j = n % kK;
    const float *col = W_e + (int64_t)half * kK * kK + j;
    const float4 v = make_float4(col[(4 * lane) * kK], col[(4 * lane + 1) * kK], col[(4 * lane + 2) * kK],
                                 col[(4 * lane + 3) * kK]);
    slice_row(v, lane, planes + n * kK, planes + (kNT + n) * kK, planes + (2 * kNT + n) * kK, e + n);
    if (lane == 0) bias2[n] = (half == 0 || !b_e) ? 0.0f : b_e[j];
}

// ------------------------------------------------------------- host side ----
using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                              const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode_i8() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}

// [rows][128] uint8 row-major, {128, box_rows} box, 128-byte swizzle
bool make_map_u8(CUtensorMap *m, const void *base, int64_t rows, int box_rows) {
    EncodeFn enc = get_encode_i8();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)kK, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)kK};
    cuuint32_t box[2] = {(cuuint32_t)kK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

size_t align256(size_t x) { return (x + 255) / 256 * 256; }

}  // namespace

size_t ggnn_i8_workspace_bytes(int64_t M) {
    return align256(3 * (size_t)M * kK) + align256(4 * (size_t)M) + align256(3 * kNT * kK) + align256(4 * kNT) +
           align256(4 * kNT);
}

cudaError_t launch_ggnn_edge_i8x(int64_t M, int32_t f, const float *H, const float *W_e, const float *b_e, void *ws,
                                 float *AB, cudaStream_t st, const char **why) {
    if (M == 0) return cudaSuccess;
    if (f != kK) {
        *why = "int8-sliced GGNN edge GEMM needs f = 128";
        return cudaErrorInvalidValue;
    }
    uint8_t *w = static_cast<uint8_t *>(ws);
    int8_t *pa = reinterpret_cast<int8_t *>(w);
    w += align256(3 * (size_t)M * kK);
    int32_t *ea = reinterpret_cast<int32_t *>(w);
    w += align256(4 * (size_t)M);
    int8_t *pb = reinterpret_cast<int8_t *>(w);
    w += align256(3 * kNT * kK);
    int32_t *eb = reinterpret_cast<int32_t *>(w);
    w += align256(4 * kNT);
    float *bias2 = reinterpret_cast<float *>(w);
    CUtensorMap ma, mb;
    if (!make_map_u8(&ma, pa, 3 * M, kBM) || !make_map_u8(&mb, pb, 3 * kNT, kNT)) {
        *why = "cuTensorMapEncodeTiled failed";
        return cudaErrorInvalidValue;
    }
    cudaError_t e = launch(k_slice_wt_ggnn, kNT * 32 / 256, 256, 0, st, W_e, b_e, pb, eb, bias2);
    if (e) return e;
    const int64_t warps = M;
    const unsigned sgrid = (unsigned)std::min<int64_t>((warps * 32 + 255) / 256, (int64_t)kNumSMs * 16);
    e = launch(k_slice_rows, sgrid, 256, 0, st, H, M, pa, ea);
    if (e) return e;
    e = cudaFuncSetAttribute(k_gemm_i8x, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e) return e;
    int dev = 0, sms = kNumSMs;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t m_tiles = (M + kBM - 1) / kBM;
    const unsigned grid = (unsigned)(m_tiles < sms ? m_tiles : sms);
    return launch(k_gemm_i8x, grid, kThreads, kSmemBytes, st, ma, mb, M, (const int32_t *)ea, (const int32_t *)eb,
                  (const float *)bias2, AB);
}

}  // namespace saga
