// gemm_tf32split.cu -- fp32-accurate ApplyEdge-by-type + ApplyVertex GRU for the
// gated layer (config C4) on the 5th-gen tensor cores.
//
// Paper: GGNN's ApplyVertex is a GRU over the gathered message and the
// vertex's own embedding (Table 1); the
// per-edge-type message weight is applied after Gather by linearity
// (sum_e H[u] W_t(e) = sum_t S_t W_t).  Two GEMMs:
//   messages:  m[M][128]   = [S_0 || .. || S_{T-1}] . [W_0; ..; W_{T-1}]   (K = 128 T)
//   gates:     G[M][4x128] = [m || h] . B_gru  with, per hidden unit j, the
//              columns gin_j (m rows only), r_j, z_j (K = 256), ghn_j (h rows
//              only) -- the MMAs skip the two zero blocks (N = 192 per K half)
//              -- followed by the PyTorch-GRUCell epilogue (reading A15):
//              h' = (1 - z) tanh(gin + b_in + r (ghn + b_hn)) + z h.
// The fp32 tolerance (1e-4) rules out single-pass TF32 (~3e-4 normwise), so
// every operand is split x = x_hi + x_lo with x_hi = tf32(x) and x_lo =
// tf32(x - x_hi) (both round-to-nearest: 22 significant bits, residual
// <= 2^-23 |x|) and A.B ~= A_hi.B_hi + A_hi.B_lo + A_lo.B_hi (3xTF32; the
// A_lo.B_lo term changed the measured worst case by < 3%).  Measured worst
// case: 7.0e-5 normwise on a 70K-in-degree hub whose per-type sums reach
// |S| ~ 130 (tests/test_gpu_parity.py zoo "hub70k"); the fp32 FFMA reference
// kernels give 2.0e-5 there.
//
// Kernel (persistent, one CTA per SM, 448 threads):
//   warp 0      TMA producer: per 16-wide K block, the fp32 A tile (128 rows,
//               64-byte swizzle; A may come from two tensors along K) and the
//               pre-split B_hi / B_lo tiles (BN rows of W^T),
//   warp 1      TMEM owner + single-thread tcgen05.mma.kind::tf32 issuer
//               (M = 128, N = BN, K = 8): 3 MMAs per K step,
//   warps 2..5  converters: A tile -> A_hi (in place) + A_lo (elementwise,
//               so the swizzled layout is preserved), fence.proxy.async,
//   warps 6..13 epilogue: tcgen05.ld, then store (messages) or the GRU; two
//               warps per TMEM lane quarter, each half of the tile's columns
//               (with one warp per quarter the GRU epilogue's dependent
//               activations were the kernel's bound: 0.21 ms of 0.29 with
//               every load, conversion and MMA switched off).
// The accumulator is double-buffered in TMEM (2 x BN columns) so the
// epilogue of one tile overlaps the MMAs of the next.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "epilogue.cuh"
#include "internal.cuh"
#include "ptx.cuh"

namespace saga {
namespace {

constexpr int kEpiWarps = 8;                // two per TMEM lane quarter, each half the columns
constexpr int kThreads = 192 + 32 * kEpiWarps;
constexpr int kBM = 128;
// K block: 16 fp32 = one 64-byte swizzle row, so a ring stage (A, A_lo,
// B_hi, B_lo) is half the 128-byte-block size and twice as many K blocks are
// in flight (the per-block producer -> converter -> MMA hand-offs, not the
// bytes, bound the message GEMMs).
constexpr int kBK = 16;
constexpr int kATile = kBM * kBK * 4;       // 8 KB
constexpr int kMaxStages = 8;
constexpr int kSmemLimit = 232448;

enum { EPI_MSG = 0, EPI_GRU = 1 };

template <int BN>
struct Layout {
    static constexpr int kBTile = BN * kBK * 4;                 // one of B_hi / B_lo
    static constexpr int kStage = 2 * kATile + 2 * kBTile;     // A(hi in place), A_lo, B_hi, B_lo
    static constexpr int kStages =
        (kSmemLimit - 2048) / kStage > kMaxStages ? kMaxStages : (kSmemLimit - 2048) / kStage;
    static constexpr int kBytes = 1024 + kStages * kStage + 1024;
    static_assert(kStages >= 2, "need a double-buffered ring");
};

struct alignas(8) Bars {
    uint64_t full[kMaxStages], conv[kMaxStages], empty[kMaxStages], tfull[2], tempty[2];
    uint32_t tmem_base;
};

struct GruEpi {
    const float *h;      // [M][128]
    const float *b_ih;   // [3][128]
    const float *b_hh;   // [3][128]
    float *out;          // [M][128]
    const float *bias;   // EPI_MSG: optional bias [N]
    int relu;            // EPI_MSG: ReLU
};

__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// sigma(x) = 1 / (1 + e^-x) with the approximate reciprocal, tanh(x) = 2 sigma(2x) - 1:
// |error| ~1e-7 absolute.  The GRU epilogue applies them to every gate output
// of every row; with IEEE division and tanhf it was the kernel's bound.
__device__ __forceinline__ float sigmoidf_(float x) { return __fdividef(1.0f, 1.0f + __expf(-x)); }
__device__ __forceinline__ float tanhf_(float x) { return 2.0f * sigmoidf_(2.0f * x) - 1.0f; }

template <int BN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_tf32split(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmA1,
                  const __grid_constant__ CUtensorMap tmBhi, const __grid_constant__ CUtensorMap tmBlo, int64_t M,
                  int KB, int KB0, int n_tiles, float *__restrict__ msg_out, int ld_out, GruEpi gru) {
    using L = Layout<BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Bars *bar = reinterpret_cast<Bars *>(smem + L::kStages * L::kStage);
    auto stage_a = [&](int s) { return smem + s * L::kStage; };
    auto stage_alo = [&](int s) { return smem + s * L::kStage + kATile; };
    auto stage_bhi = [&](int s) { return smem + s * L::kStage + 2 * kATile; };
    auto stage_blo = [&](int s) { return smem + s * L::kStage + 2 * kATile + L::kBTile; };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t m_tiles = (M + kBM - 1) / kBM;
    const int64_t ntiles = m_tiles * n_tiles;

    if (threadIdx.x == 0) {
        for (int s = 0; s < L::kStages; ++s) {
            ptx::mbar_init(&bar->full[s], 1);
            ptx::mbar_init(&bar->conv[s], 128);
            ptx::mbar_init(&bar->empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&bar->tfull[a], 1);
            ptx::mbar_init(&bar->tempty[a], 32 * kEpiWarps);
        }
        ptx::fence_mbar_init();
        ptx::prefetch_tmap(&tmA0);
        ptx::prefetch_tmap(&tmA1);
        ptx::prefetch_tmap(&tmBhi);
        ptx::prefetch_tmap(&tmBlo);
    }
    if (warp == 1) ptx::tmem_alloc<2 * BN>(&bar->tmem_base);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = bar->tmem_base;

    if (warp == 0) {
        // ============================ TMA producer ============================
        if (lane == 0) {
            const uint64_t pol_a = ptx::policy_evict_first();  // A streamed once
            const uint64_t pol_b = ptx::policy_evict_last();   // B re-read by every CTA
            griddep_wait();  // A and the split B come from the call's earlier kernels
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const int32_t m0 = (int32_t)((t / n_tiles) * kBM);
                const int32_t n0 = (int32_t)((t % n_tiles) * BN);
                for (int kb = 0; kb < KB; ++kb) {
                    ptx::mbar_wait(&bar->empty[stage], phase ^ 1);
                    ptx::mbar_arrive_expect_tx(&bar->full[stage], kATile + 2 * L::kBTile);
                    const bool first = kb < KB0;
                    ptx::tma_load_2d(stage_a(stage), first ? &tmA0 : &tmA1, &bar->full[stage],
                                     (first ? kb : kb - KB0) * kBK, m0, pol_a);
                    ptx::tma_load_2d(stage_bhi(stage), &tmBhi, &bar->full[stage], kb * kBK, n0, pol_b);
                    ptx::tma_load_2d(stage_blo(stage), &tmBlo, &bar->full[stage], kb * kBK, n0, pol_b);
                    if (++stage == L::kStages) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ============================ MMA issuer ==============================
        if (lane == 0) {
            constexpr uint32_t idesc = ptx::make_idesc(2 /*TF32*/, kBM, BN);
            // GRU tiles hold columns [gin | r | z | ghn] x 64 units: the m rows
            // of K (kb < KB0) never reach ghn and the h rows never reach gin,
            // so after the first K step (N = 256, which zeroes every column)
            // the m part runs N = 192 over [gin r z] and the h part N = 192
            // over [r z ghn] -- 25% fewer MMAs
            constexpr uint32_t idesc192 = ptx::make_idesc(2 /*TF32*/, kBM, 192);
            constexpr uint32_t kRow64 = 64 * kBK * 4;  // 64 B^T rows (whole 512-B swizzle atoms)
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
                const int acc = it & 1;
                const uint32_t aphase = (it >> 1) & 1;
                ptx::mbar_wait(&bar->tempty[acc], aphase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem + acc * BN;
                for (int kb = 0; kb < KB; ++kb) {
                    ptx::mbar_wait(&bar->conv[stage], phase);
                    ptx::tc_fence_after();
                    const uint32_t ahi = ptx::smem_u32(stage_a(stage)), alo = ptx::smem_u32(stage_alo(stage));
                    const uint32_t bhi = ptx::smem_u32(stage_bhi(stage)), blo = ptx::smem_u32(stage_blo(stage));
#pragma unroll
                    for (int k = 0; k < kBK / 8; ++k) {  // K = 8 tf32 = 32 bytes per MMA
                        const uint32_t off = k * 32;
                        if (EPI == EPI_GRU && (kb | k) != 0) {
                            const bool hpart = kb >= KB0;
                            const uint32_t dd = d + (hpart ? 64 : 0), bo = hpart ? kRow64 : 0;
                            ptx::umma_tf32(dd, ptx::make_sdesc_sw64(ahi + off), ptx::make_sdesc_sw64(bhi + bo + off),
                                           idesc192, 1);
                            ptx::umma_tf32(dd, ptx::make_sdesc_sw64(ahi + off), ptx::make_sdesc_sw64(blo + bo + off),
                                           idesc192, 1);
                            ptx::umma_tf32(dd, ptx::make_sdesc_sw64(alo + off), ptx::make_sdesc_sw64(bhi + bo + off),
                                           idesc192, 1);
                            continue;
                        }
                        ptx::umma_tf32(d, ptx::make_sdesc_sw64(ahi + off), ptx::make_sdesc_sw64(bhi + off), idesc,
                                       (kb | k) != 0);
                        ptx::umma_tf32(d, ptx::make_sdesc_sw64(ahi + off), ptx::make_sdesc_sw64(blo + off), idesc, 1);
                        ptx::umma_tf32(d, ptx::make_sdesc_sw64(alo + off), ptx::make_sdesc_sw64(bhi + off), idesc, 1);
                    }
                    ptx::umma_commit(&bar->empty[stage]);  // frees the stage when these MMAs retire
                    if (++stage == L::kStages) { stage = 0; phase ^= 1; }
                }
                ptx::umma_commit(&bar->tfull[acc]);
            }
        }
    } else if (warp < 6) {
        // ============================ converters ==============================
        const int ct = threadIdx.x - 64;  // 0..127
        int stage = 0;
        uint32_t phase = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            for (int kb = 0; kb < KB; ++kb) {
                ptx::mbar_wait(&bar->full[stage], phase);
                float4 *a = reinterpret_cast<float4 *>(stage_a(stage));
                float4 *lo = reinterpret_cast<float4 *>(stage_alo(stage));
#pragma unroll
                for (int i = 0; i < kATile / 16 / 128; ++i) {
                    const int c = i * 128 + ct;
                    const float4 x = a[c];
                    const float4 h = make_float4(tf32_rna(x.x), tf32_rna(x.y), tf32_rna(x.z), tf32_rna(x.w));
                    a[c] = h;
                    lo[c] = make_float4(tf32_rna(x.x - h.x), tf32_rna(x.y - h.y), tf32_rna(x.z - h.z),
                                        tf32_rna(x.w - h.w));
                }
                ptx::fence_proxy_async_smem();  // generic writes -> visible to the tensor core
                ptx::mbar_arrive(&bar->conv[stage]);
                if (++stage == L::kStages) { stage = 0; phase ^= 1; }
            }
        }
    } else {
        // ============================ epilogue ================================
        // warps 6 .. 6 + kEpiWarps - 1: TMEM lane quarter q = warp % 4, column half
        const int q = warp & 3;       // TMEM lane quarter this warp may access
        const int half = (warp - 6) >> 2;
        const int r = q * 32 + lane;  // row within the tile
        int it = 0;
        griddep_wait();  // before this grid's first global write
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            const int acc = it & 1;
            const uint32_t aphase = (it >> 1) & 1;
            const int64_t row = (t / n_tiles) * kBM + r;
            const int nt = (int)(t % n_tiles);
            ptx::mbar_wait(&bar->tfull[acc], aphase);
            ptx::tc_fence_after();
            const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + acc * BN;
            if (EPI == EPI_MSG) {
#pragma unroll 1
                for (int c = half; c < BN / 32; c += 2) {
                    uint32_t v[32];
                    ptx::tmem_ld32(tbase + c * 32, v);
                    ptx::tmem_ld_wait();
                    const int col0 = nt * BN + c * 32;
                    float x[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        x[j] = __uint_as_float(v[j]) + (gru.bias ? __ldg(gru.bias + col0 + j) : 0.0f);
                        if (gru.relu) x[j] = fmaxf(x[j], 0.0f);
                    }
                    // lane = row holds 32 contiguous columns: transpose 8x8 blocks of
                    // float4 within each 8-lane group so that every store instruction
                    // writes 4 whole 128-byte row segments (one per group) instead of
                    // 32 scattered 16-byte pieces
                    epi::store_rows_coalesced<8>(x, msg_out, ld_out, (t / n_tiles) * kBM + q * 32, col0, M, lane);
                }
            } else {
                // tile columns: [gin | r | z | ghn] x 64 units (unit0 = 64 nt); this warp: 32 units, 16 at a time
#pragma unroll 1
                for (int c = 2 * half; c < 2 * half + 2; ++c) {
                    const int j0 = nt * 64 + c * 16;
                    const int64_t row0 = (t / n_tiles) * kBM + q * 32;
                    float hh[16], o[16];
                    epi::load_rows_coalesced<4>(hh, gru.h, 128, row0, j0, M, lane);
                    uint32_t vr[16], vz[16], vi[16], vh[16];
                    ptx::tmem_ld16(tbase + 64 + c * 16, vr);
                    ptx::tmem_ld16(tbase + 128 + c * 16, vz);
                    ptx::tmem_ld16(tbase + c * 16, vi);
                    ptx::tmem_ld16(tbase + 192 + c * 16, vh);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const float rg = sigmoidf_(__uint_as_float(vr[j]) + __ldg(gru.b_ih + j0 + j) +
                                                   __ldg(gru.b_hh + j0 + j));
                        const float zg = sigmoidf_(__uint_as_float(vz[j]) + __ldg(gru.b_ih + 128 + j0 + j) +
                                                   __ldg(gru.b_hh + 128 + j0 + j));
                        const float n = tanhf_(__uint_as_float(vi[j]) + __ldg(gru.b_ih + 256 + j0 + j) +
                                               rg * (__uint_as_float(vh[j]) + __ldg(gru.b_hh + 256 + j0 + j)));
                        o[j] = (1.0f - zg) * n + zg * hh[j];
                    }
                    epi::store_rows_coalesced<4>(o, gru.out, 128, row0, j0, M, lane);
                }
            }
            ptx::tc_fence_before();
            ptx::mbar_arrive(&bar->tempty[acc]);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<2 * BN>(tmem);
    }
}

// B^T operands in K-major layout, split hi/lo:
//   messages: Bm[n][k] = W_type[k / f][k % f][n]             (N = f, K = T f)
//   gates:    Bg[c][k], c = 256 nt + 64 s + j (unit 64 nt + j; slot s = gin, r, z, ghn),
//             k < f from W_ih, k >= f from W_hh; gin has no h rows, ghn no m rows.
// Gate B^T element (c, k) of the GRU GEMM over [m || h] (layout above).
__device__ __forceinline__ float gru_bt(int f, const float *__restrict__ W_ih, const float *__restrict__ W_hh, int idx) {
    const int c = idx / (2 * f), k = idx % (2 * f);
    const int nt = c / 256, slot = (c % 256) / 64, j = nt * 64 + c % 64;
    const bool from_m = k < f;
    const int kk = from_m ? k : k - f;
    if (slot == 1 || slot == 2)  // r (gate 0), z (gate 1)
        return (from_m ? W_ih : W_hh)[((int64_t)(slot - 1) * f + kk) * f + j];
    if (slot == 0)               // gin: m rows only
        return from_m ? W_ih[((int64_t)2 * f + kk) * f + j] : 0.0f;
    return from_m ? 0.0f : W_hh[((int64_t)2 * f + kk) * f + j];  // ghn: h rows only
}

__global__ void k_split_weights(int f, int T, const float *__restrict__ W_type, const float *__restrict__ W_ih,
                                const float *__restrict__ W_hh, float *bm_hi, float *bm_lo, float *bg_hi,
                                float *bg_lo, double *w64) {
    griddep_wait();
    if (w64)  // the heavy rows' fp64 weights (gru_f64.cu)
        for (int64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < heavy_weights_f64_count(T, false);
             i += gridDim.x * blockDim.x)
            heavy_weights_f64_item(i, T, W_type, W_ih, W_hh, nullptr, w64);
    const int nm = f * T * f, ng = 4 * f * 2 * f;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nm + ng; i += gridDim.x * blockDim.x) {
        float x;
        float *hi, *lo;
        int idx;
        if (i < nm) {
            const int n = i / (T * f), k = i % (T * f);
            x = W_type[((int64_t)(k / f) * f + k % f) * f + n];
            hi = bm_hi; lo = bm_lo; idx = i;
        } else {
            idx = i - nm;
            x = gru_bt(f, W_ih, W_hh, idx);
            hi = bg_hi; lo = bg_lo;
        }
        const float h = tf32_rna(x);
        hi[idx] = h;
        lo[idx] = tf32_rna(x - h);
    }
}

// GGNN (NEXT-4): edge-MLP B^T [2f][f] (rows c < f: W_a = W_e[0:f] columns, c >= f:
// W_b = W_e[f:2f] columns), its bias vector [0 | b_e], and the GRU B^T.
__global__ void k_split_ggnn(int f, const float *__restrict__ W_e, const float *__restrict__ b_e,
                             const float *__restrict__ W_ih, const float *__restrict__ W_hh, float *be_hi,
                             float *be_lo, float *bias2, float *bg_hi, float *bg_lo, double *w64) {
    griddep_wait();
    if (w64)  // the heavy rows' fp64 weights (gru_f64.cu): W_ih, W_hh, W_b = W_e rows f .. 2f-1
        for (int64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < heavy_weights_f64_count(0, true);
             i += gridDim.x * blockDim.x)
            heavy_weights_f64_item(i, 0, nullptr, W_ih, W_hh, W_e + (int64_t)f * f, w64);
    const int ne = 2 * f * f, ng = 4 * f * 2 * f;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ne + ng + 2 * f; i += gridDim.x * blockDim.x) {
        if (i >= ne + ng) {
            const int c = i - ne - ng;
            bias2[c] = (c < f || !b_e) ? 0.0f : b_e[c - f];
            continue;
        }
        float x;
        float *hi, *lo;
        int idx;
        if (i < ne) {
            const int c = i / f, k = i % f;
            x = W_e[((int64_t)(c < f ? 0 : f) + k) * f + c % f];
            hi = be_hi; lo = be_lo; idx = i;
        } else {
            idx = i - ne;
            x = gru_bt(f, W_ih, W_hh, idx);
            hi = bg_hi; lo = bg_lo;
        }
        const float h = tf32_rna(x);
        hi[idx] = h;
        lo[idx] = tf32_rna(x - h);
    }
}

// R-GCN B^T in K-major layout, split hi/lo: Br[n][k], k < T f from W_type[k / f][k % f][n],
// k >= T f from W_self[k - T f][n]  (N = f_out = f, K = (T + 1) f).
__global__ void k_split_rgcn(int f, int T, const float *__restrict__ W_type, const float *__restrict__ W_self,
                             float *b_hi, float *b_lo) {
    griddep_wait();
    const int K = (T + 1) * f, total = f * K;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int n = i / K, k = i % K;
        const float x = k < T * f ? W_type[((int64_t)(k / f) * f + k % f) * f + n] : W_self[(int64_t)(k - T * f) * f + n];
        const float h = tf32_rna(x);
        b_hi[i] = h;
        b_lo[i] = tf32_rna(x - h);
    }
}

// ------------------------------------------------------------- host side ----
using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                              const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
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

// 2-D fp32 row-major [rows][cols] (row stride ld floats) with a {kBK, box_rows} box, 64B swizzle.
bool make_map_f32(CUtensorMap *m, const void *base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
    EncodeFn enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
    cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, int EPI>
cudaError_t launch_tf32split(const CUtensorMap &a0, const CUtensorMap &a1, const CUtensorMap &bhi,
                          const CUtensorMap &blo, int64_t M, int KB, int KB0, int n_tiles, float *msg_out, int ld_out,
                          const GruEpi &gru, cudaStream_t st) {
    using L = Layout<BN>;
    // per launch: the attribute is per device, and the call is cheap next to the kernel
    cudaError_t e = cudaFuncSetAttribute(k_gemm_tf32split<BN, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         L::kBytes);
    if (e) return e;
    int dev = 0, sms = kNumSMs;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t ntiles = (M + kBM - 1) / kBM * n_tiles;
    const unsigned grid = (unsigned)(ntiles < sms ? ntiles : sms);
    return launch<false>(k_gemm_tf32split<BN, EPI>, grid, kThreads, L::kBytes, st, a0, a1, bhi, blo, M, KB, KB0, n_tiles,
                  msg_out, ld_out, gru);
}

}  // namespace

size_t rgcn_tc_workspace_floats(int32_t f, int32_t T) { return (size_t)2 * f * (T + 1) * f; }

cudaError_t launch_rgcn_apply_tc(int64_t M, int32_t f, int32_t T, const float *S, const float *H, const float *W_type,
                                 const float *W_self, const float *bias, int act, float *wsplit, float *out,
                                 cudaStream_t st, const char **why) {
    if (M == 0) return cudaSuccess;
    if (f != 128 || T < 1 || T > 4) {
        *why = "tensor-core R-GCN path needs f = 128, 1 <= T <= 4";
        return cudaErrorInvalidValue;
    }
    const int K = (T + 1) * f;
    float *b_hi = wsplit, *b_lo = wsplit + (size_t)f * K;
    cudaError_t e = launch<false>(k_split_rgcn, 256, 256, 0, st, f, T, W_type, W_self, b_hi, b_lo);
    if (e) return e;
    CUtensorMap aS, aH, bh, bl;
    if (!make_map_f32(&aS, S, M, (int64_t)T * f, (int64_t)T * f, kBM) || !make_map_f32(&aH, H, M, f, f, kBM) ||
        !make_map_f32(&bh, b_hi, f, K, K, 128) || !make_map_f32(&bl, b_lo, f, K, K, 128)) {
        *why = "cuTensorMapEncodeTiled failed";
        return cudaErrorInvalidValue;
    }
    GruEpi epi{nullptr, nullptr, nullptr, nullptr, bias, act == SAGA_ACT_RELU};
    return launch_tf32split<128, EPI_MSG>(aS, aH, bh, bl, M, K / kBK, T * f / kBK, 1, out, f, epi, st);
}

size_t gated_tc_workspace_floats(int32_t f, int32_t T) { return (size_t)2 * f * T * f + (size_t)2 * 4 * f * 2 * f; }

cudaError_t launch_gated_apply_tc(int64_t M, int32_t f, int32_t T, const float *S, const float *H,
                                  const float *W_type, const float *W_ih, const float *W_hh, const float *b_ih,
                                  const float *b_hh, float *m_ws, float *wsplit, double *w64, float *out,
                                  cudaStream_t st, const char **why) {
    if (M == 0) return cudaSuccess;
    if (f != 128 || T < 1 || T > 4) {
        *why = "tensor-core gated path needs f = 128, 1 <= T <= 4";
        return cudaErrorInvalidValue;
    }
    float *bm_hi = wsplit, *bm_lo = bm_hi + (size_t)f * T * f;
    float *bg_hi = bm_lo + (size_t)f * T * f, *bg_lo = bg_hi + (size_t)4 * f * 2 * f;
    cudaError_t e = launch<false>(k_split_weights, 256, 256, 0, st, f, T, W_type, W_ih, W_hh, bm_hi, bm_lo, bg_hi, bg_lo,
                                  w64);
    if (e) return e;
    CUtensorMap aS, aM, aH, bmh, bml, bgh, bgl;
    if (!make_map_f32(&aS, S, M, (int64_t)T * f, (int64_t)T * f, kBM) || !make_map_f32(&aM, m_ws, M, f, f, kBM) ||
        !make_map_f32(&aH, H, M, f, f, kBM) || !make_map_f32(&bmh, bm_hi, f, (int64_t)T * f, (int64_t)T * f, 128) ||
        !make_map_f32(&bml, bm_lo, f, (int64_t)T * f, (int64_t)T * f, 128) ||
        !make_map_f32(&bgh, bg_hi, 4 * f, 2 * f, 2 * f, 256) || !make_map_f32(&bgl, bg_lo, 4 * f, 2 * f, 2 * f, 256)) {
        *why = "cuTensorMapEncodeTiled failed";
        return cudaErrorInvalidValue;
    }
    GruEpi none{nullptr, nullptr, nullptr, nullptr, nullptr, 0};
    e = launch_tf32split<128, EPI_MSG>(aS, aS, bmh, bml, M, T * f / kBK, T * f / kBK, 1, m_ws, f, none, st);
    if (e) return e;
    GruEpi gru{H, b_ih, b_hh, out, nullptr, 0};
    return launch_tf32split<256, EPI_GRU>(aM, aH, bgh, bgl, M, 2 * f / kBK, f / kBK, 2, nullptr, 0, gru, st);
}

size_t ggnn_tc_workspace_floats(int32_t f) { return (size_t)2 * 2 * f * f + 2 * f + (size_t)2 * 4 * f * 2 * f; }

// GGNN (NEXT-4): the GRU's split B^T (the edge-MLP projection AB runs on the
// int8-sliced exact-accumulation GEMM, gemm_i8x.cu).
cudaError_t launch_ggnn_split_weights(int32_t f, const float *W_e, const float *b_e, const float *W_ih,
                                      const float *W_hh, float *wsplit, double *w64, cudaStream_t st) {
    float *be_hi = wsplit, *be_lo = be_hi + (size_t)2 * f * f, *bias2 = be_lo + (size_t)2 * f * f;
    float *bg_hi = bias2 + 2 * f, *bg_lo = bg_hi + (size_t)4 * f * 2 * f;
    return launch<false>(k_split_ggnn, 256, 256, 0, st, f, W_e, b_e, W_ih, W_hh, be_hi, be_lo, bias2, bg_hi, bg_lo,
                         w64);
}

cudaError_t launch_ggnn_gru_tc(int64_t M, int32_t f, const float *m, const float *H, const float *b_ih,
                               const float *b_hh, const float *wsplit, float *out, cudaStream_t st, const char **why) {
    if (M == 0) return cudaSuccess;
    const float *bg_hi = wsplit + (size_t)2 * 2 * f * f + 2 * f, *bg_lo = bg_hi + (size_t)4 * f * 2 * f;
    CUtensorMap aM, aH, bgh, bgl;
    if (!make_map_f32(&aM, m, M, f, f, kBM) || !make_map_f32(&aH, H, M, f, f, kBM) ||
        !make_map_f32(&bgh, bg_hi, 4 * f, 2 * f, 2 * f, 256) || !make_map_f32(&bgl, bg_lo, 4 * f, 2 * f, 2 * f, 256)) {
        *why = "cuTensorMapEncodeTiled failed";
        return cudaErrorInvalidValue;
    }
    GruEpi gru{H, b_ih, b_hh, out, nullptr, 0};
    return launch_tf32split<256, EPI_GRU>(aM, aH, bgh, bgl, M, 2 * f / kBK, f / kBK, 2, nullptr, 0, gru, st);
}

}  // namespace saga
