// gemm_tc.cu -- ApplyVertex / pre-projection GEMM on the 5th-gen tensor cores.
//
// Paper: ApplyVertex "can be implemented by GEMM" batched over all vertices
// (Table 3).  Here: out[M][N] = A[M][K] . W
// with bf16 operands and fp32 accumulation, one persistent CTA per SM:
//   warp 0      TMA producer: 128x64 bf16 A tiles (128-byte swizzle) into an
//               S-stage mbarrier ring (A may come from two sources along K:
//               SAGE's [x || mean]),
//   warp 1      TMEM owner + single-thread tcgen05.mma issuer (M=128, N=BN,
//               K=16 per instruction), commits to mbarriers,
//   warps 2..5  epilogue: tcgen05.ld (32 lanes x 32 columns) -> fused
//               row-scale / bias+act / GAT attention dots -> bf16 -> swizzled
//               smem -> TMA store.
// W (K <= 256) stays resident in shared memory in the K-major 128-byte
// swizzled layout for the whole kernel; the accumulator is double-buffered
// in TMEM (2 x BN columns) so the epilogue of tile i overlaps the MMAs of
// tile i+1.  For the configs here the GEMM is HBM-bound (K = 256, arithmetic
// intensity 46-128 FLOP/B < the ~206 FLOP/B ridge), so the design goal is to
// keep A loads and C stores streaming at full bandwidth.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "internal.cuh"
#include "ptx.cuh"

namespace saga {
namespace {

constexpr int kThreads = 192;
constexpr int kBM = 128;
constexpr int kBK = 64;                       // 64 bf16 = 128 bytes = one swizzle row
constexpr int kATileBytes = kBM * kBK * 2;    // 16 KB
constexpr int kCStageBytes = kBM * 64 * 2;    // 16 KB: 128 rows x 64 bf16 columns
constexpr int kSmemLimit = 232448;            // 227 KB opt-in maximum

struct alignas(8) Barriers {
    uint64_t full[8], empty[8], tfull[2], tempty[2], wready;
    uint32_t tmem_base;
    float vec[256];  // epilogue vectors staged once per CTA: bias[BN], or GAT a_src[64] | a_dst[64]
    float red[4][8];  // GAT: the epilogue warps' maxima of el per head
};

template <int BN>
struct Layout {
    static constexpr int kBBytesPerKB = BN * 128;
    static constexpr int kMaxKB = 4;
    static constexpr int kBBytes = kBBytesPerKB * kMaxKB;
    static constexpr int kCBytes = 2 * kCStageBytes;
    static constexpr int kStages =
        (kSmemLimit - 1024 - (int)sizeof(Barriers) - kBBytes - kCBytes) / kATileBytes > 8
            ? 8
            : (kSmemLimit - 1024 - (int)sizeof(Barriers) - kBBytes - kCBytes) / kATileBytes;
    static constexpr int kBytes = 1024 + kBBytes + kStages * kATileBytes + kCBytes + (int)sizeof(Barriers);
    static_assert(kStages >= 2, "not enough shared memory for the A ring");
    static_assert(BN != 256 || kStages >= 4, "the BN = 256 GEMM (C5) keeps a 4-stage A ring");
};

struct EpiParams {
    int epi;
    const float *row_scale;
    const float *bias;
    int act;
    const float *a_src, *a_dst;
    float *el, *er;
    float *elmax;   // GAT: per-CTA maxima of el per head, [gridDim.x][8] (the edge softmax's shift)
    bool self_out;  // GAT: the aggregation view's output tile (GemmArgs::out2; kernel template SELF)
};

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }

__device__ __forceinline__ float act_fn(float x, int act) {
    if (act == SAGA_ACT_RELU) return fmaxf(x, 0.0f);
    if (act == SAGA_ACT_ELU) return x > 0.0f ? x : expm1f(x);
    return x;
}

// EPI (GemmEpi) and SELF (the aggregation view's self-term output tile) are
// compile-time: a runtime epilogue switch let the compiler interleave the
// modes' code and made the C5 GEMM 3.5x slower.
template <int BN, int EPI, bool SELF>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_bf16_tc(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmA1,
                   const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmO,
                   const __nv_bfloat16 *__restrict__ W, int64_t M, int KB, int KB0, EpiParams ep) {
    using L = Layout<BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *Bs = smem;
    uint8_t *As = Bs + L::kBBytes;
    uint8_t *Cs = As + L::kStages * kATileBytes;
    Barriers *bar = reinterpret_cast<Barriers *>(Cs + L::kCBytes);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t ntiles = (M + kBM - 1) / kBM;

    // ---- prologue: barriers, epilogue vectors, TMEM (W is staged by the
    // epilogue warps after the barrier, overlapping the first A loads) ----
    if (threadIdx.x == 0) {
        for (int s = 0; s < L::kStages; ++s) {
            ptx::mbar_init(&bar->full[s], 1);
            ptx::mbar_init(&bar->empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&bar->tfull[a], 1);
            ptx::mbar_init(&bar->tempty[a], 128);
        }
        ptx::mbar_init(&bar->wready, 128);
        ptx::fence_mbar_init();
        ptx::prefetch_tmap(&tmA0);
        ptx::prefetch_tmap(&tmA1);
        ptx::prefetch_tmap(&tmC);
        ptx::prefetch_tmap(&tmO);
    }
    for (int i = threadIdx.x; i < BN; i += kThreads) {
        if constexpr (EPI == EPI_BIAS_ACT) {
            bar->vec[i] = ep.bias ? ep.bias[i] : 0.0f;
        } else if constexpr (EPI == EPI_GAT) {  // BN = 64 here
            bar->vec[i] = ep.a_src[i];
            bar->vec[64 + i] = ep.a_dst[i];
        }
    }
    if (warp == 1) ptx::tmem_alloc<2 * BN>(&bar->tmem_base);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = bar->tmem_base;

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            const uint64_t pol = ptx::policy_evict_first();  // A is streamed once
            griddep_wait();  // A may come from the call's previous kernel
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const int32_t m0 = (int32_t)(t * kBM);
                for (int kb = 0; kb < KB; ++kb) {
                    ptx::mbar_wait(&bar->empty[stage], phase ^ 1);
                    ptx::mbar_arrive_expect_tx(&bar->full[stage], kATileBytes);
                    const bool first = kb < KB0;
                    ptx::tma_load_2d(As + stage * kATileBytes, first ? &tmA0 : &tmA1, &bar->full[stage],
                                     (first ? kb : kb - KB0) * kBK, m0, pol);
                    if (++stage == L::kStages) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            constexpr uint32_t idesc = ptx::make_idesc(1 /*BF16*/, kBM, BN);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            ptx::mbar_wait(&bar->wready, 0);  // W staged by the epilogue warps
            ptx::tc_fence_after();
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
                const int acc = it & 1;
                const uint32_t aphase = (it >> 1) & 1;
                ptx::mbar_wait(&bar->tempty[acc], aphase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem + acc * BN;
                for (int kb = 0; kb < KB; ++kb) {
                    ptx::mbar_wait(&bar->full[stage], phase);
                    ptx::tc_fence_after();
                    const uint32_t a_base = ptx::smem_u32(As + stage * kATileBytes);
                    const uint32_t b_base = ptx::smem_u32(Bs + kb * L::kBBytesPerKB);
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k) {
                        ptx::umma_f16(d, ptx::make_sdesc_sw128(a_base + k * 32), ptx::make_sdesc_sw128(b_base + k * 32),
                                      idesc, (kb | k) != 0);
                    }
                    ptx::umma_commit(&bar->empty[stage]);  // frees the A slot when these MMAs retire
                    if (++stage == L::kStages) { stage = 0; phase ^= 1; }
                }
                ptx::umma_commit(&bar->tfull[acc]);  // accumulator ready for the epilogue
            }
        }
    } else {
        // ===================== epilogue (warps 2..5) =====================
        const int q = warp & 3;            // TMEM lane quarter this warp may access
        const int r = q * 32 + lane;       // row within the tile
        const int et = threadIdx.x - 64;   // 0..127
        {   // W -> shared (K-major, 128-byte swizzle) while the first A tiles load.
            // One unit = an 8(k) x 8(n) block: eight independent 16-byte loads
            // along n (coalesced across threads), a register transpose, eight
            // 16-byte smem stores (one K-major chunk per n).
            if ((reinterpret_cast<uintptr_t>(W) & 15) == 0) {
                const int units = KB * 8 * (BN / 8);
                auto unit_load = [&](int c, uint4 (&v)[8]) {
                    const int n0 = (c % (BN / 8)) * 8;
                    const int k0 = (c / BN) * kBK + ((c / (BN / 8)) % 8) * 8;
#pragma unroll
                    for (int r = 0; r < 8; ++r)
                        v[r] = __ldg(reinterpret_cast<const uint4 *>(W + (int64_t)(k0 + r) * BN + n0));
                };
                auto unit_store = [&](int c, const uint4 (&v)[8]) {
                    const int n0 = (c % (BN / 8)) * 8;
                    const int kc = (c / (BN / 8)) % 8;
                    const int kb = c / BN;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const uint32_t sel = (j & 1) ? 0x7632u : 0x5410u;
                        uint32_t w[4];
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const uint32_t *a = reinterpret_cast<const uint32_t *>(&v[2 * i]);
                            const uint32_t *b = reinterpret_cast<const uint32_t *>(&v[2 * i + 1]);
                            w[i] = __byte_perm(a[j >> 1], b[j >> 1], sel);
                        }
                        const int n = n0 + j;
                        uint8_t *dst = Bs + kb * L::kBBytesPerKB + n * 128 + ((kc ^ (n & 7)) << 4);
                        *reinterpret_cast<uint4 *>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
                    }
                };
                // two units per round: 16 loads in flight per thread
                for (int c = et; c < units; c += 256) {
                    uint4 va[8], vb[8];
                    const bool two = c + 128 < units;
                    unit_load(c, va);
                    if (two) unit_load(c + 128, vb);
                    unit_store(c, va);
                    if (two) unit_store(c + 128, vb);
                }
            } else {
                const int chunks = KB * BN * 8;  // 16-byte chunks: (kb, n, kc)
                for (int c = et; c < chunks; c += 128) {
                    const int n = c % BN;
                    const int kc = (c / BN) % 8;
                    const int kb = c / (BN * 8);
                    const int k0 = kb * kBK + kc * 8;
                    uint32_t w[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        __nv_bfloat16 lo = W[(int64_t)(k0 + 2 * i) * BN + n];
                        __nv_bfloat16 hi = W[(int64_t)(k0 + 2 * i + 1) * BN + n];
                        w[i] = (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
                    }
                    uint8_t *dst = Bs + kb * L::kBBytesPerKB + n * 128 + ((kc ^ (n & 7)) << 4);
                    *reinterpret_cast<uint4 *>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
                }
            }
            ptx::fence_proxy_async_smem();  // generic stores -> visible to UMMA
            ptx::mbar_arrive(&bar->wready);
        }
        griddep_wait();  // before this grid's first global write
        int it = 0;
        uint32_t cstage = 0;
        [[maybe_unused]] float elmx[8];
        if constexpr (EPI == EPI_GAT) {
#pragma unroll
            for (int h = 0; h < 8; ++h) elmx[h] = -INFINITY;
        }
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            const int acc = it & 1;
            const uint32_t aphase = (it >> 1) & 1;
            const int64_t m0 = t * kBM;
            const int64_t row = m0 + r;
            const bool valid = row < M;
            float scale = 1.0f;
            if constexpr (EPI == EPI_ROWSCALE) scale = valid ? __ldg(ep.row_scale + row) : 0.0f;
            // GAT: a row whose only in-edge is its self-loop has one softmax term of
            // weight 1, so its output is ELU(z[v]); a row without in-edges gets 0
            const float gcoef = EPI == EPI_GAT && SELF && valid && __ldg(ep.row_scale + row) > 0.0f ? 1.0f : 0.0f;
            ptx::mbar_wait(&bar->tfull[acc], aphase);
            ptx::tc_fence_after();
            float el[8], er[8];
            if constexpr (EPI == EPI_GAT) {
#pragma unroll
                for (int h = 0; h < 8; ++h) el[h] = er[h] = 0.0f;
            }
#pragma unroll 1
            for (int c64 = 0; c64 < BN / 64; ++c64) {
                if constexpr (SELF) {
                    // GAT with the aggregation view: the z chunk and the output chunk
                    // of EVERY row -- ELU(z[v]) for a row whose only in-edge is its
                    // self-loop (one softmax term of weight 1), 0 for a row with
                    // none, from the same bf16 z the edge kernel would read; the
                    // view's rows overwrite theirs -- staged in the two buffers for
                    // two TMA tile stores (+33 MB at C3, gat_edge 205 -> 183 us).
                    // The same for GCN (act(dinv Y + b)) was measured at C5: the
                    // gather lost 0.6-0.8 ms, the GEMM gained 0.45-0.5 ms of stores
                    // (per-row stores of only the needed rows were slower still:
                    // from the epilogue warps 1.36-1.78 ms, 4 dedicated store warps
                    // 1.41, TMA scatter4 4.0, vs 1.16-1.25 for the tile stores).
                    // the previous tile's two TMA stores have finished reading both
                    // staging buffers before they are overwritten
                    if (et == 0) ptx::bulk_wait_read<0>();
                    named_bar(1, 128);
                    uint32_t yp[32], op[32];
#pragma unroll
                    for (int half = 0; half < 2; ++half) {
                        const int col0 = c64 * 64 + half * 32;
                        uint32_t v[32];
                        ptx::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + acc * BN + col0, v);
                        ptx::tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 32; ++i) {  // BN = 64: el / er from the fp32 accumulators
                            const int h = (half * 32 + i) >> 3;
                            el[h] = fmaf(__uint_as_float(v[i]), bar->vec[col0 + i], el[h]);
                            er[h] = fmaf(__uint_as_float(v[i]), bar->vec[64 + col0 + i], er[h]);
                        }
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const uint32_t y2 =
                                ptx::pack_bf16x2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
                            const float2 f = ptx::unpack_bf16x2(y2);
                            yp[half * 16 + i] = y2;
                            // ELU as the edge kernel's flush (output bf16)
                            const float a = gcoef * f.x, b = gcoef * f.y;
                            op[half * 16 + i] = ptx::pack_bf16x2(a > 0.0f ? a : __expf(a) - 1.0f,
                                                                 b > 0.0f ? b : __expf(b) - 1.0f);
                        }
#pragma unroll
                        for (int c4 = 0; c4 < 4; ++c4) {
                            const int ch = half * 4 + c4, off = r * 128 + ((ch ^ (r & 7)) << 4);
                            const int b = half * 16 + 4 * c4;
                            *reinterpret_cast<uint4 *>(Cs + off) = make_uint4(yp[b], yp[b + 1], yp[b + 2], yp[b + 3]);
                            *reinterpret_cast<uint4 *>(Cs + kCStageBytes + off) =
                                make_uint4(op[b], op[b + 1], op[b + 2], op[b + 3]);
                        }
                    }
                    ptx::fence_proxy_async_smem();
                    named_bar(1, 128);
                    if (et == 0) {
                        ptx::tma_store_2d(&tmC, Cs, c64 * 64, (int32_t)m0);
                        ptx::tma_store_2d(&tmO, Cs + kCStageBytes, c64 * 64, (int32_t)m0);
                        ptx::bulk_commit();
                    }
                    continue;
                }
                uint8_t *stg = Cs + (cstage & 1) * kCStageBytes;
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    const int col0 = c64 * 64 + half * 32;
                    uint32_t v[32];
                    ptx::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + acc * BN + col0, v);
                    ptx::tmem_ld_wait();
                    float x[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) x[i] = __uint_as_float(v[i]);
                    if constexpr (EPI == EPI_ROWSCALE) {
#pragma unroll
                        for (int i = 0; i < 32; ++i) x[i] *= scale;
                    } else if constexpr (EPI == EPI_BIAS_ACT) {
#pragma unroll
                        for (int i = 0; i < 32; ++i) x[i] = act_fn(x[i] + bar->vec[col0 + i], ep.act);
                    } else {  // EPI_GAT: heads of 8 columns; el/er from the fp32 accumulators
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            const int h = (half * 32 + i) >> 3;  // GAT runs with BN = 64 (c64 == 0)
                            el[h] = fmaf(x[i], bar->vec[col0 + i], el[h]);
                            er[h] = fmaf(x[i], bar->vec[64 + col0 + i], er[h]);
                        }
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) {  // 4 x 16-byte chunks = 32 columns
                        uint4 pk = make_uint4(ptx::pack_bf16x2(x[8 * j + 0], x[8 * j + 1]),
                                              ptx::pack_bf16x2(x[8 * j + 2], x[8 * j + 3]),
                                              ptx::pack_bf16x2(x[8 * j + 4], x[8 * j + 5]),
                                              ptx::pack_bf16x2(x[8 * j + 6], x[8 * j + 7]));
                        const int chunk = half * 4 + j;
                        *reinterpret_cast<uint4 *>(stg + r * 128 + ((chunk ^ (r & 7)) << 4)) = pk;
                    }
                }
                ptx::fence_proxy_async_smem();
                named_bar(1, 128);
                if (et == 0) {
                    ptx::tma_store_2d(&tmC, stg, c64 * 64, (int32_t)m0);
                    ptx::bulk_commit();
                    ptx::bulk_wait_read<1>();  // the other staging buffer is free again
                }
                named_bar(1, 128);
                ++cstage;
            }
            // accumulator drained: hand it back to the MMA warp
            ptx::tc_fence_before();
            ptx::mbar_arrive(&bar->tempty[acc]);
            if (EPI == EPI_GAT && valid) {
#pragma unroll
                for (int h = 0; h < 8; ++h) elmx[h] = fmaxf(elmx[h], el[h]);
                float4 *pe = reinterpret_cast<float4 *>(ep.el + row * 8);
                float4 *pr = reinterpret_cast<float4 *>(ep.er + row * 8);
                pe[0] = make_float4(el[0], el[1], el[2], el[3]);
                pe[1] = make_float4(el[4], el[5], el[6], el[7]);
                pr[0] = make_float4(er[0], er[1], er[2], er[3]);
                pr[1] = make_float4(er[4], er[5], er[6], er[7]);
            }
        }
        if constexpr (EPI == EPI_GAT) {
            // this CTA's maximum of el per head -> ep.elmax[blockIdx.x]
#pragma unroll
            for (int h = 0; h < 8; ++h) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) elmx[h] = fmaxf(elmx[h], __shfl_xor_sync(0xffffffffu, elmx[h], o));
            }
            if (lane == 0) {
#pragma unroll
                for (int h = 0; h < 8; ++h) bar->red[q][h] = elmx[h];
            }
            named_bar(1, 128);
            if (et < 8)
                ep.elmax[blockIdx.x * 8 + et] =
                    fmaxf(fmaxf(bar->red[0][et], bar->red[1][et]), fmaxf(bar->red[2][et], bar->red[3][et]));
        }
        if (et == 0) ptx::bulk_wait<0>();
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<2 * BN>(tmem);
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


template <int BN, int EPI, bool SELF>
cudaError_t launch_bn(const GemmArgs &a, const CUtensorMap &m0, const CUtensorMap &m1, const CUtensorMap &mc,
                      const CUtensorMap &mo, int KB, int KB0, const EpiParams &ep, cudaStream_t st) {
    using L = Layout<BN>;
    // per launch: the attribute is per device, and the call is cheap next to the kernel
    cudaError_t e =
        cudaFuncSetAttribute(k_gemm_bf16_tc<BN, EPI, SELF>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kBytes);
    if (e) return e;
    const unsigned grid = (unsigned)gemm_bf16_tc_grid(a.M);
    return launch(k_gemm_bf16_tc<BN, EPI, SELF>, grid, kThreads, L::kBytes, st, m0, m1, mc, mo, a.W, a.M, KB, KB0, ep);
}

}  // namespace

// persistent grid: one CTA per SM, at most one per 128-row tile
int gemm_bf16_tc_grid(int64_t M) {
    int dev = 0, sms = kNumSMs;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t ntiles = (M + kBM - 1) / kBM;
    return (int)(ntiles < sms ? ntiles : sms);
}

// 2-D bf16 row-major [rows][cols] map with a {64 col, box_rows row} box, 128B swizzle.
bool make_map_bf16(CUtensorMap *m, const void *base, int64_t rows, int64_t cols, int box_rows) {  // box_rows <= 256
    EncodeFn enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t launch_gemm_bf16_tc(const GemmArgs &a, cudaStream_t st, const char **why) {
    if (a.M == 0) return cudaSuccess;
    if (a.epi == EPI_GAT && !a.elmax) {
        *why = "GAT GEMM needs elmax";
        return cudaErrorInvalidValue;
    }
    const int K = a.K0 + a.K1;
    if (a.K0 % kBK || a.K1 % kBK || K > 256 || K == 0) {
        *why = "GEMM K must be a multiple of 64 and <= 256";
        return cudaErrorInvalidValue;
    }
    CUtensorMap m0, m1, mc, mo;
    if (!make_map_bf16(&m0, a.A0, a.M, a.K0) || !make_map_bf16(&m1, a.K1 ? a.A1 : a.A0, a.M, a.K1 ? a.K1 : a.K0) ||
        !make_map_bf16(&mc, a.out, a.M, a.N) || !make_map_bf16(&mo, a.out2 ? a.out2 : a.out, a.M, a.N)) {
        *why = "cuTensorMapEncodeTiled failed";
        return cudaErrorInvalidValue;
    }
    EpiParams ep{a.epi, a.row_scale, a.bias, a.act, a.a_src, a.a_dst, a.el, a.er, a.elmax,
                 a.epi == EPI_GAT && a.out2};
    const int KB = K / kBK, KB0 = a.K0 / kBK;
    // instantiated modes: GCN (row scale), SAGE / LSTM (bias + act), GAT (N = 64,
    // with / without the aggregation view's output tile)
    const bool self = ep.self_out;
    if (a.epi == EPI_ROWSCALE) {
        switch (a.N) {
            case 256: return launch_bn<256, EPI_ROWSCALE, false>(a, m0, m1, mc, mo, KB, KB0, ep, st);
            case 128: return launch_bn<128, EPI_ROWSCALE, false>(a, m0, m1, mc, mo, KB, KB0, ep, st);
            case 64: return launch_bn<64, EPI_ROWSCALE, false>(a, m0, m1, mc, mo, KB, KB0, ep, st);
        }
    } else if (a.epi == EPI_BIAS_ACT) {
        switch (a.N) {
            case 256: return launch_bn<256, EPI_BIAS_ACT, false>(a, m0, m1, mc, mo, KB, KB0, ep, st);
            case 128: return launch_bn<128, EPI_BIAS_ACT, false>(a, m0, m1, mc, mo, KB, KB0, ep, st);
            case 64: return launch_bn<64, EPI_BIAS_ACT, false>(a, m0, m1, mc, mo, KB, KB0, ep, st);
        }
    } else if (a.N == 64) {
        return self ? launch_bn<64, EPI_GAT, true>(a, m0, m1, mc, mo, KB, KB0, ep, st)
                    : launch_bn<64, EPI_GAT, false>(a, m0, m1, mc, mo, KB, KB0, ep, st);
    }
    *why = "GEMM N must be 64, 128 or 256";
    return cudaErrorInvalidValue;
}

}  // namespace saga
