// gather_probe.cu -- standalone probe of the raw row-gather throughput a
// B200 reaches for the C5 access pattern (development tool, not product).
// Reads col_src (int32 little-endian file), allocates an N x 256 bf16 table,
// and times kernels that only gather + sum rows (no per-row epilogue):
//   csr  : edges in CSR (destination) order, warp streams a contiguous range
//   rand : the same indices hashed to uniform random rows
// with U outstanding 16-byte loads per lane, at several occupancies.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_probe gather_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <functional>

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e_ = (x);                                                    \
        if (e_) {                                                                \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                            \
        }                                                                       \
    } while (0)

// load flavours (L2 policy experiments)
template <int POL>
__device__ __forceinline__ uint4 ldg_pol(const void *p, uint64_t pol) {
    uint4 r;
    if (POL == 0)
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    else if (POL == 1)
        asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    else if (POL == 4)
        asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    else
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
    return r;
}
template <int POL>
__device__ __forceinline__ uint64_t make_pol() {
    uint64_t p = 0;
    if (POL == 2) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    if (POL == 3) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    if (POL == 5) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 0.5;" : "=l"(p));
    return p;
}

template <int U, bool kRand, int POL>
__global__ void k_gather(const int32_t *__restrict__ col, int64_t e, int32_t n, const uint4 *__restrict__ Y,
                         int64_t per_warp, float *sink) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t b = w * per_warp;
    if (b >= e) return;
    const int64_t end = b + per_warp < e ? b + per_warp : e;
    float acc[8] = {};
    const uint64_t pol = make_pol<POL>();
    for (int64_t q0 = b; q0 < end; q0 += 32) {
        int32_t c = q0 + lane < end ? col[q0 + lane] : 0;
        if (kRand) c = (int32_t)(((uint32_t)c * 2654435761u) % (uint32_t)n);
#pragma unroll
        for (int j0 = 0; j0 < 32; j0 += U) {
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                int32_t s = __shfl_sync(0xffffffffu, c, j0 + u);
                v[u] = ldg_pol<POL>(Y + (int64_t)s * 32 + lane, pol);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                acc[0] += __uint_as_float(v[u].x << 16);
                acc[1] += __uint_as_float(v[u].x & 0xffff0000u);
                acc[2] += __uint_as_float(v[u].y << 16);
                acc[3] += __uint_as_float(v[u].y & 0xffff0000u);
                acc[4] += __uint_as_float(v[u].z << 16);
                acc[5] += __uint_as_float(v[u].z & 0xffff0000u);
                acc[6] += __uint_as_float(v[u].w << 16);
                acc[7] += __uint_as_float(v[u].w & 0xffff0000u);
            }
        }
    }
    float s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == 12345.f) sink[w] = s;
}

// hot-aware: col high bit = hot row; HOTPOL selects (hot, cold) policies:
// 0: (evict_last, evict_first)  1: (evict_last, normal)  2: (normal, evict_first)  3: (normal, no_allocate-L1)
template <int U, int HOTPOL>
__global__ void k_gather_hot(const int32_t *__restrict__ col, int64_t e, const uint4 *__restrict__ Y,
                             int64_t per_warp, float *sink) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t b = w * per_warp;
    if (b >= e) return;
    const int64_t end = b + per_warp < e ? b + per_warp : e;
    float acc[8] = {};
    uint64_t pl, pf, pn;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pn));
    const uint64_t ph = (HOTPOL <= 1) ? pl : pn;
    const uint64_t pc = (HOTPOL == 0 || HOTPOL == 2) ? pf : pn;
    for (int64_t q0 = b; q0 < end; q0 += 32) {
        int32_t c = q0 + lane < end ? col[q0 + lane] : 0;
#pragma unroll
        for (int j0 = 0; j0 < 32; j0 += U) {
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                int32_t s = __shfl_sync(0xffffffffu, c, j0 + u);
                const bool hot = s < 0;
                const uint4 *ptr = Y + (int64_t)(s & 0x7fffffff) * 32 + lane;
                asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                             : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(ptr), "l"(hot ? ph : pc));
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                acc[0] += __uint_as_float(v[u].x << 16);
                acc[1] += __uint_as_float(v[u].x & 0xffff0000u);
                acc[2] += __uint_as_float(v[u].y << 16);
                acc[3] += __uint_as_float(v[u].y & 0xffff0000u);
                acc[4] += __uint_as_float(v[u].z << 16);
                acc[5] += __uint_as_float(v[u].z & 0xffff0000u);
                acc[6] += __uint_as_float(v[u].w << 16);
                acc[7] += __uint_as_float(v[u].w & 0xffff0000u);
            }
        }
    }
    float s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == 12345.f) sink[w] = s;
}

template <int U, int HOTPOL>
float run_hot(const int32_t *col, int64_t e, const uint4 *Y, float *sink) {
    int64_t warps = (int64_t)148 * 4 * 8 * 8;
    int64_t per = (e + warps - 1) / warps;
    per = (per + 31) / 32 * 32;
    int64_t nw = (e + per - 1) / per;
    int64_t blocks = (nw * 32 + 255) / 256;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_gather_hot<U, HOTPOL><<<blocks, 256>>>(col, e, Y, per, sink);
    cudaEventRecord(a);
    for (int i = 0; i < 3; ++i) k_gather_hot<U, HOTPOL><<<blocks, 256>>>(col, e, Y, per, sink);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 3;
}

// column slice: S edges per warp step, each by 32/S lanes reading the first
// 512/S bytes of its row (a 1/S column tile of the 512-B row)
template <int U, int S>
__global__ void k_gather_cols(const int32_t *__restrict__ col, int64_t e, const uint4 *__restrict__ Y,
                              int64_t per_warp, float *sink) {
    const int lane = threadIdx.x & 31;
    const int sub = lane / (32 / S), gl = lane % (32 / S);
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t b = w * per_warp;
    if (b >= e) return;
    const int64_t end = b + per_warp < e ? b + per_warp : e;
    float acc[8] = {};
    for (int64_t q0 = b; q0 < end; q0 += 32) {
        int32_t c = q0 + lane < end ? col[q0 + lane] : 0;
#pragma unroll
        for (int j0 = 0; j0 < 32; j0 += U * S) {
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                int32_t s = __shfl_sync(0xffffffffu, c, j0 + u * S + sub);
                v[u] = __ldg(Y + (int64_t)s * 32 + gl);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                acc[0] += __uint_as_float(v[u].x << 16);
                acc[1] += __uint_as_float(v[u].x & 0xffff0000u);
                acc[2] += __uint_as_float(v[u].y << 16);
                acc[3] += __uint_as_float(v[u].y & 0xffff0000u);
                acc[4] += __uint_as_float(v[u].z << 16);
                acc[5] += __uint_as_float(v[u].z & 0xffff0000u);
                acc[6] += __uint_as_float(v[u].w << 16);
                acc[7] += __uint_as_float(v[u].w & 0xffff0000u);
            }
        }
    }
    float s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == 12345.f) sink[w] = s;
}
template <int U, int S>
float run_cols(const int32_t *col, int64_t e, const uint4 *Y, float *sink) {
    int64_t warps = (int64_t)148 * 4 * 8 * 8;
    int64_t per = (e + warps - 1) / warps;
    per = (per + 31) / 32 * 32;
    int64_t nw = (e + per - 1) / per;
    int64_t blocks = (nw * 32 + 255) / 256;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_gather_cols<U, S><<<blocks, 256>>>(col, e, Y, per, sink);
    cudaEventRecord(a);
    for (int i = 0; i < 3; ++i) k_gather_cols<U, S><<<blocks, 256>>>(col, e, Y, per, sink);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 3;
}

// TMA (bulk-copy) gather: per U-edge batch, lanes 0..U-1 each issue one
// cp.async.bulk of a 512-byte row into the warp's shared-memory stage
// (mbarrier-tracked, two stages in flight), then every lane reduces its
// 16-byte slice of the U staged rows -- the round-2 verdict's "TMA /
// shared-memory staging of feature tiles" for the gather.
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
template <int U>
__global__ void __launch_bounds__(256) k_gather_bulk(const int32_t *__restrict__ col, int64_t e, const uint4 *__restrict__ Y,
                                                   int64_t per_warp, float *sink) {
    extern __shared__ __align__(128) uint8_t sm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint4 *stage = reinterpret_cast<uint4 *>(sm + wid * (2 * U * 512));
    __shared__ __align__(8) uint64_t bars[8][2];
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t b = w * per_warp;
    if (lane == 0) {
        for (int i = 0; i < 2; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[wid][i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    if (b >= e) return;
    const int64_t end = b + per_warp < e ? b + per_warp : e;
    float acc[8] = {};
    uint32_t phase[2] = {0, 0};
    // issue batch j (U edges from chunk register c) into stage j & 1
    auto issue = [&](int32_t c, int j0, int st) {
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[wid][st])),
                         "r"(U * 512) : "memory");
        __syncwarp();
        const int32_t s = __shfl_sync(0xffffffffu, c, j0 + (lane % U));
        if (lane < U)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 512, [%2];" ::"r"(
                             smem_u32(stage + (st * U + lane) * 32)),
                         "l"(Y + (int64_t)s * 32), "r"(smem_u32(&bars[wid][st]))
                         : "memory");
    };
    int st = 0;
    for (int64_t q0 = b; q0 < end; q0 += 32) {
        const int32_t c = q0 + lane < end ? col[q0 + lane] : 0;
        issue(c, 0, st);
#pragma unroll
        for (int j0 = 0; j0 < 32; j0 += U) {
            if (j0 + U < 32) issue(c, j0 + U, st ^ 1);
            asm volatile(
                "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(
                    smem_u32(&bars[wid][st])),
                "r"(phase[st])
                : "memory");
            phase[st] ^= 1;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint4 v = stage[(st * U + u) * 32 + lane];
                acc[0] += __uint_as_float(v.x << 16);
                acc[1] += __uint_as_float(v.x & 0xffff0000u);
                acc[2] += __uint_as_float(v.y << 16);
                acc[3] += __uint_as_float(v.y & 0xffff0000u);
                acc[4] += __uint_as_float(v.z << 16);
                acc[5] += __uint_as_float(v.z & 0xffff0000u);
                acc[6] += __uint_as_float(v.w << 16);
                acc[7] += __uint_as_float(v.w & 0xffff0000u);
            }
            __syncwarp();  // the stage is read before it is refilled
            st ^= 1;
        }
    }
    float s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == 12345.f) sink[w] = s;
}
template <int U>
float run_bulk(const int32_t *col, int64_t e, const uint4 *Y, int blocks_per_sm, float *sink) {
    int64_t warps = (int64_t)148 * blocks_per_sm * 8 * 8;
    int64_t per = (e + warps - 1) / warps;
    per = (per + 31) / 32 * 32;
    int64_t nw = (e + per - 1) / per;
    int64_t blocks = (nw * 32 + 255) / 256;
    const int smem = 8 * 2 * U * 512;
    CK(cudaFuncSetAttribute(k_gather_bulk<U>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_gather_bulk<U><<<blocks, 256, smem>>>(col, e, Y, per, sink);
    CK(cudaGetLastError());
    cudaEventRecord(a);
    for (int i = 0; i < 3; ++i) k_gather_bulk<U><<<blocks, 256, smem>>>(col, e, Y, per, sink);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 3;
}

template <int U, bool kRand, int POL>
float run(const int32_t *col, int64_t e, int32_t n, const uint4 *Y, int threads, int blocks_per_sm, float *sink) {
    int64_t warps = (int64_t)148 * blocks_per_sm * (threads / 32) * 8;
    int64_t per = (e + warps - 1) / warps;
    per = (per + 31) / 32 * 32;
    int64_t nw = (e + per - 1) / per;
    int64_t blocks = (nw * 32 + threads - 1) / threads;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_gather<U, kRand, POL><<<blocks, threads>>>(col, e, n, Y, per, sink);
    cudaEventRecord(a);
    for (int i = 0; i < 3; ++i) k_gather<U, kRand, POL><<<blocks, threads>>>(col, e, n, Y, per, sink);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 3;
}

int main(int argc, char **argv) {
    if (argc < 3) {
        fprintf(stderr, "usage: gather_probe col_src.bin N\n");
        return 1;
    }
    FILE *f = fopen(argv[1], "rb");
    fseek(f, 0, SEEK_END);
    int64_t e = ftell(f) / 4;
    fseek(f, 0, SEEK_SET);
    std::vector<int32_t> h(e);
    if (fread(h.data(), 4, e, f) != (size_t)e) return 1;
    fclose(f);
    int32_t n = atoi(argv[2]);
    int32_t *col;
    uint4 *Y;
    float *sink;
    CK(cudaMalloc(&col, 4 * e));
    CK(cudaMalloc(&Y, (size_t)n * 512));
    CK(cudaMalloc(&sink, 1 << 26));
    CK(cudaMemcpy(col, h.data(), 4 * e, cudaMemcpyHostToDevice));
    CK(cudaMemset(Y, 0x3c, (size_t)n * 512));
    const double gb = e * 512.0 / 1e9;
    printf("E=%lld N=%d gathered GB per pass=%.2f\n", (long long)e, n, gb);
#define R(U, RAND, POL)                                                                             \
    {                                                                                               \
        float ms = run<U, RAND, POL>(col, e, n, Y, 256, 4, sink);                                   \
        printf("U=%2d rand=%d pol=%d  %.3f ms  %.0f GB/s requested\n", U, RAND, POL, ms, gb / ms * 1e3); \
    }
    R(8, false, 1) R(4, false, 1)
#define RB(U, BPS) { float ms = run_bulk<U>(col, e, Y, BPS, sink); printf("bulk-copy (TMA) gather U=%d, %d blocks/SM: %.3f ms  %.0f GB/s requested\n", U, BPS, ms, gb / ms * 1e3); }
    RB(4, 4) RB(8, 3) RB(8, 2) RB(4, 2)
#define RC(U, S) { float ms = run_cols<U, S>(col, e, Y, sink); printf("cols 1/%d U=%d  %.3f ms per pass, x%d passes = %.3f ms\n", S, U, ms, S, ms * S); }
    RC(8, 1) RC(8, 2) RC(4, 2) RC(8, 4) RC(4, 4) RC(8, 8) RC(4, 8)
    return 0;
}
