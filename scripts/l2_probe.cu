// l2_probe.cu -- development probe: can L2 persistence raise the hit rate of
// C5's row gather?  (Not product code.)
//
// The C5 source-frequency distribution is heavy-tailed: an LRU over 100 MB of
// rows hits ~66% of the 71M row references, a static set of the 200K most
// referenced rows ~77%.  This probe times the plain gather (all rows evict-
// normal) against:
//   win K : the K hottest rows relabelled to a contiguous block Y[n, n+K)
//           covered by a persisting cudaAccessPolicyWindow (L2 set-aside)
//   hint K: per-access createpolicy evict_last on hot rows, evict_first on the
//           rest, with and without the set-aside
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_probe l2_probe.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_) {                                                                          \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));     \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)

// MODE 0: plain ld.global.nc; 1: hot bit -> (evict_last, evict_first); 2: hot bit -> (evict_last, normal)
template <int MODE>
__global__ void k_gather(const int32_t *__restrict__ col, int64_t e, const uint4 *__restrict__ Y, int64_t per_warp,
                         float *sink) {
    constexpr int U = 8;
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
    for (int64_t q0 = b; q0 < end; q0 += 32) {
        const int32_t c = q0 + lane < end ? col[q0 + lane] : 0;
#pragma unroll
        for (int j0 = 0; j0 < 32; j0 += U) {
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int32_t s = __shfl_sync(0xffffffffu, c, j0 + u);
                const uint4 *ptr = Y + (int64_t)(s & 0x7fffffff) * 32 + lane;
                if (MODE == 0) {
                    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                                 : "l"(ptr));
                } else {
                    const uint64_t pol = s < 0 ? pl : (MODE == 1 ? pf : pn);
                    asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                                 : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                                 : "l"(ptr), "l"(pol));
                }
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

// evict L2 between timed passes
__global__ void k_flush(uint4 *buf, int64_t n16) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
        buf[i] = make_uint4((uint32_t)i, 0, 0, 0);
}

template <int MODE>
float run(cudaStream_t st, const int32_t *col, int64_t e, const uint4 *Y, float *sink, uint4 *fl, int64_t fl16) {
    const int64_t warps = (int64_t)148 * 32 * 2;
    int64_t per = (e + warps - 1) / warps;
    per = (per + 31) / 32 * 32;
    const int64_t nw = (e + per - 1) / per;
    const unsigned blocks = (unsigned)((nw * 32 + 255) / 256);
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    float tot = 0;
    for (int i = 0; i < 4; ++i) {
        k_flush<<<148 * 8, 256, 0, st>>>(fl, fl16);
        CK(cudaEventRecord(a, st));
        k_gather<MODE><<<blocks, 256, 0, st>>>(col, e, Y, per, sink);
        CK(cudaEventRecord(b, st));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (i > 0) tot += ms;  // first pass warms up
    }
    return tot / 3;
}

int main(int argc, char **argv) {
    if (argc < 3) {
        fprintf(stderr, "usage: l2_probe col_src.bin N\n");
        return 1;
    }
    FILE *f = fopen(argv[1], "rb");
    fseek(f, 0, SEEK_END);
    const int64_t e = ftell(f) / 4;
    fseek(f, 0, SEEK_SET);
    std::vector<int32_t> h(e);
    if (fread(h.data(), 4, e, f) != (size_t)e) return 1;
    fclose(f);
    const int32_t n = atoi(argv[2]);
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    printf("L2 %d MB, persistingL2CacheMaxSize %.1f MB, accessPolicyMaxWindowSize %.1f MB\n", prop.l2CacheSize >> 20,
           prop.persistingL2CacheMaxSize / 1048576.0, prop.accessPolicyMaxWindowSize / 1048576.0);

    // rows by reference count, descending
    std::vector<int64_t> freq(n, 0);
    for (int64_t i = 0; i < e; ++i) freq[h[i]]++;
    std::vector<int32_t> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return freq[a] > freq[b]; });
    std::vector<int32_t> rank(n);
    for (int32_t i = 0; i < n; ++i) rank[order[i]] = i;

    const int32_t kmax = 300000;
    int32_t *col;
    uint4 *Y, *fl;
    float *sink;
    const int64_t fl16 = (int64_t)512 << 20 >> 4;  // 512 MB flush buffer
    CK(cudaMalloc(&col, 4 * e));
    CK(cudaMalloc(&Y, ((size_t)n + kmax) * 512));
    CK(cudaMalloc(&fl, fl16 * 16));
    CK(cudaMalloc(&sink, 1 << 26));
    CK(cudaMemset(Y, 0x3c, ((size_t)n + kmax) * 512));
    cudaStream_t st;
    CK(cudaStreamCreate(&st));
    const double gb = e * 512.0 / 1e9;
    std::vector<int32_t> c2(e);

    auto upload_plain = [&]() { CK(cudaMemcpy(col, h.data(), 4 * e, cudaMemcpyHostToDevice)); };
    auto upload_hotbit = [&](int32_t K) {
        for (int64_t i = 0; i < e; ++i) c2[i] = rank[h[i]] < K ? (int32_t)(h[i] | 0x80000000u) : h[i];
        CK(cudaMemcpy(col, c2.data(), 4 * e, cudaMemcpyHostToDevice));
    };
    auto upload_window = [&](int32_t K) {  // hot rows -> Y[n + rank]
        for (int64_t i = 0; i < e; ++i) c2[i] = rank[h[i]] < K ? n + rank[h[i]] : h[i];
        CK(cudaMemcpy(col, c2.data(), 4 * e, cudaMemcpyHostToDevice));
    };
    auto set_aside = [&](size_t bytes) {
        CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, bytes));
        size_t got = 0;
        CK(cudaDeviceGetLimit(&got, cudaLimitPersistingL2CacheSize));
        return got;
    };
    auto set_window = [&](int32_t K, float ratio) {
        cudaStreamAttrValue av = {};
        if (K > 0) {
            av.accessPolicyWindow.base_ptr = (void *)(Y + (int64_t)n * 32);
            av.accessPolicyWindow.num_bytes = std::min<size_t>((size_t)K * 512, prop.accessPolicyMaxWindowSize);
            av.accessPolicyWindow.hitRatio = ratio;
            av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
            av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        }
        CK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &av));
    };
    auto report = [&](const char *what, float ms) {
        printf("%-48s %.3f ms  %.0f GB/s requested\n", what, ms, gb / ms * 1e3);
    };
    char buf[128];

    upload_plain();
    set_aside(0);
    report("plain (no set-aside)", run<0>(st, col, e, Y, sink, fl, fl16));
    for (int32_t K : {100000, 150000, 200000}) {
        std::vector<int64_t> f2(freq.begin(), freq.end());
        int64_t cov = 0;
        for (int32_t i = 0; i < K; ++i) cov += freq[order[i]];
        printf("K=%d rows (%.0f MB) cover %.3f of references\n", K, K * 512 / 1048576.0, (double)cov / e);
    }
    for (int32_t K : {100000, 150000}) {
        upload_hotbit(K);
        set_aside(0);
        snprintf(buf, sizeof buf, "hint K=%d last/first, no set-aside", K);
        report(buf, run<1>(st, col, e, Y, sink, fl, fl16));
        snprintf(buf, sizeof buf, "hint K=%d last/normal, no set-aside", K);
        report(buf, run<2>(st, col, e, Y, sink, fl, fl16));
        const size_t got = set_aside((size_t)K * 512);
        snprintf(buf, sizeof buf, "hint K=%d last/first, set-aside %.0f MB", K, got / 1048576.0);
        report(buf, run<1>(st, col, e, Y, sink, fl, fl16));
        snprintf(buf, sizeof buf, "hint K=%d last/normal, set-aside %.0f MB", K, got / 1048576.0);
        report(buf, run<2>(st, col, e, Y, sink, fl, fl16));
    }
    for (int32_t K : {60000, 100000, 150000, 200000}) {
        upload_window(K);
        for (float ratio : {1.0f, 0.6f}) {
            const size_t got = set_aside(std::min<size_t>((size_t)K * 512, prop.persistingL2CacheMaxSize));
            set_window(K, ratio);
            snprintf(buf, sizeof buf, "window K=%d ratio %.1f, set-aside %.0f MB", K, ratio, got / 1048576.0);
            report(buf, run<0>(st, col, e, Y, sink, fl, fl16));
            set_window(0, 0);
            CK(cudaCtxResetPersistingL2Cache());
        }
    }
    upload_window(150000);
    set_aside(0);
    report("window layout, no window (control)", run<0>(st, col, e, Y, sink, fl, fl16));
    return 0;
}
