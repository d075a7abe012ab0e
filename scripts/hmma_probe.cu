// hmma_probe.cu -- mma.sync m16n8k16 bf16 -> f32 throughput / latency on sm_100a (development
// probe, not product): NT independent accumulator chains of KS mmas per warp.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hmma_probe hmma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ void mma(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
// NT independent accumulator tiles, each a chain of KS mmas, per iteration
template <int NT, int KS>
__global__ void k(int iters, float *out, uint32_t seed) {
    uint32_t a[4], b[NT][KS][2];
    for (int i = 0; i < 4; ++i) a[i] = seed * (threadIdx.x + i);
    for (int t = 0; t < NT; ++t) for (int s = 0; s < KS; ++s) { b[t][s][0] = seed + t * 7 + s; b[t][s][1] = seed ^ (t + s); }
    float d[NT][4] = {};
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int s = 0; s < KS; ++s)
#pragma unroll
            for (int t = 0; t < NT; ++t) mma(d[t], a, b[t][s]);
    }
    long long t1 = clock64();
    float acc = 0; for (int t = 0; t < NT; ++t) for (int i = 0; i < 4; ++i) acc += d[t][i];
    if (acc == 1.2345f) out[0] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (float)(t1 - t0) / iters;
}
template <int NT, int KS>
void run(int warps, int blocks) {
    float *o; cudaMalloc(&o, 8);
    int iters = 2000;
    k<NT, KS><<<blocks, warps * 32>>>(iters, o, 1);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<NT, KS><<<blocks, warps * 32>>>(iters, o, 3);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    float cyc; cudaMemcpy(&cyc, o + 1, 4, cudaMemcpyDeviceToHost);
    double mmas_per_sm = (double)warps * iters * NT * KS;
    printf("NT=%d KS=%d warps/SM=%2d: %.1f cycles/iter/warp (%d mma), SM-wide %.2f cycles per mma per SMSP; %.1f TFLOP/s\n",
           NT, KS, warps, cyc, NT * KS, cyc / (NT * KS) / (warps / 4.0 > 1 ? warps / 4.0 : 1),
           mmas_per_sm * blocks * 4096.0 / (ms * 1e-3) / 1e12);
    cudaFree(o);
}
int main() {
    run<4, 8>(1, 148);
    run<4, 8>(4, 148);
    run<4, 8>(8, 148);
    run<4, 8>(16, 148);
    run<8, 8>(8, 148);
    run<16, 8>(16, 148);
    run<1, 8>(1, 148);
    return 0;
}
