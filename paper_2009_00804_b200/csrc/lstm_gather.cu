// lstm_gather.cu -- GraphSAGE-LSTM Gather as ONE
// persistent kernel over all vertices.
//
// Paper: GraphSAGE's Gather is LSTM(in_edges) (Table 1); the LSTM
// "treats the inedges of a vertex as a sequence" and DGL runs it by "degree
// traversal", one batched launch per distinct degree, which leaves the GPU
// idle up to 20x the kernel time.  Here every
// sequence runs in one launch, and the time is set by the longest sequence
// (a power-law hub: ~13K dependent steps at C7) or by the total work:
//   * the input projections P_g = X . W_ih[g] (gates i, f, g, o) are one
//     tensor-core GEMM per gate before this kernel (gemm_tc.cu), so a step
//     only gathers a 1 KB row of P and applies the recurrent GEMV h . W_hh;
//   * one CTA (512 threads, one per SM) runs one sequence at a time and
//     takes the next vertex from a queue in descending in-degree order (the
//     graph's deg_order): the longest sequences -- the critical path --
//     start first on whole SMs and the short ones fill in behind them;
//   * thread (unit j, gate g) computes z_g[j] = P_g[u][j] + b + h . W_hh[g][:, j]
//     with its row of W_hh^T (128 bf16) resident in 64 registers -- a step
//     reads only h (bf16, 256 B, broadcast) from shared memory; re-reading a
//     128 KB shared-memory W_hh every step was the bound (ncu: MIO throttle,
//     1.6K shared wavefronts per step).  Each product is one sm_100
//     mixed-precision FHFMA.BF16 (bf16 x bf16 -> fp32 accumulate);
//   * the 4 gates of unit j sit in adjacent lanes: after its activation each
//     thread gathers (i, f, g, o) with shuffles and updates c_j (fp32, kept
//     identically in the 4 lanes), and h is double-buffered, so a step has
//     one barrier (the h broadcast) instead of a gate exchange and a
//     broadcast through shared memory;
//   * the P terms of the next kAhead steps are in flight while a step runs.
// Reading A25: sequence = in-edges in CSR order, PyTorch
// LSTMCell (i, f, g, o), zero initial state, output = final h (0 without
// in-edges), stored bf16 for the ApplyVertex concat-GEMM.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.cuh"
#include "ptx.cuh"

namespace saga {
namespace {

constexpr int kF = 128;        // hidden = input width
constexpr int kThreads = 512;  // one thread per (unit, gate): 128 x 4
constexpr int kAhead = 2;      // steps of P prefetched ahead

struct LstmSmem {
    uint4 hb[2][kF / 8];       // hidden state, bf16, double-buffered (read t & 1, write (t + 1) & 1)
    int32_t v;                 // current vertex
};

// sigm(x) = 1 / (1 + e^-x) with the fast reciprocal (|error| ~1e-7, the
// output feeds bf16 h); tanh(x) = 2 sigm(2x) - 1
__device__ __forceinline__ float sigm_fast(float x) { return __fdividef(1.0f, 1.0f + __expf(-x)); }

// wt[j][g][c] = W_hh[g][8c .. 8c+7][j] (bf16): row (unit j, gate g) of W_hh^T, 256 contiguous bytes
// (thread 0 also resets the gather's work-queue head)
__global__ void k_stage_whh(const __nv_bfloat16 *__restrict__ W_hh, uint4 *wt, int32_t *queue) {
    griddep_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;  // over kF * 4 * kF / 8 chunks
    if (i == 0) *queue = 0;
    if (i >= 4 * kF * kF / 8) return;
    const int c = i % (kF / 8), g = (i / (kF / 8)) % 4, j = i / (kF / 8 * 4);
    uint32_t q[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const uint16_t lo = __bfloat16_as_ushort(W_hh[((int64_t)g * kF + 8 * c + 2 * e) * kF + j]);
        const uint16_t hi = __bfloat16_as_ushort(W_hh[((int64_t)g * kF + 8 * c + 2 * e + 1) * kF + j]);
        q[e] = (uint32_t)lo | ((uint32_t)hi << 16);
    }
    wt[i] = make_uint4(q[0], q[1], q[2], q[3]);
}

__global__ void __launch_bounds__(kThreads, 1)
    k_lstm_gather(int32_t n, const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col_src,
                  const int32_t *__restrict__ order, const __nv_bfloat16 *__restrict__ P,  // [4][n][kF]
                  const uint4 *__restrict__ wt,                                            // staged W_hh^T
                  const float *__restrict__ b_ih, const float *__restrict__ b_hh,          // [4][kF]
                  __nv_bfloat16 *__restrict__ h_out, int32_t *queue) {
    __shared__ LstmSmem S;
    griddep_wait();  // P, W_hh^T and the queue head come from the call's earlier kernels
    // thread -> (unit j, gate g): the 4 gates of a unit are adjacent lanes,
    // so the cell update gathers them with shuffles and a step needs ONE
    // barrier (the h broadcast)
    const int j = threadIdx.x / 4, g = threadIdx.x % 4;
    const int lane = threadIdx.x & 31, gbase = lane & ~3;
    uint4 w[kF / 8];  // this thread's row of W_hh^T, resident in registers
#pragma unroll
    for (int c = 0; c < kF / 8; ++c) w[c] = __ldg(wt + ((int64_t)j * 4 + g) * (kF / 8) + c);
    const float bias = __ldg(b_ih + g * kF + j) + __ldg(b_hh + g * kF + j);
    const float ks = g == 2 ? 2.0f : 1.0f;  // gate g uses tanh = 2 sigm(2x) - 1
    const __nv_bfloat16 *Pg = P + g * (int64_t)n * kF + j;

    for (;;) {
        if (threadIdx.x == 0) {
            const int32_t qi = atomicAdd(queue, 1);
            S.v = qi < n ? order[qi] : -1;
        }
        if (threadIdx.x < kF / 8) S.hb[0][threadIdx.x] = make_uint4(0, 0, 0, 0);
        __syncthreads();
        const int32_t v = S.v;
        if (v < 0) break;
        const int32_t p0 = (int32_t)row_ptr[v], p1 = (int32_t)row_ptr[v + 1];
        float c = 0.0f, hf = 0.0f;  // cell state and output of unit j (identical in its 4 lanes)
        __nv_bfloat16 ring[kAhead];
#pragma unroll
        for (int a = 0; a < kAhead; ++a)
            ring[a] = (p0 + a < p1) ? Pg[(int64_t)__ldg(col_src + p0 + a) * kF] : __float2bfloat16_rn(0.0f);
        int buf = 0;
        for (int32_t p = p0; p < p1; ++p) {
            const float pz = __bfloat162float(ring[0]);
#pragma unroll
            for (int a = 0; a + 1 < kAhead; ++a) ring[a] = ring[a + 1];
            ring[kAhead - 1] =
                (p + kAhead < p1) ? Pg[(int64_t)__ldg(col_src + p + kAhead) * kF] : __float2bfloat16_rn(0.0f);
            // z_g[j] = P_g[u][j] + b + h . W_hh[g][:, j]: 64 FHFMA.BF16 in 4 chains
            float a4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
            const uint4 *hb = S.hb[buf];
#pragma unroll
            for (int cc = 0; cc < kF / 8; ++cc) {
                const uint4 hv = hb[cc];
                ptx::fma_bf16x2_f32(a4[0], w[cc].x, hv.x);
                ptx::fma_bf16x2_f32(a4[1], w[cc].y, hv.y);
                ptx::fma_bf16x2_f32(a4[2], w[cc].z, hv.z);
                ptx::fma_bf16x2_f32(a4[3], w[cc].w, hv.w);
            }
            const float zz = (a4[0] + a4[1]) + (a4[2] + a4[3]) + pz + bias;
            const float sg = sigm_fast(ks * zz);
            const float act = g == 2 ? 2.0f * sg - 1.0f : sg;
            const float ig = __shfl_sync(0xffffffffu, act, gbase + 0);
            const float fg = __shfl_sync(0xffffffffu, act, gbase + 1);
            const float gg = __shfl_sync(0xffffffffu, act, gbase + 2);
            const float og = __shfl_sync(0xffffffffu, act, gbase + 3);
            c = fg * c + ig * gg;
            hf = og * (2.0f * sigm_fast(2.0f * c) - 1.0f);
            buf ^= 1;
            if (g == 0) reinterpret_cast<__nv_bfloat16 *>(S.hb[buf])[j] = __float2bfloat16_rn(hf);
            __syncthreads();  // new h visible; every read of the old one is done
        }
        if (g == 0) h_out[(int64_t)v * kF + j] = __float2bfloat16_rn(hf);
        __syncthreads();  // S.v and S.hb[0] are rewritten for the next sequence
    }
}

}  // namespace

// [staged W_hh^T | work-queue head]: the head lives in this region, not among
// the split-row ticket counters (which every completed call leaves zero); the
// staging kernel resets it before every gather
size_t lstm_workspace_bytes() { return sizeof(uint4) * 4 * kF * kF / 8 + 16; }

cudaError_t launch_lstm_gather(const GraphDev &g, const __nv_bfloat16 *P, const __nv_bfloat16 *W_hh,
                               const float *b_ih, const float *b_hh, __nv_bfloat16 *h_out, void *wt_ws,
                               cudaStream_t st) {
    if (g.n == 0) return cudaSuccess;
    uint4 *wt = static_cast<uint4 *>(wt_ws);
    int32_t *queue = reinterpret_cast<int32_t *>(wt + 4 * kF * kF / 8);
    cudaError_t e = launch(k_stage_whh, (4 * kF * kF / 8 + 255) / 256, 256, 0, st, W_hh, wt, queue);
    if (e) return e;
    int dev = 0, sms = kNumSMs;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = (unsigned)(g.n < sms ? g.n : sms);
    return launch(k_lstm_gather, grid, kThreads, 0, st, g.n, g.row_ptr, g.col_src, g.deg_order, P, wt, b_ih, b_hh,
                  h_out, queue);
}

}  // namespace saga
