// gemm_f32.cu -- fp32 ApplyEdge-by-type + ApplyVertex GRU for the gated
// layer (config C4), on the FP32 SIMT pipe (the fp32 tolerance 1e-4 rules
// out single-pass TF32).
//
// Paper: GGNN's ApplyVertex is a GRU over the gathered message and the
// vertex's own embedding (Table 1).
//   kernel 1:  m = [S_0 || S_1 || S_2 || S_3] . [W_0; W_1; W_2; W_3]
//              (per-type messages, summed -- linearity moves W_t after Gather)
//   kernel 2:  gate tile = [m || h] . B' with B' interleaving, per hidden unit
//              j, the columns (r_j, z_j, gin_j, ghn_j):
//                r   = m W_ir + h W_hr,   z = m W_iz + h W_hz,
//                gin = m W_in,            ghn = h W_hn
//              so every thread owns whole hidden units and the GRU epilogue
//              (PyTorch GRUCell form, reading A15) runs in registers.
// Both are 128x128x16 shared-memory tiled SGEMMs with 8x8 register tiles.
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.cuh"

namespace saga {
namespace {

constexpr int BM = 128, BN = 128, BK = 16, TM = 8, TN = 8;
constexpr int kThreads = (BM / TM) * (BN / TN);  // 256

// B element loaders --------------------------------------------------------
struct BPlain {  // row-major [K][N]
    const float *B;
    int N;
    __device__ __forceinline__ float operator()(int k, int n) const { return __ldg(B + (int64_t)k * N + n); }
};
struct BGru {  // interleaved GRU gate matrix over [m || h] (K = 2f, N = 4f)
    const float *W_ih, *W_hh;
    int f;
    __device__ __forceinline__ float operator()(int k, int n) const {
        const int j = n >> 2, g = n & 3;
        const bool from_m = k < f;
        const int kk = from_m ? k : k - f;
        switch (g) {
            case 0: return __ldg((from_m ? W_ih : W_hh) + ((int64_t)0 * f + kk) * f + j);
            case 1: return __ldg((from_m ? W_ih : W_hh) + ((int64_t)1 * f + kk) * f + j);
            case 2: return from_m ? __ldg(W_ih + ((int64_t)2 * f + kk) * f + j) : 0.0f;
            default: return from_m ? 0.0f : __ldg(W_hh + ((int64_t)2 * f + kk) * f + j);
        }
    }
};
// A element loaders ---------------------------------------------------------
struct APlain {
    const float *A;
    int K;
    __device__ __forceinline__ float operator()(int64_t m, int k) const { return __ldg(A + m * K + k); }
};
struct ACat {  // [m || h], both [M][f]
    const float *A0, *A1;
    int f;
    __device__ __forceinline__ float operator()(int64_t m, int k) const {
        return k < f ? __ldg(A0 + m * f + k) : __ldg(A1 + m * f + (k - f));
    }
};

struct EpiStore {
    float *C;
    int N;
    __device__ __forceinline__ void operator()(int64_t m, int n0, const float (&c)[TN]) const {
        float4 *p = reinterpret_cast<float4 *>(C + m * N + n0);
        p[0] = make_float4(c[0], c[1], c[2], c[3]);
        p[1] = make_float4(c[4], c[5], c[6], c[7]);
    }
};
struct EpiGru {  // columns n0..n0+7 = hidden units n0/4, n0/4 + 1 (4 gates each)
    const float *H, *b_ih, *b_hh;
    float *out;
    int f;
    __device__ __forceinline__ void operator()(int64_t m, int n0, const float (&c)[TN]) const {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int j = (n0 >> 2) + u;
            const float *g = c + 4 * u;
            const float r = 1.0f / (1.0f + expf(-(g[0] + b_ih[j] + b_hh[j])));
            const float z = 1.0f / (1.0f + expf(-(g[1] + b_ih[f + j] + b_hh[f + j])));
            const float n = tanhf(g[2] + b_ih[2 * f + j] + r * (g[3] + b_hh[2 * f + j]));
            const float h = H[m * f + j];
            out[m * f + j] = (1.0f - z) * n + z * h;
        }
    }
};

template <typename AL, typename BL, typename EP>
__global__ void __launch_bounds__(kThreads) k_sgemm(int64_t M, int N, int K, AL a, BL b, EP ep) {
    __shared__ float As[BK][BM + 4];
    __shared__ float Bs[BK][BN + 4];
    const int tid = threadIdx.x;
    const int tx = tid % (BN / TN), ty = tid / (BN / TN);
    const int64_t m0 = (int64_t)blockIdx.y * BM;
    const int n0 = blockIdx.x * BN;
    float acc[TM][TN] = {};
    for (int k0 = 0; k0 < K; k0 += BK) {
        // A tile: 128 x 16 -> As[k][m]
#pragma unroll
        for (int i = 0; i < (BM * BK) / kThreads; ++i) {
            const int idx = tid + i * kThreads;
            const int mm = idx / BK, kk = idx % BK;
            const int64_t gm = m0 + mm;
            As[kk][mm] = (gm < M && k0 + kk < K) ? a(gm, k0 + kk) : 0.0f;
        }
#pragma unroll
        for (int i = 0; i < (BN * BK) / kThreads; ++i) {
            const int idx = tid + i * kThreads;
            const int kk = idx / BN, nn = idx % BN;
            Bs[kk][nn] = (k0 + kk < K && n0 + nn < N) ? b(k0 + kk, n0 + nn) : 0.0f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            float av[TM], bv[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) av[i] = As[kk][ty * TM + i];
#pragma unroll
            for (int j = 0; j < TN; ++j) bv[j] = Bs[kk][tx * TN + j];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int64_t gm = m0 + ty * TM + i;
        if (gm < M) ep(gm, n0 + tx * TN, acc[i]);
    }
}

}  // namespace

cudaError_t launch_gated_apply(int64_t M, int32_t f, int32_t T, const float *S, const float *H, const float *W_type,
                               const float *W_ih, const float *W_hh, const float *b_ih, const float *b_hh,
                               float *m_ws, float *out, cudaStream_t st) {
    if (M == 0) return cudaSuccess;
    const unsigned gy = (unsigned)((M + BM - 1) / BM);
    // m = S[M][T f] . W_type viewed as [T f][f]
    k_sgemm<<<dim3((f + BN - 1) / BN, gy), kThreads, 0, st>>>(M, f, T * f, APlain{S, T * f}, BPlain{W_type, f},
                                                               EpiStore{m_ws, f});
    cudaError_t e = cudaGetLastError();
    if (e) return e;
    k_sgemm<<<dim3((4 * f + BN - 1) / BN, gy), kThreads, 0, st>>>(M, 4 * f, 2 * f, ACat{m_ws, H, f},
                                                                   BGru{W_ih, W_hh, f},
                                                                   EpiGru{H, b_ih, b_hh, out, f});
    return cudaGetLastError();
}

}  // namespace saga
