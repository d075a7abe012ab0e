// gru_f64.cu -- ApplyVertex of the gated (C4) and paper-form GGNN (C8) layers
// for the graph's heavy rows (in-degree >= kHeavyInDeg), in fp64 on the CUDA
// cores.
//
// Paper: GGNN's ApplyVertex is a GRU over the gathered message m and the
// vertex's own embedding (Table 1; readings
// A15/A16).  For the gated layer m[v] = sum_t S[v][t] . W_t (the per-type
// message weight applied after Gather by linearity), for GGNN m comes from the
// edge-MLP gather.
//
// Why a second path.  The split-TF32 tensor-core GEMMs (gemm_tf32split.cu)
// represent every operand with 22 significant bits but ACCUMULATE in the
// tensor core's fp32 accumulator.  m is a sum over the in-edges, so its
// magnitude grows with the in-degree (linearly for the GGNN ReLU+sum message,
// ~sqrt for the zero-mean gated sums): on a 6K-in-edge GGNN hub |m| reaches
// 1.5e4, the gate pre-activations' partial sums carry fp32 ulps of ~1e-3, and
// the GRU output of that row misses the 1e-4 fp32 bar (measured 1.35e-4;
// scripts/tc_accum_probe.py: any fp32-accumulating GEMM, cuBLAS SGEMM
// included, lands at 4e-5..8e-5 on such rows, while fp64 accumulation of the
// same fp32 m gives 2e-6..4e-6).  The error is proportional to |m|, i.e. to
// the in-degree, so the rows whose in-degree reaches kHeavyInDeg (a list the
// graph build already has: the head of deg_order, sorted by in-degree) are
// recomputed here after the tensor-core GEMMs with every product and sum in
// fp64 and the GRU nonlinearities in fp64, from messages that were never
// rounded to fp32: the gathers also write the heavy rows' sums in fp64 (Sx
// for the gated layer, mx for GGNN).  For GGNN the destination term B[v] =
// H[v] W_b + b_e enters the edge-MLP sum deg(v) times, so its fp32 tensor-core
// value (error ~1e-7) would be amplified by the in-degree too: the heavy rows'
// B is computed here in fp64 (k_ggnn_heavy_b) before the gather, which adds it
// to A[u] in fp64.  The tensor path's rows stay below 256 in-edges.  This
// kernel overwrites the heavy rows' outputs (stream-ordered after the GEMM
// that wrote them), so the result is deterministic.
//
// Cost: per heavy row (T f + 6 f) f fp64 FMAs (164K at C4) -- 834 rows at
// C4/C8 (0.64% of the vertices, 39% of the edges).  A CTA takes kR = 8 rows
// and thread j owns column j of all 8 rows (8 accumulators per output
// matrix, 48 in the gate phase), so each weight element read from shared
// memory feeds 8 FMAs and the row operands are broadcasts.  The weights
// (converted to fp64 once per call by k_weights_f64) stream through a
// two-slot shared-memory ring of 48 KB chunks filled by bulk copies
// (cp.async.bulk, one thread) while the previous chunk is consumed.
// Measured on the way (C4): weights read from L2 per FMA were latency-bound
// (60 us), fp32 weights converted per use bound the XU pipe (F2F, 66 us),
// and a (row, column-quad) thread mapping was bound by shared-memory
// wavefronts (8 x re-reads of every weight, 2-way conflicts: 107 us).
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.cuh"
#include "ptx.cuh"

namespace saga {
namespace {

constexpr int kF = 128;            // hidden width (in = out = 128, checked by the host)
constexpr int kR = 8;              // rows per CTA batch
constexpr int kRT = 4;             // rows per thread: thread = (row group of kRT rows, column)
constexpr int kThreads = kF * (kR / kRT);
constexpr int kSlot = 48 * 1024;   // ring slot (bytes): fp64 weights
constexpr int kChunkG = 8;         // gate phase: K-rows per chunk (x 6 matrices of [kF][kF] fp64)
constexpr int kChunkM = 32;        // message / B phase: K-rows per chunk of one [K][kF] fp64 matrix

struct alignas(16) Ring {
    uint64_t full[2];
};

// acc[r] += sum_k x[r0 + r][k] W[k][j] for kRT rows: x smem fp64 [kR][ldx], W a
// [K][kF] fp64 matrix streamed in chunks of kChunkM rows.  The ring's chunk
// counter `cc` continues across calls (slot = cc & 1, parity = (cc >> 1) & 1).
__device__ __forceinline__ void stream_gemm(double (&acc)[kRT], const double *x, int ldx, const double *W, int K,
                                            double *slots, Ring &ring, uint32_t &cc, int r0, int j) {
    const int nch = K / kChunkM;
    auto issue = [&](int c, uint32_t seq) {
        double *dst = slots + (seq & 1) * (kSlot / 8);
        ptx::mbar_arrive_expect_tx(&ring.full[seq & 1], kChunkM * kF * 8);
        ptx::bulk_g2s(dst, W + (int64_t)c * kChunkM * kF, kChunkM * kF * 8, &ring.full[seq & 1]);
    };
    if (threadIdx.x == 0) {
        issue(0, cc);
        if (nch > 1) issue(1, cc + 1);
    }
    for (int c = 0; c < nch; ++c, ++cc) {
        ptx::mbar_wait(&ring.full[cc & 1], (cc >> 1) & 1);
        const double *w = slots + (cc & 1) * (kSlot / 8);
#pragma unroll 2
        for (int k = 0; k < kChunkM; k += 2) {
            const double w0 = w[k * kF + j], w1 = w[(k + 1) * kF + j];
#pragma unroll
            for (int r = 0; r < kRT; ++r) {
                const double2 xv = *reinterpret_cast<const double2 *>(x + (r0 + r) * ldx + c * kChunkM + k);
                acc[r] = fma(xv.x, w0, acc[r]);
                acc[r] = fma(xv.y, w1, acc[r]);
            }
        }
        __syncthreads();  // slot consumed by every thread
        if (threadIdx.x == 0 && c + 2 < nch) issue(c + 2, cc + 2);
    }
}

// fp64 copies of the weights the heavy kernels stream: [W_type (T kF kF) | W_ih (3 kF kF) | W_hh | W_b (kF kF)]
__global__ void k_weights_f64(int32_t nt, const float *__restrict__ W_type, const float *__restrict__ W_ih,
                              const float *__restrict__ W_hh, const float *__restrict__ W_b, double *__restrict__ out) {
    griddep_wait();  // before this grid's first global write
    const int64_t a = (int64_t)nt * kF * kF, g = (int64_t)3 * kF * kF, b = W_b ? (int64_t)kF * kF : 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a + 2 * g + b;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float x = i < a ? W_type[i] : i < a + g ? W_ih[i - a] : i < a + 2 * g ? W_hh[i - a - g] : W_b[i - a - 2 * g];
        out[i] = (double)x;
    }
}

// smem: ring 2 x kSlot | a[kR][T kF] fp64 (gated) | m[kR][kF] fp64 | h[kR][kF] fp64
size_t smem_bytes(int T) { return 2 * (size_t)kSlot + sizeof(double) * ((size_t)kR * T * kF + 2 * kR * kF); }

__global__ void __launch_bounds__(kThreads, 1)
    k_gru_heavy_f64(int32_t nh, const int32_t *__restrict__ rows, int32_t T, const double *__restrict__ Sx,
                    const double *__restrict__ W64, const double *__restrict__ mx, const float *__restrict__ H,
                    const float *__restrict__ b_ih, const float *__restrict__ b_hh, float *__restrict__ out) {
    extern __shared__ __align__(16) uint8_t smem[];
    const bool gated = Sx != nullptr;
    const int K = T * kF;
    double *slots = reinterpret_cast<double *>(smem);
    const double *W_type = W64, *W_ih = W64 + (int64_t)K * kF * gated, *W_hh = W_ih + 3 * kF * kF;
    double *a = reinterpret_cast<double *>(smem + 2 * kSlot);  // [kR][K]      (gated only)
    double *m = a + (gated ? kR * K : 0);                       // [kR][kF]
    double *h = m + kR * kF;                                    // [kR][kF]
    __shared__ Ring ring;
    const int j = threadIdx.x % kF, r0 = (threadIdx.x / kF) * kRT;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&ring.full[0], 1);
        ptx::mbar_init(&ring.full[1], 1);
        ptx::fence_mbar_init();
    }
    __syncthreads();
    uint32_t cc = 0;  // chunks consumed (ring sequence)

    griddep_wait();  // Sx / mx and the tensor path's output rows come from the call's earlier kernels
    for (int32_t b0 = blockIdx.x * kR; b0 < nh; b0 += gridDim.x * kR) {
        const int nr = min(kR, nh - b0);
        for (int r = r0; r < r0 + kRT; ++r) {
            h[r * kF + j] = r < nr ? (double)H[(int64_t)rows[b0 + r] * kF + j] : 0.0;
            if (!gated) m[r * kF + j] = r < nr ? mx[(int64_t)(b0 + r) * kF + j] : 0.0;
        }
        if (gated)
            for (int i = threadIdx.x; i < kR * K; i += kThreads) a[i] = i / K < nr ? Sx[(int64_t)b0 * K + i] : 0.0;
        __syncthreads();
        if (gated) {
            // m = S . W_type  (W_type [T][kF][kF] = [K][kF])
            double acc[kRT] = {};
            stream_gemm(acc, a, K, W_type, K, slots, ring, cc, r0, j);
#pragma unroll
            for (int r = 0; r < kRT; ++r) m[(r0 + r) * kF + j] = acc[r];
            __syncthreads();
        }
        // gate pre-activations: gi[g] = m . W_ih[g], gh[g] = h . W_hh[g] (g = r, z, n); the six
        // matrices stream together in chunks of kChunkG K-rows
        double gi[3][kRT] = {}, gh[3][kRT] = {};
        {
            auto issue = [&](int c, uint32_t seq) {
                double *dst = slots + (seq & 1) * (kSlot / 8);
                ptx::mbar_arrive_expect_tx(&ring.full[seq & 1], 6 * kChunkG * kF * 8);
                for (int mat = 0; mat < 6; ++mat)
                    ptx::bulk_g2s(dst + mat * kChunkG * kF,
                                  (mat < 3 ? W_ih : W_hh) + ((int64_t)(mat % 3) * kF + c * kChunkG) * kF,
                                  kChunkG * kF * 8, &ring.full[seq & 1]);
            };
            constexpr int nch = kF / kChunkG;
            if (threadIdx.x == 0) {
                issue(0, cc);
                issue(1, cc + 1);
            }
            for (int c = 0; c < nch; ++c, ++cc) {
                ptx::mbar_wait(&ring.full[cc & 1], (cc >> 1) & 1);
                const double *w = slots + (cc & 1) * (kSlot / 8);
                for (int k = 0; k < kChunkG; k += 2) {
                    double wi[3][2], wh[3][2];
#pragma unroll
                    for (int g = 0; g < 3; ++g)
#pragma unroll
                        for (int d = 0; d < 2; ++d) {
                            wi[g][d] = w[(g * kChunkG + k + d) * kF + j];
                            wh[g][d] = w[((3 + g) * kChunkG + k + d) * kF + j];
                        }
#pragma unroll
                    for (int r = 0; r < kRT; ++r) {
                        const double2 mv = *reinterpret_cast<const double2 *>(m + (r0 + r) * kF + c * kChunkG + k);
                        const double2 hv = *reinterpret_cast<const double2 *>(h + (r0 + r) * kF + c * kChunkG + k);
#pragma unroll
                        for (int g = 0; g < 3; ++g) {
                            gi[g][r] = fma(mv.x, wi[g][0], gi[g][r]);
                            gi[g][r] = fma(mv.y, wi[g][1], gi[g][r]);
                            gh[g][r] = fma(hv.x, wh[g][0], gh[g][r]);
                            gh[g][r] = fma(hv.y, wh[g][1], gh[g][r]);
                        }
                    }
                }
                __syncthreads();
                if (threadIdx.x == 0 && c + 2 < nch) issue(c + 2, cc + 2);
            }
        }
        // PyTorch GRUCell (reading A15): r = s(gi_r + gh_r), z = s(gi_z + gh_z),
        // n = tanh(gi_n + r gh_n), h' = (1 - z) n + z h  -- in this thread's registers
        {
            const double bir = b_ih[j], biz = b_ih[kF + j], bin = b_ih[2 * kF + j];
            const double bhr = b_hh[j], bhz = b_hh[kF + j], bhn = b_hh[2 * kF + j];
#pragma unroll
            for (int r = 0; r < kRT; ++r) {
                if (r0 + r >= nr) break;
                const double rg = 1.0 / (1.0 + exp(-(gi[0][r] + bir + gh[0][r] + bhr)));
                const double zg = 1.0 / (1.0 + exp(-(gi[1][r] + biz + gh[1][r] + bhz)));
                const double n = tanh(gi[2][r] + bin + rg * (gh[2][r] + bhn));
                out[(int64_t)rows[b0 + r0 + r] * kF + j] = (float)((1.0 - zg) * n + zg * h[(r0 + r) * kF + j]);
            }
        }
        __syncthreads();  // m, h, a are rewritten by the next batch
    }
}

// GGNN heavy rows: Bx[s][j] = sum_k H[v_s][k] W_e[f + k][j] + b_e[j] in fp64
// (W_e [2f][f], source rows first; W_b = rows f .. 2f-1, converted to fp64).
__global__ void __launch_bounds__(kThreads, 1)
    k_ggnn_heavy_b(int32_t nh, const int32_t *__restrict__ rows, const float *__restrict__ H,
                   const double *__restrict__ W_b, const float *__restrict__ b_e, double *__restrict__ Bx) {
    extern __shared__ __align__(16) uint8_t smem[];
    double *slots = reinterpret_cast<double *>(smem);
    double *hs = reinterpret_cast<double *>(smem + 2 * kSlot);  // [kR][kF]
    __shared__ Ring ring;
    const int j = threadIdx.x % kF, r0 = (threadIdx.x / kF) * kRT;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&ring.full[0], 1);
        ptx::mbar_init(&ring.full[1], 1);
        ptx::fence_mbar_init();
    }
    __syncthreads();
    uint32_t cc = 0;
    griddep_wait();  // before this grid's first global write
    const double b = b_e ? (double)b_e[j] : 0.0;
    for (int32_t b0 = blockIdx.x * kR; b0 < nh; b0 += gridDim.x * kR) {
        const int nr = min(kR, nh - b0);
        for (int r = r0; r < r0 + kRT; ++r) hs[r * kF + j] = r < nr ? (double)H[(int64_t)rows[b0 + r] * kF + j] : 0.0;
        __syncthreads();
        double acc[kRT] = {};
        stream_gemm(acc, hs, kF, W_b, kF, slots, ring, cc, r0, j);
        for (int r = 0; r < kRT && r0 + r < nr; ++r) Bx[(int64_t)(b0 + r0 + r) * kF + j] = acc[r] + b;
        __syncthreads();
    }
}

unsigned grid_for_heavy(int32_t nh) {
    const int batches = (nh + kR - 1) / kR;
    return (unsigned)(batches < kNumSMs ? batches : kNumSMs);
}

}  // namespace

// [Sx (gated: n_heavy T kF) | Bx, mx (GGNN: 2 n_heavy kF) | W64: fp64 weights]
HeavyWs heavy_ws(const GraphDev &g, saga_model kind, void *base) {
    HeavyWs w;
    double *p = static_cast<double *>(base);
    const int64_t nh = g.n_heavy;
    const int T = g.trow_ptr ? g.num_etypes : 1;
    if (kind == SAGA_GATED) {
        w.Sx = p;
        w.W64 = p + nh * T * kF;
        w.T = T;
    } else {
        w.Bx = p;
        w.mx = p + nh * kF;
        w.W64 = p + 2 * nh * kF;
        w.T = 0;
    }
    return w;
}

size_t heavy_workspace_bytes(const GraphDev &g, saga_model kind, int32_t f) {
    if (f != kF || g.n_heavy == 0) return 0;
    const size_t nh = (size_t)g.n_heavy, ff = (size_t)kF * kF;
    const size_t T = g.trow_ptr ? (size_t)g.num_etypes : 1;
    if (kind == SAGA_GATED) return sizeof(double) * (nh * T * kF + (T + 6) * ff);
    if (kind == SAGA_GGNN) return sizeof(double) * (2 * nh * kF + 7 * ff);
    return 0;
}

cudaError_t launch_heavy_weights_f64(const GraphDev &g, const HeavyWs &w, const float *W_type, const float *W_ih,
                                     const float *W_hh, const float *W_e, cudaStream_t st) {
    if (g.n_heavy == 0) return cudaSuccess;
    const float *W_b = W_e ? W_e + (int64_t)kF * kF : nullptr;  // W_e [2f][f]: destination half
    return launch(k_weights_f64, 2 * kNumSMs, 256, 0, st, (int32_t)(W_type ? w.T : 0), W_type, W_ih, W_hh, W_b,
                  w.W64);
}

cudaError_t launch_ggnn_heavy_b(const GraphDev &g, const HeavyWs &w, const float *H, const float *b_e,
                                cudaStream_t st) {
    if (g.n_heavy == 0) return cudaSuccess;
    const size_t smem = smem_bytes(0) - sizeof(double) * kR * kF;  // ring + one [kR][kF] block
    cudaError_t e = cudaFuncSetAttribute(k_ggnn_heavy_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e) return e;
    return launch(k_ggnn_heavy_b, grid_for_heavy(g.n_heavy), kThreads, smem, st, g.n_heavy,
                  (const int32_t *)g.deg_order, H, (const double *)(w.W64 + 6 * kF * kF), b_e, w.Bx);
}

cudaError_t launch_gru_heavy_f64(const GraphDev &g, const HeavyWs &w, const float *H, const float *b_ih,
                                 const float *b_hh, float *out, cudaStream_t st) {
    if (g.n_heavy == 0) return cudaSuccess;
    const size_t smem = smem_bytes(w.Sx ? w.T : 0);
    cudaError_t e = cudaFuncSetAttribute(k_gru_heavy_f64, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e) return e;
    return launch(k_gru_heavy_f64, grid_for_heavy(g.n_heavy), kThreads, smem, st, g.n_heavy,
                  (const int32_t *)g.deg_order, w.Sx ? w.T : 1, (const double *)w.Sx, (const double *)w.W64,
                  (const double *)w.mx, H, b_ih, b_hh, out);
}

}  // namespace saga
