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
// C4/C8 (0.64% of the vertices, 39% of the edges).  A CTA takes kR = 8 rows,
// the M of the fp64 tensor-core MMA (mma.sync m8n8k4 f64, DMMA): warp w owns
// output columns [16 w, 16 w + 16) as two 8-column n-tiles, so one A fragment
// (8 rows x 4 k, one double per lane) feeds two MMAs and each weight double
// read from shared memory feeds 8 FMAs inside the MMA.  The operands sit in
// shared memory in fragment order -- A as [k/4][row][k%4], the weights as
// [k/4][n/8][n%8][k%4] (permuted once per call by the split-weights kernel,
// heavy_weights_f64_item) -- so every fragment load is one conflict-free
// 256-byte LDS.64.  The weights stream through a 3-slot ring of 48 KB chunks
// filled by bulk copies from a producer warp.
// Measured (C4 / C8 heavy GRU, in-step): 26.8 / 18.5 us, DMMA pipe ~42% busy
// on the 105 SMs that hold a batch.  On the way: the FFMA form with thread =
// (4 rows, column) was bound by shared-memory wavefronts (one LDS per DFMA:
// 48.9 / 24 us); before it, weights read from L2 per FMA (60 us), fp32
// weights converted per use (F2F on the XU pipe, 66 us) and a (row,
// column-quad) mapping (107 us); serial operand fills (one round trip per
// element loop) were 30% of the DMMA form's stall samples.
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.cuh"
#include "ptx.cuh"

namespace saga {
namespace {

constexpr int kF = 128;            // hidden width (in = out = 128, checked by the host)
constexpr int kR = 8;              // rows per CTA batch = the DMMA's M
constexpr int kCompute = 256;      // 8 MMA warps x 16 output columns
constexpr int kThreads = kCompute + 32;  // + one producer warp (weight chunks)
constexpr int kNT = 2;             // 8-column n-tiles per warp
constexpr int kSlot = 48 * 1024;   // ring slot (bytes): fp64 weights
constexpr int kSlots = 3;          // ring depth
constexpr int kChunkG = 8;         // gate phase: K-rows per chunk (x 6 matrices of [kF][kF] fp64)
constexpr int kChunkM = 32;        // message / B phase: K-rows per chunk of one [K][kF] fp64 matrix

struct alignas(16) Ring {
    uint64_t full[kSlots];   // chunk landed (1 arrival + tx bytes)
    uint64_t empty[kSlots];  // chunk consumed (one arrival per MMA warp)
};

// the MMA warps' own barrier (the producer warp never joins)
__device__ __forceinline__ void compute_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kCompute) : "memory"); }

// D (8 x 8) += A (8 x 4) . B (4 x 8), fp64; per lane: a = A[lane / 4][lane % 4],
// b = B[lane % 4][lane / 4], d = D[lane / 4][2 (lane % 4) + {0, 1}]
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// fragment-order position of element (r, k) of an [kR][K] A operand
__device__ __forceinline__ int afrag(int r, int k) { return (k >> 2) * 32 + r * 4 + (k & 3); }

// Operand fills (MMA warps): every global load of a thread is issued before
// the first shared-memory store -- as a loop with a store per load they were
// serial round trips (30% of the GGNN GRU's stall samples).
// dst[afrag(r, j)] = H[rows[b0 + r]][j] (0 past nr rows), [kR][kF]
__device__ __forceinline__ void fill_rows_f32(double *dst, const float *__restrict__ H, const int32_t *__restrict__ rows,
                                              int32_t b0, int nr) {
    constexpr int kPer = kR * kF / kCompute;
    float v[kPer];
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const int i = threadIdx.x + q * kCompute, rr = i / kF;
        v[q] = rr < nr ? __ldg(H + (int64_t)__ldg(rows + b0 + rr) * kF + i % kF) : 0.0f;
    }
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const int i = threadIdx.x + q * kCompute;
        dst[afrag(i / kF, i % kF)] = (double)v[q];
    }
}
// dst[afrag(r, k)] = src[r][k] (0 past nr rows), [kR][K] fp64, K a multiple of kCompute / kR
__device__ __forceinline__ void fill_f64(double *dst, const double *src, int K, int nr) {
    constexpr int kBatch = 8;
    for (int i0 = threadIdx.x; i0 < kR * K; i0 += kBatch * kCompute) {
        double v[kBatch];
#pragma unroll
        for (int q = 0; q < kBatch; ++q) {
            const int i = i0 + q * kCompute;
            v[q] = (i < kR * K && i / K < nr) ? __ldcg(src + i) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < kBatch; ++q) {
            const int i = i0 + q * kCompute;
            if (i < kR * K) dst[afrag(i / K, i % K)] = v[q];
        }
    }
}

// The weight chunks of a CTA's whole run form one sequence through the
// kSlots-deep ring: per batch, the message (or B) GEMM's chunks of kChunkM
// K-rows (n1 of them, 0 for the GGNN GRU), then the gate phase's chunks of
// kChunkG K-rows of all six gate matrices (n2).  A producer warp issues chunk
// s + kSlots as soon as every MMA warp has released chunk s -- across phases
// and batches -- so the MMA warps never wait on one another for the ring.
struct Feed {
    Ring *ring;
    double *slots;
    const double *W1;            // [K1][kF] message / B weights (fragment order)
    const double *W_ih, *W_hh;   // gate weights, [3][kF][kF] each (fragment order)
    int n1, n2;                  // chunks per batch of each phase
    uint32_t total;              // chunks of the CTA's run
    __device__ void issue(uint32_t seq) const {
        if (seq >= total) return;
        double *dst = slots + (seq % kSlots) * (kSlot / 8);
        const int local = (int)(seq % (uint32_t)(n1 + n2));
        uint64_t *bar = &ring->full[seq % kSlots];
        if (local < n1) {
            ptx::mbar_arrive_expect_tx(bar, kChunkM * kF * 8);
            ptx::bulk_g2s(dst, W1 + (int64_t)local * kChunkM * kF, kChunkM * kF * 8, bar);
            return;
        }
        const int c = local - n1;
        ptx::mbar_arrive_expect_tx(bar, 6 * kChunkG * kF * 8);
        for (int mat = 0; mat < 6; ++mat)
            ptx::bulk_g2s(dst + mat * kChunkG * kF, (mat < 3 ? W_ih : W_hh) + ((int64_t)(mat % 3) * kF + c * kChunkG) * kF,
                          kChunkG * kF * 8, bar);
    }
    // wait for chunk seq; returns its slot
    __device__ const double *wait(uint32_t seq) const {
        ptx::mbar_wait(&ring->full[seq % kSlots], (seq / kSlots) & 1);
        return slots + (seq % kSlots) * (kSlot / 8);
    }
    // this warp is done with chunk seq
    __device__ void release(uint32_t seq) const {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) ptx::mbar_arrive(&ring->empty[seq % kSlots]);
    }
    // the producer warp's loop (one thread)
    __device__ void produce() const {
        for (uint32_t seq = 0; seq < total; ++seq) {
            if (seq >= kSlots) ptx::mbar_wait(&ring->empty[seq % kSlots], ((seq / kSlots) - 1) & 1);
            issue(seq);
        }
    }
};

// acc[t] += x . W1 over K for this warp's n-tiles: x in A-fragment order, the
// [K][kF] weights arriving through the feed in chunks of kChunkM K-rows.  Two
// accumulator sets (even / odd k-steps) keep four independent MMA chains per
// warp.
__device__ __forceinline__ void stream_mma(double (&acc)[kNT][2], const double *x, int K, const Feed &fd,
                                           uint32_t &cc, int nt0, int lane) {
    const int nch = K / kChunkM;
    double odd[kNT][2] = {};
    for (int c = 0; c < nch; ++c, ++cc) {
        const double *w = fd.wait(cc);
        const double *xa = x + c * (kChunkM / 4) * 32 + lane;
#pragma unroll
        for (int kb = 0; kb < kChunkM / 4; kb += 2) {
            const double a0 = xa[kb * 32], a1 = xa[(kb + 1) * 32];
#pragma unroll
            for (int t = 0; t < kNT; ++t) {
                dmma(acc[t], a0, w[(kb * 16 + nt0 + t) * 32 + lane]);
                dmma(odd[t], a1, w[((kb + 1) * 16 + nt0 + t) * 32 + lane]);
            }
        }
        fd.release(cc);
    }
#pragma unroll
    for (int t = 0; t < kNT; ++t) {
        acc[t][0] += odd[t][0];
        acc[t][1] += odd[t][1];
    }
}

// smem: ring 2 x kSlot | a[kR][T kF] (gated) | m[kR][kF] | h[kR][kF], fp64, A-fragment order
size_t smem_bytes(int T) { return kSlots * (size_t)kSlot + sizeof(double) * ((size_t)kR * T * kF + 2 * kR * kF); }

__global__ void __launch_bounds__(kThreads, 1)
    k_gru_heavy_f64(int32_t nh, const int32_t *__restrict__ rows, int32_t T, const double *__restrict__ Sx,
                    const double *__restrict__ W64, const double *__restrict__ mx, const float *__restrict__ H,
                    const float *__restrict__ b_ih, const float *__restrict__ b_hh, float *__restrict__ out) {
    extern __shared__ __align__(16) uint8_t smem[];
    const bool gated = Sx != nullptr;
    const int K = T * kF;
    double *slots = reinterpret_cast<double *>(smem);
    const double *W_type = W64, *W_ih = W64 + (int64_t)K * kF * gated, *W_hh = W_ih + 3 * kF * kF;
    double *a = reinterpret_cast<double *>(smem + kSlots * kSlot);  // [kR][K]      (gated only)
    double *m = a + (gated ? kR * K : 0);                       // [kR][kF]
    double *h = m + kR * kF;                                    // [kR][kF]
    __shared__ Ring ring;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nt0 = warp * kNT, r = lane >> 2, c2 = (lane & 3) * 2;  // this lane's D row and column pair
    if (threadIdx.x == 0) {
        for (int i = 0; i < kSlots; ++i) {
            ptx::mbar_init(&ring.full[i], 1);
            ptx::mbar_init(&ring.empty[i], kCompute / 32);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    uint32_t cc = 0;  // chunks consumed (ring sequence)
    const int nb = (nh - (int)blockIdx.x * kR + (int)gridDim.x * kR - 1) / ((int)gridDim.x * kR);  // batches of this CTA
    const Feed fd{&ring, slots, W_type, W_ih, W_hh, gated ? K / kChunkM : 0, kF / kChunkG,
                  (uint32_t)nb * (uint32_t)((gated ? K / kChunkM : 0) + kF / kChunkG)};

    if (warp == kCompute / 32) {  // producer warp
        griddep_wait();  // the fp64 weights come from the call's split-weights kernel
        if (lane == 0) fd.produce();
        return;
    }
    // the layer's own inputs (H, the biases, the graph) before the grid dependency
    float bias[6][kNT][2];
#pragma unroll
    for (int t = 0; t < kNT; ++t)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int j = (nt0 + t) * 8 + c2 + e;
#pragma unroll
            for (int g = 0; g < 3; ++g) {
                bias[g][t][e] = b_ih[g * kF + j];
                bias[3 + g][t][e] = b_hh[g * kF + j];
            }
        }
    if ((int)blockIdx.x * kR < nh) fill_rows_f32(h, H, rows, blockIdx.x * kR, min(kR, nh - (int)blockIdx.x * kR));
    griddep_wait();  // Sx / mx and the tensor path's output rows come from the call's earlier kernels
    for (int32_t b0 = blockIdx.x * kR; b0 < nh; b0 += gridDim.x * kR) {
        const int nr = min(kR, nh - b0);
        if (b0 != (int32_t)blockIdx.x * kR) fill_rows_f32(h, H, rows, b0, nr);
        if (gated)
            fill_f64(a, Sx + (int64_t)b0 * K, K, nr);
        else
            fill_f64(m, mx + (int64_t)b0 * kF, kF, nr);
        compute_sync();
        if (gated) {
            // m = S . W_type  (W_type [T][kF][kF] = [K][kF])
            double acc[kNT][2] = {};
            stream_mma(acc, a, K, fd, cc, nt0, lane);
#pragma unroll
            for (int t = 0; t < kNT; ++t) {
                const int col = (nt0 + t) * 8 + c2;
                m[afrag(r, col)] = acc[t][0];
                m[afrag(r, col + 1)] = acc[t][1];
            }
            compute_sync();
        }
        // gate pre-activations: gi[g] = m . W_ih[g], gh[g] = h . W_hh[g] (g = r, z, n); the six
        // matrices stream together in chunks of kChunkG K-rows, [mat][kChunkG / 4][kF / 8][32] per slot
        double gi[3][kNT][2] = {}, gh[3][kNT][2] = {};
        for (int c = 0; c < kF / kChunkG; ++c, ++cc) {
            const double *w = fd.wait(cc) + lane;
#pragma unroll
            for (int kb = 0; kb < kChunkG / 4; ++kb) {
                const double am = m[(c * (kChunkG / 4) + kb) * 32 + lane];
                const double ah = h[(c * (kChunkG / 4) + kb) * 32 + lane];
#pragma unroll
                for (int t = 0; t < kNT; ++t)
#pragma unroll
                    for (int g = 0; g < 3; ++g) {
                        dmma(gi[g][t], am, w[g * kChunkG * kF + (kb * 16 + nt0 + t) * 32]);
                        dmma(gh[g][t], ah, w[(3 + g) * kChunkG * kF + (kb * 16 + nt0 + t) * 32]);
                    }
            }
            fd.release(cc);
        }
        // PyTorch GRUCell (reading A15): r = s(gi_r + gh_r), z = s(gi_z + gh_z),
        // n = tanh(gi_n + r gh_n), h' = (1 - z) n + z h  -- on this lane's D elements
        if (r < nr) {
            float *o = out + (int64_t)rows[b0 + r] * kF;
#pragma unroll
            for (int t = 0; t < kNT; ++t)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int j = (nt0 + t) * 8 + c2 + e;
                    const double rg = 1.0 / (1.0 + exp(-(gi[0][t][e] + bias[0][t][e] + gh[0][t][e] + bias[3][t][e])));
                    const double zg = 1.0 / (1.0 + exp(-(gi[1][t][e] + bias[1][t][e] + gh[1][t][e] + bias[4][t][e])));
                    const double n = tanh(gi[2][t][e] + bias[2][t][e] + rg * (gh[2][t][e] + bias[5][t][e]));
                    o[j] = (float)((1.0 - zg) * n + zg * h[afrag(r, j)]);
                }
        }
        compute_sync();  // m, h, a are rewritten by the next batch
    }
}

// GGNN heavy rows: Bx[s][j] = sum_k H[v_s][k] W_e[f + k][j] + b_e[j] in fp64
// (W_e [2f][f], source rows first; W_b = rows f .. 2f-1, converted to fp64).
__global__ void __launch_bounds__(kThreads, 1)
    k_ggnn_heavy_b(int32_t nh, const int32_t *__restrict__ rows, const float *__restrict__ H,
                   const double *__restrict__ W_b, const float *__restrict__ b_e, double *__restrict__ Bx) {
    extern __shared__ __align__(16) uint8_t smem[];
    double *slots = reinterpret_cast<double *>(smem);
    double *hs = reinterpret_cast<double *>(smem + kSlots * kSlot);  // [kR][kF], A-fragment order
    __shared__ Ring ring;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nt0 = warp * kNT, r = lane >> 2, c2 = (lane & 3) * 2;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kSlots; ++i) {
            ptx::mbar_init(&ring.full[i], 1);
            ptx::mbar_init(&ring.empty[i], kCompute / 32);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    uint32_t cc = 0;
    const int nb = (nh - (int)blockIdx.x * kR + (int)gridDim.x * kR - 1) / ((int)gridDim.x * kR);
    const Feed fd{&ring, slots, W_b, nullptr, nullptr, kF / kChunkM, 0, (uint32_t)nb * (uint32_t)(kF / kChunkM)};
    if (warp == kCompute / 32) {  // producer warp
        griddep_wait();  // the fp64 weights come from the call's split-weights kernel
        if (lane == 0) fd.produce();
        return;
    }
    for (int32_t b0 = blockIdx.x * kR; b0 < nh; b0 += gridDim.x * kR) {
        const int nr = min(kR, nh - b0);
        fill_rows_f32(hs, H, rows, b0, nr);  // the layer input: before the grid dependency
        if (b0 == (int32_t)blockIdx.x * kR) griddep_wait();  // before this grid's first global write
        compute_sync();
        double acc[kNT][2] = {};
        stream_mma(acc, hs, kF, fd, cc, nt0, lane);
        if (r < nr)
#pragma unroll
            for (int t = 0; t < kNT; ++t)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int j = (nt0 + t) * 8 + c2 + e;
                    Bx[(int64_t)(b0 + r) * kF + j] = acc[t][e] + (b_e ? (double)b_e[j] : 0.0);
                }
        compute_sync();
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
