// lstm_gather.cu -- GraphSAGE-LSTM Gather: every
// sequence of the layer in one forked pair of persistent kernels.
//
// Paper: GraphSAGE's Gather is LSTM(in_edges) (Table 1); the LSTM
// "treats the inedges of a vertex as a sequence" and DGL runs it by "degree
// traversal", one batched launch per distinct degree, which leaves the GPU
// idle up to 20x the kernel time.  Here the input
// projections P_g = X . W_ih[g] (gates i, f, g, o) are tensor-core GEMMs
// before this file's kernels, so a step gathers one 1 KB row of P and applies
// the recurrent GEMV h . W_hh.  Two bounds meet (C7: 1.05M steps; one hub
// of 6,614 dependent steps): the per-SM step count and the longest chain, so
// the work is split by sequence length (the graph's deg_order, descending):
//   * k_lstm_cluster -- sequences of >= kLongDeg steps, each on a 2-CTA
//     cluster: CTA r owns 64 units, thread (unit, gate) with its W_hh^T row
//     in 64 registers (128 FHFMA.BF16 per step), and the two halves of h are
//     exchanged every step through distributed shared memory (st.async +
//     mbarrier, no cluster-wide barrier): the chain's step takes ~0.55 us
//     instead of 0.66-0.74 on one SM;
//   * k_lstm_mma -- the rest, 8 sequences per CTA on the tensor cores
//     (mma.sync m16n8k16 with W_hh^T as the A operand and the 8 sequences as
//     N): one step of 8 sequences issues what one sequence's FHFMA GEMV does.
// The two run concurrently (the caller's stream and a library stream, forked
// and joined with events).  Reading A25: sequence = in-edges in
// CSR order, PyTorch LSTMCell (i, f, g, o), zero initial state, output =
// final h (0 without in-edges), stored bf16 for the ApplyVertex concat-GEMM.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <mutex>

#include "internal.cuh"
#include "ptx.cuh"

namespace saga {
namespace {

constexpr int kF = 128;        // hidden = input width
constexpr int kThreads = 512;  // one thread per (unit, gate): 128 x 4
constexpr int kAhead = 2;      // steps of P prefetched ahead

// sigm(x) = 1 / (1 + e^-x) with the fast reciprocal (|error| ~1e-7, the
// output feeds bf16 h); tanh(x) = 2 sigm(2x) - 1
__device__ __forceinline__ float sigm_fast(float x) { return __fdividef(1.0f, 1.0f + __expf(-x)); }

// wt[j][g][c] = W_hh[g][8c .. 8c+7][j] (bf16): row (unit j, gate g) of W_hh^T, 256 contiguous bytes
// (thread 0 also resets the gather's work-queue head)
__global__ void k_stage_whh(const __nv_bfloat16 *__restrict__ W_hh, uint4 *wt, int32_t *queue) {
    griddep_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;  // over kF * 4 * kF / 8 chunks
    if (i == 0) queue[0] = queue[1] = 0;
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

// ------------------------------------------------------------------------
// The long sequences on CTA pairs (a 2-CTA cluster per sequence): CTA r owns
// the units [64 r, 64 r + 64) -- thread (unit, gate) with its W_hh^T row in
// registers -- so a step's FHFMA work per SM halves (512
// issue cycles per SMSP instead of 1,024).  Each CTA keeps the full h in its
// shared memory: after a step every warp sends its 8 new h values (16 bytes)
// into the peer's copy with st.async, completing bytes on the peer's
// mbarrier for that h buffer, so a step waits for the peer's half of h on
// an mbarrier (no cluster-wide barrier per step).  The pair takes items from
// queue[0] while they have at least min_deg steps.
struct alignas(16) PairSmem {
    uint4 hb[2][kF / 8];   // h (bf16), double-buffered by step parity; this CTA's half written locally
    uint64_t hfull[2];     // the peer's 128-byte half of hb[b] arrived
    int32_t v;
};

__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_peer(uint32_t local_addr, uint32_t peer) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(peer));
    return r;
}

// CS CTAs per sequence (2 or 4; the cluster shape is given at launch)
template <int CS>
__global__ void __launch_bounds__(512 / CS, 1)
    k_lstm_cluster(int32_t n, const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col_src,
                   const int32_t *__restrict__ order, const __nv_bfloat16 *__restrict__ P,  // [4][n][kF]
                   const uint4 *__restrict__ wt,                                            // staged W_hh^T
                   const float *__restrict__ b_ih, const float *__restrict__ b_hh,          // [4][kF]
                   __nv_bfloat16 *__restrict__ h_out, int32_t *queue, int32_t min_deg) {
    constexpr int kU = kF / CS;                  // units per CTA
    constexpr uint32_t kPeerBytes = (CS - 1) * kU * 2;  // h bytes arriving from the other CTAs per step
    __shared__ PairSmem S;
    const uint32_t rank = cluster_ctarank();
    const int jl = threadIdx.x / 4, g = threadIdx.x % 4;  // local unit, gate
    const int j = kU * (int)rank + jl;
    const int lane = threadIdx.x & 31, gbase = lane & ~3, warp = threadIdx.x >> 5;
    const int chunk = (kU / 8) * (int)rank + warp;  // this warp's 8 units: 16 bytes of hb
    if (threadIdx.x == 0) {
        ptx::mbar_init(&S.hfull[0], 1);
        ptx::mbar_init(&S.hfull[1], 1);
        ptx::fence_mbar_init();
        ptx::mbar_arrive_expect_tx(&S.hfull[0], kPeerBytes);  // armed: each phase takes the other CTAs' units
        ptx::mbar_arrive_expect_tx(&S.hfull[1], kPeerBytes);
    }
    griddep_wait();  // P, W_hh^T and the queue head come from the call's earlier kernels
    uint4 w[kF / 8];
#pragma unroll
    for (int c = 0; c < kF / 8; ++c) w[c] = __ldg(wt + ((int64_t)j * 4 + g) * (kF / 8) + c);
    const float bias = __ldg(b_ih + g * kF + j) + __ldg(b_hh + g * kF + j);
    const float ks = g == 2 ? 2.0f : 1.0f;
    const __nv_bfloat16 *Pg = P + g * (int64_t)n * kF + j;
    // the other CTAs' copies of this warp's chunk of hb[b] and their mbarriers
    uint32_t rh[2][CS - 1], rb[2][CS - 1];
#pragma unroll
    for (int q = 0; q < CS - 1; ++q) {
        const uint32_t pr = (rank + 1 + q) % CS;
        rh[0][q] = map_peer(ptx::smem_u32(&S.hb[0][chunk]), pr);
        rh[1][q] = map_peer(ptx::smem_u32(&S.hb[1][chunk]), pr);
        rb[0][q] = map_peer(ptx::smem_u32(&S.hfull[0]), pr);
        rb[1][q] = map_peer(ptx::smem_u32(&S.hfull[1]), pr);
    }
    uint32_t par[2] = {0u, 0u};
    cluster_sync_all();  // every CTA's barriers are initialised before any remote arrival
    for (;;) {
        if (rank == 0 && threadIdx.x == 0) {
            const int32_t qi = atomicAdd(queue, 1);
            int32_t vv = qi < n ? order[qi] : -1;
            if (vv >= 0 && row_ptr[vv + 1] - row_ptr[vv] < min_deg) vv = -1;
            S.v = vv;
#pragma unroll
            for (int q = 1; q < CS; ++q)
                asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(map_peer(ptx::smem_u32(&S.v), (uint32_t)q)),
                             "r"(vv)
                             : "memory");
        }
        if (threadIdx.x < kF / 8) S.hb[1][threadIdx.x] = make_uint4(0, 0, 0, 0);  // h(-1) = 0, every unit
        cluster_sync_all();
        const int32_t v = S.v;
        if (v < 0) break;
        const int32_t p0 = (int32_t)row_ptr[v], p1 = (int32_t)row_ptr[v + 1];
        float c = 0.0f, hf = 0.0f;
        __nv_bfloat16 ring[kAhead];
#pragma unroll
        for (int a = 0; a < kAhead; ++a)
            ring[a] = (p0 + a < p1) ? Pg[(int64_t)__ldg(col_src + p0 + a) * kF] : __float2bfloat16_rn(0.0f);
        // the source of step p + kAhead, loaded a step before its P row (so no
        // step waits on a col_src load)
        int32_t un = (p0 + kAhead < p1) ? __ldg(col_src + p0 + kAhead) : 0;
        for (int32_t p = p0; p < p1; ++p) {
            const int t = p - p0, bi = (t + 1) & 1, bo = t & 1;  // read h(t-1) from hb[bi], write h(t) to hb[bo]
            if (t > 0) {  // the other CTAs' units of h(t-1); then re-armed for h(t+1), which they
                          // send only after they have this CTA's h(t), sent after this point
                ptx::mbar_wait(&S.hfull[bi], par[bi]);
                par[bi] ^= 1u;
                if (threadIdx.x == 0) ptx::mbar_arrive_expect_tx(&S.hfull[bi], kPeerBytes);
            }
            const float pz = __bfloat162float(ring[0]);
#pragma unroll
            for (int a = 0; a + 1 < kAhead; ++a) ring[a] = ring[a + 1];
            ring[kAhead - 1] = (p + kAhead < p1) ? Pg[(int64_t)un * kF] : __float2bfloat16_rn(0.0f);
            un = (p + kAhead + 1 < p1) ? __ldg(col_src + p + kAhead + 1) : 0;
            float a4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
            const uint4 *hb = S.hb[bi];
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
            if (g == 0) reinterpret_cast<__nv_bfloat16 *>(S.hb[bo])[j] = __float2bfloat16_rn(hf);
            __syncwarp();
            if (lane == 0) {  // this warp's 8 units of h(t) into the other CTAs' hb[bo]
                const uint4 x = S.hb[bo][chunk];
#pragma unroll
                for (int q = 0; q < CS - 1; ++q)
                    asm volatile(
                        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, "
                        "[%5];" ::"r"(bo ? rh[1][q] : rh[0][q]),
                        "r"(x.x), "r"(x.y), "r"(x.z), "r"(x.w), "r"(bo ? rb[1][q] : rb[0][q])
                        : "memory");
            }
            __syncthreads();  // this CTA's units of h(t) are visible; every read of hb[bi] is done
        }
        if (g == 0) h_out[(int64_t)v * kF + j] = __float2bfloat16_rn(hf);
        // the other CTAs' units of the last h arrived (keeps the barrier phases in step)
        const int tl = p1 - p0 - 1, bl = tl & 1;
        ptx::mbar_wait(&S.hfull[bl], par[bl]);
        par[bl] ^= 1u;
        if (threadIdx.x == 0) ptx::mbar_arrive_expect_tx(&S.hfull[bl], kPeerBytes);
        __syncthreads();
    }
    cluster_sync_all();  // no CTA exits while another may still write into it
}

// ------------------------------------------------------------------------
// The sequences shorter than kLongDeg in batches on the tensor cores
// (mma.sync m16n8k16, bf16 -> fp32), concurrently with k_lstm_cluster on the
// long ones.  The recurrent GEMV of a step is computed transposed, G^T =
// W_hh^T . H^T: the 512 gate rows are the MMA's M (W_hh^T resident in
// registers as A fragments, 64 per thread) and up to 8 sequences (the CTA's
// slots) its N, so one step of 8 sequences is 512 HMMA per SM -- measured at
// 8 cycles per HMMA per SMSP, the issue time of ONE sequence's FHFMA GEMV.
// Gate rows are unit-major (m = 4 j + g): a unit's four gate pre-activations
// are one float4 of the step's gate block G in shared memory, and thread
// (slot s, units j0, j0 + 64) adds P + b, applies the gates and keeps c.
// Each slot walks its own 8-item chunk of the queue (queue[1]; the long items
// at its head are skipped) and loads its next item while the current one
// runs, so the next sequence's first P row is prefetched like any step's.
constexpr int kLongDeg = 2048;  // sequences of at least this many steps go to k_lstm_cluster
constexpr int kLongCluster = 2;  // CTAs per long sequence (a cluster; h exchanged through DSMEM; 4: slower)
constexpr int kLongCtas = 32;     // CTAs for them (16 pairs, one CTA per SM); the batches take the other SMs
constexpr int kSlots = 8;
constexpr int kHP = kF + 8;          // H row pitch (bf16): the B-fragment loads hit 32 distinct banks
constexpr int kGP = 4 * kF + 4;      // G row pitch (fp32): conflict-free C stores, 16-B rows
struct alignas(16) MmaSmem {
    __nv_bfloat16 H[kSlots][kHP];    // h of each slot (bf16): read by the MMAs, written by the activations
    float G[kSlots][kGP];            // the step's gate pre-activations, unit-major
};

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__global__ void __launch_bounds__(kThreads, 1)
    k_lstm_mma(int32_t n, const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col_src,
               const int32_t *__restrict__ order, const __nv_bfloat16 *__restrict__ P,  // [4][n][kF]
               const __nv_bfloat16 *__restrict__ W_hh,                                  // [4][kF (k)][kF (j)]
               const float *__restrict__ b_ih, const float *__restrict__ b_hh, __nv_bfloat16 *__restrict__ h_out,
               int32_t long_deg) {
    __shared__ MmaSmem S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gr = lane >> 2, gc = lane & 3;  // fragment group / thread-in-group
    // A fragments: W_hh^T rows m = 32 warp + 16 t + {gr, gr + 8}, k = 16 ks + 2 gc (+8)
    uint32_t a[2][kF / 16][4];
    auto wt = [&](int m, int k) -> uint32_t {
        return __bfloat16_as_ushort(W_hh[((int64_t)(m & 3) * kF + k) * kF + (m >> 2)]);
    };
#pragma unroll
    for (int t = 0; t < 2; ++t) {
#pragma unroll
        for (int ks = 0; ks < kF / 16; ++ks) {
            const int m0 = 32 * warp + 16 * t + gr, m1 = m0 + 8, k0 = 16 * ks + 2 * gc, k1 = k0 + 8;
            a[t][ks][0] = wt(m0, k0) | (wt(m0, k0 + 1) << 16);
            a[t][ks][1] = wt(m1, k0) | (wt(m1, k0 + 1) << 16);
            a[t][ks][2] = wt(m0, k1) | (wt(m0, k1 + 1) << 16);
            a[t][ks][3] = wt(m1, k1) | (wt(m1, k1 + 1) << 16);
        }
    }
    // activation role: slot s (threads 64 s .. 64 s + 63: two warps), units j0 and j0 + 64
    const int s = threadIdx.x >> 6, j0 = threadIdx.x & 63;
    float bias[2][4];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int g = 0; g < 4; ++g) bias[u][g] = b_ih[g * kF + j0 + 64 * u] + b_hh[g * kF + j0 + 64 * u];
    for (int i = threadIdx.x; i < kSlots * kHP; i += kThreads) (&S.H[0][0])[i] = __float2bfloat16_rn(0.0f);
    griddep_wait();  // P and the queue heads come from the call's earlier kernels

    // slot state, identical in the slot's 64 threads: current item (v, p, p1),
    // the next one (nv, np, np1: loaded while the current one runs), the
    // slot's chunk of the queue [cb, ce)
    // slot state, identical in the slot's 64 threads.  Items are dealt to the
    // slots round-robin in queue order (descending in-degree: every slot gets
    // a similar share), so a slot knows its next items without any atomic:
    // the current one (v, p, p1), the next one (nv, np, np1: its row_ptr loads
    // issued when the previous item started) and the vertex after it (nnv),
    // so a sequence switch never waits on a load.
    const int32_t nslots = (int32_t)gridDim.x * kSlots;
    int32_t kn = (int32_t)blockIdx.x * kSlots + s;  // the slot's next queue index to fetch
    auto fetch_v = [&]() -> int32_t {
        const int32_t r = kn < n ? __ldg(order + kn) : -1;
        kn += nslots;
        return r;
    };
    int32_t v = fetch_v(), p = 0, p1 = 0;
    if (v >= 0) { p = (int32_t)__ldg(row_ptr + v); p1 = (int32_t)__ldg(row_ptr + v + 1); }
    int32_t nv = fetch_v(), np = 0, np1 = 0;
    if (nv >= 0) { np = (int32_t)__ldg(row_ptr + nv); np1 = (int32_t)__ldg(row_ptr + nv + 1); }
    int32_t nnv = fetch_v();
    float c[2] = {0.0f, 0.0f};
    // P values of a step, raw bf16 (unit u, gate g at [4 u + g]): loaded a
    // whole step before their use and converted only then, in two register
    // sets that swap roles every step (a register copy would wait on the load)
    uint16_t pa[8], pb[8];
    auto load_p = [&](int32_t q, uint16_t (&dst)[8]) {
        const int32_t u = __ldg(col_src + q);
#pragma unroll
        for (int uu = 0; uu < 2; ++uu)
#pragma unroll
            for (int g = 0; g < 4; ++g)
                dst[4 * uu + g] = __ldg(reinterpret_cast<const unsigned short *>(P) + ((int64_t)g * n + u) * kF + j0 +
                                        64 * uu);
    };
    auto shift = [&]() {
        v = nv; p = np; p1 = np1;
        nv = nnv;
        if (nv >= 0) { np = (int32_t)__ldg(row_ptr + nv); np1 = (int32_t)__ldg(row_ptr + nv + 1); }
        nnv = fetch_v();
    };
    // make the first runnable item current: empty ones (in-degree 0: h = 0)
    // are finished here, the long ones belong to the CTA pairs
    auto settle = [&]() {
        while (v >= 0 && (p1 == p || p1 - p >= long_deg)) {
            if (p1 == p) {
                h_out[(int64_t)v * kF + j0] = __float2bfloat16_rn(0.0f);
                h_out[(int64_t)v * kF + j0 + 64] = __float2bfloat16_rn(0.0f);
            }
            shift();
        }
    };
    settle();
    if (v >= 0) load_p(p, pa);
    __syncthreads();  // H is zero before the first MMA reads it
    // one step: cur holds this step's P, nxt receives the next step's
    auto step = [&](uint16_t (&cur)[8], uint16_t (&nxt)[8]) -> bool {
        bool pre = false;  // the next step's P is in flight
        if (v >= 0) {
            if (p + 1 < p1) {
                load_p(p + 1, nxt);
                pre = true;
            } else if (nv >= 0 && np1 > np && np1 - np < long_deg) {
                load_p(np, nxt);
                pre = true;
            }
        }
        // ---- MMA: G^T[gate rows][slots] = W_hh^T . H^T ----
        {
            uint32_t b[kF / 16][2];
#pragma unroll
            for (int ks = 0; ks < kF / 16; ++ks) {
                const uint32_t *hr = reinterpret_cast<const uint32_t *>(&S.H[gr][16 * ks + 2 * gc]);
                b[ks][0] = hr[0];
                b[ks][1] = hr[4];
            }
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                float d[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
                for (int ks = 0; ks < kF / 16; ++ks) mma_bf16_16816(d, a[t][ks], b[ks][0], b[ks][1]);
                const int m = 32 * warp + 16 * t + gr;
                S.G[2 * gc][m] = d[0];
                S.G[2 * gc + 1][m] = d[1];
                S.G[2 * gc][m + 8] = d[2];
                S.G[2 * gc + 1][m + 8] = d[3];
            }
        }
        __syncthreads();
        // ---- activations of slot s, units j0 and j0 + 64 ----
        if (v >= 0) {
            const bool last = p + 1 == p1;
#pragma unroll
            for (int uu = 0; uu < 2; ++uu) {
                const int j = j0 + 64 * uu;
                const float4 z = *reinterpret_cast<const float4 *>(&S.G[s][4 * j]);
                auto pv = [&](int g) { return __uint_as_float((uint32_t)cur[4 * uu + g] << 16); };
                const float ig = sigm_fast(z.x + pv(0) + bias[uu][0]);
                const float fg = sigm_fast(z.y + pv(1) + bias[uu][1]);
                const float gg = 2.0f * sigm_fast(2.0f * (z.z + pv(2) + bias[uu][2])) - 1.0f;
                const float og = sigm_fast(z.w + pv(3) + bias[uu][3]);
                c[uu] = fg * c[uu] + ig * gg;
                const float h = og * (2.0f * sigm_fast(2.0f * c[uu]) - 1.0f);
                const __nv_bfloat16 hb = __float2bfloat16_rn(h);
                if (!last) {
                    S.H[s][j] = hb;
                } else {
                    h_out[(int64_t)v * kF + j] = hb;
                    S.H[s][j] = __float2bfloat16_rn(0.0f);  // the next sequence starts from h = 0
                    c[uu] = 0.0f;
                }
            }
            if (!last) {
                ++p;
            } else {
                shift();
                settle();
                if (v >= 0 && !pre) load_p(p, nxt);  // (the prefetched item was skipped)
            }
        }
        return __syncthreads_or(v >= 0);
    };
    for (;;) {
        if (!step(pa, pb)) break;
        if (!step(pb, pa)) break;
    }
}

}  // namespace

// [staged W_hh^T | work-queue head]: the head lives in this region, not among
// the split-row ticket counters (which every completed call leaves zero); the
// staging kernel resets it before every gather
size_t lstm_workspace_bytes() { return sizeof(uint4) * 4 * kF * kF / 8 + 16; }

namespace {
// A library stream per device for the second half of a forked launch pair, with
// its fork / join events (created once; the enqueue of a fork-join is
// serialised across host threads, so concurrent calls do not interleave the
// event records).
struct SideStream {
    cudaStream_t st = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
std::mutex g_side_mu;
SideStream &side_stream(int dev) {
    static SideStream ss[64];
    SideStream &x = ss[dev & 63];
    if (!x.st) {
        cudaStreamCreateWithFlags(&x.st, cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming);
    }
    return x;
}
}  // namespace

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
    if (g.max_in_deg < kLongDeg) {  // no long sequence: the batches alone
        const unsigned grid = (unsigned)(g.n < sms ? g.n : sms);
        return launch(k_lstm_mma, grid, kThreads, 0, st, g.n, g.row_ptr, g.col_src, g.deg_order, P, W_hh, b_ih,
                      b_hh, h_out, INT32_MAX);
    }
    // the long sequences on kLongCtas SMs (k_lstm_cluster, the caller's stream)
    // and the batches on the others (k_lstm_mma, a library stream forked and
    // joined with events, so the pair also captures into a CUDA graph)
    std::lock_guard<std::mutex> lock(g_side_mu);
    SideStream &ss = side_stream(dev);
    if (!ss.st || !ss.fork || !ss.join) return cudaErrorInitializationError;
    if ((e = cudaEventRecord(ss.fork, st))) return e;
    if ((e = cudaStreamWaitEvent(ss.st, ss.fork, 0))) return e;
    {
        constexpr int CS = kLongCluster;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)kLongCtas);
        cfg.blockDim = dim3(512 / CS);
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = CS;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, k_lstm_cluster<CS>, g.n, (const int64_t *)g.row_ptr, (const int32_t *)g.col_src,
                               (const int32_t *)g.deg_order, P, (const uint4 *)wt, b_ih, b_hh, h_out, queue,
                               (int32_t)kLongDeg);
    }
    if (e) return e;
    e = launch<false>(k_lstm_mma, (unsigned)std::max(1, sms - kLongCtas), kThreads, 0, ss.st, g.n, g.row_ptr,
                      g.col_src, g.deg_order, P, W_hh, b_ih, b_hh, h_out, kLongDeg);
    if (e) return e;
    if ((e = cudaEventRecord(ss.join, ss.st))) return e;
    return cudaStreamWaitEvent(st, ss.join, 0);
}

}  // namespace saga
