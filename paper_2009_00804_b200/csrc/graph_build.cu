// graph_build.cu -- S0 (COO -> destination-sorted CSR), S1 (per-vertex norms)
// and S6 (merge-path load-balance schedule) on the GPU.
//
// Definition followed: PAPER.md line 130 (the layer input is the graph as an
// adjacency matrix) and lines 351-354 (row = destination vertex, nonzero =
// in-edge); reading A7: rows ordered by destination, ties in
// ascending COO index.  Stability comes from an LSD radix sort on dst whose
// payload starts as the COO index (each pass is a stable scatter), so the
// result is bit-exact and independent of scheduling -- no atomics decide any
// position.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "internal.cuh"

namespace saga {
namespace {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

constexpr int kSortThreads = 256;
constexpr int kSortRounds = 16;
constexpr int kSortTile = kSortThreads * kSortRounds;  // 4096 keys per block
constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;

// ------------------------------------------------------------ range check ----
// S0 range check fused with S2 degree counting: in-range edges count into the
// degrees (integer atomics: order-independent result), out-of-range ones
// report their lowest COO index.
__global__ void k_range_degrees(int32_t n, int64_t e, const int32_t *__restrict__ src,
                                const int32_t *__restrict__ dst, const int32_t *__restrict__ etype, int32_t T,
                                unsigned long long *first_bad, int32_t *in_deg, int32_t *out_deg) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t s = src[i], d = dst[i];
        bool bad = s < 0 || s >= n || d < 0 || d >= n;
        if (etype) {
            const int32_t t = etype[i];
            bad |= t < 0 || t >= T;
        }
        if (bad) {
            atomicMin(first_bad, (unsigned long long)i);
        } else {
            atomicAdd(in_deg + d, 1);
            atomicAdd(out_deg + s, 1);
        }
    }
}

// max in-degree (read back with the range-check result)
// max in-degree and the number of heavy rows (in-degree >= kHeavyInDeg), read
// back with the range check
__global__ void k_max_deg(int32_t n, const int32_t *__restrict__ in_deg, unsigned long long *out) {
    int32_t m = 0, heavy = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        m = max(m, in_deg[i]);
        heavy += in_deg[i] >= kHeavyInDeg;
    }
    for (int o = 16; o > 0; o >>= 1) {
        m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        heavy += __shfl_xor_sync(0xffffffffu, heavy, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(out, (unsigned long long)m);
        if (heavy) atomicAdd(out + 1, (unsigned long long)heavy);
    }
}

// ------------------------------------------------------------------- scan ----
// Exclusive scan of `count` non-negative integers into int64 out[0..count]
// (out[count] = total).  Three phases: tile sums -> scan of sums -> tiles.
template <typename Tin>
__device__ __forceinline__ int64_t block_scan_excl(int64_t v, int64_t *warp_sums, int64_t *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int64_t w = lane < (blockDim.x >> 5) ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int64_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        warp_sums[lane] = w;  // inclusive
    }
    __syncthreads();
    int64_t before = warp ? warp_sums[warp - 1] : 0;
    if (total) *total = warp_sums[(blockDim.x >> 5) - 1];
    int64_t r = before + x - v;
    __syncthreads();
    return r;
}

template <typename Tin>
__global__ void k_scan_tile_sums(const Tin *__restrict__ in, int64_t count, int64_t *sums) {
    __shared__ int64_t ws[32];
    int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    int64_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i)
        if (base + i < count) s += (int64_t)in[base + i];
    int64_t tot;
    block_scan_excl<Tin>(s, ws, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

template <typename Tin>
__global__ void k_scan_tiles(const Tin *__restrict__ in, int64_t count, const int64_t *__restrict__ tile_offs,
                             int64_t *out) {
    __shared__ int64_t ws[32];
    int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    int64_t v[kScanItems];
    int64_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        v[i] = base + i < count ? (int64_t)in[base + i] : 0;
        s += v[i];
    }
    int64_t tot;
    int64_t run = block_scan_excl<Tin>(s, ws, &tot) + tile_offs[blockIdx.x];
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        if (base + i < count) out[base + i] = run;
        run += v[i];
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == blockDim.x - 1) out[count] = run;
}

template <typename Tin>
cudaError_t scan_exclusive(const Tin *in, int64_t count, int64_t *out, cudaStream_t st) {
    if (count == 0) return cudaMemsetAsync(out, 0, sizeof(int64_t), st);
    int64_t tiles = (count + kScanTile - 1) / kScanTile;
    if (tiles == 1) {
        int64_t *zero;
        cudaError_t err = cudaMallocAsync(&zero, sizeof(int64_t), st);
        if (err) return err;
        cudaMemsetAsync(zero, 0, sizeof(int64_t), st);
        k_scan_tiles<Tin><<<1, kScanThreads, 0, st>>>(in, count, zero, out);
        cudaFreeAsync(zero, st);
        return cudaGetLastError();
    }
    int64_t *sums = nullptr, *offs = nullptr;
    cudaError_t err = cudaMallocAsync(&sums, sizeof(int64_t) * tiles, st);
    if (!err) err = cudaMallocAsync(&offs, sizeof(int64_t) * (tiles + 1), st);
    if (!err) {
        k_scan_tile_sums<Tin><<<(unsigned)tiles, kScanThreads, 0, st>>>(in, count, sums);
        err = scan_exclusive<int64_t>(sums, tiles, offs, st);
    }
    if (!err) {
        k_scan_tiles<Tin><<<(unsigned)tiles, kScanThreads, 0, st>>>(in, count, offs, out);
        err = cudaGetLastError();
    }
    if (sums) cudaFreeAsync(sums, st);  // every buffer allocated so far, also on failure
    if (offs) cudaFreeAsync(offs, st);
    return err;
}

// ------------------------------------------------------------- radix sort ----
// One LSD pass over digit (key >> shift) & 255.  Histogram layout is
// digit-major: hist[d * nblocks + b], so its exclusive scan gives every
// (digit, block) its global output offset; within a block, keys keep their
// input order (rank = #earlier equal digits), so the pass is stable.
__global__ void k_radix_hist(const int32_t *__restrict__ keys, int64_t e, int shift, int32_t *hist,
                             int64_t nblocks) {
    __shared__ int32_t h[kRadix];
    for (int i = threadIdx.x; i < kRadix; i += blockDim.x) h[i] = 0;
    __syncthreads();
    int64_t base = (int64_t)blockIdx.x * kSortTile;
    for (int r = 0; r < kSortRounds; ++r) {
        int64_t i = base + r * kSortThreads + threadIdx.x;
        if (i < e) atomicAdd(&h[(keys[i] >> shift) & (kRadix - 1)], 1);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kRadix; i += blockDim.x) hist[(int64_t)i * nblocks + blockIdx.x] = h[i];
}

__global__ void __launch_bounds__(kSortThreads) k_radix_scatter(const int32_t *__restrict__ keys_in,
                                                                const int32_t *__restrict__ vals_in, int64_t e,
                                                                int shift, const int64_t *__restrict__ offs,
                                                                int64_t nblocks, int32_t *keys_out,
                                                                int32_t *vals_out) {
    constexpr int kWarps = kSortThreads / 32;
    __shared__ int32_t wcnt[kWarps][kRadix];
    __shared__ int64_t gofs[kRadix];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int d = tid; d < kRadix; d += kSortThreads) gofs[d] = offs[(int64_t)d * nblocks + blockIdx.x];
    const uint32_t lt_mask = (1u << lane) - 1u;
    int64_t base = (int64_t)blockIdx.x * kSortTile;
    for (int r = 0; r < kSortRounds; ++r) {
        for (int w = 0; w < kWarps; ++w) wcnt[w][tid] = 0;  // kSortThreads == kRadix
        __syncthreads();
        int64_t i = base + r * kSortThreads + tid;
        bool valid = i < e;
        int32_t key = valid ? keys_in[i] : 0;
        int32_t val = valid ? (vals_in ? vals_in[i] : (int32_t)i) : 0;
        int digit = (key >> shift) & (kRadix - 1);
        uint32_t peers = __match_any_sync(0xffffffffu, valid ? digit : (kRadix + lane));
        int rank = __popc(peers & lt_mask);
        if (valid && rank == 0) wcnt[warp][digit] = __popc(peers);
        __syncthreads();
        {   // per digit: exclusive prefix over warps (warp order == input order)
            int64_t run = 0;
            int32_t cnts[kWarps];
#pragma unroll
            for (int w = 0; w < kWarps; ++w) cnts[w] = wcnt[w][tid];
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                wcnt[w][tid] = (int32_t)run;
                run += cnts[w];
            }
            __syncthreads();
            if (valid) {
                int64_t pos = gofs[digit] + wcnt[warp][digit] + rank;
                keys_out[pos] = key;
                vals_out[pos] = val;
            }
            __syncthreads();
            gofs[tid] += run;
        }
        __syncthreads();
    }
}

__global__ void k_iota(int32_t *p, int64_t e) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = (int32_t)i;
}

// ell[v][i] = the i-th source of row v (CSR order), -1 past the row's end
__global__ void k_build_ell(int64_t cells, int32_t w, const int64_t *__restrict__ row_ptr,
                            const int32_t *__restrict__ col_src, int32_t *__restrict__ ell) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= cells) return;
    const int64_t v = c / w, i = c % w;
    const int64_t q = row_ptr[v] + i;
    ell[c] = q < row_ptr[v + 1] ? col_src[q] : -1;
}

__global__ void k_gather_csr(int64_t e, const int32_t *__restrict__ edge_id, const int32_t *__restrict__ src,
                             const int32_t *__restrict__ etype, int32_t *col_src, int32_t *etype_csr) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < e; p += (int64_t)gridDim.x * blockDim.x) {
        int32_t id = edge_id[p];
        col_src[p] = src[id];
        if (etype) etype_csr[p] = etype[id];
    }
}

// S1: dinv = deg^-1/2 (GCN, reading A1), inv_deg = 1/deg (SAGE mean); 0 for deg 0 (A12).
__global__ void k_norms(int32_t n, const int32_t *__restrict__ in_deg, float *dinv, float *inv_deg) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        int32_t d = in_deg[v];
        float fd = (float)d;
        dinv[v] = d > 0 ? 1.0f / sqrtf(fd) : 0.0f;
        inv_deg[v] = d > 0 ? 1.0f / fd : 0.0f;
    }
}

// S6: merge-path coordinates.  Items: row v's edges are items
// row_ptr[v] + v .. row_ptr[v+1] + v - 1, its end marker is item
// row_ptr[v+1] + v.  Task k starts at diagonal d = min(kT, E+N) at row
// v = #rows whose end item is < d, edge position p = d - v.
__global__ void k_merge_path(int32_t n, int64_t e, const int64_t *__restrict__ row_ptr, int64_t T, int64_t ntasks,
                             int32_t *task_v, int64_t *task_p) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k > ntasks) return;
    int64_t d = min(k * T, e + (int64_t)n);
    int32_t lo = 0, hi = n;  // smallest v in [0, n] with v == n or row_ptr[v+1] + v >= d
    while (lo < hi) {
        int32_t mid = lo + ((hi - lo) >> 1);
        if (row_ptr[mid + 1] + mid >= d)
            hi = mid;
        else
            lo = mid + 1;
    }
    task_v[k] = lo;
    task_p[k] = d - lo;
}

unsigned grid_for(int64_t work, int threads) {
    int64_t b = (work + threads - 1) / threads;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)kNumSMs * 32));
}

}  // namespace

#define SAGA_TRY(x)                                   \
    do {                                              \
        cudaError_t _e = (x);                         \
        if (_e != cudaSuccess) {                      \
            *why = cudaGetErrorString(_e);            \
            return _e == cudaErrorMemoryAllocation ? SAGA_ENOMEM : SAGA_ECUDA; \
        }                                             \
    } while (0)

// Stable LSD radix sort of `count` non-negative int32 keys (< 2^key_bits):
// writes to `order` the item indices in key order, ties in index order.
static cudaError_t radix_sort_index(const int32_t *keys, int64_t count, int key_bits, int32_t *order,
                                    cudaStream_t st) {
    const int passes = (key_bits + kRadixBits - 1) / kRadixBits;
    if (passes == 0) {
        k_iota<<<grid_for(count, 256), 256, 0, st>>>(order, count);
        return cudaGetLastError();
    }
    const int64_t nblocks = (count + kSortTile - 1) / kSortTile;
    int32_t *kbuf[2] = {nullptr, nullptr}, *vbuf[2] = {nullptr, nullptr}, *hist = nullptr;
    int64_t *offs = nullptr;
    cudaError_t err = cudaMallocAsync(&kbuf[0], sizeof(int32_t) * count, st);
    if (!err) err = cudaMallocAsync(&kbuf[1], sizeof(int32_t) * count, st);
    if (!err) err = cudaMallocAsync(&vbuf[0], sizeof(int32_t) * count, st);
    if (!err) err = cudaMallocAsync(&vbuf[1], sizeof(int32_t) * count, st);
    if (!err) err = cudaMallocAsync(&hist, sizeof(int32_t) * kRadix * nblocks, st);
    if (!err) err = cudaMallocAsync(&offs, sizeof(int64_t) * (kRadix * nblocks + 1), st);
    const int32_t *kin = keys;
    const int32_t *vin = nullptr;  // pass 0 payload = item index
    for (int pass = 0; pass < passes && !err; ++pass) {
        const int shift = pass * kRadixBits;
        int32_t *kout = kbuf[pass & 1], *vout = (pass == passes - 1) ? order : vbuf[pass & 1];
        k_radix_hist<<<(unsigned)nblocks, kSortThreads, 0, st>>>(kin, count, shift, hist, nblocks);
        if ((err = cudaGetLastError())) break;
        if ((err = scan_exclusive<int32_t>(hist, kRadix * nblocks, offs, st))) break;
        k_radix_scatter<<<(unsigned)nblocks, kSortThreads, 0, st>>>(kin, vin, count, shift, offs, nblocks, kout, vout);
        err = cudaGetLastError();
        kin = kout;
        vin = vout;
    }
    // every buffer allocated so far, also when a later allocation failed
    for (void *p : {(void *)kbuf[0], (void *)kbuf[1], (void *)vbuf[0], (void *)vbuf[1], (void *)hist, (void *)offs})
        if (p) cudaFreeAsync(p, st);
    return err;
}

__global__ void k_typed_keys(int64_t e, const int32_t *__restrict__ dst, const int32_t *__restrict__ etype, int32_t T,
                             int32_t *keys, int32_t *tdeg) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t k = dst[i] * T + etype[i];
        keys[i] = k;
        atomicAdd(tdeg + k, 1);  // integer atomics: order-independent result
    }
}

__global__ void k_gather_src(int64_t e, const int32_t *__restrict__ order, const int32_t *__restrict__ src,
                             int32_t *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = src[order[i]];
}

__global__ void k_inv(int64_t m, const int32_t *__restrict__ deg, float *inv) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        inv[i] = deg[i] > 0 ? 1.0f / (float)deg[i] : 0.0f;
}

// Merge-path task starts over (rows' edges + row-end markers) of a CSR.
static cudaError_t merge_path_schedule(int32_t n, int64_t e, const int64_t *row_ptr, int64_t *T_out,
                                       int64_t *ntasks_out, int32_t **task_v, int64_t **task_p, cudaStream_t st,
                                       int tasks_per_sm = 32) {
    static const int sms = [] {
        int dev = 0, c = kNumSMs;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
        return c;
    }();
    const int64_t items = e + (int64_t)n;
    const int64_t target = (int64_t)sms * tasks_per_sm;
    const int64_t T = std::max<int64_t>(8, (items + target - 1) / target);
    const int64_t ntasks = items > 0 ? (items + T - 1) / T : 0;
    *T_out = T;
    *ntasks_out = ntasks;
    cudaError_t err;
    if ((err = cudaMallocAsync(task_v, sizeof(int32_t) * (ntasks + 1), st))) return err;
    if ((err = cudaMallocAsync(task_p, sizeof(int64_t) * (ntasks + 1), st))) return err;
    if (n > 0)
        k_merge_path<<<(unsigned)((ntasks + 1 + 255) / 256), 256, 0, st>>>(n, e, row_ptr, T, ntasks, *task_v, *task_p);
    return cudaGetLastError();
}

// heavy_slot[deg_order[s]] = s for the n_heavy vertices of largest in-degree
// (deg_order's head: in-degree >= kHeavyInDeg); -1 elsewhere (memset)
__global__ void k_heavy_slots(int32_t nh, const int32_t *__restrict__ deg_order, int32_t *heavy_slot) {
    const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s < nh) heavy_slot[deg_order[s]] = s;
}

// Step 8 (aggregation view): per vertex, whether its in-edges are nothing but
// one self-loop (or none): then the GCN output needs no gather.
__global__ void k_epi_flags(int32_t n, const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col_src,
                            const int32_t *__restrict__ in_deg, int32_t *aflag) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int32_t d = in_deg[v];
        aflag[v] = (d == 0 || (d == 1 && col_src[row_ptr[v]] == (int32_t)v)) ? 0 : 1;
    }
}
__global__ void k_compact_rows(int32_t n, const int32_t *__restrict__ aflag, const int64_t *__restrict__ apos,
                               const int32_t *__restrict__ in_deg, const float *__restrict__ dinv, int32_t *arow,
                               int32_t *adeg, float *adinv) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        if (!aflag[v]) continue;
        const int64_t i = apos[v];
        arow[i] = (int32_t)v;
        adeg[i] = in_deg[v];
        adinv[i] = dinv[v];
    }
}
// warp per compact row: its in-edges, in CSR order
// the complement of the aggregation rows: erow[v - apos[v]] = v where aflag[v] == 0
__global__ void k_compact_epi_rows(int32_t n, const int32_t *__restrict__ aflag, const int64_t *__restrict__ apos,
                                   int32_t *erow) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        if (!aflag[v]) erow[v - apos[v]] = (int32_t)v;
}

__global__ void k_compact_edges(int32_t an, const int32_t *__restrict__ arow, const int64_t *__restrict__ row_ptr,
                                const int32_t *__restrict__ col_src, const int64_t *__restrict__ arow_ptr,
                                int32_t *acol_src) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < an;
         i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t b = row_ptr[arow[i]], d = arow_ptr[i + 1] - arow_ptr[i], o = arow_ptr[i];
        for (int64_t k = lane; k < d; k += 32) acol_src[o + k] = col_src[b + k];
    }
}

// keys max_deg - in_deg: ascending keys = descending degree, in bit_length(max_deg) bits
__global__ void k_degree_desc_keys(int32_t n, const int32_t *__restrict__ in_deg, int32_t max_deg, int32_t *keys) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        keys[i] = max_deg - in_deg[i];
}

saga_status build_graph(int32_t n, int64_t e, const int32_t *src, const int32_t *dst, const int32_t *etype,
                        int32_t num_etypes, cudaStream_t st, GraphDev *g, int64_t *first_bad, const char **why) {
    g->n = n;
    g->e = e;
    g->num_etypes = etype ? num_etypes : 1;
    g->stream = st;
    *first_bad = -1;

    const size_t nn = (size_t)std::max(n, 1), ne = (size_t)std::max<int64_t>(e, 1);
    SAGA_TRY(cudaMallocAsync(&g->row_ptr, sizeof(int64_t) * (nn + 1), st));
    SAGA_TRY(cudaMallocAsync(&g->col_src, sizeof(int32_t) * ne, st));
    SAGA_TRY(cudaMallocAsync(&g->edge_id, sizeof(int32_t) * ne, st));
    if (etype) SAGA_TRY(cudaMallocAsync(&g->etype, sizeof(int32_t) * ne, st));
    SAGA_TRY(cudaMallocAsync(&g->in_deg, sizeof(int32_t) * nn, st));
    SAGA_TRY(cudaMallocAsync(&g->out_deg, sizeof(int32_t) * nn, st));
    SAGA_TRY(cudaMallocAsync(&g->dinv, sizeof(float) * nn, st));
    SAGA_TRY(cudaMallocAsync(&g->inv_deg, sizeof(float) * nn, st));
    SAGA_TRY(cudaMemsetAsync(g->in_deg, 0, sizeof(int32_t) * nn, st));
    SAGA_TRY(cudaMemsetAsync(g->out_deg, 0, sizeof(int32_t) * nn, st));

    // 1+2. range check and degrees in one pass, max in-degree; read back
    // together (the library's only host sync)
    {
        unsigned long long *rb_d;  // [first bad edge, max in-degree, heavy rows]
        SAGA_TRY(cudaMallocAsync(&rb_d, 3 * sizeof(unsigned long long), st));
        SAGA_TRY(cudaMemsetAsync(rb_d, 0xFF, sizeof(unsigned long long), st));
        SAGA_TRY(cudaMemsetAsync(rb_d + 1, 0, 2 * sizeof(unsigned long long), st));
        if (e > 0)
            k_range_degrees<<<grid_for(e, 256), 256, 0, st>>>(n, e, src, dst, etype, num_etypes, rb_d, g->in_deg,
                                                              g->out_deg);
        if (n > 0) k_max_deg<<<grid_for(n, 256), 256, 0, st>>>(n, g->in_deg, rb_d + 1);
        SAGA_TRY(cudaGetLastError());
        unsigned long long rb_h[3] = {0, 0, 0};
        SAGA_TRY(cudaMemcpyAsync(rb_h, rb_d, sizeof rb_h, cudaMemcpyDeviceToHost, st));
        SAGA_TRY(cudaStreamSynchronize(st));
        cudaFreeAsync(rb_d, st);
        if (rb_h[0] != ~0ull) {
            *first_bad = (int64_t)rb_h[0];
            *why = "COO entry out of range";
            return SAGA_ERANGE;
        }
        g->max_in_deg = (int32_t)rb_h[1];
        g->n_heavy = (int32_t)rb_h[2];
    }

    // 3. row_ptr
    SAGA_TRY(scan_exclusive<int32_t>(g->in_deg, n, g->row_ptr, st));

    // 4. stable LSD radix sort of (dst, COO index)
    if (e > 0) {
        int bits = 0;
        while (bits < 31 && (int64_t(1) << bits) < (int64_t)n) ++bits;   // keys < n <= 2^bits
        SAGA_TRY(radix_sort_index(dst, e, bits, g->edge_id, st));
        k_gather_csr<<<grid_for(e, 256), 256, 0, st>>>(e, g->edge_id, src, etype, g->col_src, g->etype);
        SAGA_TRY(cudaGetLastError());
    }
    if (n > 0) k_norms<<<grid_for(n, 256), 256, 0, st>>>(n, g->in_deg, g->dinv, g->inv_deg);
    SAGA_TRY(cudaGetLastError());

    // 4b. ELL view of a graph with small in-degrees (the row-wise fp32 GCN),
    //     when its padding stays bounded (at most 4 E cells, or 1M)
    const int32_t ell_w = std::max(4, (g->max_in_deg + 3) / 4 * 4);
    if (n > 0 && g->max_in_deg <= kEllMaxDeg && (int64_t)n * ell_w <= std::max<int64_t>(4 * e, 1 << 20)) {
        g->ell_w = ell_w;
        const int64_t cells = (int64_t)n * g->ell_w;
        SAGA_TRY(cudaMallocAsync(&g->ell, sizeof(int32_t) * (size_t)cells, st));
        k_build_ell<<<grid_for(cells, 256), 256, 0, st>>>(cells, g->ell_w, g->row_ptr, g->col_src, g->ell);
        SAGA_TRY(cudaGetLastError());
    }

    // 5. vertices by in-degree, descending (ties by id): the LSTM gather's
    //    work queue (longest sequences first)
    SAGA_TRY(cudaMallocAsync(&g->deg_order, sizeof(int32_t) * nn, st));
    if (n > 0) {
        int32_t *keys;
        SAGA_TRY(cudaMallocAsync(&keys, sizeof(int32_t) * nn, st));
        k_degree_desc_keys<<<grid_for(n, 256), 256, 0, st>>>(n, g->in_deg, g->max_in_deg, keys);
        SAGA_TRY(cudaGetLastError());
        int kbits = 0;
        while (kbits < 31 && (int64_t(1) << kbits) <= (int64_t)g->max_in_deg) ++kbits;  // keys <= max_deg < 2^kbits
        SAGA_TRY(radix_sort_index(keys, n, kbits, g->deg_order, st));
        cudaFreeAsync(keys, st);
    }
    // heavy rows (in-degree >= kHeavyInDeg): the fp64 ApplyVertex of the gated / GGNN layers
    SAGA_TRY(cudaMallocAsync(&g->heavy_slot, sizeof(int32_t) * nn, st));
    SAGA_TRY(cudaMemsetAsync(g->heavy_slot, 0xFF, sizeof(int32_t) * nn, st));
    if (g->n_heavy > 0) {
        k_heavy_slots<<<(g->n_heavy + 255) / 256, 256, 0, st>>>(g->n_heavy, g->deg_order, g->heavy_slot);
        SAGA_TRY(cudaGetLastError());
    }

    // 6. merge-path schedules: exactly one task per resident warp (the
    // gathers run 4 blocks x 8 warps per SM: 32 tasks per SM, one full wave)
    // for the sum/mean/typed gathers -- 1.5-11% faster than 2 per warp at C2,
    // C4, C5, C6, C8 (fewer split-row tickets and task prologues); 24 or 40
    // per SM (a partial wave) are 5-40% slower at C5 -- and 4 per warp for
    // GAT, whose per-item cost varies (7% faster than 1 per warp at C3)
    SAGA_TRY(merge_path_schedule(n, e, g->row_ptr, &g->task_items, &g->ntasks, &g->task_v, &g->task_p, st, 32));
    SAGA_TRY(merge_path_schedule(n, e, g->row_ptr, &g->ftask_items, &g->fntasks, &g->ftask_v, &g->ftask_p, st, 128));

    // 8. aggregation view (see GraphDev): rows with only a self-loop or no
    //    in-edge are finished outside the gather (GAT: the GEMM epilogue;
    //    GCN: a streaming pass over their list erow); a compacted CSR of the
    //    others (a second host sync, for its sizes)
    if (n > 0) {
        int32_t *aflag, *adeg = nullptr;
        int64_t *apos;
        SAGA_TRY(cudaMallocAsync(&aflag, sizeof(int32_t) * nn, st));
        SAGA_TRY(cudaMallocAsync(&apos, sizeof(int64_t) * (nn + 1), st));
        k_epi_flags<<<grid_for(n, 256), 256, 0, st>>>(n, g->row_ptr, g->col_src, g->in_deg, aflag);
        SAGA_TRY(cudaGetLastError());
        SAGA_TRY(scan_exclusive<int32_t>(aflag, n, apos, st));
        int64_t an = 0;
        SAGA_TRY(cudaMemcpyAsync(&an, apos + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        SAGA_TRY(cudaStreamSynchronize(st));
        if (an < n) {
            g->an = (int32_t)an;
            const size_t na = (size_t)std::max<int64_t>(an, 1);
            SAGA_TRY(cudaMallocAsync(&g->arow, sizeof(int32_t) * na, st));
            SAGA_TRY(cudaMallocAsync(&g->adinv, sizeof(float) * na, st));
            SAGA_TRY(cudaMallocAsync(&g->arow_ptr, sizeof(int64_t) * (na + 1), st));
            SAGA_TRY(cudaMallocAsync(&adeg, sizeof(int32_t) * na, st));
            k_compact_rows<<<grid_for(n, 256), 256, 0, st>>>(n, aflag, apos, g->in_deg, g->dinv, g->arow, adeg,
                                                             g->adinv);
            SAGA_TRY(cudaGetLastError());
            SAGA_TRY(scan_exclusive<int32_t>(adeg, an, g->arow_ptr, st));
            // every skipped row with an in-edge has exactly one (its self-loop)
            int64_t skipped_edges = 0;
            {
                int64_t tot = 0;
                SAGA_TRY(cudaMemcpyAsync(&tot, g->arow_ptr + an, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
                SAGA_TRY(cudaStreamSynchronize(st));
                g->ae = tot;
                skipped_edges = e - tot;
                (void)skipped_edges;
            }
            SAGA_TRY(cudaMallocAsync(&g->acol_src, sizeof(int32_t) * (size_t)std::max<int64_t>(g->ae, 1), st));
            if (an > 0)
                k_compact_edges<<<grid_for(an * 32, 256), 256, 0, st>>>(g->an, g->arow, g->row_ptr, g->col_src,
                                                                        g->arow_ptr, g->acol_src);
            SAGA_TRY(cudaGetLastError());
            SAGA_TRY(merge_path_schedule(g->an, g->ae, g->arow_ptr, &g->aftask_items, &g->afntasks, &g->aftask_v,
                                         &g->aftask_p, st, 128));
            SAGA_TRY(merge_path_schedule(g->an, g->ae, g->arow_ptr, &g->atask_items, &g->antasks, &g->atask_v,
                                         &g->atask_p, st, 32));
            g->ne = (int32_t)(n - an);
            SAGA_TRY(cudaMallocAsync(&g->erow, sizeof(int32_t) * (size_t)std::max<int32_t>(g->ne, 1), st));
            k_compact_epi_rows<<<grid_for(n, 256), 256, 0, st>>>(n, aflag, apos, g->erow);
            SAGA_TRY(cudaGetLastError());
            cudaFreeAsync(adeg, st);
        }
        cudaFreeAsync(aflag, st);
        cudaFreeAsync(apos, st);
    }

    // 7. typed view: rows (v, t), edges in (dst, type, COO index) order
    if (etype && n > 0) {
        const int32_t T = g->num_etypes;
        const int64_t nt = (int64_t)n * T;
        if (nt >= (int64_t(1) << 31)) {
            *why = "n * num_etypes must be < 2^31";
            return SAGA_EINVAL;
        }
        int32_t *keys, *tdeg, *order;
        SAGA_TRY(cudaMallocAsync(&g->trow_ptr, sizeof(int64_t) * (nt + 1), st));
        SAGA_TRY(cudaMallocAsync(&g->tcol_src, sizeof(int32_t) * ne, st));
        SAGA_TRY(cudaMallocAsync(&g->tinv_deg, sizeof(float) * nt, st));
        SAGA_TRY(cudaMallocAsync(&tdeg, sizeof(int32_t) * nt, st));
        SAGA_TRY(cudaMemsetAsync(tdeg, 0, sizeof(int32_t) * nt, st));
        if (e > 0) {
            SAGA_TRY(cudaMallocAsync(&keys, sizeof(int32_t) * e, st));
            SAGA_TRY(cudaMallocAsync(&order, sizeof(int32_t) * e, st));
            k_typed_keys<<<grid_for(e, 256), 256, 0, st>>>(e, dst, etype, T, keys, tdeg);
            SAGA_TRY(cudaGetLastError());
            int bits = 0;
            while (bits < 31 && (int64_t(1) << bits) < nt) ++bits;
            SAGA_TRY(radix_sort_index(keys, e, bits, order, st));
            k_gather_src<<<grid_for(e, 256), 256, 0, st>>>(e, order, src, g->tcol_src);
            SAGA_TRY(cudaGetLastError());
            cudaFreeAsync(keys, st);
            cudaFreeAsync(order, st);
        }
        SAGA_TRY(scan_exclusive<int32_t>(tdeg, nt, g->trow_ptr, st));
        k_inv<<<grid_for(nt, 256), 256, 0, st>>>(nt, tdeg, g->tinv_deg);
        SAGA_TRY(cudaGetLastError());
        cudaFreeAsync(tdeg, st);
        SAGA_TRY(merge_path_schedule((int32_t)nt, e, g->trow_ptr, &g->ttask_items, &g->tntasks, &g->ttask_v,
                                     &g->ttask_p, st));
    }
    return SAGA_OK;
}

void free_graph(GraphDev *g) {
    cudaStream_t st = g->stream;
    void *ptrs[] = {g->row_ptr,  g->col_src,  g->edge_id,  g->etype,   g->in_deg,  g->out_deg, g->dinv,
                    g->inv_deg,  g->task_v,   g->task_p,   g->deg_order, g->heavy_slot, g->arow, g->arow_ptr,
                    g->acol_src, g->adinv, g->aftask_v, g->aftask_p, g->trow_ptr, g->tcol_src, g->tinv_deg,
                    g->ttask_v, g->ttask_p, g->ftask_v, g->ftask_p, g->atask_v, g->atask_p, g->erow, g->ell};
    for (void *p : ptrs)
        if (p) cudaFreeAsync(p, st);
}

}  // namespace saga
