// epilogue.cuh -- row-per-lane accumulator tiles <-> coalesced global rows,
// shared by the tcgen05 GEMM epilogues (gemm_tf32split.cu, gemm_i8x.cu).
#pragma once
#include <cstdint>

namespace saga {
namespace epi {

// Row-per-lane tiles <-> coalesced row segments.  A warp holds rows row0 + lane
// (lane 0..31) of a [M][ld] fp32 matrix, G float4 (columns col0 .. col0+4G-1)
// per lane in x[4G].  transpose_groups<G> transposes each G-lane group's G x G
// block of float4 with log2(G) butterfly stages (shfl_xor 1, 2, 4): afterwards
// lane j of group g holds float4 j of rows G g .. G g + G-1 (slot k = row G g + k);
// it is its own inverse.  The store / load below then move whole 16G-byte row
// segments per instruction (32/G rows each) instead of 32 scattered 16-byte
// pieces.  Rows >= M are skipped (loads give 0).
template <int G>
__device__ __forceinline__ void transpose_groups(float (&x)[4 * G], int lane) {
    const int j = lane & (G - 1);
#pragma unroll
    for (int s = 1; s < G; s <<= 1) {
        const bool hi = (j & s) != 0;
#pragma unroll
        for (int k = 0; k < G; ++k) {
            if (k & s) continue;
            // the slot of the pair (k, k|s) whose bit s differs from the lane's
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float send = hi ? x[4 * k + e] : x[4 * (k | s) + e];
                const float recv = __shfl_xor_sync(0xffffffffu, send, s);
                if (hi)
                    x[4 * k + e] = recv;
                else
                    x[4 * (k | s) + e] = recv;
            }
        }
    }
}

template <int G>
__device__ __forceinline__ void store_rows_coalesced(float (&x)[4 * G], float *out, int ld, int64_t row0, int col0,
                                                     int64_t M, int lane) {
    transpose_groups<G>(x, lane);
    const int j = lane & (G - 1), g = lane / G;
#pragma unroll
    for (int k = 0; k < G; ++k) {
        const int64_t row = row0 + G * g + k;
        if (row < M)
            reinterpret_cast<float4 *>(out + row * ld + col0)[j] =
                make_float4(x[4 * k], x[4 * k + 1], x[4 * k + 2], x[4 * k + 3]);
    }
}

template <int G>
__device__ __forceinline__ void load_rows_coalesced(float (&x)[4 * G], const float *in, int ld, int64_t row0,
                                                    int col0, int64_t M, int lane) {
    const int j = lane & (G - 1), g = lane / G;
#pragma unroll
    for (int k = 0; k < G; ++k) {
        const int64_t row = row0 + G * g + k;
        const float4 v = row < M ? __ldg(reinterpret_cast<const float4 *>(in + row * ld + col0) + j)
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
        x[4 * k] = v.x; x[4 * k + 1] = v.y; x[4 * k + 2] = v.z; x[4 * k + 3] = v.w;
    }
    transpose_groups<G>(x, lane);
}

}  // namespace epi
}  // namespace saga
