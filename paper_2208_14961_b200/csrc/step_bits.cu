// step_bits.cu -- device half of the bit-stream transfer of hga_step_host_bits
// (host half: host_bits.cpp).  The host moves the caller's int8 (4N, m, m)
// population as a flat bit stream, bit e = 1 iff byte e is -1 (word e / 32,
// bit e % 32); these kernels convert it to / from the resident packed column
// records (hga_common.cuh) for orders m = 4..64, m % 4 == 0.
#include "hga_common.cuh"

namespace hga {

// Thread (matrix k, column j): column j's W words from the m row positions
// k m^2 + r m + j of the stream (neighbouring threads read neighbouring bits,
// the words come from L1).  Also the GA-invariant check of the pack kernels
// (k_pack_quads): column 0 all +1, every other column balanced.
template <int M>
__global__ void k_bits_to_cols(const uint32_t* __restrict__ bits, int64_t n, uint32_t* __restrict__ cols,
                               int32_t* flag) {
    constexpr int W = (M + 31) / 32;
    constexpr int64_t MM = (int64_t)M * M;
    uint32_t not_ga = 0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * M; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = t / M;
        const int j = (int)(t - k * M);
        const int64_t e0 = k * MM + j;
        uint32_t w[W];
#pragma unroll
        for (int x = 0; x < W; ++x) w[x] = 0;
#pragma unroll
        for (int r = 0; r < M; ++r) {
            const int64_t e = e0 + (int64_t)r * M;
            w[r >> 5] |= ((__ldg(bits + (e >> 5)) >> (e & 31)) & 1u) << (r & 31);
        }
        int neg = 0;
#pragma unroll
        for (int x = 0; x < W; ++x) {
            cols[t * W + x] = w[x];
            neg += __popc(w[x]);
        }
        not_ga |= (uint32_t)(neg != (j == 0 ? 0 : M / 2));
    }
    if (not_ga && flag) atomicOr(flag, (int32_t)HGA_FLAG_NOT_GA);
}

// Thread per stream word w in [w0, w1): its 32 entries walk (k, r, j) in
// row-major order; entries past the population are 0.  Nothing is written
// when `skip` holds a rejection flag (the host then leaves its arrays alone).
template <int M>
__global__ void k_cols_to_bits(const uint32_t* __restrict__ cols, int64_t n, int64_t w0, int64_t w1,
                               uint32_t* __restrict__ bits, const int32_t* __restrict__ skip) {
    if (skip && (*skip & (HGA_FLAG_NOT_SIGN | HGA_FLAG_NOT_GA))) return;
    constexpr int W = (M + 31) / 32;
    constexpr int64_t MM = (int64_t)M * M;
    for (int64_t w = w0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < w1; w += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = 32 * w;
        int64_t k = e / MM;
        const int rem = (int)(e - k * MM);
        int r = rem / M, j = rem - (rem / M) * M;
        uint32_t out = 0;
#pragma unroll 8
        for (int b = 0; b < 32; ++b) {
            if (k < n) out |= ((__ldg(cols + (k * M + j) * W + (r >> 5)) >> (r & 31)) & 1u) << b;
            if (++j == M) {
                j = 0;
                if (++r == M) {
                    r = 0;
                    ++k;
                }
            }
        }
        bits[w] = out;
    }
}

static int grid_words(int64_t work) {
    const int64_t g = (work + 255) / 256;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)sm_count_cached() * 16));
}

#define HGA_BITS_ORDERS(X) X(4) X(8) X(12) X(16) X(20) X(24) X(28) X(32) X(36) X(40) X(44) X(48) X(52) X(56) X(60) X(64)

int bits_to_cols(const uint32_t* bits, int64_t n, int32_t m, uint32_t* cols, int32_t* flag, cudaStream_t st) {
    if (n <= 0) return HGA_OK;
    switch (m) {
#define X(M)                                                                             \
    case M:                                                                              \
        k_bits_to_cols<M><<<grid_words(n * M), 256, 0, st>>>(bits, n, cols, flag);      \
        break;
        HGA_BITS_ORDERS(X)
#undef X
        default: return HGA_E_UNSUPPORTED;
    }
    return to_rc(cudaGetLastError());
}

int cols_to_bits(const uint32_t* cols, int64_t n, int32_t m, int64_t w0, int64_t w1, uint32_t* bits,
                 const int32_t* skip, cudaStream_t st) {
    if (w1 <= w0) return HGA_OK;
    switch (m) {
#define X(M)                                                                                      \
    case M:                                                                                       \
        k_cols_to_bits<M><<<grid_words(w1 - w0), 256, 0, st>>>(cols, n, w0, w1, bits, skip);      \
        break;
        HGA_BITS_ORDERS(X)
#undef X
        default: return HGA_E_UNSUPPORTED;
    }
    return to_rc(cudaGetLastError());
}

}  // namespace hga
