// step_bits.cu -- device half of the bit-stream transfer of hga_step_host_bits
// (host half: host_bits.cpp).  The host moves the caller's int8 (4N, m, m)
// population as a flat bit stream, bit e = 1 iff byte e is -1 (word e / 32,
// bit e % 32); these kernels convert it to / from the resident packed column
// records (hga_common.cuh) for orders m = 4..64, m % 4 == 0.
#include "hga_common.cuh"

namespace hga {

// Both directions are a bit transpose per matrix done with warp ballots.  A
// CTA of 8 warps takes a group of 8 (m > 16) or 16 (m <= 16: two matrices
// per warp, lanes 0-15 / 16-31) consecutive matrices; the group's part of
// the stream is word aligned (m^2 is a multiple of 16 and a group holds an
// even number of matrices) and is staged in shared memory.  Lane l holds
// row l (and l + 32) of its matrix as a row mask; ballot over the rows of
// "bit j of my row" is column j's word, and ballot over the columns of
// "bit r of my column" is row r's mask.
template <int M>
struct BitsGeom {
    static constexpr int W = (M + 31) / 32;
    static constexpr int MPW = M <= 16 ? 2 : 1;  // matrices per warp
    static constexpr int WARPS = 8;
    static constexpr int MPC = WARPS * MPW;      // matrices per CTA group (even)
    static constexpr int SEG = MPC * M * M / 32;  // stream words per group
    static constexpr int LPM = 32 / MPW;          // lanes per matrix
};

// Row `row` of the matrix whose bits start at bit `e0` of the staged segment s.
template <int M>
__device__ __forceinline__ uint64_t seg_row(const uint32_t* s, int e0, int row) {
    const int e = e0 + row * M;
    const int w = e >> 5, sh = e & 31;
    uint64_t v = ((uint64_t)s[w + 1] << 32 | s[w]) >> sh;
    if (M + 31 > 64 && sh + M > 64) v |= (uint64_t)s[w + 2] << (64 - sh);
    return M == 64 ? v : (v & ((1ull << M) - 1));
}

template <int M>
__global__ void __launch_bounds__(256) k_bits_to_cols(const uint32_t* __restrict__ bits, int64_t n, int64_t nwords,
                                                      uint32_t* __restrict__ cols, int32_t* flag) {
    using G = BitsGeom<M>;
    __shared__ uint32_t s[G::SEG + 3];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int sub = lane / G::LPM, r = lane % G::LPM;  // matrix of this warp, row / column of this lane
    const int mat = wid * G::MPW + sub;
    uint32_t not_ga = 0;
    for (int64_t grp = blockIdx.x; grp * G::MPC < n; grp += gridDim.x) {
        const int64_t k0 = grp * G::MPC, base = k0 * M * M / 32;
        for (int i = threadIdx.x; i < G::SEG + 3; i += blockDim.x)
            s[i] = (i < G::SEG && base + i < nwords) ? __ldg(bits + base + i) : 0u;
        __syncthreads();
        const bool live = k0 + mat < n;
        const int e0 = mat * M * M;
        const uint64_t rlo = (live && r < M) ? seg_row<M>(s, e0, r) : 0ull;
        const uint64_t rhi = (G::W > 1 && live && r + 32 < M) ? seg_row<M>(s, e0, r + 32) : 0ull;
        uint32_t c0 = 0, c1 = 0, c2 = 0, c3 = 0;  // columns (lane) and (lane + 32): words 0 / 1
#pragma unroll
        for (int j = 0; j < M; ++j) {
            const uint32_t b0 = __ballot_sync(0xffffffffu, (rlo >> j) & 1u);
            const uint32_t v0 = G::MPW == 2 ? (b0 >> (16 * sub)) & 0xFFFFu : b0;
            if (G::W == 1) {
                if ((j % G::LPM) == r) c0 = v0;
            } else {
                const uint32_t b1 = __ballot_sync(0xffffffffu, (rhi >> j) & 1u);
                if (j < 32 && j == r) c0 = v0, c1 = b1;
                if (j >= 32 && j - 32 == r) c2 = v0, c3 = b1;
            }
        }
        if (live && r < M) {
            uint32_t* q = cols + ((k0 + mat) * M + r) * G::W;
            if (G::W == 1) {
                q[0] = c0;
                not_ga |= (uint32_t)(__popc(c0) != (r == 0 ? 0 : M / 2));
            } else {
                q[0] = c0;
                q[1] = c1;
                not_ga |= (uint32_t)(__popc(c0) + __popc(c1) != (r == 0 ? 0 : M / 2));
                if (r + 32 < M) {
                    q[32 * G::W] = c2;
                    q[32 * G::W + 1] = c3;
                    not_ga |= (uint32_t)(__popc(c2) + __popc(c3) != M / 2);
                }
            }
        }
        __syncthreads();
    }
    if (not_ga && flag) atomicOr(flag, (int32_t)HGA_FLAG_NOT_GA);
}

// Nothing is written when `skip` holds a rejection flag (the host then
// leaves its arrays alone).
template <int M>
__global__ void __launch_bounds__(256) k_cols_to_bits(const uint32_t* __restrict__ cols, int64_t n, int64_t nwords,
                                                      uint32_t* __restrict__ bits, const int32_t* __restrict__ skip) {
    using G = BitsGeom<M>;
    if (skip && (*skip & (HGA_FLAG_NOT_SIGN | HGA_FLAG_NOT_GA))) return;
    __shared__ uint32_t s[G::SEG + 3];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int sub = lane / G::LPM, c = lane % G::LPM;
    const int mat = wid * G::MPW + sub;
    for (int64_t grp = blockIdx.x; grp * G::MPC < n; grp += gridDim.x) {
        const int64_t k0 = grp * G::MPC, base = k0 * M * M / 32;
        for (int i = threadIdx.x; i < G::SEG + 3; i += blockDim.x) s[i] = 0u;
        __syncthreads();
        const bool live = k0 + mat < n;
        uint32_t w0 = 0, w1 = 0, w2 = 0, w3 = 0;  // column c (words 0 / 1) and column c + 32
        if (live && c < M) {
            const uint32_t* q = cols + ((k0 + mat) * M + c) * G::W;
            w0 = __ldg(q);
            if (G::W > 1) {
                w1 = __ldg(q + 1);
                if (c + 32 < M) w2 = __ldg(q + 32 * G::W), w3 = __ldg(q + 32 * G::W + 1);
            }
        }
        uint64_t rlo = 0, rhi = 0;  // rows (lane) and (lane + 32)
#pragma unroll
        for (int r = 0; r < M; ++r) {
            const uint32_t src = r < 32 ? w0 : w1, src2 = r < 32 ? w2 : w3;
            const uint32_t b0 = __ballot_sync(0xffffffffu, (src >> (r & 31)) & 1u);
            if (G::W == 1) {
                const uint32_t v = G::MPW == 2 ? (b0 >> (16 * sub)) & 0xFFFFu : b0;
                if ((r % G::LPM) == c) rlo = v;
            } else {
                const uint32_t b1 = __ballot_sync(0xffffffffu, (src2 >> (r & 31)) & 1u);
                const uint64_t v = (uint64_t)b1 << 32 | b0;
                if (r < 32 && r == c) rlo = v;
                if (r >= 32 && r - 32 == c) rhi = v;
            }
        }
        // rows into the staged segment (shared atomics: neighbouring rows share words)
        auto put = [&](int row, uint64_t v) {
            const int e = mat * M * M + row * M, w = e >> 5, sh = e & 31;
            const uint64_t lo = v << sh;
            atomicOr(&s[w], (uint32_t)lo);
            if (sh + M > 32) atomicOr(&s[w + 1], (uint32_t)(lo >> 32));
            if (sh + M > 64) atomicOr(&s[w + 2], (uint32_t)(v >> (64 - sh)));
        };
        if (live && c < M) put(c, rlo);
        if (G::W > 1 && live && c + 32 < M) put(c + 32, rhi);
        __syncthreads();
        for (int i = threadIdx.x; i < G::SEG; i += blockDim.x)
            if (base + i < nwords) bits[base + i] = s[i];
        __syncthreads();
    }
}

#define HGA_BITS_ORDERS(X) X(4) X(8) X(12) X(16) X(20) X(24) X(28) X(32) X(36) X(40) X(44) X(48) X(52) X(56) X(60) X(64)

static int grid_groups(int64_t n, int mpc) {
    const int64_t g = (n + mpc - 1) / mpc;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)sm_count_cached() * 8));
}

int bits_to_cols(const uint32_t* bits, int64_t n, int32_t m, uint32_t* cols, int32_t* flag, cudaStream_t st) {
    if (n <= 0) return HGA_OK;
    const int64_t nwords = (n * m * m + 31) / 32;
    switch (m) {
#define X(M)                                                                                                   \
    case M:                                                                                                    \
        k_bits_to_cols<M><<<grid_groups(n, BitsGeom<M>::MPC), 256, 0, st>>>(bits, n, nwords, cols, flag);      \
        break;
        HGA_BITS_ORDERS(X)
#undef X
        default: return HGA_E_UNSUPPORTED;
    }
    return to_rc(cudaGetLastError());
}

int cols_to_bits(const uint32_t* cols, int64_t n, int32_t m, uint32_t* bits, const int32_t* skip, cudaStream_t st) {
    if (n <= 0) return HGA_OK;
    const int64_t nwords = (n * m * m + 31) / 32;
    switch (m) {
#define X(M)                                                                                                   \
    case M:                                                                                                    \
        k_cols_to_bits<M><<<grid_groups(n, BitsGeom<M>::MPC), 256, 0, st>>>(cols, n, nwords, bits, skip);      \
        break;
        HGA_BITS_ORDERS(X)
#undef X
        default: return HGA_E_UNSUPPORTED;
    }
    return to_rc(cudaGetLastError());
}

}  // namespace hga

extern "C" int hga_bits_to_cols(const uint32_t* bits, int64_t n, int32_t m, uint32_t* cols, int32_t* flag,
                                void* stream) {
    if (n < 0 || m < 4 || m > 64 || (m & 3)) return n < 0 ? HGA_E_INVALID : HGA_E_UNSUPPORTED;
    return hga::bits_to_cols(bits, n, m, cols, flag, (cudaStream_t)stream);
}

extern "C" int hga_cols_to_bits(const uint32_t* cols, int64_t n, int32_t m, uint32_t* bits, void* stream) {
    if (n < 0 || m < 4 || m > 64 || (m & 3)) return n < 0 ? HGA_E_INVALID : HGA_E_UNSUPPORTED;
    return hga::cols_to_bits(cols, n, m, bits, nullptr, (cudaStream_t)stream);
}
