// hga_common.cuh -- shared device helpers for the sm_100a GA kernels.
//
// Population layout in HBM ("packed"): for each matrix k, m column records of
// W = ceil(m/32) uint32 words; bit (r % 32) of word (r / 32) of column j is 1
// iff entry (r, j) == -1.  Matrix k starts at word k * m * W.  Column 0 of a
// GA individual is therefore 0, and every other column has popcount m/2.
// The reference's own layout, int8 (n, m, m) row-major (engine.py:1-21), is
// accepted and produced at the API edge (pack / unpack / *_i8 kernels).
#pragma once

#include <algorithm>
#include <cooperative_groups.h>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/hga.h"

namespace hga {

// ----------------------------------------------------------------- constants
constexpr int kMaxRegWords = 4;  // register-resident column words (m <= 128)
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kSeedSalt = 0x5851F42D4C957F2DULL;
constexpr uint64_t kStreamSalt = 0x14057B7EF767814FULL;

// stream purposes, reference engine.py:71-77
constexpr uint64_t kPInit = 1, kPSelect = 2, kPCrossover = 3, kPMutCol = 4, kPMutRowA = 5,
                   kPMutRowB = 6, kPRestart = 7;

__host__ __device__ inline int words_for(int m) { return (m + 31) >> 5; }

// ------------------------------------------------ reference counter streams
// splitmix64 finalizer and key derivation, reference rand.py:39-77.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ uint64_t stream_key(uint64_t seed, uint64_t sid) {
    return mix64(mix64(seed ^ kSeedSalt) ^ mix64(sid * kGolden + kStreamSalt));
}
__host__ __device__ __forceinline__ uint64_t stream_key_from_seedmix(uint64_t seedmix, uint64_t sid) {
    return mix64(seedmix ^ mix64(sid * kGolden + kStreamSalt));
}
__host__ __device__ __forceinline__ uint64_t stream_word(uint64_t key, uint64_t counter) {
    return mix64(key + counter * kGolden);
}
// purpose | generation | matrix | column packed 4 | 28 | 20 | 12 (engine.py:60-90)
__host__ __device__ __forceinline__ uint64_t sid(uint64_t purpose, uint64_t gen, uint64_t mat,
                                                 uint64_t col) {
    return (purpose << 60) | (gen << 32) | (mat << 12) | col;
}
// word % span for span < 2^32, exact (what numpy's uint64 % does).
__device__ __forceinline__ uint32_t mod_u64_u32(uint64_t w, uint32_t span) {
    return (uint32_t)(w % (uint64_t)span);
}

// ---------------------------------------------------------- Philox4x32-10
struct U4 {
    uint32_t x, y, z, w;
};
__device__ __forceinline__ U4 philox(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}
// Lemire multiply-shift: uniform in [0, span) from 32 random bits.
__device__ __forceinline__ uint32_t bounded(uint32_t r, uint32_t span) {
    return (uint32_t)(((uint64_t)r * span) >> 32);
}

// -------------------------------------------------------------- bit columns
template <int W>
struct Col {
    uint32_t w[W];
};

template <int W>
__device__ __forceinline__ uint32_t get_bit(const Col<W>& c, int r) {
    uint32_t v = 0;
#pragma unroll
    for (int i = 0; i < W; ++i)
        if ((r >> 5) == i) v = (c.w[i] >> (r & 31)) & 1u;
    return v;
}
template <int W>
__device__ __forceinline__ void flip_bit(Col<W>& c, int r) {
#pragma unroll
    for (int i = 0; i < W; ++i)
        if ((r >> 5) == i) c.w[i] ^= 1u << (r & 31);
}
// Swap rows a and b of the column (== negate both when they differ, which is
// the reference's conditional pair flip, engine.py:361-373).
template <int W>
__device__ __forceinline__ void swap_rows(Col<W>& c, int a, int b) {
    if (get_bit(c, a) != get_bit(c, b)) {
        flip_bit(c, a);
        flip_bit(c, b);
    }
}

// ------------------------------------------------------ penalty accumulators
// Variants: bit 0 = F1 (sum |g|), bit 1 = F2 (count g != 0), bit 2 = ORTH
// (count g == 0, derived from the F2 count), bit 3 = SQ (sum g^2).
struct Acc {
    uint32_t s1, s2, s4;
};

template <int VM>
__device__ __forceinline__ void acc_pair(Acc& a, int p, int m, int half) {
    const int g = m - 2 * p;
    if (VM & HGA_VAR_F1) a.s1 += (uint32_t)abs(g);
    if (VM & (HGA_VAR_F2 | HGA_VAR_ORTH)) a.s2 += (p != half);
    if (VM & HGA_VAR_SQ) a.s4 += (uint32_t)(g * g);
}

// Finished per-matrix penalties from the i<j partial sums.
__device__ __forceinline__ void write_penalties(uint32_t vm, int m, int64_t idx, uint64_t s1,
                                                uint64_t s2, uint64_t s4, int64_t* f1,
                                                int64_t* f2, int64_t* orth, int64_t* sq) {
    if ((vm & HGA_VAR_F1) && f1) f1[idx] = 2 * (int64_t)s1;
    if ((vm & HGA_VAR_F2) && f2) f2[idx] = 2 * (int64_t)s2;
    if ((vm & HGA_VAR_ORTH) && orth) orth[idx] = (int64_t)m * (m - 1) / 2 - (int64_t)s2;
    if ((vm & HGA_VAR_SQ) && sq) sq[idx] = 2 * (int64_t)s4;
}

// Number of circulant pair steps for column i: (i, i+d mod m) for
// d = 1..(m-1)/2, plus d = m/2 when m is even and i < m/2.  Every unordered
// column pair is visited exactly once across the m columns.
__device__ __forceinline__ int pair_steps(int m, int i) {
    return (m - 1) / 2 + (((m & 1) == 0 && i < m / 2) ? 1 : 0);
}

int sm_count_cached();

// Launch setup that is a property of the device (function attributes,
// occupancy) is cached per device index: a process that drives several GPUs
// sets it up on each of them.  Concurrent first calls write identical values.
constexpr int kMaxDevices = 64;
inline int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return (d >= 0 && d < kMaxDevices) ? d : 0;
}

inline int to_rc(cudaError_t e) { return e == cudaSuccess ? HGA_OK : (int)HGA_E_CUDA_BASE + (int)e; }

}  // namespace hga
