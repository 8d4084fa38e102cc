// run_common.cuh -- pieces shared by the persistent generation loops:
// Philox draws, the Feistel bijection of the select permutation, the Philox
// balanced-column init, and the grid barrier.
#pragma once

#include "hga_common.cuh"

namespace hga {

// ======================================================== Philox helpers
__device__ __forceinline__ U4 draw4(uint64_t seed, uint32_t a, uint32_t b, uint64_t gen, uint32_t purpose) {
    return philox(U4{a, b, (uint32_t)gen, (purpose << 24) ^ (uint32_t)(gen >> 32)}, (uint32_t)seed,
                  (uint32_t)(seed >> 32));
}
__device__ __forceinline__ uint32_t pick(const U4& v, int i) {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7FEB352Du;
    x ^= x >> 15;
    x *= 0x846CA68Bu;
    x ^= x >> 16;
    return x;
}

// Keyed bijection on [0, n) (4-round balanced Feistel + cycle walking).
__device__ __forceinline__ uint32_t feistel(uint32_t x, uint32_t n, int hb, const U4& k) {
    const uint32_t mask = (1u << hb) - 1u;
    do {
        uint32_t L = x >> hb, R = x & mask;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const uint32_t f = hash32(R ^ pick(k, r)) & mask;
            const uint32_t nl = R;
            R = L ^ f;
            L = nl;
        }
        x = (L << hb) | R;
    } while (x >= n);
    return x;
}

// Philox balanced column (Fisher-Yates over the m rows with Lemire draws).
template <int W>
__device__ __forceinline__ void philox_column(uint64_t seed, uint32_t purpose, uint64_t gen, int64_t slot,
                                              int m, int c, Col<W>& col) {
#pragma unroll
    for (int w = 0; w < W; ++w) col.w[w] = 0;
    if (c == 0) return;
    const int h = m / 2;
#pragma unroll
    for (int w = 0; w < W; ++w) {
        const int lo = 32 * w, hi = min(32 * w + 32, h);
        if (hi > lo) col.w[w] = (hi - lo == 32) ? 0xFFFFFFFFu : ((1u << (hi - lo)) - 1u);
    }
    U4 r{0, 0, 0, 0};
    for (int a = 0; a + 1 < m; ++a) {
        if ((a & 3) == 0)
            r = draw4(seed, (uint32_t)slot, (uint32_t)c | ((uint32_t)(a >> 2) << 12) | ((uint32_t)(slot >> 32) << 24), gen, purpose);
        const int b = a + (int)bounded(pick(r, a & 3), (uint32_t)(m - a));
        swap_rows<W>(col, a, b);
    }
}

// ======================================================== grid barrier
struct Barrier {
    unsigned int count;
    unsigned int gen;
};

__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned int atom_add_acq_rel_gpu(unsigned int* p, unsigned int v) {
    unsigned int old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void st_release_gpu(unsigned int* p, unsigned int v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// One-atomic grid barrier.  Every CTA adds to one counter: CTA 0 adds
// 2^31 - (nb - 1), the others 1, so a round adds exactly 2^31 and flips the
// top bit precisely when the last CTA arrives (the low 31 bits return to 0,
// so no reset store is needed).  bar.sync orders the CTA's writes before
// thread 0's acq_rel arrive; waiters poll the top bit with acquire loads.
// A CTA that races ahead into the next round cannot flip the bit back before
// every CTA has arrived there too.  `gen` is unused (layout kept).
__device__ __forceinline__ void grid_sync(Barrier* b) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int inc = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1u) : 1u;
        const unsigned int old = atom_add_acq_rel_gpu(&b->count, inc);
        while (((ld_acquire_gpu(&b->count) ^ old) & 0x80000000u) == 0u) {
        }
    }
    __syncthreads();
}

}  // namespace hga
