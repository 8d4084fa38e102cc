// fitness_v2.cuh -- thread-per-matrix fused penalty kernels for GA orders
// (m = 4, 8, ..., 64).  Replaces engine._fitness_batch (engine.py:200-213).
//
// int8 input (the reference layout): a 128-thread CTA streams its 128
// matrices through shared memory four rows at a time with cp.async (double
// buffered, 16-byte pieces, coalesced per matrix), every thread turns its
// own matrix's staged bytes into column bit words (one shift + one LOP3 per
// entry, compile-time positions) and validates the bytes are +-1, then runs
// the unrolled XOR+POPC pair chain.  Packed input: the CTA stages its 128
// matrices' words the same way and each thread loads its own record.
#pragma once

#include <type_traits>

#include "tile.cuh"

namespace hga {

constexpr int kV2Threads = 128;

template <int M>
struct I8Geom {
    static constexpr int R = 4;                       // rows per chunk
    static constexpr int CH = R * M;                  // bytes per matrix per chunk
    static constexpr int ST = ((CH / 16) & 1) ? CH : CH + 16;  // odd # of 16B units: conflict-free LDS.128
    static constexpr int NCH = M / R;
    static constexpr int BUF = kV2Threads * ST;
    static constexpr int SMEM = 2 * BUF;
};

template <int M>
__device__ __forceinline__ void issue_chunk(int8_t* buf, const int8_t* __restrict__ pop, int64_t k0, int cnt, int ch) {
    using G = I8Geom<M>;
    constexpr int PARTS = G::CH / 16;
    for (int q = threadIdx.x; q < cnt * PARTS; q += kV2Threads) {
        const int k = q / PARTS, part = q - (q / PARTS) * PARTS;
        cp_async16(buf + k * G::ST + part * 16, pop + (k0 + k) * (int64_t)(M * M) + ch * G::CH + part * 16);
    }
}

template <int M>
constexpr int i8_min_blocks() {
    return M > 32 ? 3 : 1;  // cap registers (<= 168) so three CTAs fit per SM at m >= 36
}

template <int M, int VM>
__global__ void __launch_bounds__(kV2Threads, i8_min_blocks<M>()) k_fit_i8_v2(const int8_t* __restrict__ pop, int64_t n, uint32_t vm_out,
                                                        int64_t* __restrict__ f1, int64_t* __restrict__ f2,
                                                        int64_t* __restrict__ orth, int64_t* __restrict__ sq,
                                                        int32_t* bad_flag) {
    using G = I8Geom<M>;
    constexpr int W = Order<M>::W;
    extern __shared__ __align__(16) int8_t sm8[];
    const int t = threadIdx.x;
    uint32_t bad = 0;
    int64_t k0 = (int64_t)blockIdx.x * kV2Threads;
    if (k0 < n) issue_chunk<M>(sm8, pop, k0, (int)min((int64_t)kV2Threads, n - k0), 0);
    cp_async_commit();
    int buf = 0;
    for (; k0 < n; k0 += (int64_t)gridDim.x * kV2Threads) {
        const int cnt = (int)min((int64_t)kV2Threads, n - k0);
        const int64_t k1 = k0 + (int64_t)gridDim.x * kV2Threads;
        uint32_t c[M * W];
#pragma unroll
        for (int i = 0; i < M * W; ++i) c[i] = 0;
        int sum_sq = 0, sum_v = 0;
        // one staged chunk: prefetch the next one (or the next tile's first), wait, extract
        auto step = [&](int ch, auto wsel) {
            constexpr int WS = decltype(wsel)::value;
            if (ch + 1 < G::NCH)
                issue_chunk<M>(sm8 + (buf ^ 1) * G::BUF, pop, k0, cnt, ch + 1);
            else if (k1 < n)
                issue_chunk<M>(sm8 + (buf ^ 1) * G::BUF, pop, k1, (int)min((int64_t)kV2Threads, n - k1), 0);
            cp_async_commit();
            cp_async_wait<1>();
            __syncthreads();
            if (t < cnt) extract_chunk<M, G::R, WS>(sm8 + buf * G::BUF + t * G::ST, c, sum_sq, sum_v);
            __syncthreads();
            buf ^= 1;
        };
        constexpr int RW0 = M < 32 ? M : 32;
        for (int ch = 0; ch < RW0 / G::R; ++ch) step(ch, std::integral_constant<int, 0>{});
        if constexpr (RW0 < 32) {
#pragma unroll
            for (int col = 0; col < M; ++col) c[col * W] >>= (32 - RW0);
        }
        if constexpr (W > 1) {
            constexpr int RW1 = M - 32;
            for (int ch = 8; ch < 8 + RW1 / G::R; ++ch) step(ch, std::integral_constant<int, 1>{});
            if constexpr (RW1 < 32) {
#pragma unroll
                for (int col = 0; col < M; ++col) c[col * W + 1] >>= (32 - RW1);
            }
        }
        if (t < cnt) {
            int nneg = 0;
#pragma unroll
            for (int i = 0; i < M * W; ++i) nneg += __popc(c[i]);
            bad |= (sum_sq != M * M) | (sum_v != M * M - 2 * nneg);
            Sums s{0, 0, 0, 0};
            pair_sums<M, VM, 0>(c, s);
            write_all<M>(vm_out, k0 + t, s, Order<M>::PAIRS, f1, f2, orth, sq);
        }
    }
    cp_async_wait<0>();
    if (bad_flag) {
        const int any = __syncthreads_or(bad != 0);
        if (any && t == 0) atomicOr(bad_flag, HGA_FLAG_NOT_SIGN);
    }
}

template <int M>
struct PkGeom {
    static constexpr int W = Order<M>::W;
    static constexpr int MW = M * W;                          // words per matrix
    static constexpr int U = (MW + 3) / 4;                    // 16B units per matrix
    static constexpr int STU = (U & 1) ? U : U + 1;           // odd: conflict-free LDS.128
    static constexpr int BUF = kV2Threads * STU * 16;         // bytes
    static constexpr int NBUF = (2 * BUF <= 96 * 1024) ? 2 : 1;
    static constexpr int SMEM = NBUF * BUF;
};

template <int M>
__device__ __forceinline__ void issue_packed(uint8_t* buf, const uint32_t* __restrict__ cols, int64_t k0, int cnt) {
    using G = PkGeom<M>;
    // matrix records are MW words; copy whole 16B units when MW % 4 == 0,
    // which holds for every order here (M multiple of 4)
    for (int q = threadIdx.x; q < cnt * G::U; q += kV2Threads) {
        const int k = q / G::U, part = q - (q / G::U) * G::U;
        cp_async16(buf + (k * G::STU + part) * 16, cols + (k0 + k) * (int64_t)G::MW + part * 4);
    }
}

template <int M, int VM, int FIRST>
__global__ void __launch_bounds__(kV2Threads) k_fit_packed_v2(const uint32_t* __restrict__ cols, int64_t n,
                                                            uint32_t vm_out, int64_t* __restrict__ f1,
                                                            int64_t* __restrict__ f2, int64_t* __restrict__ orth,
                                                            int64_t* __restrict__ sq) {
    using G = PkGeom<M>;
    constexpr int W = Order<M>::W;
    static_assert(G::MW % 4 == 0, "packed records must be 16B granular");
    extern __shared__ __align__(16) uint8_t smp[];
    const int t = threadIdx.x;
    int buf = 0;
    int64_t k0 = (int64_t)blockIdx.x * kV2Threads;
    if (G::NBUF == 2 && k0 < n) issue_packed<M>(smp, cols, k0, (int)min((int64_t)kV2Threads, n - k0));
    cp_async_commit();
    for (; k0 < n; k0 += (int64_t)gridDim.x * kV2Threads) {
        const int cnt = (int)min((int64_t)kV2Threads, n - k0);
        const int64_t k1 = k0 + (int64_t)gridDim.x * kV2Threads;
        if (G::NBUF == 1) issue_packed<M>(smp, cols, k0, cnt);
        else if (k1 < n) issue_packed<M>(smp + (buf ^ 1) * G::BUF, cols, k1, (int)min((int64_t)kV2Threads, n - k1));
        cp_async_commit();
        if (G::NBUF == 2) cp_async_wait<1>();
        else cp_async_wait<0>();
        __syncthreads();
        uint32_t c[M * W];
        if (t < cnt) {
            const uint4* src = reinterpret_cast<const uint4*>(smp + (G::NBUF == 2 ? buf : 0) * G::BUF + t * G::STU * 16);
#pragma unroll
            for (int u = 0; u < G::U; ++u) {
                const uint4 q = src[u];
                c[4 * u] = q.x;
                c[4 * u + 1] = q.y;
                c[4 * u + 2] = q.z;
                c[4 * u + 3] = q.w;
            }
        }
        __syncthreads();
        if (t < cnt) {
            Sums s{0, 0, 0, 0};
            pair_sums<M, VM, FIRST>(c, s);
            write_all<M>(vm_out, k0 + t, s, Order<M>::PAIRS, f1, f2, orth, sq);
        }
        buf ^= 1;
    }
    cp_async_wait<0>();
}

// launcher shared by the per-range instantiation files
template <int M>
int launch_fit_v2_m(bool from_i8, const void* src, int64_t n, uint32_t v, int64_t* f1, int64_t* f2, int64_t* orth,
                    int64_t* sq, int32_t* bad, cudaStream_t st) {
    void (*ki)(const int8_t*, int64_t, uint32_t, int64_t*, int64_t*, int64_t*, int64_t*, int32_t*);
    void (*kp)(const uint32_t*, int64_t, uint32_t, int64_t*, int64_t*, int64_t*, int64_t*);
    if ((v & ~(HGA_VAR_F2 | HGA_VAR_ORTH)) == 0) {
        ki = k_fit_i8_v2<M, HGA_VAR_F2 | HGA_VAR_ORTH>;
        kp = k_fit_packed_v2<M, HGA_VAR_F2 | HGA_VAR_ORTH, 0>;
    } else if (v == HGA_VAR_F1) {
        ki = k_fit_i8_v2<M, HGA_VAR_F1>;
        kp = k_fit_packed_v2<M, HGA_VAR_F1, 0>;
    } else {
        ki = k_fit_i8_v2<M, HGA_VAR_ALL>;
        kp = k_fit_packed_v2<M, HGA_VAR_ALL, 0>;
    }
    const void* kern = from_i8 ? (const void*)ki : (const void*)kp;
    const int smem = from_i8 ? I8Geom<M>::SMEM : PkGeom<M>::SMEM;
    static int attr_done[3] = {0, 0, 0};
    const int slot = (v == HGA_VAR_F1) ? 1 : ((v & ~(HGA_VAR_F2 | HGA_VAR_ORTH)) == 0 ? 0 : 2);
    if (smem > 48 * 1024 && !(attr_done[slot] & (from_i8 ? 1 : 2))) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return to_rc(e);
        attr_done[slot] |= from_i8 ? 1 : 2;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kV2Threads, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t tiles = (n + kV2Threads - 1) / kV2Threads;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sm_count_cached() * per_sm));
    if (from_i8)
        ki<<<(unsigned)grid, kV2Threads, smem, st>>>((const int8_t*)src, n, v, f1, f2, orth, sq, bad);
    else
        kp<<<(unsigned)grid, kV2Threads, smem, st>>>((const uint32_t*)src, n, v, f1, f2, orth, sq);
    return to_rc(cudaGetLastError());
}

// one explicit instantiation per order lives in fit_m<M>.cu (parallel build)
#define HGA_V2_ORDERS(X) X(4) X(8) X(12) X(16) X(20) X(24) X(28) X(32) X(36) X(40) X(44) X(48) X(52) X(56) X(60) X(64)
#define HGA_V2_EXTERN(M)                                                                                         \
    extern template int launch_fit_v2_m<M>(bool, const void*, int64_t, uint32_t, int64_t*, int64_t*, int64_t*, \
                                           int64_t*, int32_t*, cudaStream_t);

inline bool v2_order(int m) { return m >= 4 && m <= 64 && (m % 4) == 0; }

}  // namespace hga
