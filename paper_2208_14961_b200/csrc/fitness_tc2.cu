// fitness_tc2.cu -- int8 fitness on the tcgen05 tensor cores for orders
// m = 36..64 (engine._fitness_batch / evaluate, reference engine.py:200-230).
//
// Same formulation as the reference: G = Q^T Q per matrix (exact s8 x s8 ->
// s32 on tcgen05.mma.kind::i8, accumulators in TMEM), F1 = sum|G| - m^2,
// F2 = nnz(G) - m; ORTH and SQ from the same pass.  Round-2 design, built to
// cut the issue slots per matrix (the round-1 kernel, fitness_tc.cu, spent
// ~680 warp instructions per matrix at m = 64 and sat at 0.34-0.48 of HBM):
//
//   * Loads.  m % 16 == 0 (48, 64): TMA, one 3-D box (16 columns x 64 rows x
//     1 matrix, rows >= m zero-filled) per column group straight into the
//     canonical no-swizzle MN-major layout.  Other orders (36..60): ONE 1-D
//     bulk copy per unit (8 consecutive matrices = 8 m^2 contiguous bytes;
//     m^2 is a multiple of 16) into a raw staging area; the check warps,
//     which must read every byte anyway for the +-1 contract, re-lay the
//     rows into the canonical tiles as they check them (no per-piece
//     cp.async; DRAM sees whole 8 m^2 byte runs).
//   * +-1 check with three dp4a per 4-byte word: for every byte v (signed)
//     with unsigned reading u, v^2 - v - 2[v<0] = v^2 - (127 v + u) / 128 is
//     >= 0 and 0 iff v in {-1, 0, 1}; so  128 sum v^2 == sum(127 v + u)  and
//     sum v^2 == m^2  <=>  every entry is +-1.  (Round 1: ~9 ALU ops / word.)
//   * Tiles.  A = B = the same tile.  At NCG = 3 column groups (m = 36..48)
//     the tile pitch is 3 KB: the M = 64 A operand's fourth column group is
//     the NEXT tile's first one, so Gram rows 48..63 are garbage -- no
//     quarter reads them (rows >= m of a real tile are zero padding).
//   * Epilogue: 4 groups x 4 warps (one per TMEM lane quarter); group g takes
//     MMA pair g of every unit, so all groups work on the same TMEM slot and
//     two slots double-buffer.  The slot is released as soon as the
//     tcgen05.ld's have landed.  Quarter q reads the Gram blocks (q, q+d mod
//     NCG), d = 0..NCG/2, each off-diagonal block counted twice -- 10 of 16
//     blocks at NCG = 4, 6 of 9 at NCG = 3 (quarter 3 idle).  Per element:
//     F2 counts nonzeros with a carry chain (add.cc g + 0xffffffff; addc),
//     2 instructions; F1 |g| (IABS + IADD3, 1.5); SQ one IMAD.
//   * Per-matrix totals without barriers: the 16-lane partials go to shared
//     memory with atomics; the LAST warp of the pair to arrive (a counter)
//     writes the penalties and resets the accumulators (3-deep ring, safe
//     because a warp cannot start unit it+3 before every epilogue warp has
//     loaded unit it+1 -- the TMEM slot handshake).
//
// Roofline: HBM, m^2 + 8 bytes per matrix (int8 in, int64 out).
#include <cuda.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "hga_common.cuh"
#include "tcgen05.cuh"

namespace hga {
namespace tc2 {

using namespace tcx;

constexpr int kB = 4;                 // MMA pairs (2 matrices each) per pipeline unit
constexpr int kUnit = 2 * kB;         // matrices per unit
constexpr int kGroups = kB;           // epilogue group g takes pair g of every unit
constexpr int kEpiWarps = 4 * kGroups;
constexpr int kCheckWarps = 4;        // check warp w takes matrices 2w, 2w + 1 of every unit
constexpr int kProdWarp = kEpiWarps + kCheckWarps;
constexpr int kMmaWarp = kProdWarp + 1;
constexpr int kThreads = (kMmaWarp + 1) * 32;
constexpr int kSlots = 2;             // TMEM accumulator slots
constexpr int kBufs = 3;              // finalisation ring depth (see header)
constexpr int kSmemBytes = 220 * 1024;
constexpr int kMaxStages = 12;

template <int M>
struct Geo {
    static_assert(M >= 36 && M <= 64 && M % 4 == 0, "orders 36..64");
    static constexpr int NCG = (M + 15) / 16;        // 16-column groups
    static constexpr int N = 16 * NCG;               // MMA N (Gram columns)
    static constexpr int TILE = NCG * 1024;          // tile pitch: NCG groups x 64 K-rows x 16 B
    static constexpr bool TMA = (M % 16) == 0;
    static constexpr int RAW = M * M;                // raw matrix bytes (bulk path)
    static constexpr int STAGE_TILES = kUnit * TILE;
    static constexpr int STAGE = (STAGE_TILES + (TMA ? 0 : kUnit * RAW) + 1023) & ~1023;
    static constexpr int STAGES = ((kSmemBytes - 1024) / STAGE) > kMaxStages ? kMaxStages
                                                                               : (kSmemBytes - 1024) / STAGE;
    static constexpr int SMEM = STAGES * STAGE + 1024;  // + the fourth-group overhang of the last tile
    static constexpr int SLOT = kB * N;              // TMEM columns per slot
    static constexpr int NQ = NCG == 3 ? 3 : 4;      // lane quarters holding real Gram rows
    static constexpr int LASTW = (M - 16 * (NCG - 1)) / 4;  // valid 4-byte words of the last group
    static constexpr int MR = (M + 7) & ~7;          // rows per group in the relayout walk
    static constexpr uint32_t IDESC = (2u << 4)                    // D: s32
                                      | (1u << 7) | (1u << 10)     // A, B: signed 8-bit
                                      | (1u << 15) | (1u << 16)    // A, B: MN-major
                                      | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(64 >> 4) << 24);
    static_assert(2 * SLOT <= 512, "two TMEM slots");
    static_assert(STAGES >= 2, "at least two stages");
};

// nonzero count: carry of g + 0xffffffff is [g != 0]
__device__ __forceinline__ uint32_t add_nonzero(uint32_t acc, uint32_t g) {
    uint32_t t;
    asm("add.cc.u32 %1, %2, 0xffffffff;\n\taddc.u32 %0, %0, 0;" : "+r"(acc), "=r"(t) : "r"(g));
    return acc;
}

// per-byte +-1 check sums of one 4-byte word (see header)
__device__ __forceinline__ void check_word(uint32_t x, int& sq, int& lin) {
    sq = __dp4a((int)x, (int)x, sq);
    lin = __dp4a((int)x, 0x7F7F7F7F, lin);
    lin = (int)__dp4a(x, 0x01010101u, (unsigned)lin);
}

// Row sums of quarter Q over its Gram blocks (q, q + d mod NCG), d = 0..NB-1.
template <int M, int VM, int Q>
__device__ __forceinline__ void quarter_sums(uint32_t taddr, uint32_t& s1, uint32_t& s2, uint32_t& s4) {
    using G = Geo<M>;
    constexpr int NB = G::NCG == 4 ? (Q < 2 ? 3 : 2) : 2;
    uint32_t v[NB][16];
#pragma unroll
    for (int d = 0; d < NB; ++d) tmem_ld16(taddr + (uint32_t)(16 * ((Q + d) % G::NCG)), v[d]);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    s1 = s2 = s4 = 0;
#pragma unroll
    for (int d = 0; d < NB; ++d) {
        uint32_t a = 0, z = 0, q = 0;
#pragma unroll
        for (int e = 0; e < 16; e += 2) {
            const int g0 = (int)v[d][e], g1 = (int)v[d][e + 1];
            if constexpr ((VM & HGA_VAR_F1) != 0) a += (uint32_t)abs(g0) + (uint32_t)abs(g1);
            if constexpr ((VM & (HGA_VAR_F2 | HGA_VAR_ORTH)) != 0) z = add_nonzero(add_nonzero(z, (uint32_t)g0), (uint32_t)g1);
            if constexpr ((VM & HGA_VAR_SQ) != 0) q += (uint32_t)(g0 * g0) + (uint32_t)(g1 * g1);
        }
        const uint32_t w = d == 0 ? 1u : 2u;
        s1 += w * a;
        s2 += w * z;
        s4 += w * q;
    }
}

template <int M, int VM>
__global__ void __launch_bounds__(kThreads, 1)
    k_fit_i8_tc2(const int8_t* __restrict__ pop, int64_t n, uint32_t vm_out, int64_t* __restrict__ f1,
                 int64_t* __restrict__ f2, int64_t* __restrict__ orth, int64_t* __restrict__ sq, int32_t* bad_flag,
                 const __grid_constant__ CUtensorMap tmap) {
    using G = Geo<M>;
    extern __shared__ __align__(1024) uint8_t smem[];  // STAGES x [kUnit tiles | kUnit raw matrices]
    __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages], ready[kMaxStages], tfull[kSlots],
        tempty[kSlots];
    __shared__ uint32_t tmem_base;
    __shared__ uint32_t eacc[kBufs][kGroups][2][3];
    __shared__ uint32_t ecnt[kBufs][kGroups];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t nunits = (n + kUnit - 1) / kUnit;

    // zero everything once: tile padding (rows >= m, columns >= m) is never written again
    for (int i = tid; i < G::SMEM / 16; i += kThreads) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0u, 0u, 0u, 0u);
    for (int i = tid; i < kBufs * kGroups * 6; i += kThreads) (&eacc[0][0][0][0])[i] = 0;
    if (tid < kBufs * kGroups) (&ecnt[0][0])[tid] = 0;
    if (tid == 0) {
        for (int s = 0; s < G::STAGES; ++s) {
            mbar_init(&full[s], 1);                                  // producer's expect_tx arrival
            mbar_init(&empty[s], G::TMA ? 1 + kCheckWarps : 1);      // MMA commit (+ check warps, TMA path)
            mbar_init(&ready[s], kCheckWarps);                       // bulk path: relayout + check done
        }
        for (int a = 0; a < kSlots; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], kGroups * G::NQ);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tmem_base)),
                     "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = tmem_base;
    const uint32_t sbase = saddr(smem);

    if (warp == kProdWarp) {
        // ---------------------------------------------------------------- producer
        if (lane == 0) {
            int it = 0;
            for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
                const int s = it % G::STAGES;
                mbar_wait(&empty[s], ((it / G::STAGES) & 1) ^ 1);
                const uint32_t st = sbase + (uint32_t)(s * G::STAGE);
                if constexpr (G::TMA) {
                    // matrices >= n are out of bounds: zero-filled, bytes still counted
                    mbar_expect_tx(&full[s], (uint32_t)(kUnit * G::NCG * 1024));
#pragma unroll
                    for (int t = 0; t < kUnit; ++t)
#pragma unroll
                        for (int cg = 0; cg < G::NCG; ++cg)
                            tma_load_cg(st + (uint32_t)(t * G::TILE + cg * 1024), &tmap, 16 * cg, kUnit * u + t,
                                        &full[s]);
                } else {
                    const int64_t k0 = kUnit * u;
                    const uint32_t bytes = (uint32_t)(min((int64_t)kUnit, n - k0) * G::RAW);
                    mbar_expect_tx(&full[s], bytes);
                    bulk_g2s(st + (uint32_t)G::STAGE_TILES, pop + k0 * G::RAW, bytes, &full[s]);
                }
            }
        }
    } else if (warp == kMmaWarp) {
        // ---------------------------------------------------------------- MMA issuer
        int it = 0;
        for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
            const int s = it % G::STAGES, a = it & 1;
            mbar_wait(G::TMA ? &full[s] : &ready[s], (it / G::STAGES) & 1);
            mbar_wait(&tempty[a], ((it >> 1) & 1) ^ 1);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (lane == 0) {
                const uint32_t st = sbase + (uint32_t)(s * G::STAGE);
#pragma unroll
                for (int t = 0; t < kUnit; ++t) {  // pair t / 2, matrix t % 2 at TMEM lane offset 16
                    const uint32_t tile = st + (uint32_t)(t * G::TILE);
                    const uint32_t d = tbase + (uint32_t)(a * G::SLOT + (t >> 1) * G::N) + ((uint32_t)(16 * (t & 1)) << 16);
#pragma unroll
                    for (int ks = 0; ks < 2; ++ks) {
                        const uint64_t desc = sdesc(tile + (uint32_t)(ks * 512), 128u, 1024u);
                        mma_i8(d, desc, desc, G::IDESC, ks > 0 ? 1u : 0u);
                    }
                }
                mma_commit(&empty[s]);
                mma_commit(&tfull[a]);
            }
            __syncwarp();
        }
    } else if (warp >= kEpiWarps) {
        // ---------------------------------------------------------------- check (+ relayout) warps
        const int w = warp - kEpiWarps;
        uint32_t bad = 0;
        int it = 0;
        for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
            const int s = it % G::STAGES;
            mbar_wait(&full[s], (it / G::STAGES) & 1);
            const uint8_t* st = smem + (size_t)s * G::STAGE;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int t = 2 * w + j;
                const int64_t k = kUnit * u + t;
                if (k >= n) continue;  // warp-uniform
                uint8_t* tile = const_cast<uint8_t*>(st) + t * G::TILE;
                int sq = 0, lin = 0;
                if constexpr (G::TMA) {
                    // canonical chunks (group cg, row r < m): 16 B at cg*1024 + (r/8)*128 + (r%8)*16
                    for (int c = lane; c < G::NCG * M; c += 32) {
                        const int cg = c / M, r = c - cg * M;
                        const uint4 x = *reinterpret_cast<const uint4*>(tile + cg * 1024 + (r >> 3) * 128 + (r & 7) * 16);
                        check_word(x.x, sq, lin);
                        check_word(x.y, sq, lin);
                        check_word(x.z, sq, lin);
                        check_word(x.w, sq, lin);
                    }
                } else {
                    // raw row r of the matrix -> canonical chunks; the last group keeps its
                    // LASTW valid words and zeroes the rest (they belong to the next row)
                    const uint8_t* raw = st + G::STAGE_TILES + t * G::RAW;
                    for (int c = lane; c < G::NCG * G::MR; c += 32) {
                        const int cg = c / G::MR, r = c - cg * G::MR;
                        if (r >= M) continue;
                        const uint8_t* src = raw + r * M + 16 * cg;
                        uint32_t x[4] = {0u, 0u, 0u, 0u};
                        const int nw = cg == G::NCG - 1 ? G::LASTW : 4;
                        if constexpr (M % 8 == 0) {
                            // 8-byte aligned rows: two 8-byte loads (conflict-free for odd m / 8)
                            const uint2 lo = *reinterpret_cast<const uint2*>(src);
                            x[0] = lo.x;
                            x[1] = lo.y;
                            if (nw > 2) {
                                const uint2 hi = *reinterpret_cast<const uint2*>(src + 8);
                                x[2] = hi.x;
                                x[3] = hi.y;
                            }
                        } else {
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                if (q < nw) x[q] = *reinterpret_cast<const uint32_t*>(src + 4 * q);
                        }
#pragma unroll
                        for (int q = 0; q < 4; ++q) check_word(x[q], sq, lin);
                        *reinterpret_cast<uint4*>(tile + cg * 1024 + (r >> 3) * 128 + (r & 7) * 16) =
                            make_uint4(x[0], x[1], x[2], x[3]);
                    }
                }
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    sq += __shfl_xor_sync(0xffffffffu, sq, o);
                    lin += __shfl_xor_sync(0xffffffffu, lin, o);
                }
                if (128ll * sq != (long long)lin || sq != M * M) bad = 1;
            }
            if constexpr (!G::TMA) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // tiles -> MMA
            __syncwarp();
            if (lane == 0) mbar_arrive(G::TMA ? &empty[s] : &ready[s]);
        }
        if (bad && lane == 0 && bad_flag) atomicOr(bad_flag, HGA_FLAG_NOT_SIGN);
    } else {
        // ---------------------------------------------------------------- epilogue
        const int g = warp >> 2, q = warp & 3;
        if (q < G::NQ) {
            const int j = lane >> 4;  // lanes 0-15: matrix 0 of the pair, 16-31: matrix 1
            int it = 0;
            for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
                const int a = it & 1, buf = it % kBufs;
                mbar_wait(&tfull[a], (it >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t taddr = tbase + (uint32_t)(a * G::SLOT + g * G::N) + ((uint32_t)(32 * q) << 16);
                uint32_t s1, s2, s4;
                switch (q) {
                    case 0: quarter_sums<M, VM, 0>(taddr, s1, s2, s4); break;
                    case 1: quarter_sums<M, VM, 1>(taddr, s1, s2, s4); break;
                    case 2: quarter_sums<M, VM, 2>(taddr, s1, s2, s4); break;
                    default: quarter_sums<M, VM, 3>(taddr, s1, s2, s4); break;
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[a]);  // registers hold the data: release the slot now
#pragma unroll
                for (int o = 8; o; o >>= 1) {
                    if constexpr ((VM & HGA_VAR_F1) != 0) s1 += __shfl_xor_sync(0xffffffffu, s1, o);
                    if constexpr ((VM & (HGA_VAR_F2 | HGA_VAR_ORTH)) != 0) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
                    if constexpr ((VM & HGA_VAR_SQ) != 0) s4 += __shfl_xor_sync(0xffffffffu, s4, o);
                }
                if ((lane & 15) == 0) {
                    if constexpr ((VM & HGA_VAR_F1) != 0) atomicAdd(&eacc[buf][g][j][0], s1);
                    if constexpr ((VM & (HGA_VAR_F2 | HGA_VAR_ORTH)) != 0) atomicAdd(&eacc[buf][g][j][1], s2);
                    if constexpr ((VM & HGA_VAR_SQ) != 0) atomicAdd(&eacc[buf][g][j][2], s4);
                }
                __syncwarp();
                __threadfence_block();
                uint32_t prev = 0;
                if (lane == 0) prev = atomicAdd(&ecnt[buf][g], 1u);
                prev = __shfl_sync(0xffffffffu, prev, 0);
                if (prev == (uint32_t)(G::NQ - 1)) {
                    // last quarter of this pair: finalise both matrices, reset the ring entry
                    __threadfence_block();
                    if (lane < 2) {
                        volatile uint32_t* e = &eacc[buf][g][lane][0];
                        const uint32_t ta = e[0], tn = e[1], ts = e[2];
                        e[0] = 0u;
                        e[1] = 0u;
                        e[2] = 0u;
                        const int64_t k = kUnit * u + 2 * g + lane;
                        if (k < n) {
                            const int64_t nz_off = (int64_t)tn - M;  // diagonal g_ii = m (checked)
                            if ((vm_out & HGA_VAR_F1) && f1) f1[k] = (int64_t)ta - (int64_t)M * M;
                            if ((vm_out & HGA_VAR_F2) && f2) f2[k] = nz_off;
                            if ((vm_out & HGA_VAR_ORTH) && orth) orth[k] = ((int64_t)M * (M - 1) - nz_off) / 2;
                            if ((vm_out & HGA_VAR_SQ) && sq) sq[k] = (int64_t)ts - (int64_t)M * M * M;
                        }
                    }
                    if (lane == 0) *(volatile uint32_t*)&ecnt[buf][g] = 0u;
                    __threadfence_block();
                }
            }
        }
    }

    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512) : "memory");
}

template <int M, int VM>
static int launch(const int8_t* pop, int64_t n, uint32_t v, int64_t* f1, int64_t* f2, int64_t* orth, int64_t* sq,
                  int32_t* bad, cudaStream_t st) {
    using G = Geo<M>;
    auto kern = k_fit_i8_tc2<M, VM>;
    int dev = 0;
    cudaGetDevice(&dev);
    static bool attr[64] = {};  // per device: the attribute is a property of the device's module
    if (dev < 0 || dev >= 64 || !attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
        if (e != cudaSuccess) return to_rc(e);
        if (dev >= 0 && dev < 64) attr[dev] = true;
    }
    const int64_t nunits = (n + kUnit - 1) / kUnit;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(nunits, sm_count_cached()));
    CUtensorMap map;
    std::memset(&map, 0, sizeof(map));
    if constexpr (G::TMA) {
        const int rc = encode_pop_map(&map, pop, n, M, 64);
        if (rc != 0) return rc;
    }
    kern<<<grid, kThreads, G::SMEM, st>>>(pop, n, v, f1, f2, orth, sq, bad, map);
    return to_rc(cudaGetLastError());
}

template <int M>
static int launch_m(const int8_t* pop, int64_t n, uint32_t v, int64_t* f1, int64_t* f2, int64_t* orth, int64_t* sq,
                    int32_t* bad, cudaStream_t st) {
    if ((v & ~(HGA_VAR_F2 | HGA_VAR_ORTH)) == 0)
        return launch<M, HGA_VAR_F2 | HGA_VAR_ORTH>(pop, n, v, f1, f2, orth, sq, bad, st);
    if (v == HGA_VAR_F1) return launch<M, HGA_VAR_F1>(pop, n, v, f1, f2, orth, sq, bad, st);
    if (v == HGA_VAR_SQ) return launch<M, HGA_VAR_SQ>(pop, n, v, f1, f2, orth, sq, bad, st);
    return launch<M, HGA_VAR_ALL>(pop, n, v, f1, f2, orth, sq, bad, st);
}

}  // namespace tc2

bool fit_tc2_order(int m) { return m % 4 == 0 && m >= 36 && m <= 64; }

int launch_fit_tc2(int m, const int8_t* pop, int64_t n, uint32_t v, int64_t* f1, int64_t* f2, int64_t* orth,
                   int64_t* sq, int32_t* bad, cudaStream_t st) {
    switch (m) {
#define HGA_TC2_CASE(M) \
    case M: return tc2::launch_m<M>(pop, n, v, f1, f2, orth, sq, bad, st);
        HGA_TC2_CASE(36) HGA_TC2_CASE(40) HGA_TC2_CASE(44) HGA_TC2_CASE(48)
        HGA_TC2_CASE(52) HGA_TC2_CASE(56) HGA_TC2_CASE(60) HGA_TC2_CASE(64)
#undef HGA_TC2_CASE
        default: return HGA_E_UNSUPPORTED;
    }
}

}  // namespace hga
