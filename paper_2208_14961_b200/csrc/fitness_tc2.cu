// fitness_tc2.cu -- int8 fitness on the tcgen05 tensor cores for orders
// m = 36..64 (engine._fitness_batch / evaluate, reference engine.py:200-230).
//
// Same formulation as the reference: G = Q^T Q per matrix (exact s8 x s8 ->
// s32 on tcgen05.mma.kind::i8, accumulators in TMEM), F1 = sum|G| - m^2,
// F2 = nnz(G) - m; ORTH and SQ from the same pass.  Round-2 design, built to
// cut the issue slots per matrix (the round-1 kernel, fitness_tc.cu, spent
// ~680 warp instructions per matrix at m = 64 and sat at 0.34-0.48 of HBM):
//
//   * Loads: ONE 1-D bulk copy (cp.async.bulk) per unit -- 8 consecutive
//     matrices = 8 m^2 contiguous bytes (m^2 is a multiple of 16) -- into a
//     raw staging ring.  The check warps, which must read every byte anyway
//     for the +-1 contract, re-lay the rows into the canonical no-swizzle
//     MN-major tiles (16-column groups of 64 K-rows x 16 B) as they check
//     them.  (Measured: the round-1 kernel's 3-D TMA boxes are 16 bytes wide
//     -- one 16-byte row segment per request -- and the TMA unit, not DRAM,
//     set the pace: ~1.3 us per 8 matrices at m = 48.)  Separate raw and
//     tile rings: raw stages are freed as soon as they are re-laid, so up to
//     12 units of loads stay in flight.
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
//   * Per-matrix totals without barriers: one REDUX per matrix and variant,
//     red.shared of the partials and one acq_rel counter increment per warp;
//     the quarter that arrives LAST writes the penalties and resets the
//     accumulators (kSlots+1-deep ring, safe because a warp cannot start
//     unit it+kSlots+1 before every epilogue warp has loaded unit it+1 --
//     the TMEM slot handshake).  (Shuffle trees + SC fences here cost ~25 % at m = 48.)
//   * Two half-size CTAs per SM (kB = 2 pairs per unit, 256 TMEM columns,
//     108 KB shared memory each): each CTA's handshake latencies hide behind
//     the other's work (+15-20 % at every order over one full-size CTA).
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

#ifndef HGA_TC2_SPIN
#define HGA_TC2_SPIN 0  // 1: epilogue / MMA waits busy-poll (test_wait); 2: + check warps
#endif
#ifndef HGA_TC2_M128
#define HGA_TC2_M128 0
#endif
#ifndef HGA_TC2_FLAGS
#define HGA_TC2_FLAGS 0
#endif
#ifndef HGA_TC2_KB
#define HGA_TC2_KB 2
#endif
constexpr int kB = HGA_TC2_KB;        // MMA pairs (2 matrices each) per pipeline unit
#ifndef HGA_TC2_CPS
#define HGA_TC2_CPS 2
#endif
constexpr int kCtasPerSm = HGA_TC2_CPS;  // CTAs sharing an SM (TMEM and shared memory split between them)
constexpr int kUnit = 2 * kB;         // matrices per unit
constexpr int kGroups = kB;           // epilogue group g takes pair g of every unit
constexpr int kEpiWarps = 4 * kGroups;
#ifndef HGA_TC2_CHECK
#define HGA_TC2_CHECK 4
#endif
#ifndef HGA_TC2_TST
#define HGA_TC2_TST 2
#endif
constexpr int kCheckWarps = HGA_TC2_CHECK;  // check warp w takes matrices kMpw*w .. kMpw*w + kMpw-1 of every unit
constexpr int kMpw = 2 * kB / kCheckWarps;
static_assert(kMpw * kCheckWarps == 2 * kB, "check warps divide the unit");
constexpr int kProdWarp = kEpiWarps + kCheckWarps;
constexpr int kMmaWarp = kProdWarp + 1;
constexpr int kThreads = (kMmaWarp + 1) * 32;
constexpr int kSmemBytes = kCtasPerSm == 4 ? 52 * 1024 : (kCtasPerSm == 2 ? 108 * 1024 : 220 * 1024);
constexpr int kTmemCols = 512 / kCtasPerSm;
constexpr int kPairCols = HGA_TC2_M128 ? 128 : 64;  // TMEM columns per MMA pair
constexpr int kSlots = kTmemCols / (kB * kPairCols) > 4 ? 4 : kTmemCols / (kB * kPairCols);  // accumulator slots
constexpr int kBufs = kSlots + 1;     // finalisation ring depth (see header)
constexpr int kMaxStages = 12;

template <int M>
struct Geo {
    static_assert(M >= 36 && M <= 64 && M % 4 == 0, "orders 36..64");
    static constexpr int NCG = (M + 15) / 16;        // 16-column groups
    // MMA N: 64 even at NCG = 3 -- measured (scripts/probe.py, rotating tiles) a
    // 64 x 48 x 32 MMA takes 92 clocks, 64 x 64 x 32 only 77; the extra Gram
    // columns 48..63 (B's fourth group = the next tile's first) are never read
    // M128 mode: one M = 128, N = 128 MMA per K step covers a PAIR -- A = B =
    // the pair's two 4-group tiles back to back, the diagonal 64 x 64 blocks of
    // D are the two Grams (same instruction time as 64 x 64, measured)
    static constexpr bool M128 = HGA_TC2_M128 != 0;
    static constexpr int N = M128 ? 128 : 64;
    static constexpr int MM = M128 ? 128 : 64;       // MMA M
    static constexpr int TILE = M128 ? 4096 : NCG * 1024;  // tile pitch: groups x 64 K-rows x 16 B
    static constexpr int RAW = M * M;                // raw matrix bytes (a multiple of 16)
    static constexpr int TSTAGE = kUnit * TILE;      // canonical tiles of one unit
    static constexpr int RSTAGE = (kUnit * RAW + 127) & ~127;  // raw bytes of one unit
    static constexpr int TSTAGES = HGA_TC2_TST;
    static constexpr int RS_FIT = (kSmemBytes - 1024 - TSTAGES * TSTAGE) / RSTAGE;
    static constexpr int RSTAGES = RS_FIT > kMaxStages ? kMaxStages : RS_FIT;
    static constexpr int SMEM = TSTAGES * TSTAGE + RSTAGES * RSTAGE + 1024;
    static constexpr int SLOT = kB * N;              // TMEM columns per slot
    static constexpr int NQ = (M128 || NCG == 4) ? 4 : 3;  // lane quarters with Gram rows
    static constexpr int LASTW = (M - 16 * (NCG - 1)) / 4;  // valid 4-byte words of the last group
    static constexpr int MR = (M + 7) & ~7;          // rows per group in the relayout walk
    static constexpr int CHUNKS = NCG * MR;          // relayout slots per matrix
    static constexpr int ITER = (CHUNKS + 31) / 32;  // per lane
    static constexpr uint32_t IDESC = (2u << 4)                    // D: s32
                                      | (1u << 7) | (1u << 10)     // A, B: signed 8-bit
                                      | (1u << 15) | (1u << 16)    // A, B: MN-major
                                      | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(MM >> 4) << 24);
    static_assert(kSlots >= 2 && kSlots * SLOT <= kTmemCols, "at least two TMEM slots");
    static_assert(RSTAGES >= 2, "at least two raw stages");
};

// nonzero count: carry of g + 0xffffffff is [g != 0]
__device__ __forceinline__ uint32_t add_nonzero(uint32_t acc, uint32_t g) {
    asm("{\n\t.reg .u32 t;\n\tadd.cc.u32 t, %1, 0xffffffff;\n\taddc.u32 %0, %0, 0;\n\t}" : "+r"(acc) : "r"(g));
    return acc;
}

// per-byte +-1 check sums of one 4-byte word (see header)
__device__ __forceinline__ void check_word(uint32_t x, int& sq, int& lin) {
    sq = __dp4a((int)x, (int)x, sq);
    lin = __dp4a((int)x, 0x7F7F7F7F, lin);
    lin = (int)__dp4a(x, 0x01010101u, (unsigned)lin);
}

// Row sums of quarter Q over its Gram blocks (q, q + d mod NCG), d = 0..NB-1.
// M128 layout: lane = Gram row; HALF 0 = rows 0..31 (row blocks 0, 1), HALF 1 =
// rows 32..63.  HALF 0 reads column blocks 0, 1 (weight 1: both diagonal blocks
// and the {0,1} pair from both sides) and 2 .. NCG-1 (weight 2); HALF 1 reads
// column blocks 2 .. NCG-1 with weight 1 (rows >= m are zero).
template <int M, int VM, int HALF>
__device__ __forceinline__ void half_sums(uint32_t taddr, uint32_t& s1, uint32_t& s2, uint32_t& s4) {
    using G = Geo<M>;
    constexpr int C0 = HALF == 0 ? 0 : 2;
    constexpr int NB = G::NCG - C0;
    uint32_t v[NB][16];
#pragma unroll
    for (int d = 0; d < NB; ++d) tmem_ld16(taddr + (uint32_t)(16 * (C0 + d)), v[d]);
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
        const uint32_t w = (HALF == 0 && C0 + d >= 2) ? 2u : 1u;
        s1 += w * a;
        s2 += w * z;
        s4 += w * q;
    }
}

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
__global__ void __launch_bounds__(kThreads, kCtasPerSm)
    k_fit_i8_tc2(const int8_t* __restrict__ pop, int64_t n, uint32_t vm_out, int64_t* __restrict__ f1,
                 int64_t* __restrict__ f2, int64_t* __restrict__ orth, int64_t* __restrict__ sq, int32_t* bad_flag) {
    // role ablation for bottleneck experiments (compile time: -DHGA_TC2_FLAGS=..., results invalid;
    // 0 in production): 2 = skip the MMAs, 4 = skip the epilogue, 8 = skip the relayout + check
    constexpr int flags = HGA_TC2_FLAGS;
    using G = Geo<M>;
    // dynamic shared memory: [TSTAGES x kUnit canonical tiles][RSTAGES x kUnit raw matrices][1 KB]
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t rfull[kMaxStages], rempty[kMaxStages], tready[G::TSTAGES],
        tfree[G::TSTAGES], tfull[kSlots], tempty[kSlots];
    __shared__ uint32_t tmem_base;
    __shared__ uint32_t eacc[kBufs][kGroups][2][3];
    __shared__ uint32_t ecnt[kBufs][kGroups];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t nunits = (n + kUnit - 1) / kUnit;

    // zero the tiles once: their padding (rows >= m, columns >= m) is never written again
    for (int i = tid; i < G::TSTAGES * G::TSTAGE / 16; i += kThreads)
        reinterpret_cast<uint4*>(smem)[i] = make_uint4(0u, 0u, 0u, 0u);
    for (int i = tid; i < kBufs * kGroups * 6; i += kThreads) (&eacc[0][0][0][0])[i] = 0;
    if (tid < kBufs * kGroups) (&ecnt[0][0])[tid] = 0;
    if (tid == 0) {
        for (int s = 0; s < G::RSTAGES; ++s) {
            mbar_init(&rfull[s], 1);             // producer's expect_tx arrival
            mbar_init(&rempty[s], kCheckWarps);  // check warps done reading the raw bytes
        }
        for (int s = 0; s < G::TSTAGES; ++s) {
            mbar_init(&tready[s], kCheckWarps);  // canonical tiles written
            mbar_init(&tfree[s], 1);             // MMA commit: tiles read
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
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = tmem_base;
    const uint32_t sbase = saddr(smem);
    uint8_t* const raw0 = smem + G::TSTAGES * G::TSTAGE;

    if (warp == kProdWarp) {
        // ---------------------------------------------------------------- producer: one bulk copy per unit
        if (lane == 0) {
            int it = 0;
            for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
                const int s = it % G::RSTAGES;
                mbar_wait(&rempty[s], ((it / G::RSTAGES) & 1) ^ 1);
                const int64_t k0 = kUnit * u;
                const uint32_t bytes = (uint32_t)(min((int64_t)kUnit, n - k0) * G::RAW);
                mbar_expect_tx(&rfull[s], bytes);
                bulk_g2s(saddr(raw0 + s * G::RSTAGE), pop + k0 * G::RAW, bytes, &rfull[s]);
            }
        }
    } else if (warp == kMmaWarp) {
        // ---------------------------------------------------------------- MMA issuer
        int it = 0;
        for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
            const int ts = it % G::TSTAGES, a = it % kSlots;
            if constexpr (HGA_TC2_SPIN >= 1) {
                mbar_wait_spin(&tready[ts], (it / G::TSTAGES) & 1);
                mbar_wait_spin(&tempty[a], ((it / kSlots) & 1) ^ 1);
            } else {
                mbar_wait(&tready[ts], (it / G::TSTAGES) & 1);
                mbar_wait(&tempty[a], ((it / kSlots) & 1) ^ 1);
            }
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (lane == 0) {
                const uint32_t st = sbase + (uint32_t)(ts * G::TSTAGE);
                if constexpr (G::M128) {
                    // pair b: tiles 2b, 2b+1 back to back = one 128-row operand; D columns b * 128
#pragma unroll
                    for (int ks = 0; ks < 2; ++ks)
#pragma unroll
                        for (int b = 0; b < kB; ++b) {
                            const uint64_t desc = sdesc(st + (uint32_t)(2 * b * G::TILE + ks * 512), 128u, 1024u);
                            if constexpr (!(flags & 2))
                                mma_i8(tbase + (uint32_t)(a * G::SLOT + b * 128), desc, desc, G::IDESC, ks > 0 ? 1u : 0u);
                        }
                } else {
                // K step 0 of every tile, then K step 1: consecutive MMAs never feed the
                // same accumulator (a dependent pair would wait for the first's result)
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
#pragma unroll
                    for (int t = 0; t < kUnit; ++t) {  // pair t / 2, matrix t % 2 at TMEM lane offset 16
                        const uint32_t tile = st + (uint32_t)(t * G::TILE);
                        const uint32_t d =
                            tbase + (uint32_t)(a * G::SLOT + (t >> 1) * G::N) + ((uint32_t)(16 * (t & 1)) << 16);
                        const uint64_t desc = sdesc(tile + (uint32_t)(ks * 512), 128u, 1024u);
                        if constexpr (!(flags & 2)) mma_i8(d, desc, desc, G::IDESC, ks > 0 ? 1u : 0u);
                    }
                }
                }
                mma_commit(&tfree[ts]);
                mma_commit(&tfull[a]);
            }
            __syncwarp();
        }
    } else if (warp >= kEpiWarps) {
        // ---------------------------------------------------------------- check + relayout warps
        // Warp w takes matrices 2w, 2w + 1 of each unit: raw row r, column group cg
        // (16 bytes, the last group's LASTW valid words, the rest zero: they belong
        // to the next row) -> canonical chunk cg*1024 + (r/8)*128 + (r%8)*16, and
        // the three dp4a sums of every word (independent accumulators per word
        // position: no long dependency chains).
        const int w = warp - kEpiWarps;
        uint32_t bad = 0;
        int it = 0;
        for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
            const int rs = it % G::RSTAGES, ts = it % G::TSTAGES;
            if constexpr (HGA_TC2_SPIN >= 2) {
                mbar_wait_spin(&rfull[rs], (it / G::RSTAGES) & 1);
                mbar_wait_spin(&tfree[ts], ((it / G::TSTAGES) & 1) ^ 1);
            } else {
                mbar_wait(&rfull[rs], (it / G::RSTAGES) & 1);
                mbar_wait(&tfree[ts], ((it / G::TSTAGES) & 1) ^ 1);
            }
            const uint8_t* rawu = raw0 + rs * G::RSTAGE;
            uint8_t* tileu = smem + ts * G::TSTAGE;
            int sqa[kMpw][4], lna[kMpw][4];
#pragma unroll
            for (int j = 0; j < kMpw; ++j)
#pragma unroll
                for (int q = 0; q < 4; ++q) sqa[j][q] = lna[j][q] = 0;
#pragma unroll
            for (int i = 0; i < G::ITER; ++i) {
                int cg, r;
                bool on;
                if constexpr (M == 64) {
                    // rows at a 64-byte pitch: lane (l & 7) reads row 8*blk + (l & 7) at column
                    // group ((l & 7) / 2 + i) % 4, so the 8 lanes of a 16-byte wavefront hit 8
                    // distinct bank quads for the raw read AND the tile write
                    r = 8 * ((lane >> 3) + 4 * (i >> 2)) + (lane & 7);
                    cg = (((lane & 7) >> 1) + i) & 3;
                    on = true;
                } else {
                    const int c = lane + 32 * i;
                    cg = c / G::MR;
                    r = c - cg * G::MR;
                    on = c < G::CHUNKS && r < M;
                }
                const int nw = cg == G::NCG - 1 ? G::LASTW : 4;
#pragma unroll
                for (int j = 0; j < kMpw; ++j) {
                    const int t = kMpw * w + j;
                    const uint8_t* src = rawu + t * G::RAW + r * M + 16 * cg;
                    uint32_t x[4] = {0u, 0u, 0u, 0u};
                    if (on && !(flags & 8)) {
                        if constexpr (M % 16 == 0) {
                            const uint4 v = *reinterpret_cast<const uint4*>(src);
                            x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
                        } else if constexpr (M % 8 == 0) {
                            const uint2 lo = *reinterpret_cast<const uint2*>(src);
                            x[0] = lo.x; x[1] = lo.y;
                            if (nw > 2) {
                                const uint2 hi = *reinterpret_cast<const uint2*>(src + 8);
                                x[2] = hi.x; x[3] = hi.y;
                            }
                        } else {
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                if (q < nw) x[q] = *reinterpret_cast<const uint32_t*>(src + 4 * q);
                        }
                        *reinterpret_cast<uint4*>(tileu + t * G::TILE + cg * 1024 + (r >> 3) * 128 + (r & 7) * 16) =
                            make_uint4(x[0], x[1], x[2], x[3]);
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) check_word(x[q], sqa[j][q], lna[j][q]);
                }
            }
            // raw bytes consumed, tiles written (generic proxy -> async proxy for the MMA)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&rempty[rs]);
                mbar_arrive(&tready[ts]);
            }
#pragma unroll
            for (int j = 0; j < kMpw; ++j) {
                const int s2 = __reduce_add_sync(0xffffffffu, (sqa[j][0] + sqa[j][1]) + (sqa[j][2] + sqa[j][3]));
                const int l2 = __reduce_add_sync(0xffffffffu, (lna[j][0] + lna[j][1]) + (lna[j][2] + lna[j][3]));
                if (kUnit * u + kMpw * w + j < n && (128ll * s2 != (long long)l2 || s2 != M * M)) bad = 1;
            }
        }
        if (bad && lane == 0 && bad_flag) atomicOr(bad_flag, HGA_FLAG_NOT_SIGN);
    } else {
        // ---------------------------------------------------------------- epilogue
        const int g = warp >> 2, q = warp & 3;
        if (q < G::NQ) {
            const int j = lane >> 4;  // lanes 0-15: matrix 0 of the pair, 16-31: matrix 1
            int it = 0;
            for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
                const int a = it % kSlots, buf = it % kBufs;
                if constexpr (HGA_TC2_SPIN >= 1) mbar_wait_spin(&tfull[a], (it / kSlots) & 1);
                else mbar_wait(&tfull[a], (it / kSlots) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t taddr = G::M128
                                           ? tbase + (uint32_t)(a * G::SLOT + g * 128 + 64 * (q >> 1)) + ((uint32_t)(32 * q) << 16)
                                           : tbase + (uint32_t)(a * G::SLOT + g * G::N) + ((uint32_t)(32 * q) << 16);
                uint32_t s1 = 0, s2 = 0, s4 = 0;
                if constexpr ((flags & 4) != 0) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[a]);
                    continue;
                }
                if constexpr (G::M128) {
                    if (q & 1) half_sums<M, VM, 1>(taddr, s1, s2, s4);
                    else half_sums<M, VM, 0>(taddr, s1, s2, s4);
                } else {
                    switch (q) {
                        case 0: quarter_sums<M, VM, 0>(taddr, s1, s2, s4); break;
                        case 1: quarter_sums<M, VM, 1>(taddr, s1, s2, s4); break;
                        case 2: quarter_sums<M, VM, 2>(taddr, s1, s2, s4); break;
                        default: quarter_sums<M, VM, 3>(taddr, s1, s2, s4); break;
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[a]);  // registers hold the data: release the slot now
                // per-matrix partials of this quarter: one REDUX per matrix and variant
                uint32_t p[2][3] = {{0u, 0u, 0u}, {0u, 0u, 0u}};
#pragma unroll
                for (int jj = 0; jj < 2; ++jj) {
                    // M128: the whole warp is one matrix (q / 2); else lanes 16-31 are matrix 1
                    const bool mine = G::M128 ? (q >> 1) == jj : j == jj;
                    if constexpr ((VM & HGA_VAR_F1) != 0) p[jj][0] = __reduce_add_sync(0xffffffffu, mine ? s1 : 0u);
                    if constexpr ((VM & (HGA_VAR_F2 | HGA_VAR_ORTH)) != 0)
                        p[jj][1] = __reduce_add_sync(0xffffffffu, mine ? s2 : 0u);
                    if constexpr ((VM & HGA_VAR_SQ) != 0) p[jj][2] = __reduce_add_sync(0xffffffffu, mine ? s4 : 0u);
                }
                if (lane == 0) {
                    // red.shared of the partials, then ONE acq_rel counter increment: the
                    // quarter that arrives last sees every partial and finalises the pair
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj)
#pragma unroll
                        for (int v = 0; v < 3; ++v)
                            if (v == 0 ? (VM & HGA_VAR_F1) != 0
                                       : (v == 1 ? (VM & (HGA_VAR_F2 | HGA_VAR_ORTH)) != 0 : (VM & HGA_VAR_SQ) != 0))
                                asm volatile("red.relaxed.cta.shared::cta.add.u32 [%0], %1;" ::"r"(
                                                 saddr(&eacc[buf][g][jj][v])),
                                             "r"(p[jj][v])
                                             : "memory");
                    uint32_t prev;
                    asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                                 : "=r"(prev)
                                 : "r"(saddr(&ecnt[buf][g]))
                                 : "memory");
                    if (prev == (uint32_t)(G::NQ - 1)) {
                        // last quarter of this pair: finalise both matrices, reset the ring entry
#pragma unroll
                        for (int jj = 0; jj < 2; ++jj) {
                            volatile uint32_t* e = &eacc[buf][g][jj][0];
                            const uint32_t ta = e[0], tn = e[1], ts = e[2];
                            e[0] = 0u;
                            e[1] = 0u;
                            e[2] = 0u;
                            const int64_t k = kUnit * u + 2 * g + jj;
                            if (k < n) {
                                const int64_t nz_off = (int64_t)tn - M;  // diagonal g_ii = m (checked)
                                if ((vm_out & HGA_VAR_F1) && f1) f1[k] = (int64_t)ta - (int64_t)M * M;
                                if ((vm_out & HGA_VAR_F2) && f2) f2[k] = nz_off;
                                if ((vm_out & HGA_VAR_ORTH) && orth) orth[k] = ((int64_t)M * (M - 1) - nz_off) / 2;
                                if ((vm_out & HGA_VAR_SQ) && sq) sq[k] = (int64_t)ts - (int64_t)M * M * M;
                            }
                        }
                        *(volatile uint32_t*)&ecnt[buf][g] = 0u;
                    }
                }
                __syncwarp();
            }
        }
    }

    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(kTmemCols) : "memory");
}

template <int M, int VM>
static int launch(const int8_t* pop, int64_t n, uint32_t v, int64_t* f1, int64_t* f2, int64_t* orth, int64_t* sq,
                  int32_t* bad, cudaStream_t st) {
    using G = Geo<M>;
    auto kern = k_fit_i8_tc2<M, VM>;
    static bool attr[kMaxDevices] = {};  // per device: the attribute is a property of the device's module
    const int dev = current_device();
    if (!attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
        if (e != cudaSuccess) return to_rc(e);
        attr[dev] = true;
    }
    const int64_t nunits = (n + kUnit - 1) / kUnit;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(nunits, (int64_t)kCtasPerSm * sm_count_cached()));
    kern<<<grid, kThreads, G::SMEM, st>>>(pop, n, v, f1, f2, orth, sq, bad);
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
