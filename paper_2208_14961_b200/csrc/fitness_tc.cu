// fitness_tc.cu -- int8 fitness on the 5th-generation tensor cores for
// orders m = 4..64 (engine._fitness_batch, reference engine.py:200-213).
//
// The reference forms the column Gram G = Q^T Q of every matrix with a
// batched float32 matmul and reduces it to F1 = sum|G| - m^2 / F2 = nnz(G) - m.
// Here G comes from tcgen05.mma.kind::i8 (s8 x s8 -> s32, exact), straight
// from the reference's int8 bytes:
//
//   * Q (row-major, r = K index, c = MN index) is read as an MN-major
//     operand; A and B are the SAME shared-memory tile.  Loader warps move
//     the matrix bytes with cp.async (16/8/4-byte pieces, the widest the
//     order's row pitch allows) straight into the canonical no-swizzle
//     layout: 16-column groups of KP (= 64) rows x 16 bytes, core matrices
//     of 8 rows contiguous (LBO = 128 B between K groups, SBO = KP*16 B
//     between column groups).  Padding (rows >= m, columns >= m, the fourth
//     column group at m <= 48) is never written and stays zero, so padded
//     Gram entries are exactly 0.
//   * Two matrices per MMA pair: M = 64 MMAs (K = 32 per instruction, two
//     K steps) whose accumulators interleave in TMEM (the second at lane
//     offset 16), so each of the four epilogue warps (one per TMEM lane
//     quarter) gets 16 Gram rows of each matrix: the work is balanced for
//     every order.  Units of kB = 4 pairs, two accumulator slots (512 TMEM
//     columns) and 6 (K = 64) / 12 (K = 32) shared-memory stages keep loads,
//     MMAs and epilogues overlapped.
//   * Epilogue: tcgen05.ld 32x32b.x16 -> registers; each lane sums |g|,
//     [g != 0] and g^2 over its row; 16-lane shuffles and a 4-warp combine
//     give the matrix totals.
//   * +-1 contract of the v2 kernels (HGA_FLAG_NOT_SIGN otherwise): check
//     warps scan each staged matrix for bytes outside {0x00, 0x01, 0xFF} and
//     count the nonzero ones (m^2 iff no entry is 0).
//
// Roofline: HBM (m^2 + 8 bytes per matrix).  Per matrix the tensor pipe
// does 2 * 64 * N * 64 MACs (N = 16 ceil(m/16)) and the epilogue ~2 * 64 * N
// integer ops, both far below the HBM time at these orders.
#include <cuda.h>  // CUtensorMap (types only; the encoder comes from cudaGetDriverEntryPoint)

#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "hga_common.cuh"
#include "tcgen05.cuh"

namespace hga {
namespace tc {

using namespace tcx;

constexpr int kStageBytes = 192 * 1024;  // all stages; > 114 KB keeps one CTA (and one TMEM owner) per SM
constexpr int kMaxStages = 48;
#ifndef HGA_TC_KB
#define HGA_TC_KB 4
#endif
// MMA pairs per pipeline unit (one barrier round trip per unit).  Measured
// (B200, 10^6 matrices, F2): kB = 1 / 2 / 4 -> m = 48: 5.4 / 8.4 / 9.7e8,
// m = 64: 4.4 / 6.7 / 7.7e8 evals/s -- the per-unit costs (mbarrier round
// trips, group barrier, finalisation) dominate small units; kB = 4 leaves 2
// accumulator slots of 256 TMEM columns, so 2 epilogue groups.
constexpr int kB = HGA_TC_KB;
constexpr int kSlotCols = kB * 64;
constexpr int kSlots = 512 / kSlotCols;  // TMEM accumulator slots
// epilogue groups of 4 warps (one per TMEM lane quarter); group g takes units it = g mod kEpiGroups.
// A group starts waiting on a slot's mbarrier only after finishing unit it - kEpiGroups, so the slot's
// previous phase (unit it - kSlots) is complete iff kSlots >= kEpiGroups: parity waits stay unambiguous.
constexpr int kEpiGroups = kSlots >= 3 ? 3 : kSlots;
static_assert(kSlots >= kEpiGroups, "parity waits need kSlots >= kEpiGroups");
constexpr int kEpiWarps = 4 * kEpiGroups;
constexpr int kLoadWarps = 4;  // two per tile of the pair
constexpr int kCheckWarps = kLoadWarps;  // check warp w re-reads what loader warp w copied
constexpr int kThreads = (kEpiWarps + kLoadWarps + kCheckWarps + 1) * 32;
constexpr int kMmaWarp = kEpiWarps + kLoadWarps + kCheckWarps;

// A tile is the M = 64 MMA operand: 4 column groups of 16.  Orders <= 16 put
// four matrices side by side in it (P = 4), orders 17..32 two (P = 2), larger
// orders one (zero-padded).  With P > 1 the MMA also forms the cross-matrix
// blocks; the epilogue reads only each matrix's own diagonal block.
template <int M>
struct Geo {
    static_assert(M >= 4 && M <= 64 && M % 4 == 0, "tensor-core path covers orders 4..64");
    static constexpr int KP = M <= 32 ? 32 : 64;        // padded K (rows)
    static constexpr int NCG = (M + 15) / 16;           // column groups per matrix
    static constexpr int P = M <= 16 ? 4 : (M <= 32 ? 2 : 1);  // matrices per tile
    static constexpr int MPP = 2 * P;                   // matrices per MMA pair (two tiles)
    static constexpr int N = P > 1 ? 64 : 16 * NCG;     // MMA N
    static constexpr int COLS = 16 * NCG;               // Gram columns read per lane
    static constexpr int QPM = P > 1 ? NCG : 4;         // TMEM lane quarters summed per matrix
    static constexpr int TILE = 4 * KP * 16;
    static constexpr int GR = (M % 16 == 0) ? 16 : ((M % 8 == 0) ? 8 : 4);  // cp.async piece
    static constexpr int NG = M * M / GR;               // pieces per matrix
    static constexpr int PER = (P * NG + 64 - 1) / 64;  // pieces per lane (two loader warps per tile)
    static constexpr int SBO = KP * 16;
    static constexpr int STAGES = kStageBytes / (2 * kB * TILE);  // 12 (KP = 64) or 24 (KP = 32)
    static constexpr uint32_t IDESC = (2u << 4)          // D: s32
                                      | (1u << 7) | (1u << 10)   // A, B: signed 8-bit
                                      | (1u << 15) | (1u << 16)  // A, B: MN-major
                                      | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(64 >> 4) << 24);
};

template <int M, int VM, bool OW>
__global__ void __launch_bounds__(kThreads, 1)
    k_fit_i8_tc(const int8_t* __restrict__ pop, int64_t n, uint32_t vm_out, int64_t* __restrict__ f1,
                int64_t* __restrict__ f2, int64_t* __restrict__ orth, int64_t* __restrict__ sq, int32_t* bad_flag,
                int flags, const __grid_constant__ CUtensorMap tmap) {
    // flags (A/B and bottleneck experiments, HGA_TC_FLAGS; 0 in production): 1 = legacy piece
    // order; 2 = skip the MMAs, 4 = skip the epilogue reductions, 8 = skip the +-1 check (results invalid)
    using G = Geo<M>;
    // Orders 48 and 64 (row pitch a multiple of 16 B, one matrix per tile): the
    // stages are filled by TMA, one bulk tensor copy per column group, issued by
    // one thread; the other orders use cp.async pieces from four loader warps.
    constexpr bool kTma = G::P == 1 && M % 16 == 0;
    const bool rowmajor = flags & 1;
    constexpr int UT = 2 * kB;  // tiles per pipeline unit
    extern __shared__ __align__(1024) uint8_t smem[];  // G::STAGES x UT x G::TILE
    __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages], tfull[kSlots], tempty[kSlots];
    __shared__ uint32_t tmem_base;
    __shared__ uint32_t part[kEpiGroups][2][kB][2][4][3];  // [group][iteration parity][pair][tile][quarter][sum]

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t nunits = (n + kB * G::MPP - 1) / (kB * G::MPP);

    // zero the stages once: padding bytes are never written again
    for (int i = tid; i < G::STAGES * UT * G::TILE / 16; i += kThreads)
        reinterpret_cast<uint4*>(smem)[i] = make_uint4(0u, 0u, 0u, 0u);
    if (tid == 0) {
        for (int s = 0; s < G::STAGES; ++s) {
            // TMA: one expect_tx arrival; cp.async: one asynchronous arrival per loader lane
            mbar_init(&full[s], kTma ? 1 : kLoadWarps * 32);
            mbar_init(&empty[s], 1 + kCheckWarps);  // MMA commit + the check warps
        }
        for (int a = 0; a < kSlots; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // zeroed stages -> async proxy (MMA reads)
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

    if (warp >= kEpiWarps && warp < kMmaWarp) {
        // ------------------------------------------------------------ loaders / byte checkers
        const bool checker = warp >= kEpiWarps + kLoadWarps;
        const int lw = (warp - kEpiWarps) % kLoadWarps, j = lw & 1, half = lw >> 1;
        // per-lane piece table: (source byte offset) | (tile byte offset << 16)
        uint32_t tab[G::PER];
#pragma unroll
        for (int i = 0; i < G::PER; ++i) {
            const int g = (i * 2 + half) * 32 + lane;  // piece of the tile's P consecutive matrices
            int e, r, c;
            if (rowmajor) {  // legacy order (A/B switch): pieces in source order
                const int src = g * G::GR;
                e = src / (M * M);
                const int o = src - e * (M * M);
                r = o / M;
                c = o - r * M;
            } else {
                // Bank-conflict-free order: within each block of 8 rows, column group
                // by column group, row by row, then the 16-byte row segment's pieces.
                // The lanes of one shared-memory phase (8 x 16 B, 16 x 8 B or 32 x 4 B)
                // then write / read the 128 contiguous bytes of one core-matrix column
                // (8 rows x 16 B) instead of the same 16 bytes of 4 column groups
                // (4-way conflicts); a warp still covers whole 8-row blocks of the
                // source, so global accesses stay coalesced.
                constexpr int SUB = 16 / G::GR, RB = 8 * (M / G::GR);  // pieces per full 16-B segment / row block
                e = g / G::NG;
                const int o = g - e * G::NG;
                const int rb = o / RB, o2 = o - rb * RB;
                const int rows = min(8, M - 8 * rb);
                const int cg = o2 / (rows * SUB), o3 = o2 - cg * (rows * SUB);
                const int subs = min(16, M - 16 * cg) / G::GR;
                const int rl = o3 / subs;
                r = 8 * rb + rl;
                c = 16 * cg + (o3 - rl * subs) * G::GR;
            }
            const int src = e * (M * M) + r * M + c;
            const int dst = e * G::NCG * G::SBO + (c >> 4) * G::SBO + (r >> 3) * 128 + (r & 7) * 16 + (c & 15);
            tab[i] = g < G::P * G::NG ? ((uint32_t)src | ((uint32_t)dst << 16)) : 0xFFFFFFFFu;
        }
        // check warps: this lane's 16-byte chunks (column group, row < m) of one matrix
        constexpr int kCH = G::NCG * M, kChk = (kCH + 31) / 32;
        uint32_t coff[kChk];
#pragma unroll
        for (int i = 0; i < kChk; ++i) {
            const int idx = i * 32 + lane, cg = idx / M, r = idx - (idx / M) * M;
            coff[i] = idx < kCH ? (uint32_t)((cg * G::KP + r) * 16) : 0x80000000u;
        }
        uint32_t bad = 0;
        int it = 0;
        for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
            const int s = it % G::STAGES;
            if (checker) {
                // Check of the staged tiles (check warp lw takes tiles lw, lw + 4, ..;
                // tile tt = pair tt / 2, interleave tt % 2): every byte of each matrix's rows < m and column
                // groups must be 0x00, 0x01 or 0xFF (entries in {-1, 0, +1}; padding is
                // 0), and the nonzero bytes (bit 0 set) must number m^2 -- so no entry
                // is 0.  16-byte chunks of the canonical layout, contiguous per lane
                // group: conflict-free, independent of the loaders' piece order.
                mbar_wait(&full[s], (it / G::STAGES) & 1);
                for (int tt = lw; tt < ((flags & 8) ? 0 : UT); tt += kCheckWarps) {
                    const uint8_t* tile = smem + (size_t)(s * UT + tt) * G::TILE;
                    const int b = tt >> 1, j = tt & 1;
#pragma unroll
                    for (int e = 0; e < G::P; ++e) {
                        uint32_t cnt = 0;
#pragma unroll
                        for (int i = 0; i < kChk; ++i) {
                            // lanes past the last chunk re-read chunk 0 and mask it to zero (no
                            // branch: all loads of the matrix can be in flight together)
                            const uint4 x = *reinterpret_cast<const uint4*>(tile + e * (G::NCG * G::KP * 16) +
                                                                            (coff[i] & 0xFFFFu));
                            const uint32_t mk = coff[i] >> 31 ? 0u : 0xFFFFFFFFu;
                            const uint32_t w4[4] = {x.x & mk, x.y & mk, x.z & mk, x.w & mk};
#pragma unroll
                            for (int v4 = 0; v4 < 4; ++v4) {
                                const uint32_t a8 = w4[v4], h8 = a8 & 0xFEFEFEFEu;
                                // bits 1..7 equal, and 0xFE excluded (bits 1..7 set => bit 0 set)
                                bad |= ((h8 ^ (h8 << 1)) & 0xFCFCFCFCu) | ((a8 >> 1) & ~a8 & 0x01010101u);
                                cnt += a8 & 0x01010101u;  // per-byte counts, <= 4 * 8 < 256
                            }
                        }
                        cnt = (cnt * 0x01010101u) >> 24;  // sum of the four byte counts
#pragma unroll
                        for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
                        const int64_t k = (int64_t)G::MPP * (kB * u + b) + (int64_t)G::P * j + e;
                        if (k < n && cnt != (uint32_t)(M * M)) bad = 1;
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
                continue;
            }
            if constexpr (kTma) {
                if (lw != 0) break;
                if (lane == 0) {
                    mbar_wait(&empty[s], ((it / G::STAGES) & 1) ^ 1);
                    mbar_expect_tx(&full[s], (uint32_t)(UT * G::NCG * G::KP * 16));
#pragma unroll
                    for (int t = 0; t < UT; ++t) {  // tile t = pair t / 2, interleave t % 2
                        // matrices >= n are fully out of bounds: zero-filled, bytes still counted
                        const int64_t k = (int64_t)G::MPP * (kB * u + (t >> 1)) + (t & 1);
                        const uint32_t dst = sbase + (uint32_t)((s * UT + t) * G::TILE);
#pragma unroll
                        for (int cg = 0; cg < G::NCG; ++cg)
                            tma_load_cg(dst + (uint32_t)(cg * G::SBO), &tmap, 16 * cg, k, &full[s]);
                    }
                }
                __syncwarp();
                continue;
            }
            mbar_wait(&empty[s], ((it / G::STAGES) & 1) ^ 1);
#pragma unroll
            for (int b = 0; b < kB; ++b) {
                const int64_t k0 = (int64_t)G::MPP * (kB * u + b) + (int64_t)G::P * j;
                if (k0 >= n) continue;
                const int8_t* src = pop + k0 * (int64_t)(M * M);
                const uint32_t lim = (uint32_t)min((int64_t)G::P, n - k0) * (uint32_t)(M * M);
                const uint32_t dst = sbase + (uint32_t)((s * UT + 2 * b + j) * G::TILE);
#pragma unroll
                for (int i = 0; i < G::PER; ++i) {
                    if (tab[i] != 0xFFFFFFFFu && (tab[i] & 0xFFFFu) < lim) {
                        const void* gp = src + (tab[i] & 0xFFFFu);
                        const uint32_t sp = dst + (tab[i] >> 16);
                        if constexpr (G::GR == 16) cp_async_piece16(sp, gp);
                        else if constexpr (G::GR == 8) cp_async_piece8(sp, gp);
                        else cp_async_piece4(sp, gp);
                    }
                }
            }
            // arrives on full[s] once this lane's copies above have landed (no blocking wait:
            // up to STAGES units stay in flight per CTA)
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(saddr(&full[s])) : "memory");
        }
        if (bad && bad_flag) atomicOr(bad_flag, HGA_FLAG_NOT_SIGN);
    } else if (warp == kMmaWarp) {
        // ------------------------------------------------------------ MMA issuer
        int it = 0;
        for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
            const int s = it % G::STAGES, a = it % kSlots;
            mbar_wait(&full[s], (it / G::STAGES) & 1);
            mbar_wait(&tempty[a], ((it / kSlots) & 1) ^ 1);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // cp.async data -> MMA operand reads
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (lane == 0) {
#pragma unroll
                for (int t = 0; t < ((flags & 2) ? 0 : UT); ++t) {  // tile t = pair t/2, interleave t%2
                    const uint32_t tile = sbase + (uint32_t)((s * UT + t) * G::TILE);
                    const uint32_t d =
                        tbase + (uint32_t)(a * kSlotCols + (t >> 1) * 64) + ((uint32_t)(16 * (t & 1)) << 16);
#pragma unroll
                    for (int ks = 0; ks < G::KP / 32; ++ks) {
                        const uint64_t desc = sdesc(tile + (uint32_t)(ks * 512), 128u, (uint32_t)G::SBO);
                        mma_i8(d, desc, desc, G::IDESC, ks > 0 ? 1u : 0u);
                    }
                }
                mma_commit(&empty[s]);
                mma_commit(&tfull[a]);
            }
            __syncwarp();
        }
    } else {
        // ------------------------------------------------------------ epilogue (warps 0 .. kEpiWarps-1)
        // Several groups so that each SM sub-partition has kEpiGroups epilogue
        // warps to interleave (one warp alone is latency-bound on the reductions).
        const int q = warp & 3, grp = warp >> 2;  // TMEM lane quarter, epilogue group
        const int jj = lane >> 4;
        // Gram symmetry: each unordered pair of 16-row/16-column blocks {i, j} is
        // read once, off-diagonal blocks counted twice.  Quarter q holds row
        // block lq of its matrix and may read any column block of it (block
        // (q, j) is the transpose of (j, q)).  Packed tiles (P > 1) read the
        // upper triangle, cb >= lq.  One matrix per tile (m = 36..64,
        // NCG = 3 or 4): quarter q reads the cyclic blocks q, q+1, .. q+NCG/2
        // (mod NCG; the d = NCG/2 block of an even NCG only for q < NCG/2), so
        // the quarters read 2/2/2/0 (NCG = 3) or 3/3/2/2 (NCG = 4) blocks per
        // matrix instead of 3/2/1/0 or 4/3/2/1 -- the slowest warp of the group
        // sets the pace.
        const int lq = G::P > 1 ? q % G::NCG : q;
        const int cs = G::P > 1 ? G::COLS * (q / G::NCG) : 0;  // this quarter's matrix block
        constexpr int NB = G::P > 1 ? G::NCG : G::NCG / 2 + 1;  // block slots per pair
        // (column block, weight) of slot d for this quarter; weight 0 = skip
        int bcol[NB];
        uint32_t bw[NB];
#pragma unroll
        for (int d = 0; d < NB; ++d) {
            if constexpr (G::P > 1) {
                bcol[d] = d;
                bw[d] = d < lq ? 0u : (d == lq ? 1u : 2u);
            } else {
                bcol[d] = (q + d) % G::NCG;
                const bool on = q < G::NCG && (d < G::NCG / 2 || (G::NCG & 1) || q < G::NCG / 2);
                bw[d] = on ? (d == 0 ? 1u : 2u) : 0u;
            }
        }
        // one tcgen05.wait::ld per unit when both pairs' blocks fit in registers
        constexpr bool kOneWait = OW && G::P == 1 && kB * NB <= 4;
        for (int it = grp;; it += kEpiGroups) {
            const int64_t u = (int64_t)blockIdx.x + (int64_t)it * gridDim.x;
            if (u >= nunits) break;
            const int a = it % kSlots;
            mbar_wait(&tfull[a], (it / kSlots) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (flags & 4) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[a]);
                continue;
            }
            uint32_t(&pp)[kB][2][4][3] = part[grp][(it / kEpiGroups) & 1];
            uint32_t vall[kOneWait ? kB : 1][NB][16];
            if constexpr (kOneWait) {
#pragma unroll
                for (int b = 0; b < kB; ++b) {
                    const uint32_t taddr = tbase + (uint32_t)(a * kSlotCols + b * 64) + ((uint32_t)(32 * q) << 16);
#pragma unroll
                    for (int d = 0; d < NB; ++d)
                        if (bw[d]) tmem_ld16(taddr + (uint32_t)(16 * bcol[d]), vall[b][d]);
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            }
#pragma unroll
            for (int b = 0; b < kB; ++b) {
                uint32_t(&v)[NB][16] = vall[kOneWait ? b : 0];
                if constexpr (!kOneWait) {
                    const uint32_t taddr = tbase + (uint32_t)(a * kSlotCols + b * 64 + cs) + ((uint32_t)(32 * q) << 16);
#pragma unroll
                    for (int d = 0; d < NB; ++d)
                        if (bw[d]) tmem_ld16(taddr + (uint32_t)(16 * bcol[d]), v[d]);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                }
                // weighted row sums over the chosen blocks (padded entries are 0)
                uint32_t pa[4] = {0, 0, 0, 0}, pn[4] = {0, 0, 0, 0}, ps[4] = {0, 0, 0, 0};  // 4 chains for ILP
#pragma unroll
                for (int d = 0; d < NB; ++d) {
                    if (!bw[d]) continue;
                    const uint32_t wgt = bw[d];
                    uint32_t ba[4] = {0, 0, 0, 0}, bn[4] = {0, 0, 0, 0}, bs[4] = {0, 0, 0, 0};
#pragma unroll
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        const int g = (int)v[d][e];
                        if constexpr ((VM & HGA_VAR_F1) != 0) ba[e & 3] += (uint32_t)abs(g);
                        if constexpr ((VM & (HGA_VAR_F2 | HGA_VAR_ORTH)) != 0) bn[e & 3] += (g != 0);
                        if constexpr ((VM & HGA_VAR_SQ) != 0) bs[e & 3] += (uint32_t)(g * g);
                    }
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        pa[c] += wgt * ba[c];
                        pn[c] += wgt * bn[c];
                        ps[c] += wgt * bs[c];
                    }
                }
                uint32_t s_abs = (pa[0] + pa[1]) + (pa[2] + pa[3]);
                uint32_t s_nz = (pn[0] + pn[1]) + (pn[2] + pn[3]);
                uint32_t s_sq = (ps[0] + ps[1]) + (ps[2] + ps[3]);
#pragma unroll
                for (int o = 8; o; o >>= 1) {
                    s_abs += __shfl_xor_sync(0xffffffffu, s_abs, o);
                    s_nz += __shfl_xor_sync(0xffffffffu, s_nz, o);
                    s_sq += __shfl_xor_sync(0xffffffffu, s_sq, o);
                }
                if ((lane & 15) == 0) {
                    pp[b][jj][q][0] = s_abs;
                    pp[b][jj][q][1] = s_nz;
                    pp[b][jj][q][2] = s_sq;
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[a]);
            asm volatile("bar.sync %0, 128;" ::"r"(1 + grp) : "memory");  // the group's 4 warps
            if (q == 3 && lane < kB * G::MPP) {  // quarter 3 reads the fewest blocks: it finalises
                const int b = lane / G::MPP, ml = lane - b * G::MPP;
                const int64_t k = (int64_t)G::MPP * (kB * u + b) + ml;
                if (k < n) {
                    const int jm = ml / G::P, q0 = G::P > 1 ? (ml % G::P) * G::NCG : 0;
                    uint32_t ta = 0, tn = 0, ts = 0;
#pragma unroll
                    for (int w = 0; w < G::QPM; ++w) {
                        ta += pp[b][jm][q0 + w][0];
                        tn += pp[b][jm][q0 + w][1];
                        ts += pp[b][jm][q0 + w][2];
                    }
                    // diagonal: g_ii = m for +-1 entries (checked by the check warps)
                    const int64_t nz_off = (int64_t)tn - M;
                    if ((vm_out & HGA_VAR_F1) && f1) f1[k] = (int64_t)ta - (int64_t)M * M;
                    if ((vm_out & HGA_VAR_F2) && f2) f2[k] = nz_off;
                    if ((vm_out & HGA_VAR_ORTH) && orth) orth[k] = ((int64_t)M * (M - 1) - nz_off) / 2;
                    if ((vm_out & HGA_VAR_SQ) && sq) sq[k] = (int64_t)ts - (int64_t)M * M * M;
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

template <int M, int VM, bool OW>
static int launch_tc(const int8_t* pop, int64_t n, uint32_t v, int64_t* f1, int64_t* f2, int64_t* orth, int64_t* sq,
                     int32_t* bad, cudaStream_t st) {
    auto kern = k_fit_i8_tc<M, VM, OW>;
    constexpr int smem = Geo<M>::STAGES * 2 * kB * Geo<M>::TILE;
    static bool attr[kMaxDevices] = {};
    const int dev = current_device();
    if (!attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return to_rc(e);
        attr[dev] = true;
    }
    const int64_t nunits = (n + kB * Geo<M>::MPP - 1) / (kB * Geo<M>::MPP);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(nunits, sm_count_cached()));
    static const int flags = [] {
        const char* e = std::getenv("HGA_TC_FLAGS");
        return e ? std::atoi(e) : 0;
    }();
    CUtensorMap map;
    std::memset(&map, 0, sizeof(map));
    if constexpr (Geo<M>::P == 1 && M % 16 == 0) {
        int rc = encode_pop_map(&map, pop, n, M, Geo<M>::KP);
        if (rc != 0) return rc;
    }
    kern<<<grid, kThreads, smem, st>>>(pop, n, v, f1, f2, orth, sq, bad, flags, map);
    return to_rc(cudaGetLastError());
}

template <int M>
static int launch_tc_m(const int8_t* pop, int64_t n, uint32_t v, int64_t* f1, int64_t* f2, int64_t* orth,
                       int64_t* sq, int32_t* bad, cudaStream_t st) {
    // HGA_TC_ONEWAIT: one tcgen05.wait::ld per unit at NCG = 3 (A/B switch)
    static const bool ow = std::getenv("HGA_TC_ONEWAIT") != nullptr;
    if constexpr (Geo<M>::P == 1 && Geo<M>::NCG == 3) {
        if (ow) {
            if ((v & ~(HGA_VAR_F2 | HGA_VAR_ORTH)) == 0)
                return launch_tc<M, HGA_VAR_F2 | HGA_VAR_ORTH, true>(pop, n, v, f1, f2, orth, sq, bad, st);
            if (v == HGA_VAR_F1) return launch_tc<M, HGA_VAR_F1, true>(pop, n, v, f1, f2, orth, sq, bad, st);
            return launch_tc<M, HGA_VAR_ALL, true>(pop, n, v, f1, f2, orth, sq, bad, st);
        }
    }
    if ((v & ~(HGA_VAR_F2 | HGA_VAR_ORTH)) == 0)
        return launch_tc<M, HGA_VAR_F2 | HGA_VAR_ORTH, false>(pop, n, v, f1, f2, orth, sq, bad, st);
    if (v == HGA_VAR_F1) return launch_tc<M, HGA_VAR_F1, false>(pop, n, v, f1, f2, orth, sq, bad, st);
    return launch_tc<M, HGA_VAR_ALL, false>(pop, n, v, f1, f2, orth, sq, bad, st);
}

}  // namespace tc

// Orders routed to the tensor cores by default: measured faster than the
// XOR+POPC kernels from m = 48 on (B200, 10^6 matrices, F2: m = 48 8.4e8 vs
// 6.3e8 evals/s, m = 64 6.8e8 vs 3.7e8; at m = 44 XOR+POPC wins, 9.1e8 vs
// 8.6e8); HGA_FITNESS_TC=all routes every order 4..64, HGA_FITNESS_TC=0 none.
bool fit_tc_order(int m, bool all) { return (m % 4) == 0 && m >= (all ? 4 : 48) && m <= 64; }

int launch_fit_tc(int m, const int8_t* pop, int64_t n, uint32_t v, int64_t* f1, int64_t* f2, int64_t* orth,
                  int64_t* sq, int32_t* bad, cudaStream_t st) {
    switch (m) {
#define HGA_TC_CASE(M) \
    case M: return tc::launch_tc_m<M>(pop, n, v, f1, f2, orth, sq, bad, st);
        HGA_TC_CASE(4) HGA_TC_CASE(8) HGA_TC_CASE(12) HGA_TC_CASE(16) HGA_TC_CASE(20) HGA_TC_CASE(24)
        HGA_TC_CASE(28) HGA_TC_CASE(32) HGA_TC_CASE(36) HGA_TC_CASE(40) HGA_TC_CASE(44) HGA_TC_CASE(48)
        HGA_TC_CASE(52) HGA_TC_CASE(56) HGA_TC_CASE(60) HGA_TC_CASE(64)
#undef HGA_TC_CASE
        default: return HGA_E_UNSUPPORTED;
    }
}

}  // namespace hga
