// run_v2.cuh -- the production generation loop for GA orders m = 4..64
// (step / run_search, reference engine.py:449-538, with Philox streams).
//
// One persistent cooperative kernel runs a batch of generations; each
// generation is three grid-barrier-separated phases:
//   B  every CTA reads the select histogram of the current population (built
//      during the previous generation, keys = fitness >> granule, exact
//      because every balanced GA matrix has F1 = 0 mod 8, F2 = 0 mod 2,
//      SQ = 0 mod 32), finds the threshold tau and the tie quota for the 2N
//      survivors (lowest index first on ties, engine.py:245), and counts
//      (F < tau, F == tau) over its contiguous index range
//   D  survivor ranks (CTA prefix + block scan, index order) -> parent slot
//      through a keyed Feistel bijection (uniformly random placement,
//      engine.py:246); survivors' keys go into the NEXT generation's
//      histogram
//   E  offspring tiles, one thread per offspring: the CTA gathers the 64
//      pairs' parents into shared memory (and writes them to the new
//      population's parent slots), each thread assembles its child's columns
//      (column-block crossover, engine.py:257-277), applies its Philox
//      mutation plan to them in shared memory (engine.py:339-373), loads the
//      M column words into registers and runs the unrolled XOR+POPC pair
//      chain (column 0 is all +1 in every GA individual, so its pairs are 0)
//   F  bookkeeping replicated in every CTA (trace, best, stop, stall restart)
#pragma once

#include <cstdlib>

#include "run_common.cuh"
#include "tile.cuh"

namespace hga {

constexpr int kR2Threads = 128;
constexpr int kTeam = 4;                          // threads (warps) per offspring in the pair chain
constexpr int kTileOff = kR2Threads / kTeam;      // 32 offspring per tile
constexpr int kR2Pairs = kTileOff / 2;            // 16 parent pairs per tile
constexpr int kSelItems = 8;                      // fitness values per thread in the select scans
constexpr int kR2Bins = 32768;
constexpr int kR2MaxGrid = 2048;
constexpr int kR2MaxPlan = 128;  // nc + 2 nr <= (m - 1) + m
constexpr int kRng = 64;          // items per key range (one-barrier select)
constexpr int kMaxRng = 2048;     // one-barrier select up to 4N = 131,072 matrices
// internal run flags (experiments): L2 bulk prefetch at launch of the population / of fitness + histogram
constexpr uint32_t kRunPrefetchPop = 1u << 20;
constexpr uint32_t kRunPrefetchFit = 1u << 21;
constexpr uint32_t kRunPlainLaunch = 1u << 22;
// internal (hga_step_host): do nothing when the uploaded population was rejected
// (RunWs2::host_flag has HGA_FLAG_NOT_SIGN / HGA_FLAG_NOT_GA) -- no host round trip
constexpr uint32_t kRunHostCheck = 1u << 23;

// Per-slot state: the two-barrier loop uses slots gen & 1, the one-barrier
// loop gen % 3 (see k_run_v3).
struct RunWs2 {
    Barrier bar;
    unsigned long long best_key[3];
    unsigned long long par_key[3];
    unsigned long long restart_key;
    int32_t host_flag;  // hga_step_host: HGA_FLAG_* of the uploaded population
    uint32_t kmin[3];
    uint32_t kmax[3];
    uint32_t cnt_lt[kR2MaxGrid];
    uint32_t cnt_eq[kR2MaxGrid];
    alignas(16) uint32_t hist[3][kR2Bins];  // 16-byte aligned: bulk-prefetched into L2 at launch
    unsigned long long tstamp[64][20];  // HGA_RUN_TIMING: %globaltimer at phase boundaries (CTA 0)
    // followed by lt_list[4N], eq_list[4N] (uint64 (F << 32) | index): each CTA's survivors, compacted in index
    // order (two-barrier loop), then keys[2][run2_key_stride] (uint16 F >> granule per slot, padded with 0xFFFF;
    // one-barrier loop)
};

__host__ __device__ inline int64_t run2_key_stride(int64_t n_pairs) { return (4 * n_pairs + kRng - 1) / kRng * kRng; }
__host__ __device__ inline bool run2_onebar(int64_t n_pairs) { return 4 * n_pairs <= (int64_t)kMaxRng * kRng; }

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__host__ __device__ inline size_t run_ws2_head() { return (sizeof(RunWs2) + 255) & ~(size_t)255; }

template <int M>
struct RunGeom {
    static constexpr int W = Order<M>::W;
    static constexpr int MW = M * W;
    static constexpr int U = MW / 4;                      // 16B units per matrix (M multiple of 4)
    static constexpr int STU = (U & 1) ? U : U + 1;       // odd stride: conflict-free per-thread LDS.128
    static constexpr int ROWS = kTileOff * STU * 16;      // parent rows, turned into the children in place
    static constexpr int SMEM = ROWS;
    static constexpr int NP = (M - 1) * (M - 2) / 2;      // pairs with column 0 skipped
};

// ------------------------------------------------------------ helpers
__device__ __forceinline__ void group_sync(int g) {
    asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(kR2Threads) : "memory");
}

__device__ __forceinline__ uint32_t ld_cg_u32(const uint32_t* p) { return __ldcg(p); }

// Block-wide: first bin b (in [0, bins)) where the inclusive prefix of h
// reaches k; also the count strictly below b.  h is read with ld.cg.
__device__ inline void kth_bin_cg(const uint32_t* h, int bins, uint64_t k, int* out_bin, uint64_t* out_below,
                           uint64_t* scratch) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int per = (bins + nt - 1) / nt;
    const int b0 = tid * per;
    uint64_t mine = 0;
    for (int b = b0; b < min(bins, b0 + per); ++b) mine += ld_cg_u32(h + b);
    uint64_t x = mine;
    const int lane = tid & 31, wid = tid >> 5;
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) scratch[wid] = x;
    __syncthreads();
    if (tid == 0) {
        uint64_t run = 0;
        for (int w = 0; w < nt / 32; ++w) {
            const uint64_t t = scratch[w];
            scratch[w] = run;
            run += t;
        }
    }
    __syncthreads();
    const uint64_t excl = scratch[wid] + x - mine;
    if (excl < k && excl + mine >= k) {
        uint64_t run = excl;
        for (int b = b0; b < min(bins, b0 + per); ++b) {
            const uint32_t hb = ld_cg_u32(h + b);
            if (run + hb >= k) {
                *out_bin = b;
                *out_below = run;
                break;
            }
            run += hb;
        }
    }
    __syncthreads();
}

// One warp: first bin b (in [0, bins)) where the inclusive prefix of h
// reaches k (1 <= k <= total), and the count strictly below b.  Bins are
// loaded 128 at a time (four independent loads per lane in flight) so a
// typical key window costs one L2 round trip.
__device__ inline void kth_bin_warp(const uint32_t* h, int bins, uint64_t k, int* out_bin, uint64_t* out_below) {
    const int lane = threadIdx.x & 31;
    uint64_t run = 0;
    for (int c0 = 0; c0 < bins; c0 += 128) {
        uint32_t v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int b = c0 + 32 * u + lane;
            v[u] = b < bins ? __ldcg(h + b) : 0u;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int b = c0 + 32 * u + lane;
            uint64_t x = v[u];
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            const bool hit = (run + x >= k) && (run + x - v[u] < k);
            const unsigned m = __ballot_sync(0xffffffffu, hit);
            if (m) {
                if (lane == __ffs(m) - 1) {
                    *out_bin = b;
                    *out_below = run + x - v[u];
                }
                return;
            }
            run += __shfl_sync(0xffffffffu, x, 31);
        }
    }
}

// Warp-aggregated histogram + key-range update for the next generation.
__device__ __forceinline__ void hist_add(RunWs2* ws, int slot, bool valid, uint32_t key) {
    const unsigned act = __ballot_sync(0xffffffffu, valid);
    if (!act) return;
    const unsigned peers = __match_any_sync(0xffffffffu, valid ? key : 0xffffffffu);
    if (valid && (__ffs(peers & act) - 1) == (int)(threadIdx.x & 31))
        atomicAdd(&ws->hist[slot][key], (uint32_t)__popc(peers & act));
    uint32_t mn = valid ? key : 0xffffffffu, mx = valid ? key : 0u;
    mn = __reduce_min_sync(0xffffffffu, mn);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&ws->kmin[slot], mn);
        atomicMax(&ws->kmax[slot], mx);
    }
}

// Per-CTA accumulation of the next generation's histogram (shared-memory
// window around the current minimum key, global atomics outside it), key
// range and best keys; flushed once per CTA per phase instead of one global
// atomic per warp on a handful of hot addresses.
constexpr int kWin = 1024;

struct LocalAcc {
    uint32_t* s_hist;   // [kWin]
    uint32_t wbase;     // key of s_hist[0]
    uint32_t kmin, kmax;
    unsigned long long best;   // min (F << 32 | slot) over this thread's parents + children
    unsigned long long pbest;  // same over parents only
};

__device__ __forceinline__ void local_hist_add(LocalAcc& L, RunWs2* ws, int slot, bool valid, uint32_t key) {
    if (valid) {
        L.kmin = min(L.kmin, key);
        L.kmax = max(L.kmax, key);
    }
    const uint32_t rel = key - L.wbase;
    const bool in_win = valid && rel < (uint32_t)kWin;
    const unsigned peers = __match_any_sync(0xffffffffu, valid ? key : 0xffffffffu);
    const unsigned act = __ballot_sync(0xffffffffu, valid);
    if (valid && (__ffs(peers & act) - 1) == (int)(threadIdx.x & 31)) {
        if (in_win) atomicAdd(&L.s_hist[rel], (uint32_t)__popc(peers & act));
        else atomicAdd(&ws->hist[slot][key], (uint32_t)__popc(peers & act));
    }
}

__device__ __forceinline__ void key_min_warp(unsigned long long* dst, unsigned long long k) {
    for (int o = 16; o; o >>= 1) k = min(k, __shfl_xor_sync(0xffffffffu, k, o));
    if ((threadIdx.x & 31) == 0 && k != ~0ull) atomicMin(dst, k);
}

// kSelItems consecutive fitness values (16-byte loads; i0 is a multiple of
// kSelItems, so aligned), zero past `hi`.
__device__ __forceinline__ void load_items(const int64_t* f, int64_t i0, int64_t hi, int64_t (&out)[kSelItems]) {
    if (i0 + kSelItems <= hi) {
#pragma unroll
        for (int u = 0; u < kSelItems / 2; ++u) {
            const longlong2 v = __ldcg(reinterpret_cast<const longlong2*>(f + i0) + u);
            out[2 * u] = v.x;
            out[2 * u + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int u = 0; u < kSelItems; ++u) out[u] = (i0 + u < hi) ? __ldcg(f + i0 + u) : 0;
    }
}

// Keyed bijection on [0, n): a six-round alternating Feistel network on
// Z_a x Z_b with a = ceil(sqrt n), b = ceil(n / a) (each round adds a
// Lemire-bounded hash of the other half modulo its own radix), plus cycle
// walking -- the domain a*b < n + b, so almost every point maps in one walk.
struct FeistelKey {
    uint32_t k[6];
    uint32_t n, a, b;
};

__device__ __forceinline__ FeistelKey make_feistel_key(const U4& r, uint32_t n) {
    FeistelKey f;
    f.k[0] = r.x;
    f.k[1] = r.y;
    f.k[2] = r.z;
    f.k[3] = r.w;
    f.k[4] = hash32(r.x ^ 0x68E31DA4u);
    f.k[5] = hash32(r.y ^ 0xB5297A4Du);
    f.n = n < 1 ? 1 : n;
    uint32_t a = (uint32_t)ceilf(sqrtf((float)f.n));
    while ((uint64_t)a * a < f.n) ++a;
    f.a = a;
    f.b = (f.n + a - 1) / a;
    return f;
}

__device__ __forceinline__ uint32_t feistel2(uint32_t x, const FeistelKey& f) {
    uint32_t L = x / f.b, R = x - (x / f.b) * f.b;
    do {
#pragma unroll
        for (int r = 0; r < 6; r += 2) {
            L += bounded(hash32(R ^ f.k[r]), f.a);
            L -= L >= f.a ? f.a : 0u;
            R += bounded(hash32(L ^ f.k[r + 1]), f.b);
            R -= R >= f.b ? f.b : 0u;
        }
    } while (L * f.b + R >= f.n);
    return L * f.b + R;
}

__device__ __forceinline__ uint32_t feistel2_inv(uint32_t y, const FeistelKey& f) {
    uint32_t L = y / f.b, R = y - (y / f.b) * f.b;
    do {
#pragma unroll
        for (int r = 4; r >= 0; r -= 2) {
            const uint32_t tr = bounded(hash32(L ^ f.k[r + 1]), f.b);
            R = R >= tr ? R - tr : R + f.b - tr;
            const uint32_t tl = bounded(hash32(R ^ f.k[r]), f.a);
            L = L >= tl ? L - tl : L + f.a - tl;
        }
    } while (L * f.b + R >= f.n);
    return L * f.b + R;
}

struct Run2Params {
    hga_run_args a;
    int gshift;  // granule shift of the selection keys
};

template <int M, int VM, int F, int B0, int... Ps>
__device__ __forceinline__ void pair_seq_at(const uint32_t (&c)[M * Order<M>::W], Sums& s,
                                            std::integer_sequence<int, Ps...>) {
    (pair_one<M, VM, pair_i(M, F, B0 + Ps), pair_j(M, F, B0 + Ps)>(c, s), ...);
}

// Team member K's quarter of the pair list (column 0 skipped).
template <int M, int VM, int K>
__device__ __forceinline__ void pair_part(const uint32_t (&c)[M * Order<M>::W], Sums& s) {
    constexpr int NP = RunGeom<M>::NP;
    constexpr int B0 = NP * K / kTeam, B1 = NP * (K + 1) / kTeam;
    pair_seq_at<M, VM, 1, B0>(c, s, std::make_integer_sequence<int, B1 - B0>{});
}

constexpr int kPlanStride = kR2MaxPlan + 4;  // 33 words: plan rows of 32 children hit 32 banks

struct TileShared {  // one per 128-thread tile group
    int16_t point[kR2Pairs];
    int32_t pidx[2 * kR2Pairs];  // old-population index of parent row 2q (A) / 2q+1 (B)
    uint16_t pkey[2 * kR2Pairs]; // its selection key (one-barrier lookup)
    int8_t plan[kTileOff][kPlanStride];
    uint32_t part[kTeam][4][kTileOff];  // child-minor: conflict-free
};

// Survivor lists: CTA b's lt survivors (F < tau) and eq candidates (F == tau)
// are compacted in index order at [b * chunk, ...); rank order is all lt
// survivors (CTA-major), then the first `quota` eq candidates.  Any fixed
// bijection works here because the Feistel permutation randomises the slots.
struct SelView {
    const uint32_t* lt_pre;  // [nb + 1] exclusive prefix, in shared memory (one-barrier: [nrng + 1] over key ranges)
    const uint32_t* eq_pre;
    int nb;                  // CTAs (two-barrier) or key ranges (one-barrier)
    int64_t chunk;
    const unsigned long long* lt_list;
    const unsigned long long* eq_list;
    uint32_t total_lt;
    const uint16_t* keys;    // one-barrier: selection keys of the old population
    uint32_t tau_key;
};

__device__ __forceinline__ int upper_bound_u32(const uint32_t* a, int n, uint32_t v) {
    int lo = 0, hi = n;  // first index with a[i] > v
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] <= v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ unsigned long long survivor_by_rank(const SelView& V, uint32_t r) {
    if (r < V.total_lt) {
        const int b = upper_bound_u32(V.lt_pre, V.nb + 1, r) - 1;
        return __ldcg(V.lt_list + (int64_t)b * V.chunk + (r - V.lt_pre[b]));
    }
    const uint32_t e = r - V.total_lt;
    const int b = upper_bound_u32(V.eq_pre, V.nb + 1, e) - 1;
    return __ldcg(V.eq_list + (int64_t)b * V.chunk + (e - V.eq_pre[b]));
}

// One 128-thread tile group runs its tiles (16 pairs -> 32 children each)
// as a two-stage pipeline: while tile i is crossed, mutated and evaluated,
// tile i+1's parents are already being gathered with cp.async into the other
// row buffer.  Parent slot s (p for A, N + p for B) holds the survivor of rank
// Feistel^-1(s); rows 2q / 2q+1 receive parents A / B of pair q, are copied to
// the new population's parent slots, and swapping the columns j >= point turns
// them into O1 / O2 in place (engine.py:257-277).  Mutation is column-parallel
// (engine.py:339-373); four warps each run a quarter of every child's pairs.
struct TileCtx {
    const hga_run_args* A;
    RunWs2* ws;
    const SelView* V;
    const FeistelKey* fkey;
    const uint32_t* pop_old;
    uint32_t* pop_new;
    int64_t* f_new;
    int64_t N;
    int nc, nr;
    uint64_t gen;
    int gp, gshift, g;
    unsigned long long* ts;  // HGA_RUN_TIMING stamps of this generation (CTA 0, group 0), else null
    uint16_t* keys_new;      // one-barrier: selection keys of the new population, else null
    int hslot;               // histogram slot of the new population
};

// 8 uint16 keys: (count < tk) | (count == tk) << 16
__device__ __forceinline__ uint32_t count8(const uint4& v, uint32_t tk) {
    const uint32_t t2 = tk | (tk << 16);
    const uint32_t lt = __popc(__vcmpltu2(v.x, t2)) + __popc(__vcmpltu2(v.y, t2)) + __popc(__vcmpltu2(v.z, t2)) +
                        __popc(__vcmpltu2(v.w, t2));
    const uint32_t eq = __popc(__vcmpeq2(v.x, t2)) + __popc(__vcmpeq2(v.y, t2)) + __popc(__vcmpeq2(v.z, t2)) +
                        __popc(__vcmpeq2(v.w, t2));
    return (lt >> 4) | ((eq >> 4) << 16);
}

// One-barrier select, warp 0 of a tile group: the parent of each of the
// `noff` parent rows is the survivor of rank Feistel^-1(slot).  Lane o finds
// the key range holding that rank (binary search of the range prefixes in
// shared memory); then 8-lane teams resolve four lookups per step from the
// ranges' 64 keys (one 16-byte load per lane, all eight loads in flight).
__device__ __forceinline__ void select_lookup(const TileCtx& C, TileShared& S, int noff, int64_t slot, bool act) {
    const SelView& V = *C.V;
    const int o = threadIdx.x & 31, h = o >> 3, sub = o & 7;
    int rb = 0;
    uint32_t rk = 0;
    bool req = false;
    if (act) {
        const uint32_t r = feistel2_inv((uint32_t)slot, *C.fkey);
        if (r < V.total_lt) {
            rb = upper_bound_u32(V.lt_pre, V.nb + 1, r) - 1;
            rk = r - V.lt_pre[rb];
        } else {
            const uint32_t e = r - V.total_lt;
            req = true;
            rb = upper_bound_u32(V.eq_pre, V.nb + 1, e) - 1;
            rk = e - V.eq_pre[rb];
        }
    }
    uint4 kv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int j = 4 * i + h;
        const int bj = __shfl_sync(0xffffffffu, rb, j);
        kv[i] = j < noff ? __ldcg(reinterpret_cast<const uint4*>(V.keys + (int64_t)bj * kRng) + sub)
                         : make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
    }
    const uint32_t t2 = V.tau_key | (V.tau_key << 16);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int j = 4 * i + h;
        const uint32_t kj = __shfl_sync(0xffffffffu, rk, j);
        const bool eqj = __shfl_sync(0xffffffffu, req, j);
        const int bj = __shfl_sync(0xffffffffu, rb, j);
        const uint32_t w[4] = {kv[i].x, kv[i].y, kv[i].z, kv[i].w};
        uint32_t mask = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t c = eqj ? __vcmpeq2(w[u], t2) : __vcmpltu2(w[u], t2);
            mask |= ((c & 1u) << (2 * u)) | (((c >> 16) & 1u) << (2 * u + 1));
        }
        const uint32_t cnt = __popc(mask);
        uint32_t incl = cnt;
#pragma unroll
        for (int d = 1; d < 8; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d, 8);
            if (sub >= d) incl += y;
        }
        const uint32_t excl = incl - cnt;
        if (j < noff && kj >= excl && kj < incl) {
            uint32_t mm = mask;
            for (uint32_t z = kj - excl; z > 0; --z) mm &= mm - 1u;
            const int u = __ffs(mm) - 1;
            S.pidx[j] = bj * kRng + 8 * sub + u;
            S.pkey[j] = (uint16_t)(w[u >> 1] >> (16 * (u & 1)));
        }
    }
    __syncwarp();
}

__device__ __forceinline__ void tile_stamp(const TileCtx& C, int slot) {
    if (C.ts != nullptr && (threadIdx.x & (kR2Threads - 1)) == 0) C.ts[slot] = gtimer();
}

// Step a: parents by rank (warp 0), crossover points (warp 3), mutation plans (warps 1-3).
template <int M, bool ONE>
__device__ __forceinline__ void tile_prepare(const TileCtx& C, TileShared& S, int64_t p0, int cnt, LocalAcc& L) {
    const int t = threadIdx.x & (kR2Threads - 1), k = t >> 5, o = t & 31;
    const int noff = 2 * cnt;
    const int per_off = C.nc + 2 * C.nr;
    const int nblk = (per_off + 3) >> 2;
    const int64_t N = C.N;
    if (k == 0) {
        const bool act = o < noff;
        const int64_t slot = (int64_t)(o & 1) * N + p0 + (o >> 1);
        int64_t f = 0;
        if constexpr (ONE) {
            select_lookup(C, S, noff, slot, act);
            if (act) {
                const uint16_t pk = S.pkey[o];
                f = (int64_t)pk << C.gshift;
                C.keys_new[slot] = pk;
            }
        } else if (act) {
            const unsigned long long kv = survivor_by_rank(*C.V, feistel2_inv((uint32_t)slot, *C.fkey));
            S.pidx[o] = (int32_t)(kv & 0xffffffffu);
            f = (int64_t)(kv >> 32);
        }
        if (act) {
            C.f_new[slot] = f;
            const unsigned long long key = ((unsigned long long)f << 32) | (unsigned long long)slot;
            L.best = min(L.best, key);
            L.pbest = min(L.pbest, key);
        }
        local_hist_add(L, C.ws, C.hslot, act, (uint32_t)(f >> C.gshift));
    } else {
        if (k == kTeam - 1 && o < cnt) {
            const int64_t p = p0 + o;
            const U4 r = draw4(C.A->seed, (uint32_t)p, (uint32_t)(p >> 32), C.gen, (uint32_t)kPCrossover);
            S.point[o] = (int16_t)(1 + bounded(r.x, (uint32_t)(M - 1)));
        }
        for (int x = t - 32; x < noff * nblk; x += kR2Threads - 32) {
            const int ol = x / nblk, blk = x - (x / nblk) * nblk;
            const int q = ol >> 1;
            int64_t prow = (ol & 1) ? N + p0 + q : p0 + q;  // plan row as engine.py: O1 -> p, O2 -> N + p
            if (C.A->strategy == HGA_MUT_SHARED) prow = 0;
            const U4 r = draw4(C.A->seed, (uint32_t)prow, (uint32_t)blk | ((uint32_t)(prow >> 32) << 16), C.gen,
                               (uint32_t)kPMutCol);
#pragma unroll
            for (int e4 = 0; e4 < 4; ++e4) {
                const int e = blk * 4 + e4;
                if (e < per_off)
                    S.plan[ol][e] = (int8_t)(e < C.nc ? 1 + bounded(pick(r, e4), (uint32_t)(M - 1))
                                                      : bounded(pick(r, e4), (uint32_t)M));
            }
        }
    }
}

// Step b: async gather of the 2 cnt parents into rows (one commit group).
template <int M>
__device__ __forceinline__ void tile_gather(const TileCtx& C, const TileShared& S, uint4* rows, int cnt) {
    using G = RunGeom<M>;
    const int t = threadIdx.x & (kR2Threads - 1);
    for (int x = t; x < 2 * cnt * G::U; x += kR2Threads) {
        const int pi = x / G::U, u = x - (x / G::U) * G::U;
        cp_async16(rows + pi * G::STU + u, reinterpret_cast<const uint4*>(C.pop_old + (int64_t)S.pidx[pi] * G::MW) + u);
    }
}

// Steps b'-g on landed rows; ends with a group barrier.
template <int M, int VM>
__device__ __forceinline__ void tile_compute(const TileCtx& C, TileShared& S, uint4* rows, int64_t p0, int cnt,
                                             LocalAcc& L) {
    using G = RunGeom<M>;
    constexpr int W = G::W;
    const int64_t N = C.N;
    const int t = threadIdx.x & (kR2Threads - 1), k = t >> 5, o = t & 31;
    const int noff = 2 * cnt;
    const int nc = C.nc, nr = C.nr;
    const int g = C.g;
    // b'. parents to the new population's parent slots (block A, then block B)
    for (int x = t; x < noff * G::U; x += kR2Threads) {
        const int b = x / (cnt * G::U);
        const int r = x - b * cnt * G::U;
        const int q = r / G::U, u = r - q * G::U;
        reinterpret_cast<uint4*>(C.pop_new + ((int64_t)b * N + p0 + q) * G::MW)[u] = rows[(2 * q + b) * G::STU + u];
    }
    group_sync(g);
    tile_stamp(C, 14);
    // c. column-block crossover in place
    for (int x = t; x < cnt * M; x += kR2Threads) {
        const int q = x / M, j = x - q * M;
        if (j >= S.point[q]) {
            uint32_t* ra = reinterpret_cast<uint32_t*>(rows + (2 * q) * G::STU) + j * W;
            uint32_t* rb = reinterpret_cast<uint32_t*>(rows + (2 * q + 1) * G::STU) + j * W;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                const uint32_t tmp = ra[w];
                ra[w] = rb[w];
                rb[w] = tmp;
            }
        }
    }
    group_sync(g);
    tile_stamp(C, 15);
    // d. mutation: thread (k, o) handles plan entries jc = k, k + 4, ...; an
    //    entry whose column already appeared earlier is skipped, and the first
    //    occurrence applies the column's row-pair sequence once per occurrence
    //    (plan order per column == the reference's sequential order)
    if (o < noff) {
        uint32_t* row = reinterpret_cast<uint32_t*>(rows + o * G::STU);
        const int8_t* pl = S.plan[o];
        for (int jc = k; jc < nc; jc += kTeam) {
            const int col = pl[jc];
            bool first = true;
            for (int j2 = 0; j2 < jc; ++j2) first &= pl[j2] != col;
            if (!first) continue;
            int reps = 1;
            for (int j2 = jc + 1; j2 < nc; ++j2) reps += pl[j2] == col;
            // the column's words live in registers for the whole row-pair sequence:
            // one shared-memory load and store per word instead of a
            // read-modify-write per swap
            uint32_t* cw = row + col * W;
            uint32_t w0 = cw[0], w1 = W > 1 ? cw[W > 1 ? 1 : 0] : 0u;
            for (int rep = 0; rep < reps; ++rep) {
                for (int ir = 0; ir < nr; ++ir) {
                    const int ra = pl[nc + ir], rb = pl[nc + nr + ir];
                    const uint32_t va = (W > 1 && (ra >> 5)) ? w1 : w0, vb = (W > 1 && (rb >> 5)) ? w1 : w0;
                    const uint32_t flip = ((va >> (ra & 31)) ^ (vb >> (rb & 31))) & 1u;  // rows differ: swap
                    const uint32_t ma = flip << (ra & 31), mb = flip << (rb & 31);
                    if (W > 1 && (ra >> 5)) w1 ^= ma;
                    else w0 ^= ma;
                    if (W > 1 && (rb >> 5)) w1 ^= mb;
                    else w0 ^= mb;
                }
            }
            cw[0] = w0;
            if constexpr (W > 1) cw[1] = w1;
        }
    }
    group_sync(g);
    tile_stamp(C, 16);
    // e. pair chain, a quarter per warp
    if (o < noff) {
        uint32_t c[G::MW];
#pragma unroll
        for (int u = 0; u < G::U; ++u) {
            const uint4 v = rows[o * G::STU + u];
            c[4 * u] = v.x;
            c[4 * u + 1] = v.y;
            c[4 * u + 2] = v.z;
            c[4 * u + 3] = v.w;
        }
        Sums s{0, 0, 0, 0};
        switch (k) {
            case 0: pair_part<M, VM, 0>(c, s); break;
            case 1: pair_part<M, VM, 1>(c, s); break;
            case 2: pair_part<M, VM, 2>(c, s); break;
            default: pair_part<M, VM, 3>(c, s); break;
        }
        S.part[k][0][o] = s.s1;
        S.part[k][1][o] = s.s2;
        S.part[k][2][o] = s.sp;
        S.part[k][3][o] = s.spp;
    }
    group_sync(g);
    tile_stamp(C, 17);
    // f. warp 0: children's fitness, best key, next histogram
    if (k == 0) {
        const bool active = o < noff;
        int64_t value = 0;
        if (active) {
            Sums s{0, 0, 0, 0};
#pragma unroll
            for (int kk = 0; kk < kTeam; ++kk) {
                s.s1 += S.part[kk][0][o];
                s.s2 += S.part[kk][1][o];
                s.sp += S.part[kk][2][o];
                s.spp += S.part[kk][3][o];
            }
            value = variant_value<M, VM>(s, G::NP);
            const int64_t slot = 2 * N + (int64_t)(o & 1) * N + p0 + (o >> 1);
            C.f_new[slot] = value;
            if (C.keys_new != nullptr) C.keys_new[slot] = (uint16_t)(value >> C.gshift);
            L.best = min(L.best, ((unsigned long long)value << 32) | (unsigned long long)slot);
        }
        local_hist_add(L, C.ws, C.hslot, active, (uint32_t)(value >> C.gshift));
    }
    tile_stamp(C, 18);
    // g. coalesced store of the children (O1 block, then O2 block)
    for (int x = t; x < noff * G::U; x += kR2Threads) {
        const int b = x / (cnt * G::U);
        const int r = x - b * cnt * G::U;
        const int q = r / G::U, u = r - q * G::U;
        reinterpret_cast<uint4*>(C.pop_new + (2 * N + (int64_t)b * N + p0 + q) * G::MW)[u] = rows[(2 * q + b) * G::STU + u];
    }
    group_sync(g);
    tile_stamp(C, 19);
}

template <int M, int VM, bool ONE>
__device__ __forceinline__ void group_tiles(const TileCtx& C, int64_t first, int64_t stride, int64_t ntiles,
                                            uint4* rows0, uint4* rows1, TileShared* S0, TileShared* S1,
                                            LocalAcc& L) {
    if (first >= ntiles) return;
    const int64_t N = C.N;
    uint4* rows[2] = {rows0, rows1};
    TileShared* S[2] = {S0, S1};
    auto cnt_of = [&](int64_t tile) { return (int)min((int64_t)kR2Pairs, N - tile * kR2Pairs); };
    tile_prepare<M, ONE>(C, *S[0], first * kR2Pairs, cnt_of(first), L);
    group_sync(C.g);
    tile_stamp(C, 12);
    tile_gather<M>(C, *S[0], rows[0], cnt_of(first));
    cp_async_commit();
    int cur = 0;
    TileCtx Cs = C;
    for (int64_t tile = first; tile < ntiles; tile += stride) {
        const int64_t nxt = tile + stride;
        if (nxt < ntiles) tile_prepare<M, ONE>(C, *S[cur ^ 1], nxt * kR2Pairs, cnt_of(nxt), L);
        group_sync(C.g);
        if (nxt < ntiles) tile_gather<M>(C, *S[cur ^ 1], rows[cur ^ 1], cnt_of(nxt));
        cp_async_commit();
        cp_async_wait<1>();
        group_sync(C.g);
        if (tile == first) tile_stamp(C, 13);
        tile_compute<M, VM>(Cs, *S[cur], rows[cur], tile * kR2Pairs, cnt_of(tile), L);
        Cs.ts = nullptr;  // stamps for the first tile only
        cur ^= 1;
    }
    cp_async_wait<0>();
}

// ---------------------------------------------------------------- throughput tiles
// Orders 24..40 (the default there): one thread per child.  Every warp runs the whole straight-line pair chain of its own 32
// children, so all warps of the SM execute the same instruction stream (the
// team-of-4 split makes four warps run four different 10-20 KB code regions,
// which misses the instruction cache at these orders); a tile is 64 pairs =
// 128 children = the 128 threads of a group.  Same survivors, crossover
// points, plans and operator order as the team tiles: identical populations.
constexpr int kTPPairs = 64;
constexpr int kTPOff = 2 * kTPPairs;
constexpr int kTPPlanStride = 68;  // nc + 2 nr <= 64 (else the team tiles are used)

struct TileSharedTP {
    int16_t point[kTPPairs];
    int32_t pidx[kTPOff];
};

template <int M>
__device__ __forceinline__ void tp_prepare(const TileCtx& C, TileSharedTP& S, int64_t p0, int cnt, LocalAcc& L) {
    const int t = threadIdx.x & (kR2Threads - 1);
    const int64_t N = C.N;
    const bool act = t < 2 * cnt;
    const int64_t slot = (int64_t)(t & 1) * N + p0 + (t >> 1);
    int64_t f = 0;
    if (act) {
        const unsigned long long kv = survivor_by_rank(*C.V, feistel2_inv((uint32_t)slot, *C.fkey));
        S.pidx[t] = (int32_t)(kv & 0xffffffffu);
        f = (int64_t)(kv >> 32);
        C.f_new[slot] = f;
        const unsigned long long key = ((unsigned long long)f << 32) | (unsigned long long)slot;
        L.best = min(L.best, key);
        L.pbest = min(L.pbest, key);
    }
    local_hist_add(L, C.ws, C.hslot, act, (uint32_t)(f >> C.gshift));
    if (t < cnt) {
        const int64_t p = p0 + t;
        const U4 r = draw4(C.A->seed, (uint32_t)p, (uint32_t)(p >> 32), C.gen, (uint32_t)kPCrossover);
        S.point[t] = (int16_t)(1 + bounded(r.x, (uint32_t)(M - 1)));
    }
}

template <int M>
__device__ __forceinline__ void tp_gather(const TileCtx& C, const TileSharedTP& S, uint4* rows, int cnt) {
    using G = RunGeom<M>;
    const int t = threadIdx.x & (kR2Threads - 1);
    for (int x = t; x < 2 * cnt * G::U; x += kR2Threads) {
        const int pi = x / G::U, u = x - (x / G::U) * G::U;
        cp_async16(rows + pi * G::STU + u, reinterpret_cast<const uint4*>(C.pop_old + (int64_t)S.pidx[pi] * G::MW) + u);
    }
}

template <int M, int VM>
__device__ __forceinline__ void tp_compute(const TileCtx& C, const TileSharedTP& S, int8_t* plan, uint4* rows,
                                           int64_t p0, int cnt, LocalAcc& L) {
    using G = RunGeom<M>;
    constexpr int W = G::W;
    const int64_t N = C.N;
    const int t = threadIdx.x & (kR2Threads - 1);
    const int noff = 2 * cnt;
    const int nc = C.nc, nr = C.nr;
    const int g = C.g;
    // b'. parents to the new population's parent slots (block A, then block B)
    for (int x = t; x < noff * G::U; x += kR2Threads) {
        const int b = x / (cnt * G::U);
        const int r = x - b * cnt * G::U;
        const int q = r / G::U, u = r - q * G::U;
        reinterpret_cast<uint4*>(C.pop_new + ((int64_t)b * N + p0 + q) * G::MW)[u] = rows[(2 * q + b) * G::STU + u];
    }
    group_sync(g);
    // c. column-block crossover in place
    for (int x = t; x < cnt * M; x += kR2Threads) {
        const int q = x / M, j = x - q * M;
        if (j >= S.point[q]) {
            uint32_t* ra = reinterpret_cast<uint32_t*>(rows + (2 * q) * G::STU) + j * W;
            uint32_t* rb = reinterpret_cast<uint32_t*>(rows + (2 * q + 1) * G::STU) + j * W;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                const uint32_t tmp = ra[w];
                ra[w] = rb[w];
                rb[w] = tmp;
            }
        }
    }
    group_sync(g);
    // d. this thread's child: its Philox plan, then the mutation in plan order
    //    (engine.py:361-373: columns outer, row pairs inner), then e. its pair chain
    const bool active = t < noff;
    int64_t value = 0;
    const int64_t slot = 2 * N + (int64_t)(t & 1) * N + p0 + (t >> 1);
    if (active) {
        const int per_off = nc + 2 * nr;
        const int q = t >> 1;
        int64_t prow = (t & 1) ? N + p0 + q : p0 + q;  // plan row as engine.py: O1 -> p, O2 -> N + p
        if (C.A->strategy == HGA_MUT_SHARED) prow = 0;
        int8_t* pl = plan + t * kTPPlanStride;
        for (int blk = 0; blk * 4 < per_off; ++blk) {
            const U4 r = draw4(C.A->seed, (uint32_t)prow, (uint32_t)blk | ((uint32_t)(prow >> 32) << 16), C.gen,
                               (uint32_t)kPMutCol);
#pragma unroll
            for (int e4 = 0; e4 < 4; ++e4) {
                const int e = blk * 4 + e4;
                if (e < per_off)
                    pl[e] = (int8_t)(e < nc ? 1 + bounded(pick(r, e4), (uint32_t)(M - 1)) : bounded(pick(r, e4), (uint32_t)M));
            }
        }
        uint32_t* row = reinterpret_cast<uint32_t*>(rows + t * G::STU);
        for (int jc = 0; jc < nc; ++jc) {
            uint32_t* cw = row + pl[jc] * W;
            uint32_t w0 = cw[0], w1 = W > 1 ? cw[W > 1 ? 1 : 0] : 0u;
            for (int ir = 0; ir < nr; ++ir) {
                const int ra = pl[nc + ir], rb = pl[nc + nr + ir];
                const uint32_t va = (W > 1 && (ra >> 5)) ? w1 : w0, vb = (W > 1 && (rb >> 5)) ? w1 : w0;
                const uint32_t flip = ((va >> (ra & 31)) ^ (vb >> (rb & 31))) & 1u;  // rows differ: swap
                const uint32_t ma = flip << (ra & 31), mb = flip << (rb & 31);
                if (W > 1 && (ra >> 5)) w1 ^= ma;
                else w0 ^= ma;
                if (W > 1 && (rb >> 5)) w1 ^= mb;
                else w0 ^= mb;
            }
            cw[0] = w0;
            if constexpr (W > 1) cw[1] = w1;
        }
        uint32_t c[G::MW];
#pragma unroll
        for (int u = 0; u < G::U; ++u) {
            const uint4 v = rows[t * G::STU + u];
            c[4 * u] = v.x;
            c[4 * u + 1] = v.y;
            c[4 * u + 2] = v.z;
            c[4 * u + 3] = v.w;
        }
        Sums s{0, 0, 0, 0};
        pair_sums<M, VM, 1>(c, s);
        value = variant_value<M, VM>(s, G::NP);
        C.f_new[slot] = value;
        L.best = min(L.best, ((unsigned long long)value << 32) | (unsigned long long)slot);
    }
    local_hist_add(L, C.ws, C.hslot, active, (uint32_t)(value >> C.gshift));
    group_sync(g);
    // g. coalesced store of the children (O1 block, then O2 block)
    for (int x = t; x < noff * G::U; x += kR2Threads) {
        const int b = x / (cnt * G::U);
        const int r = x - b * cnt * G::U;
        const int q = r / G::U, u = r - q * G::U;
        reinterpret_cast<uint4*>(C.pop_new + (2 * N + (int64_t)b * N + p0 + q) * G::MW)[u] = rows[(2 * q + b) * G::STU + u];
    }
    group_sync(g);
}

template <int M, int VM>
__device__ __forceinline__ void group_tiles_tp(const TileCtx& C, int64_t first, int64_t stride, int64_t ntiles,
                                               uint4* rows0, uint4* rows1, TileSharedTP* S0, TileSharedTP* S1,
                                               int8_t* plan, LocalAcc& L) {
    if (first >= ntiles) return;
    const int64_t N = C.N;
    uint4* rows[2] = {rows0, rows1};
    TileSharedTP* S[2] = {S0, S1};
    auto cnt_of = [&](int64_t tile) { return (int)min((int64_t)kTPPairs, N - tile * kTPPairs); };
    tp_prepare<M>(C, *S[0], first * kTPPairs, cnt_of(first), L);
    group_sync(C.g);
    tp_gather<M>(C, *S[0], rows[0], cnt_of(first));
    cp_async_commit();
    int cur = 0;
    for (int64_t tile = first; tile < ntiles; tile += stride) {
        const int64_t nxt = tile + stride;
        if (nxt < ntiles) tp_prepare<M>(C, *S[cur ^ 1], nxt * kTPPairs, cnt_of(nxt), L);
        group_sync(C.g);
        if (nxt < ntiles) tp_gather<M>(C, *S[cur ^ 1], rows[cur ^ 1], cnt_of(nxt));
        cp_async_commit();
        cp_async_wait<1>();
        group_sync(C.g);
        tp_compute<M, VM>(C, *S[cur], plan, rows[cur], tile * kTPPairs, cnt_of(tile), L);
        cur ^= 1;
    }
    cp_async_wait<0>();
}

// dynamic shared memory of one tile group
template <int M, bool TP>
__host__ __device__ constexpr size_t run_rows_bytes() {
    return (size_t)(TP ? kTPOff : kTileOff) * RunGeom<M>::STU * 16;
}
template <int M, bool TP>
__host__ __device__ constexpr size_t run_group_bytes() {
    return TP ? 2 * run_rows_bytes<M, TP>() + 2 * ((sizeof(TileSharedTP) + 15) & ~(size_t)15) +
                    (size_t)kTPOff * kTPPlanStride
              : 2 * run_rows_bytes<M, TP>() + 2 * ((sizeof(TileShared) + 15) & ~(size_t)15);
}

constexpr int kMaxNb = 512;  // prefix scan: one pass of <= 16 warps

// Block-wide exclusive prefix of packed per-range counts (lt | eq << 16) into
// lt_pre / eq_pre[0..n]; entry n holds the totals.  Ends without a barrier.
__device__ inline void scan_ranges(const uint32_t* cnt, int n, uint32_t* lt_pre, uint32_t* eq_pre, uint64_t* sscr) {
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
    const int per = (n + nt - 1) / nt;
    const int r0 = min(n, tid * per), r1 = min(n, r0 + per);
    uint64_t mine = 0;
    for (int r = r0; r < r1; ++r) {
        const uint32_t c = cnt[r];
        mine += ((uint64_t)(c & 0xffffu) << 32) | (c >> 16);
    }
    uint64_t x = mine;
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sscr[wid] = x;
    __syncthreads();
    uint64_t run = x - mine, tot = 0;
    for (int w = 0; w < nw; ++w) {
        const uint64_t t = sscr[w];
        if (w < wid) run += t;
        tot += t;
    }
    for (int r = r0; r < r1; ++r) {
        lt_pre[r] = (uint32_t)(run >> 32);
        eq_pre[r] = (uint32_t)run;
        const uint32_t c = cnt[r];
        run += ((uint64_t)(c & 0xffffu) << 32) | (c >> 16);
    }
    if (tid == 0) {
        lt_pre[n] = (uint32_t)(tot >> 32);
        eq_pre[n] = (uint32_t)tot;
    }
}

// ONE = one grid barrier per generation (HGA_RUN_ONE_BARRIER, 4N <= kMaxRng * kRng): the tiles
// also store each new matrix's 16-bit selection key; after the barrier every
// CTA reads ALL keys (2 bytes per matrix, L2 resident), so every CTA knows
// the per-range survivor counts of the whole population and the survivor
// lists never need to be materialised (and no second barrier is needed to
// publish them).  Per-generation slots rotate mod 3 so that the histogram /
// key range / best keys being read, being accumulated and being retired are
// always different slots.  Both variants select the same survivors with the
// same ranks, so they produce identical runs.  Measured: ONE is slower at
// order 20 (22.8 vs 17.2 us/generation: reading all keys and the 8-lane
// lookups cost more than the second barrier saves), so it is opt-in.
template <int M, int VM, int GROUPS, bool ONE, bool TP>
__global__ void __launch_bounds__(kR2Threads* GROUPS, 1) k_run_v3(Run2Params P) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint64_t sscr[32];
    __shared__ int s_bin;
    __shared__ uint64_t s_below;
    __shared__ uint32_t s_hist[kWin];
    __shared__ uint32_t s_kmin, s_kmax;
    __shared__ unsigned long long s_best, s_pbest;
    __shared__ uint32_t s_ltpre[kMaxRng + 1], s_eqpre[kMaxRng + 1];
    __shared__ uint32_t s_cnt[ONE ? kMaxRng : 1];

    using G = RunGeom<M>;
    const hga_run_args& A = P.a;
    RunWs2* ws = reinterpret_cast<RunWs2*>(A.ws);
    unsigned long long* lt_list = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(A.ws) + run_ws2_head());
    const int64_t N = A.n_pairs, half = 2 * N, total = 4 * N;
    unsigned long long* eq_list = lt_list + total;
    uint16_t* keys_base = reinterpret_cast<uint16_t*>(eq_list + total);
    const int64_t kstride = run2_key_stride(N);
    const int nrng = (int)(kstride / kRng);
    const int nb = gridDim.x, bid = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
    const int g = tid / kR2Threads;
    const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
    const int64_t chunk = (((total + nb - 1) / nb) + kSelItems - 1) / kSelItems * kSelItems;
    const int64_t lo = min(total, (int64_t)bid * chunk), hi = min(total, lo + chunk);
    const int nc = A.strategy == HGA_MUT_MULTI ? A.nc : 1;
    const int nr = A.strategy == HGA_MUT_MULTI ? A.nr : 1;
    const int gshift = P.gshift;
    const int64_t ntiles = TP ? (N + kTPPairs - 1) / kTPPairs : (N + kR2Pairs - 1) / kR2Pairs;
    // warps taking part in the select scans (the rest only meet the barriers)
    const int pw_sel = (int)min((int64_t)nw, (chunk / kSelItems + 31) / 32);
    const int pw_pre = (nb + 31) / 32;  // nb <= kMaxNb = 32 * 32
    // dynamic shared memory: per group, two row buffers and two tile records
    constexpr size_t kRowsBytes = run_rows_bytes<M, TP>();
    constexpr size_t kGroupBytes = run_group_bytes<M, TP>();
    unsigned char* gbase = smem + (size_t)g * kGroupBytes;
    uint4* rows0 = reinterpret_cast<uint4*>(gbase);
    uint4* rows1 = reinterpret_cast<uint4*>(gbase + kRowsBytes);
    TileShared* S0 = reinterpret_cast<TileShared*>(gbase + 2 * kRowsBytes);
    TileShared* S1 = reinterpret_cast<TileShared*>(gbase + 2 * kRowsBytes + ((sizeof(TileShared) + 15) & ~(size_t)15));
    constexpr size_t kTPS = (sizeof(TileSharedTP) + 15) & ~(size_t)15;
    TileSharedTP* T0 = reinterpret_cast<TileSharedTP*>(gbase + 2 * kRowsBytes);
    TileSharedTP* T1 = reinterpret_cast<TileSharedTP*>(gbase + 2 * kRowsBytes + kTPS);
    int8_t* tplan = reinterpret_cast<int8_t*>(gbase + 2 * kRowsBytes + 2 * kTPS);

    if ((A.flags & HGA_RUN_TIMING) && bid == 0 && tid == 0) ws->tstamp[63][0] = gtimer();  // kernel entry
    if ((A.flags & kRunHostCheck) && (__ldcg(&ws->host_flag) & (HGA_FLAG_NOT_SIGN | HGA_FLAG_NOT_GA)))
        return;  // uniform over the grid: no barrier has been entered
    int64_t iter = A.state[0], best = A.state[1], last_restart = A.state[2];
    int parity = (int)A.state[3];
    if (A.flags & (kRunPrefetchPop | kRunPrefetchFit)) {
        // Cold launches (one generation per launch, L2 flushed by whatever ran before):
        // bulk-prefetch the current population and / or its fitness + the select
        // histogram into L2 at once, spread over all CTAs (experiment flags).
        const int64_t pieces[3] = {(A.flags & kRunPrefetchPop) ? total * (int64_t)G::MW * 4 : 0,
                                   (A.flags & kRunPrefetchFit) ? total * 8 : 0,
                                   (A.flags & kRunPrefetchFit) ? (int64_t)kR2Bins * 4 : 0};
        const char* bases[3] = {reinterpret_cast<const char*>(A.pop[parity]),
                                reinterpret_cast<const char*>(A.fit[parity]),
                                reinterpret_cast<const char*>(&ws->hist[ONE ? (int)((iter + 1) % 3) : (int)((iter + 1) & 1)][0])};
        constexpr int64_t kPiece = 4096;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const int64_t np = (pieces[r] + kPiece - 1) / kPiece;
            for (int64_t pc = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pc < np; pc += (int64_t)gridDim.x * blockDim.x) {
                const int64_t off = pc * kPiece;
                const uint32_t len = (uint32_t)min(kPiece, pieces[r] - off) & ~15u;
                if (len)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(bases[r] + off), "r"(len) : "memory");
            }
        }
    }
    int64_t run = A.state[6], last_val = A.state[7];
    const bool force = (A.flags & HGA_RUN_FORCE) != 0;
    bool stop = !force && A.state[5] != 0;
    const bool timing = (A.flags & HGA_RUN_TIMING) != 0 && bid == 0 && tid == 0;
    const bool timing_blk = (A.flags & HGA_RUN_TIMING) != 0 && bid == 0;
    uint32_t next_kmin = 0, next_kmax = 0;
    bool have_krange = false;
    int64_t fpre[kSelItems];  // first batch of the select scan's fitness values, prefetched after barrier 2
    bool have_fpre = false;

    for (int64_t gi = 0; gi < A.gens_this_call && !stop; ++gi) {
        const int64_t gen = iter + 1;
        const int gp = (int)(gen & 1);  // histogram / key slot of the population entering `gen`
        const int s0 = (int)(gen % 3), s1 = (int)((gen + 1) % 3), s2 = (int)((gen + 2) % 3);
        const int rslot = ONE ? s0 : gp;        // select histogram of the population entering gen
        const int hslot = ONE ? s1 : (gp ^ 1);  // histogram / key range of the new population
        const int bslot = ONE ? s1 : gp;        // best / parent-best keys of the new population
        const uint16_t* kold = keys_base + (int64_t)parity * kstride;
        const uint32_t* pop_old = A.pop[parity];
        uint32_t* pop_new = A.pop[parity ^ 1];
        const int64_t* f_old = A.fit[parity];
        int64_t* f_new = A.fit[parity ^ 1];
        if (timing && gi < 64) {
            ws->tstamp[gi][0] = gtimer();
            ws->tstamp[gi][10] = clock64();
        }

        uint32_t kmin = 0, kmax = 0, tau_key = 0;
        if constexpr (ONE) {
            // ---- one-barrier select: threshold, per-range counts of the whole population
            const int team = wid * 4 + (lane >> 3), sub = lane & 7, nteam = nw * 4;
            uint4 kb[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int r = team + nteam * i;
                kb[i] = r < nrng ? __ldcg(reinterpret_cast<const uint4*>(kold + (int64_t)r * kRng) + sub)
                                 : make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
            }
            if (!have_krange) {
                next_kmin = __ldcg(&ws->kmin[rslot]);
                next_kmax = __ldcg(&ws->kmax[rslot]);
            }
            kmin = next_kmin;
            kmax = next_kmax;
            uint32_t zmin = 1u, zmax = 0u;  // CTA 0 retires slot s2 (last read before the previous barrier)
            if (bid == 0) {
                zmin = __ldcg(&ws->kmin[s2]);
                zmax = __ldcg(&ws->kmax[s2]);
            }
            if (wid == 0) kth_bin_warp(&ws->hist[rslot][kmin], (int)(kmax - kmin + 1), (uint64_t)half, &s_bin, &s_below);
            __syncthreads();
            if (timing && gi < 64) ws->tstamp[gi][3] = gtimer();
            tau_key = kmin + (uint32_t)s_bin;
            if (bid == 0 && zmin <= zmax)
                for (uint32_t b = zmin + tid; b <= zmax; b += nt) ws->hist[s2][b] = 0;
            for (int r0 = 0; r0 < nrng; r0 += nteam * 8) {
                if (r0 > 0) {
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int r = r0 + team + nteam * i;
                        kb[i] = r < nrng ? __ldcg(reinterpret_cast<const uint4*>(kold + (int64_t)r * kRng) + sub)
                                         : make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
                    }
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    uint32_t c = count8(kb[i], tau_key);
                    c += __shfl_xor_sync(0xffffffffu, c, 4);
                    c += __shfl_xor_sync(0xffffffffu, c, 2);
                    c += __shfl_xor_sync(0xffffffffu, c, 1);
                    const int r = r0 + team + nteam * i;
                    if (sub == 0 && r < nrng) s_cnt[r] = c;
                }
            }
            __syncthreads();
            scan_ranges(s_cnt, nrng, s_ltpre, s_eqpre, sscr);
            __syncthreads();
            if (bid == 0 && tid == 0) {
                ws->kmin[s2] = 0xffffffffu;
                ws->kmax[s2] = 0u;
                ws->best_key[s2] = ~0ull;
                ws->par_key[s2] = ~0ull;
            }
            if (timing && gi < 64) ws->tstamp[gi][2] = ws->tstamp[gi][1] = gtimer();
        } else {
            // ---- B: threshold, tie quota, local survivor lists
            // first batch of fitness values: independent of tau, so load it under the histogram scan
            if (!have_fpre && wid < pw_sel) load_items(f_old, lo + (int64_t)tid * kSelItems, hi, fpre);
            have_fpre = false;
            if (!have_krange) {  // otherwise read with the bookkeeping loads of the previous generation
                next_kmin = __ldcg(&ws->kmin[rslot]);
                next_kmax = __ldcg(&ws->kmax[rslot]);
            }
            kmin = next_kmin;
            kmax = next_kmax;
            if (wid == 0) kth_bin_warp(&ws->hist[rslot][kmin], (int)(kmax - kmin + 1), (uint64_t)half, &s_bin, &s_below);
            __syncthreads();
            if (timing && gi < 64) ws->tstamp[gi][3] = gtimer();
            const int64_t tau = (int64_t)(kmin + (uint32_t)s_bin) << gshift;
            const uint32_t quota = (uint32_t)((uint64_t)half - s_below);
            {
                uint32_t lt_run = 0, eq_run = 0;
                const int64_t span = (int64_t)pw_sel * 32 * kSelItems;
                for (int64_t b0 = lo; b0 < hi; b0 += span) {
                    const int64_t i0 = b0 + (int64_t)tid * kSelItems;
                    int64_t f[kSelItems];
                    uint32_t v = 0, x = 0;
                    if (wid < pw_sel) {
                        if (b0 == lo) {
    #pragma unroll
                            for (int u = 0; u < kSelItems; ++u) f[u] = fpre[u];
                        } else {
                            load_items(f_old, i0, hi, f);
                        }
    #pragma unroll
                        for (int u = 0; u < kSelItems; ++u) {
                            const bool in = i0 + u < hi;
                            v += (in && f[u] < tau) ? 0x10000u : 0u;
                            v += (in && f[u] == tau) ? 1u : 0u;
                        }
                        x = v;
                        for (int o = 1; o < 32; o <<= 1) {
                            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                            if (lane >= o) x += y;
                        }
                        if (lane == 31) sscr[wid] = x;
                    }
                    __syncthreads();
                    uint32_t wbase = 0, tot = 0;
                    for (int w = 0; w < pw_sel; ++w) {
                        const uint32_t tw = (uint32_t)sscr[w];
                        if (w < wid) wbase += tw;
                        tot += tw;
                    }
                    if (wid < pw_sel) {
                        uint32_t excl = wbase + x - v;
    #pragma unroll
                        for (int u = 0; u < kSelItems; ++u) {
                            const bool in = i0 + u < hi;
                            const unsigned long long kv = ((unsigned long long)f[u] << 32) | (unsigned long long)(i0 + u);
                            if (in && f[u] < tau) lt_list[lo + lt_run + (excl >> 16)] = kv;
                            if (in && f[u] == tau) eq_list[lo + eq_run + (excl & 0xffffu)] = kv;
                            excl += ((in && f[u] < tau) ? 0x10000u : 0u) + ((in && f[u] == tau) ? 1u : 0u);
                        }
                    }
                    lt_run += tot >> 16;
                    eq_run += tot & 0xffffu;
                    __syncthreads();
                }
                if (tid == 0) {
                    ws->cnt_lt[bid] = lt_run;
                    ws->cnt_eq[bid] = eq_run;
                }
            }
            if (timing && gi < 64) ws->tstamp[gi][1] = gtimer();
            grid_sync(&ws->bar);
            if (timing && gi < 64) ws->tstamp[gi][2] = gtimer();

            // ---- E: prefix of the survivor counts, then the offspring tiles
            if (bid == 0) {
                for (uint32_t b = kmin + tid; b <= kmax; b += nt) ws->hist[rslot][b] = 0;
            }
            {
                // exclusive prefix of cnt_lt / cnt_eq over the nb CTAs (nb <= kMaxNb), pw_pre warps
                uint64_t x = 0, v = 0;
                const int b = tid;
                if (wid < pw_pre) {
                    const uint32_t a = b < nb ? __ldcg(&ws->cnt_lt[b]) : 0u;
                    const uint32_t e = b < nb ? __ldcg(&ws->cnt_eq[b]) : 0u;
                    x = v = ((uint64_t)a << 32) | e;
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
                        if (lane >= o) x += y;
                    }
                    if (lane == 31) sscr[wid] = x;
                }
                __syncthreads();
                if (wid < pw_pre) {
                    uint64_t wbase = 0, tot = 0;
                    for (int w = 0; w < pw_pre; ++w) {
                        if (w < wid) wbase += sscr[w];
                        tot += sscr[w];
                    }
                    const uint64_t excl = wbase + x - v;
                    if (b < nb) {
                        s_ltpre[b] = (uint32_t)(excl >> 32);
                        s_eqpre[b] = (uint32_t)(excl & 0xffffffffu);
                    }
                    if (tid == 0) {
                        s_ltpre[nb] = (uint32_t)(tot >> 32);
                        s_eqpre[nb] = (uint32_t)(tot & 0xffffffffu);
                    }
                }
            }
        }
        if (timing && gi < 64) ws->tstamp[gi][5] = gtimer();
        LocalAcc L;
        L.s_hist = s_hist;
        L.wbase = kmin > 256u ? kmin - 256u : 0u;
        L.kmin = 0xffffffffu;
        L.kmax = 0u;
        L.best = ~0ull;
        L.pbest = ~0ull;
        for (int b = tid; b < kWin; b += nt) s_hist[b] = 0;
        if (tid == 0) {
            s_kmin = 0xffffffffu;
            s_kmax = 0u;
            s_best = ~0ull;
            s_pbest = ~0ull;
        }
        __syncthreads();
        SelView V = ONE ? SelView{s_ltpre, s_eqpre, nrng, 0, nullptr, nullptr, s_ltpre[nrng], kold, tau_key}
                        : SelView{s_ltpre, s_eqpre, nb, chunk, lt_list, eq_list, s_ltpre[nb], nullptr, 0u};
        const FeistelKey fkey = make_feistel_key(draw4(A.seed, 0, 0, (uint64_t)gen, (uint32_t)kPSelect), (uint32_t)half);
        if (timing && gi < 64) ws->tstamp[gi][7] = gtimer();
        {
            TileCtx C{&A, ws, &V, &fkey, pop_old, pop_new, f_new, N, nc, nr, (uint64_t)gen, gp, gshift, g,
                      (timing_blk && g == 0 && gi < 64) ? ws->tstamp[gi] : nullptr,
                      ONE ? keys_base + (int64_t)(parity ^ 1) * kstride : nullptr, hslot};
            if constexpr (TP)
                group_tiles_tp<M, VM>(C, (int64_t)bid * GROUPS + g, (int64_t)nb * GROUPS, ntiles, rows0, rows1, T0, T1,
                                      tplan, L);
            else
                group_tiles<M, VM, ONE>(C, (int64_t)bid * GROUPS + g, (int64_t)nb * GROUPS, ntiles, rows0, rows1, S0, S1,
                                        L);
        }
        if (timing && gi < 64) ws->tstamp[gi][8] = gtimer();
        // flush the CTA's histogram window, key range and best keys
        {
            unsigned long long kb = L.best, pb = L.pbest;
            for (int o = 16; o; o >>= 1) {
                kb = min(kb, __shfl_xor_sync(0xffffffffu, kb, o));
                pb = min(pb, __shfl_xor_sync(0xffffffffu, pb, o));
            }
            const uint32_t mn = __reduce_min_sync(0xffffffffu, L.kmin);
            const uint32_t mx = __reduce_max_sync(0xffffffffu, L.kmax);
            if (lane == 0) {
                atomicMin(&s_best, kb);
                atomicMin(&s_pbest, pb);
                atomicMin(&s_kmin, mn);
                atomicMax(&s_kmax, mx);
            }
            __syncthreads();
            for (int b = tid; b < kWin; b += nt)
                if (s_hist[b]) atomicAdd(&ws->hist[hslot][L.wbase + b], s_hist[b]);
            if (tid == 0) {
                if (s_best != ~0ull) atomicMin(&ws->best_key[bslot], s_best);
                if (s_pbest != ~0ull) atomicMin(&ws->par_key[bslot], s_pbest);
                if (s_kmin != 0xffffffffu) atomicMin(&ws->kmin[hslot], s_kmin);
                atomicMax(&ws->kmax[hslot], s_kmax);
            }
        }
        if (timing && gi < 64) ws->tstamp[gi][9] = gtimer();
        grid_sync(&ws->bar);
        if (timing && gi < 64) {
            ws->tstamp[gi][4] = gtimer();
            ws->tstamp[gi][11] = clock64();
        }

        // ---- F: bookkeeping (identical in every CTA)
        {
            // next generation's first select batch and key range, under the bookkeeping loads
            // (not in a launch's last generation: the kernel would wait for them at exit)
            const bool more = gi + 1 < A.gens_this_call;
            if (!ONE && more && wid < pw_sel) {
                load_items(f_new, lo + (int64_t)tid * kSelItems, hi, fpre);
                have_fpre = true;
            }
            const unsigned long long key = __ldcg(&ws->best_key[bslot]);
            if (more) {
                next_kmin = __ldcg(&ws->kmin[hslot]);
                next_kmax = __ldcg(&ws->kmax[hslot]);
            }
            have_krange = more;
            const int64_t v = (int64_t)(key >> 32);
            const int64_t idx = (int64_t)(key & 0xffffffffu);
            iter = gen;
            parity ^= 1;
            run = (v == last_val) ? run + 1 : 1;
            last_val = v;
            const bool improved = v < best;
            if (improved) best = v;
            if (bid == 0) {
                if (gen < A.trace_capacity) A.trace[gen] = v;
                if (improved) {
                    for (int64_t t2 = tid; t2 < G::MW; t2 += nt) A.best_matrix[t2] = __ldcg(pop_new + idx * G::MW + t2);
                    if (tid == 0) A.state[4] = idx;
                }
                if (!ONE && tid == 0) {
                    ws->best_key[gp ^ 1] = ~0ull;
                    ws->par_key[gp ^ 1] = ~0ull;
                    ws->kmin[gp] = 0xffffffffu;
                    ws->kmax[gp] = 0u;
                }
            }
            stop = !force && (best == 0 || iter >= A.max_generation);
            if (!stop && !force && A.stall_window > 0 && iter - last_restart >= A.stall_window &&
                run >= A.stall_window && last_val > 0) {
                // stall restart (engine.py:482-494): fresh offspring, parents kept,
                // next-generation histogram rebuilt from scratch
                const int ngp = hslot;
                const uint32_t omin = __ldcg(&ws->kmin[ngp]), omax = __ldcg(&ws->kmax[ngp]);
                grid_sync(&ws->bar);
                if (bid == 0) {
                    for (uint32_t b = omin + tid; b <= omax; b += nt) ws->hist[ngp][b] = 0;
                    if (tid == 0) {
                        ws->kmin[ngp] = 0xffffffffu;
                        ws->kmax[ngp] = 0u;
                    }
                }
                const int64_t work = half * M;
                for (int64_t t0 = (int64_t)bid * nt; t0 < work; t0 += (int64_t)nb * nt) {
                    const int64_t tt = t0 + tid;
                    if (tt < work) {
                        const int64_t s = half + tt / M;
                        const int c = (int)(tt % M);
                        Col<G::W> col;
                        philox_column<G::W>(A.seed, (uint32_t)kPRestart, (uint64_t)iter, s, M, c, col);
#pragma unroll
                        for (int w = 0; w < G::W; ++w) pop_new[s * G::MW + (int64_t)c * G::W + w] = col.w[w];
                    }
                }
                grid_sync(&ws->bar);
                // evaluate all 4N (fresh offspring; parents unchanged) and rebuild the histogram
                for (int64_t k0 = (int64_t)bid * nt; k0 < total; k0 += (int64_t)nb * nt) {
                    const int64_t k = k0 + tid;
                    const bool ok = k < total;
                    int64_t fv = 0;
                    if (ok) {
                        if (k >= half) {
                            uint32_t c[G::MW];
#pragma unroll
                            for (int u = 0; u < G::U; ++u) {
                                const uint4 v4 = __ldcg(reinterpret_cast<const uint4*>(pop_new + k * G::MW) + u);
                                c[4 * u] = v4.x;
                                c[4 * u + 1] = v4.y;
                                c[4 * u + 2] = v4.z;
                                c[4 * u + 3] = v4.w;
                            }
                            Sums s{0, 0, 0, 0};
                            pair_sums<M, VM, 1>(c, s);
                            fv = variant_value<M, VM>(s, G::NP);
                            f_new[k] = fv;
                            if constexpr (ONE) keys_base[(int64_t)parity * kstride + k] = (uint16_t)(fv >> gshift);
                        } else {
                            fv = __ldcg(f_new + k);
                        }
                    }
                    hist_add(ws, ngp, ok, (uint32_t)(fv >> gshift));
                    key_min_warp(&ws->restart_key,
                                 ok && k >= half ? (((unsigned long long)fv << 32) | (unsigned long long)k) : ~0ull);
                }
                grid_sync(&ws->bar);
                const unsigned long long rk = __ldcg(&ws->restart_key);
                const unsigned long long pk = __ldcg(&ws->par_key[bslot]);
                const unsigned long long k2 = min(rk, pk);
                const int64_t v2 = (int64_t)(k2 >> 32);
                if (v2 < best) {
                    best = v2;
                    if (bid == 0) {
                        const int64_t id2 = (int64_t)(k2 & 0xffffffffu);
                        for (int64_t t2 = tid; t2 < G::MW; t2 += nt) A.best_matrix[t2] = __ldcg(pop_new + id2 * G::MW + t2);
                        if (tid == 0) A.state[4] = id2;
                    }
                }
                last_restart = iter;
                have_fpre = false;  // offspring fitness was rewritten
                grid_sync(&ws->bar);
                if (bid == 0 && tid == 0) ws->restart_key = ~0ull;
                stop = best == 0;
                have_krange = false;  // the histogram was rebuilt
            }
        }
    }
    if (bid == 0 && tid == 0) {
        A.state[0] = iter;
        A.state[1] = best;
        A.state[2] = last_restart;
        A.state[3] = parity;
        A.state[5] = (best == 0 || iter >= A.max_generation) ? 1 : 0;
        A.state[6] = run;
        A.state[7] = last_val;
        if (A.flags & HGA_RUN_TIMING) ws->tstamp[63][1] = gtimer();  // CTA 0 done
    }
}

int run2_granule_shift(uint32_t fit_var);
bool run2_supported(const hga_run_args* a);
constexpr uint32_t kRunTeamTiles = 1u << 16;  // internal (tests, timing): team-of-four tiles instead of throughput tiles
inline bool run2_use_onebar(const hga_run_args* a) {
    return run2_onebar(a->n_pairs) && (a->flags & HGA_RUN_ONE_BARRIER) != 0;
}

template <int M>
int launch_run_v2_m(const hga_run_args* a, cudaStream_t st);

#define HGA_R2_ORDERS(X) X(4) X(8) X(12) X(16) X(20) X(24) X(28) X(32) X(36) X(40) X(44) X(48) X(52) X(56) X(60) X(64)
#define HGA_R2_EXTERN(M) extern template int launch_run_v2_m<M>(const hga_run_args*, cudaStream_t);

template <int M>
constexpr int run_groups() {
    // tile groups per CTA (one CTA per SM): 640 threads leave <= 102 registers,
    // 512 threads <= 128; more groups = fewer tiles per group at small N
    return M <= 24 ? 5 : (M <= 36 ? 4 : 2);
}

template <int M>
constexpr int run_groups_tp() {
    // one thread per child holds the whole chain's live values: ~125 registers
    // at m = 24 (four groups fit), ~250 at m = 28..40 (two groups)
    return M <= 24 ? 4 : 2;
}

template <int M, int VM, bool ONE, bool TP = false>
int launch_run_v2_k(const hga_run_args* a, cudaStream_t st) {
    constexpr int GROUPS = TP ? run_groups_tp<M>() : run_groups<M>();
    Run2Params P;
    P.a = *a;
    P.gshift = run2_granule_shift(a->fit_var);
    const int smem = GROUPS * (int)run_group_bytes<M, TP>();
    auto kern = k_run_v3<M, VM, GROUPS, ONE, TP>;
    static bool attr[kMaxDevices] = {};
    static int per_sm_dev[kMaxDevices] = {};  // 0 = not yet queried on that device
    const int dev = current_device();
    if (!attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return to_rc(e);
        attr[dev] = true;
    }
    if (per_sm_dev[dev] == 0) {
        int v = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, kR2Threads * GROUPS, smem);
        if (e != cudaSuccess) return to_rc(e);
        per_sm_dev[dev] = v > 0 ? v : -1;
    }
    const int per_sm = per_sm_dev[dev];
    if (per_sm < 1) return HGA_E_UNSUPPORTED;
    int grid = std::min(std::min(sm_count_cached() * std::min(per_sm, 2), kMaxNb), GROUPS * kR2Threads);
    static const int grid_cap = [] {  // HGA_RUN_GRID=<ctas>: experiment, cap the loop's grid (results identical)
        const char* e = std::getenv("HGA_RUN_GRID");
        return e ? std::atoi(e) : 0;
    }();
    if (grid_cap > 0) grid = std::min(grid, grid_cap);
    void* params[] = {&P};
    if (a->flags & kRunPlainLaunch)  // experiment: ordinary launch (co-residency by construction: grid <= resident CTAs)
        return to_rc(cudaLaunchKernel((const void*)kern, dim3(grid), dim3(kR2Threads * GROUPS), params, smem, st));
    return to_rc(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(kR2Threads * GROUPS), params, smem, st));
}

// Definition used by the per-order instantiation files run_m<M>.cu.
template <int M, int VM>
int launch_run_v2_mv(const hga_run_args* a, cudaStream_t st) {
    if (run2_use_onebar(a)) return launch_run_v2_k<M, VM, true>(a, st);
    if constexpr (M >= 24 && M <= 40) {
        // throughput tiles unless the plan does not fit their per-child slot
        // (kRunTeamTiles forces the team tiles: A/B timing, tests).  Measured
        // (scripts/tp_threshold.py): faster from m = 24 on (m = 28, 4N = 125,000:
        // 35.7 -> 27.7 us/generation; m = 36, 4N = 1.25M: 481 -> 425), slower
        // at m = 20 (17.0 -> 18.6), where the team tiles stay.
        const int nc = a->strategy == HGA_MUT_MULTI ? a->nc : 1, nr = a->strategy == HGA_MUT_MULTI ? a->nr : 1;
        const bool fits = nc + 2 * nr <= kTPPlanStride - 4;
        if (fits && !(a->flags & kRunTeamTiles)) return launch_run_v2_k<M, VM, false, true>(a, st);
    }
    return launch_run_v2_k<M, VM, false>(a, st);
}

template <int M>
int launch_run_v2_m(const hga_run_args* a, cudaStream_t st) {
    switch (a->fit_var) {
        case HGA_VAR_F1: return launch_run_v2_mv<M, HGA_VAR_F1>(a, st);
        case HGA_VAR_SQ:
            if constexpr (M <= 32) return launch_run_v2_mv<M, HGA_VAR_SQ>(a, st);
            return HGA_E_UNSUPPORTED;
        default: return launch_run_v2_mv<M, HGA_VAR_F2>(a, st);
    }
}

}  // namespace hga
