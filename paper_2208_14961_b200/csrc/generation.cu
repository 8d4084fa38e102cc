// generation.cu -- one GA generation on the packed resident population.
//
//  * hga_generation_explicit: crossover + mutation + fitness with explicit
//    plans (the reference-stream replay path; select is done beforehand by
//    hga_select_order + hga_ref_permutation + hga_compose_gather).
//  * hga_run / hga_run_init: the production loop (engine.py:449-538 with
//    Philox streams): ONE persistent cooperative kernel runs many
//    generations; phases are separated by a grid barrier, and the host only
//    polls an 8-word state block.  Per generation:
//      A  radix-select histogram of the 4N fitness values (coarse, 4096 bins)
//      B  threshold tau + tie quota (2N lowest, lowest index first on ties;
//         engine.py:245), fine histogram if the coarse bin is not exact,
//         per-CTA counts of (F < tau, F == tau) over contiguous index ranges
//      D  stable winner ranks by CTA prefix + block scan; rank -> parent slot
//         through a keyed Feistel bijection (uniformly random placement,
//         engine.py:246); src[slot] = winner, F_new[slot] = F[winner]
//      E  fused offspring tiles (generation.cuh) from src[], with the
//         parents copied to the new buffer (out-of-place gather, engine.py:247)
//      F  trace / best / stop / stall-restart bookkeeping, replicated in every
//         CTA from the same global values so all CTAs agree without a barrier
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "generation.cuh"
#include "run_common.cuh"
#include "run_v2.cuh"

#include <cstddef>
#include <cstring>

namespace hga {

// ======================================================== explicit plans
template <int W, int VM>
__global__ void __launch_bounds__(kGenThreads)
    k_generation_explicit(uint32_t* pop, int64_t* fit, int64_t N, int m, int ppb,
                          const int64_t* __restrict__ points, const int64_t* __restrict__ cols,
                          const int64_t* __restrict__ ra, const int64_t* __restrict__ rb, int nc, int nr,
                          uint32_t fit_var, unsigned long long* best_key) {
    extern __shared__ __align__(16) unsigned char smem[];
    const TileSmem s = carve_tile(smem, m, W, ppb, nc, nr);
    const int64_t mw = (int64_t)m * W;
    for (int64_t p0 = (int64_t)blockIdx.x * ppb; p0 < N; p0 += (int64_t)gridDim.x * ppb) {
        const int cnt = (int)min((int64_t)ppb, N - p0);
        for (int t = threadIdx.x; t < ppb; t += blockDim.x) {
            if (t < cnt) {
                s.point[t] = (int16_t)points[p0 + t];
                s.poff[2 * t] = (p0 + t) * mw;
                s.poff[2 * t + 1] = (N + p0 + t) * mw;
            }
        }
        for (int t = threadIdx.x; t < 2 * ppb * (nc + 2 * nr); t += blockDim.x) {
            const int ol = t / (nc + 2 * nr), e = t - ol * (nc + 2 * nr);
            const int q = ol % ppb;
            if (q >= cnt) continue;
            const int64_t row = (ol < ppb) ? p0 + q : N + p0 + q;
            if (e < nc) s.pcol[ol * nc + e] = (int16_t)cols[row * nc + e];
            else if (e < nc + nr) s.pra[ol * nr + e - nc] = (int16_t)ra[row * nr + e - nc];
            else s.prb[ol * nr + e - nc - nr] = (int16_t)rb[row * nr + e - nc - nr];
        }
        __syncthreads();
        offspring_tile<W, VM, false>(s, pop, pop, fit, N, p0, cnt, ppb, m, nc, nr, fit_var, best_key);
    }
}

// ======================================================== run workspace
constexpr int kHistBins = 4096;
constexpr int kMaxGrid = 4096;

struct RunWs {
    Barrier bar;
    unsigned long long best_key[2];   // per generation parity: min over new population
    unsigned long long par_key[2];    // min over the parents only (restart bookkeeping)
    unsigned long long restart_key;
    uint32_t hist1[kHistBins];
    uint32_t hist2[kHistBins];
    uint32_t cnt_lt[kMaxGrid];
    uint32_t cnt_eq[kMaxGrid];
    // followed by src[2N] (int64)
};

__host__ __device__ inline size_t run_ws_head() { return (sizeof(RunWs) + 255) & ~(size_t)255; }

// Block-wide: find the first bin b where the inclusive prefix of h reaches
// k (1 <= k <= total).  Returns b and the count strictly below b.
__device__ void find_kth_bin(const uint32_t* h, int bins, uint64_t k, int* out_bin, uint64_t* out_below,
                             uint64_t* scratch /* >= blockDim/32 + 2 */) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int per = (bins + nt - 1) / nt;
    const int b0 = tid * per;
    uint64_t mine = 0;
    for (int b = b0; b < min(bins, b0 + per); ++b) mine += h[b];
    // exclusive scan of `mine`
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
        for (int w = 0; w < (nt + 31) / 32; ++w) {
            const uint64_t t = scratch[w];
            scratch[w] = run;
            run += t;
        }
    }
    __syncthreads();
    const uint64_t excl = scratch[wid] + x - mine;
    __syncthreads();
    if (excl < k && excl + mine >= k) {
        uint64_t run = excl;
        for (int b = b0; b < min(bins, b0 + per); ++b) {
            if (run + h[b] >= k) {
                *out_bin = b;
                *out_below = run;
                break;
            }
            run += h[b];
        }
    }
    __syncthreads();
}

struct RunParams {
    hga_run_args a;
    int W;
    int ppb;
    int shift;       // coarse histogram shift
    int hb;          // Feistel half bits
};

template <int W, int VM>
__global__ void __launch_bounds__(kGenThreads) k_run(RunParams P) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t shist[kHistBins];
    __shared__ uint64_t sscr[40];
    __shared__ int s_bin;
    __shared__ uint64_t s_below;

    const hga_run_args& A = P.a;
    RunWs* ws = reinterpret_cast<RunWs*>(A.ws);
    int64_t* src = reinterpret_cast<int64_t*>(reinterpret_cast<char*>(A.ws) + run_ws_head());
    const int64_t N = A.n_pairs, half = 2 * N, total = 4 * N;
    const int m = A.m;
    const int64_t mw = (int64_t)m * W;
    const int nb = gridDim.x, bid = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
    const int64_t chunk = (total + nb - 1) / nb;
    const int64_t lo = min(total, (int64_t)bid * chunk), hi = min(total, lo + chunk);
    const int nc = A.strategy == HGA_MUT_MULTI ? A.nc : 1;
    const int nr = A.strategy == HGA_MUT_MULTI ? A.nr : 1;
    const TileSmem ts = carve_tile(smem, m, W, P.ppb, nc, nr);

    // replicated bookkeeping state (identical in every CTA)
    int64_t iter = A.state[0], best = A.state[1], last_restart = A.state[2];
    int parity = (int)A.state[3];
    int64_t run = A.state[6], last_val = A.state[7];
    const bool force = (A.flags & HGA_RUN_FORCE) != 0;
    bool stop = !force && A.state[5] != 0;

    for (int64_t gi = 0; gi < A.gens_this_call && !stop; ++gi) {
        const int64_t gen = iter + 1;
        const int gp = (int)(gen & 1);
        const uint32_t* pop_old = A.pop[parity];
        uint32_t* pop_new = A.pop[parity ^ 1];
        const int64_t* f_old = A.fit[parity];
        int64_t* f_new = A.fit[parity ^ 1];

        // ---- A: coarse histogram
        for (int b = tid; b < kHistBins; b += nt) shist[b] = 0;
        __syncthreads();
        for (int64_t i = lo + tid; i < hi; i += nt) atomicAdd(&shist[min((int64_t)kHistBins - 1, f_old[i] >> P.shift)], 1u);
        __syncthreads();
        for (int b = tid; b < kHistBins; b += nt)
            if (shist[b]) atomicAdd(&ws->hist1[b], shist[b]);
        grid_sync(&ws->bar);

        // ---- B: threshold, tie quota, per-CTA counts
        find_kth_bin(ws->hist1, kHistBins, (uint64_t)half, &s_bin, &s_below, sscr);
        int64_t tau;
        uint64_t quota;
        if (P.shift == 0) {
            tau = s_bin;
            quota = (uint64_t)half - s_below;
        } else {
            const int64_t bucket = s_bin;
            const uint64_t below = s_below;
            for (int b = tid; b < kHistBins; b += nt) shist[b] = 0;
            __syncthreads();
            const int64_t fmask = (1ll << P.shift) - 1;
            for (int64_t i = lo + tid; i < hi; i += nt) {
                const int64_t f = f_old[i];
                if ((f >> P.shift) == bucket) atomicAdd(&shist[f & fmask], 1u);
            }
            __syncthreads();
            for (int b = tid; b < kHistBins; b += nt)
                if (shist[b]) atomicAdd(&ws->hist2[b], shist[b]);
            grid_sync(&ws->bar);
            find_kth_bin(ws->hist2, kHistBins, (uint64_t)half - below, &s_bin, &s_below, sscr);
            tau = (bucket << P.shift) | s_bin;
            quota = (uint64_t)half - below - s_below;
        }
        {
            uint32_t nlt = 0, neq = 0;
            for (int64_t i = lo + tid; i < hi; i += nt) {
                const int64_t f = f_old[i];
                nlt += f < tau;
                neq += f == tau;
            }
            nlt = __reduce_add_sync(0xffffffffu, nlt);
            neq = __reduce_add_sync(0xffffffffu, neq);
            if ((tid & 31) == 0) {
                sscr[tid >> 5] = ((uint64_t)nlt << 32) | neq;
            }
            __syncthreads();
            if (tid == 0) {
                uint64_t a = 0, e = 0;
                for (int w = 0; w < nt / 32; ++w) {
                    a += sscr[w] >> 32;
                    e += sscr[w] & 0xffffffffu;
                }
                ws->cnt_lt[bid] = (uint32_t)a;
                ws->cnt_eq[bid] = (uint32_t)e;
            }
        }
        grid_sync(&ws->bar);

        // ---- D: stable ranks -> Feistel slots
        {
            uint64_t lt_b = 0, eq_b = 0;
            for (int b = tid; b < bid; b += nt) {
                lt_b += ws->cnt_lt[b];
                eq_b += ws->cnt_eq[b];
            }
            for (int o = 16; o; o >>= 1) {
                lt_b += __shfl_xor_sync(0xffffffffu, lt_b, o);
                eq_b += __shfl_xor_sync(0xffffffffu, eq_b, o);
            }
            __syncthreads();
            if ((tid & 31) == 0) sscr[tid >> 5] = (lt_b << 32) | eq_b;
            __syncthreads();
            uint64_t lt_run = 0, eq_run = 0;
            for (int w = 0; w < nt / 32; ++w) {
                lt_run += sscr[w] >> 32;
                eq_run += sscr[w] & 0xffffffffu;
            }
            __syncthreads();
            const U4 fk = draw4(A.seed, 0, 0, (uint64_t)gen, (uint32_t)kPSelect);
            const int lane = tid & 31, wid = tid >> 5;
            unsigned long long kbest = ~0ull;
            for (int64_t i0 = lo; i0 < hi; i0 += nt) {
                const int64_t i = i0 + tid;
                int64_t f = 0;
                uint32_t is_lt = 0, is_eq = 0;
                if (i < hi) {
                    f = f_old[i];
                    is_lt = f < tau;
                    is_eq = f == tau;
                }
                // block exclusive scan of (is_lt, is_eq) packed in 16 | 16 bits
                const uint32_t v = (is_lt << 16) | is_eq;
                uint32_t x = v;
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                if (lane == 31) sscr[wid] = x;
                __syncthreads();
                uint32_t wbase = 0, tot = 0;
                for (int w = 0; w < nt / 32; ++w) {
                    const uint32_t t = (uint32_t)sscr[w];
                    if (w < wid) wbase += t;
                    tot += t;
                }
                const uint32_t excl = wbase + x - v;
                const uint64_t lt_rank = lt_run + (excl >> 16);
                const uint64_t eq_rank = eq_run + (excl & 0xffffu);
                if (is_lt || (is_eq && eq_rank < quota)) {
                    const uint64_t rank = lt_rank + min(eq_rank, quota);
                    const uint32_t slot = feistel((uint32_t)rank, (uint32_t)half, P.hb, fk);
                    src[slot] = i;
                    f_new[slot] = f;
                    kbest = min(kbest, ((unsigned long long)f << 32) | slot);
                }
                lt_run += tot >> 16;
                eq_run += tot & 0xffffu;
                __syncthreads();
            }
            for (int o = 16; o; o >>= 1) kbest = min(kbest, __shfl_xor_sync(0xffffffffu, kbest, o));
            if (lane == 0 && kbest != ~0ull) {
                atomicMin(&ws->best_key[gp], kbest);
                atomicMin(&ws->par_key[gp], kbest);
            }
        }
        grid_sync(&ws->bar);

        // ---- E: offspring tiles
        if (bid == 0) {
            for (int b = tid; b < kHistBins; b += nt) {
                ws->hist1[b] = 0;
                ws->hist2[b] = 0;
            }
        }
        {
            const int ppb = P.ppb;
            const int per_off = nc + 2 * nr;
            const int blocks4 = (per_off + 3) / 4;
            for (int64_t p0 = (int64_t)bid * ppb; p0 < N; p0 += (int64_t)nb * ppb) {
                const int cnt = (int)min((int64_t)ppb, N - p0);
                if (tid < cnt) {
                    const int64_t p = p0 + tid;
                    const U4 r = draw4(A.seed, (uint32_t)p, (uint32_t)(p >> 32), (uint64_t)gen, (uint32_t)kPCrossover);
                    ts.point[tid] = (int16_t)(1 + bounded(r.x, (uint32_t)(m - 1)));
                    ts.poff[2 * tid] = src[p] * mw;
                    ts.poff[2 * tid + 1] = src[N + p] * mw;
                }
                for (int t = tid; t < 2 * ppb * blocks4; t += nt) {
                    const int ol = t / blocks4, blk = t - ol * blocks4;
                    const int q = ol % ppb;
                    if (q >= cnt) continue;
                    int64_t o = (ol < ppb) ? p0 + q : N + p0 + q;  // plan row, as engine.py
                    if (A.strategy == HGA_MUT_SHARED) o = 0;
                    const U4 r = draw4(A.seed, (uint32_t)o, (uint32_t)blk | ((uint32_t)(o >> 32) << 16), (uint64_t)gen,
                                       (uint32_t)kPMutCol);
#pragma unroll
                    for (int e4 = 0; e4 < 4; ++e4) {
                        const int e = blk * 4 + e4;
                        const uint32_t rv = pick(r, e4);
                        if (e < nc) ts.pcol[ol * nc + e] = (int16_t)(1 + bounded(rv, (uint32_t)(m - 1)));
                        else if (e < nc + nr) ts.pra[ol * nr + e - nc] = (int16_t)bounded(rv, (uint32_t)m);
                        else if (e < per_off) ts.prb[ol * nr + e - nc - nr] = (int16_t)bounded(rv, (uint32_t)m);
                    }
                }
                __syncthreads();
                offspring_tile<W, VM, true>(ts, pop_old, pop_new, f_new, N, p0, cnt, ppb, m, nc, nr, A.fit_var,
                                            &ws->best_key[gp]);
            }
        }
        grid_sync(&ws->bar);

        // ---- F: bookkeeping (every CTA computes the same decisions)
        {
            const unsigned long long key = *(volatile unsigned long long*)&ws->best_key[gp];
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
                    for (int64_t t = tid; t < mw; t += nt) A.best_matrix[t] = pop_new[idx * mw + t];
                    if (tid == 0) A.state[4] = idx;
                }
                if (tid == 0) {
                    ws->best_key[gp ^ 1] = ~0ull;
                    ws->par_key[gp ^ 1] = ~0ull;
                }
            }
            stop = !force && (best == 0 || iter >= A.max_generation);
            // stall restart (engine.py:472-494, 518-525)
            if (!stop && !force && A.stall_window > 0 && iter - last_restart >= A.stall_window && run >= A.stall_window &&
                last_val > 0) {
                // refill offspring slots of the new population, evaluate them
                uint32_t* cur = pop_new;
                int64_t* fcur = f_new;
                const int64_t work = half * m;
                for (int64_t t0 = (int64_t)bid * nt; t0 < work; t0 += (int64_t)nb * nt) {
                    const int64_t t = t0 + tid;
                    if (t < work) {
                        const int64_t s = half + t / m;
                        const int c = (int)(t % m);
                        Col<W> col;
                        philox_column<W>(A.seed, (uint32_t)kPRestart, (uint64_t)iter, s, m, c, col);
#pragma unroll
                        for (int w = 0; w < W; ++w) cur[s * mw + (int64_t)c * W + w] = col.w[w];
                    }
                }
                grid_sync(&ws->bar);
                // evaluate fresh offspring with the fitness tile (pairs of slots)
                {
                    const int mpb = 2 * P.ppb;  // matches the tile's shared-memory carve
                    const int kl = tid / m, i = tid - kl * m;
                    const int hlf = (m & 1) ? -1 : m / 2;
                    for (int64_t k0 = half + (int64_t)bid * mpb; k0 < total; k0 += (int64_t)nb * mpb) {
                        const int cnt = (int)min((int64_t)mpb, total - k0);
                        const bool act = kl < cnt && kl < mpb;
                        Col<W> c;
                        if (act) {
#pragma unroll
                            for (int w = 0; w < W; ++w) c.w[w] = cur[(k0 + kl) * mw + (int64_t)i * W + w];
                            uint32_t* d = ts.col + ((int64_t)kl * 2 * m + i) * W;
#pragma unroll
                            for (int w = 0; w < W; ++w) {
                                d[w] = c.w[w];
                                d[(int64_t)m * W + w] = c.w[w];
                            }
                        }
                        if (tid < mpb * 3) ts.acc[tid] = 0;
                        __syncthreads();
                        Acc a{0, 0, 0};
                        if (act) {
                            const uint32_t* base = ts.col + ((int64_t)kl * 2 * m + i) * W;
                            const int steps = pair_steps(m, i);
                            for (int d = 1; d <= steps; ++d) {
                                int p = 0;
#pragma unroll
                                for (int w = 0; w < W; ++w) p += __popc(c.w[w] ^ base[d * W + w]);
                                acc_pair<VM>(a, p, m, hlf);
                            }
                        }
                        if (act) {
                            if (VM & HGA_VAR_F1) atomicAdd(&ts.acc[kl * 3 + 0], a.s1);
                            if (VM & HGA_VAR_F2) atomicAdd(&ts.acc[kl * 3 + 1], a.s2);
                            if (VM & HGA_VAR_SQ) atomicAdd(&ts.acc[kl * 3 + 2], a.s4);
                        }
                        __syncthreads();
                        if (tid < cnt) {
                            const uint32_t* ac = ts.acc + tid * 3;
                            const int64_t fv = 2 * (int64_t)(A.fit_var == HGA_VAR_F1 ? ac[0] : A.fit_var == HGA_VAR_SQ ? ac[2] : ac[1]);
                            fcur[k0 + tid] = fv;
                            atomicMin(&ws->restart_key, ((unsigned long long)fv << 32) | (unsigned long long)(k0 + tid));
                        }
                        __syncthreads();
                    }
                }
                grid_sync(&ws->bar);
                const unsigned long long rk = *(volatile unsigned long long*)&ws->restart_key;
                const unsigned long long pk = *(volatile unsigned long long*)&ws->par_key[gp];
                const unsigned long long k2 = min(rk, pk);
                const int64_t v2 = (int64_t)(k2 >> 32);
                if (v2 < best) {
                    best = v2;
                    if (bid == 0) {
                        const int64_t id2 = (int64_t)(k2 & 0xffffffffu);
                        for (int64_t t = tid; t < mw; t += nt) A.best_matrix[t] = cur[id2 * mw + t];
                        if (tid == 0) A.state[4] = id2;
                    }
                }
                last_restart = iter;
                grid_sync(&ws->bar);
                if (bid == 0 && tid == 0) ws->restart_key = ~0ull;
                stop = best == 0;
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
    }
}

// ======================================================== run init
template <int W>
__global__ void k_philox_init(uint64_t seed, uint32_t purpose, uint64_t gen, int64_t first_slot, int64_t count, int m,
                              uint32_t* __restrict__ cols) {
    const int64_t total = count * m;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = first_slot + t / m;
        const int c = (int)(t % m);
        Col<W> col;
        philox_column<W>(seed, purpose, gen, s, m, c, col);
#pragma unroll
        for (int w = 0; w < W; ++w) cols[(s * m + c) * W + w] = col.w[w];
    }
}

__global__ void k_run_finish_init(hga_run_args a, int W, unsigned long long* key, RunWs* ws) {
    const unsigned long long k = *key;
    const int64_t v = (int64_t)(k >> 32), idx = (int64_t)(k & 0xffffffffu);
    const int64_t mw = (int64_t)a.m * W;
    for (int64_t t = threadIdx.x; t < mw; t += blockDim.x) a.best_matrix[t] = a.pop[0][idx * mw + t];
    if (threadIdx.x == 0) {
        a.state[0] = 0;
        a.state[1] = v;
        a.state[2] = 0;
        a.state[3] = 0;
        a.state[4] = idx;
        a.state[5] = v == 0 ? 1 : 0;
        a.state[6] = 1;
        a.state[7] = v;
        if (a.trace_capacity > 0) a.trace[0] = v;
        ws->bar.count = 0;
        ws->bar.gen = 0;
        ws->best_key[0] = ws->best_key[1] = ~0ull;
        ws->par_key[0] = ws->par_key[1] = ~0ull;
        ws->restart_key = ~0ull;
    }
    for (int b = threadIdx.x; b < kHistBins; b += blockDim.x) {
        ws->hist1[b] = 0;
        ws->hist2[b] = 0;
    }
}

__global__ void k_argmin_key2(const int64_t* __restrict__ f, int64_t n, unsigned long long* key) {
    unsigned long long best = ~0ull;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        best = min(best, ((unsigned long long)f[i] << 32) | (unsigned long long)i);
    for (int o = 16; o; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0) atomicMin(key, best);
}

static int bit_length(uint64_t x) {
    int b = 0;
    while (x) {
        ++b;
        x >>= 1;
    }
    return b;
}

static uint64_t max_fitness(int m, uint32_t v) {
    const uint64_t M = (uint64_t)m;
    if (v == HGA_VAR_F1) return M * M * (M - 1);
    if (v == HGA_VAR_SQ) return M * M * M * (M - 1);
    return M * (M - 1);
}

template <int W, int VM>
static int launch_run(const hga_run_args* a, cudaStream_t st) {
    RunParams P;
    P.a = *a;
    P.W = W;
    const int nc = a->strategy == HGA_MUT_MULTI ? a->nc : 1;
    const int nr = a->strategy == HGA_MUT_MULTI ? a->nr : 1;
    P.ppb = kGenThreads / (2 * a->m);
    const int bits = bit_length(max_fitness(a->m, a->fit_var));
    P.shift = bits > 12 ? bits - 12 : 0;
    const int dom_bits = std::max(2, bit_length((uint64_t)(2 * a->n_pairs - 1)));
    P.hb = (dom_bits + 1) / 2;
    const size_t smem = tile_smem_bytes(a->m, W, P.ppb, nc, nr);
    auto kern = k_run<W, VM>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return to_rc(e);
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kGenThreads, smem);
    if (e != cudaSuccess) return to_rc(e);
    if (per_sm < 1) return HGA_E_UNSUPPORTED;
    int grid = sm_count_cached() * std::min(per_sm, 2);
    grid = std::min(grid, kMaxGrid);
    const int64_t want = std::max<int64_t>(1, (a->n_pairs + P.ppb - 1) / P.ppb);
    grid = (int)std::min<int64_t>(grid, std::max<int64_t>(want, 1));
    void* params[] = {&P};
    e = cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(kGenThreads), params, smem, st);
    return to_rc(e);
}

template <int W>
static int launch_run_w(const hga_run_args* a, cudaStream_t st) {
    switch (a->fit_var) {
        case HGA_VAR_F1: return launch_run<W, HGA_VAR_F1>(a, st);
        case HGA_VAR_SQ: return launch_run<W, HGA_VAR_SQ>(a, st);
        default: return launch_run<W, HGA_VAR_F2>(a, st);
    }
}

template <int W, int VM>
static int launch_explicit(uint32_t* pop, int64_t* fit, int64_t N, int m, const int64_t* points, const int64_t* cols,
                           const int64_t* ra, const int64_t* rb, int nc, int nr, uint32_t fit_var,
                           unsigned long long* best_key, cudaStream_t st) {
    const int ppb = kGenThreads / (2 * m);
    const size_t smem = tile_smem_bytes(m, W, ppb, nc, nr);
    auto kern = k_generation_explicit<W, VM>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return to_rc(e);
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kGenThreads, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t tiles = (N + ppb - 1) / ppb;
    const int64_t grid = std::min<int64_t>(tiles, (int64_t)sm_count_cached() * per_sm);
    kern<<<(unsigned)grid, kGenThreads, smem, st>>>(pop, fit, N, m, ppb, points, cols, ra, rb, nc, nr, fit_var, best_key);
    return to_rc(cudaGetLastError());
}

template <int W>
static int launch_explicit_w(uint32_t* pop, int64_t* fit, int64_t N, int m, const int64_t* points,
                             const int64_t* cols, const int64_t* ra, const int64_t* rb, int nc, int nr,
                             uint32_t fit_var, unsigned long long* best_key, cudaStream_t st) {
    switch (fit_var) {
        case HGA_VAR_F1: return launch_explicit<W, HGA_VAR_F1>(pop, fit, N, m, points, cols, ra, rb, nc, nr, fit_var, best_key, st);
        case HGA_VAR_SQ: return launch_explicit<W, HGA_VAR_SQ>(pop, fit, N, m, points, cols, ra, rb, nc, nr, fit_var, best_key, st);
        default: return launch_explicit<W, HGA_VAR_F2>(pop, fit, N, m, points, cols, ra, rb, nc, nr, fit_var, best_key, st);
    }
}

HGA_R2_ORDERS(HGA_R2_EXTERN)

int run2_granule_shift(uint32_t fit_var) { return fit_var == HGA_VAR_F1 ? 3 : (fit_var == HGA_VAR_SQ ? 5 : 1); }

bool run2_supported(const hga_run_args* a) {
    const int m = a->m;
    if (m < 4 || m > 64 || (m & 3)) return false;
    if (a->fit_var == HGA_VAR_SQ && m > 32) return false;
    const int nc = a->strategy == HGA_MUT_MULTI ? a->nc : 1, nr = a->strategy == HGA_MUT_MULTI ? a->nr : 1;
    if (nc + 2 * nr > kR2MaxPlan) return false;
    return (max_fitness(m, a->fit_var) >> run2_granule_shift(a->fit_var)) < (uint64_t)kR2Bins;
}

static int launch_run_v2(const hga_run_args* a, cudaStream_t st) {
    switch (a->m) {
#define HGA_R2_CASE(M) \
    case M: return launch_run_v2_m<M>(a, st);
        HGA_R2_ORDERS(HGA_R2_CASE)
#undef HGA_R2_CASE
        default: return HGA_E_UNSUPPORTED;
    }
}

// Rebuild the select histogram of pop/fit[parity] (state[3]) and reset keys:
// needed after init and whenever the population was replaced from outside.
__global__ void k_run2_prepare_zero(RunWs2* ws) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < 3 * kR2Bins; b += gridDim.x * blockDim.x)
        (&ws->hist[0][0])[b] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ws->bar.count = 0;
        ws->bar.gen = 0;
        ws->restart_key = ~0ull;
        for (int k = 0; k < 3; ++k) {
            ws->best_key[k] = ~0ull;
            ws->par_key[k] = ~0ull;
            ws->kmin[k] = 0xffffffffu;
            ws->kmax[k] = 0u;
        }
    }
}

// Histogram (and, for the one-barrier loop, the 16-bit key array padded with
// 0xFFFF) of pop/fit[state[3]], the population entering generation state[0]+1.
__global__ void k_run2_prepare_hist_state(RunWs2* ws, hga_run_args a, int gshift, int onebar) {
    const int64_t gen = a.state[0] + 1;
    const int slot = onebar ? (int)(gen % 3) : (int)(gen & 1);
    const int parity = (int)a.state[3];
    const int64_t* fit = a.fit[parity];
    const int64_t total = 4 * a.n_pairs;
    const int64_t kstride = run2_key_stride(a.n_pairs);
    uint16_t* keys = reinterpret_cast<uint16_t*>(reinterpret_cast<char*>(a.ws) + run_ws2_head() + 16 * total);
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < kstride; i0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = i0 + threadIdx.x;
        const bool ok = i < total;
        const uint32_t key = ok ? (uint32_t)(fit[i] >> gshift) : 0u;
        if (onebar && i < kstride) {
            keys[(int64_t)parity * kstride + i] = ok ? (uint16_t)key : (uint16_t)0xFFFF;
            if (!ok) keys[(int64_t)(parity ^ 1) * kstride + i] = (uint16_t)0xFFFF;
        }
        hist_add(ws, slot, ok, key);
    }
}

static int run2_prepare(const hga_run_args* a, cudaStream_t st) {
    RunWs2* ws = (RunWs2*)a->ws;
    const int64_t total = 4 * a->n_pairs;
    k_run2_prepare_zero<<<64, 256, 0, st>>>(ws);
    const int64_t kstride = run2_key_stride(a->n_pairs);
    const int grid = (int)std::min<int64_t>((std::max(total, kstride) + 255) / 256, (int64_t)sm_count_cached() * 8);
    k_run2_prepare_hist_state<<<std::max(grid, 1), 256, 0, st>>>(ws, *a, run2_granule_shift(a->fit_var),
                                                                   run2_use_onebar(a) ? 1 : 0);
    return to_rc(cudaGetLastError());
}

}  // namespace hga

namespace hga {
int unpack_i8_guarded(const uint32_t* cols, int64_t n, int32_t m, int8_t* pop, const int32_t* flag, cudaStream_t st);
// step_bits.cu / host_bits.cpp: the bit-stream transfer of hga_step_host_bits
int bits_to_cols(const uint32_t* bits, int64_t n, int32_t m, uint32_t* cols, int32_t* flag, cudaStream_t st);
int cols_to_bits(const uint32_t* cols, int64_t n, int32_t m, uint32_t* bits, const int32_t* skip, cudaStream_t st);
int host_pack_pieces(const int8_t* src, int64_t nbytes, uint32_t* dst, const int64_t* wlo, int k,
                     int (*started)(void*), int (*on_piece)(void*, int), void* ctx);
int host_unpack_pieces(const uint32_t* src, int8_t* dst, int64_t nbytes, const int64_t* wlo, int k,
                       int (*landed)(void*, int), void* ctx);
int host_pool_threads();

// hga_step_host on a rejected upload: the fitness copy-back returns the uploaded values
__global__ void k_fit_restore_if(const int64_t* __restrict__ src, int64_t* __restrict__ dst, int64_t n,
                                 const int32_t* __restrict__ flag) {
    if (!(*flag & (HGA_FLAG_NOT_SIGN | HGA_FLAG_NOT_GA))) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

// state block of a host-driven step: iteration, best, last restart, parity 0,
// best index 0, stop 0, run length, last trace value
__global__ void k_set_state(int64_t* s, int64_t it, int64_t best, int64_t last_restart, int64_t run, int64_t last) {
    const int64_t v[8] = {it, best, last_restart, 0, 0, 0, run, last};
    if (threadIdx.x < 8) s[threadIdx.x] = v[threadIdx.x];
}

// ---------------------------------------------------------------- hga_step_host_bits
constexpr int kStepBitsMaxChunks = 16;
constexpr size_t kStepBitsTail = 256;  // pinned staging of the 8-value state block after the stream

// Pieces of the population: whole groups of 16 matrices (word aligned in the
// stream, whole CTA groups of the bit kernels), the last piece to the end.
struct StepPieces {
    int k;
    int64_t mlo[kStepBitsMaxChunks + 1], wlo[kStepBitsMaxChunks + 1];
    StepPieces(int64_t total, int m, int chunks) {
        k = (int)std::max<int64_t>(1, std::min<int64_t>(std::min(chunks, kStepBitsMaxChunks), total / 16));
        for (int i = 0; i <= k; ++i) {
            mlo[i] = i == k ? total : ((total * i / k) & ~(int64_t)15);
            wlo[i] = i == k ? (total * m * m + 31) / 32 : mlo[i] * m * m / 32;
        }
    }
};

// The device half of one host-state step after the upload, fixed for given
// buffers: captured once into a CUDA graph (one launch instead of ~20 API
// calls per step).  Kernels run on a private stream ks; inside the graph each
// piece's download depends only on its own stream->bits kernel, so the copies
// overlap the remaining kernels.
struct StepBitsGraph {
    hga_run_args a;
    uint32_t *host_bits, *dev_bits;
    int64_t* state_out;
    int32_t* flag_out;
    int k;
    int dev;
    bool want_graph;
    cudaStream_t ks = nullptr, side = nullptr;
    cudaGraphExec_t exec = nullptr;
    // up[i]: piece i uploaded; down[i]: piece i downloaded; flag; gend: graph done; end; join; cap0/1: capture fork/join
    cudaEvent_t up[kStepBitsMaxChunks] = {}, down[kStepBitsMaxChunks] = {};
    cudaEvent_t flag = nullptr, gend = nullptr, end = nullptr, join = nullptr, cap0 = nullptr, cap1 = nullptr;
    cudaEvent_t fitup = nullptr;  // the fitness is uploaded
};

// the pinned 8-value state block in the tail of the host staging (128-byte aligned)
static int64_t* step_state_stage(uint32_t* host_bits, int64_t nwords) {
    return reinterpret_cast<int64_t*>(reinterpret_cast<char*>(host_bits) + (((size_t)nwords * 4 + 127) & ~(size_t)127));
}

static cudaError_t record(cudaEvent_t ev, cudaStream_t st, bool capturing) {
    return capturing ? cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal) : cudaEventRecord(ev, st);
}

// flag down, generation, new population -> stream -> host piece by piece, state down
static cudaError_t step_bits_tail(StepBitsGraph* g, bool capturing) {
    const hga_run_args* a = &g->a;
    const int m = a->m;
    const int64_t total = 4 * a->n_pairs;
    const StepPieces P(total, m, g->k);
    cudaStream_t ks = g->ks, sd = g->side;
    int32_t* dflag = &reinterpret_cast<RunWs2*>(a->ws)->host_flag;
    cudaError_t e = cudaMemcpyAsync(g->flag_out, dflag, sizeof(int32_t), cudaMemcpyDeviceToHost, ks);
    if (e == cudaSuccess) e = record(g->flag, ks, capturing);
    if (e != cudaSuccess) return e;
    hga_run_args r = *a;
    r.gens_this_call = 1;
    r.flags |= HGA_RUN_FORCE | kRunHostCheck;  // exactly one generation: the new population is in buffer 1
    const int rc = hga_run(&r, ks);  // (its select histogram was rebuilt during the upload)
    if (rc) return rc >= HGA_E_CUDA_BASE ? (cudaError_t)(rc - HGA_E_CUDA_BASE) : cudaErrorInvalidValue;
    const int W = words_for(m);
    for (int i = 0; i < P.k && e == cudaSuccess; ++i) {
        if (cols_to_bits(a->pop[1] + P.mlo[i] * m * W, P.mlo[i + 1] - P.mlo[i], m, g->dev_bits + P.wlo[i], dflag, ks))
            return cudaGetLastError();
        // the download of piece i waits for its own kernel only
        e = cudaEventRecord(g->cap0, ks);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(sd, g->cap0, 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(g->host_bits + P.wlo[i], g->dev_bits + P.wlo[i], (P.wlo[i + 1] - P.wlo[i]) * 4,
                                cudaMemcpyDeviceToHost, sd);
        if (e == cudaSuccess) e = record(g->down[i], sd, capturing);
    }
    if (e != cudaSuccess) return e;
    // a rejected population (NOT_GA): the fitness copy-back returns the uploaded values
    k_fit_restore_if<<<(unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)sm_count_cached() * 4), 256, 0, ks>>>(
        a->fit[0], a->fit[1], total, dflag);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(g->state_out, a->state, 8 * sizeof(int64_t), cudaMemcpyDeviceToHost, ks);
    if (e == cudaSuccess) e = cudaEventRecord(g->cap1, sd);  // join the download branch back
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ks, g->cap1, 0);
    return e;  // the fitness goes down outside the graph: the caller's array may not be page-locked
}

static void step_bits_free(StepBitsGraph* g) {
    if (g->exec) cudaGraphExecDestroy(g->exec);
    for (cudaEvent_t ev : g->up)
        if (ev) cudaEventDestroy(ev);
    for (cudaEvent_t ev : g->down)
        if (ev) cudaEventDestroy(ev);
    for (cudaEvent_t ev : {g->flag, g->gend, g->end, g->join, g->cap0, g->cap1, g->fitup})
        if (ev) cudaEventDestroy(ev);
    if (g->ks) cudaStreamDestroy(g->ks);
    if (g->side) cudaStreamDestroy(g->side);
    delete g;
}

// Cached per thread by every input of the device half (buffers, config,
// seed, piece count, device): a cached graph is exactly the work it stands for.
static StepBitsGraph* step_bits_graph(const hga_run_args* a, uint32_t* host_bits, uint32_t* dev_bits,
                                      int64_t* state_out, int32_t* flag_out, int k) {
    thread_local std::vector<StepBitsGraph*> cache;
    const int dev = current_device();
    // HGA_STEP_GRAPH=0 enqueues the same work call by call instead
    const char* env = std::getenv("HGA_STEP_GRAPH");
    const bool want_graph = !(env && env[0] == '0');
    for (size_t i = 0; i < cache.size(); ++i) {
        StepBitsGraph* g = cache[i];
        if (g->dev == dev && g->k == k && g->want_graph == want_graph && g->host_bits == host_bits &&
            g->dev_bits == dev_bits && g->state_out == state_out && g->flag_out == flag_out &&
            std::memcmp(&g->a, a, sizeof(hga_run_args)) == 0) {
            if (i) std::swap(cache[i], cache[0]);  // most recent first
            return g;
        }
    }
    StepBitsGraph* g = new StepBitsGraph();
    g->a = *a;
    g->host_bits = host_bits;
    g->dev_bits = dev_bits;
    g->state_out = state_out;
    g->flag_out = flag_out;
    g->k = k;
    g->dev = dev;
    g->want_graph = want_graph;
    bool ok = cudaStreamCreateWithFlags(&g->ks, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&g->side, cudaStreamNonBlocking) == cudaSuccess;
    for (int i = 0; i < kStepBitsMaxChunks && ok; ++i)
        ok = cudaEventCreateWithFlags(&g->up[i], cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&g->down[i], cudaEventDisableTiming) == cudaSuccess;
    for (cudaEvent_t* ev : {&g->flag, &g->gend, &g->end, &g->join, &g->cap0, &g->cap1, &g->fitup})
        ok = ok && cudaEventCreateWithFlags(ev, cudaEventDisableTiming) == cudaSuccess;
    if (!ok) {
        step_bits_free(g);
        cudaGetLastError();
        return nullptr;
    }
    if (want_graph) {
        cudaGraph_t graph = nullptr;
        if (cudaStreamBeginCapture(g->ks, cudaStreamCaptureModeRelaxed) == cudaSuccess) {
            const cudaError_t ce = step_bits_tail(g, true);
            const cudaError_t ee = cudaStreamEndCapture(g->ks, &graph);
            cudaError_t ie = cudaErrorUnknown;
            if (ce == cudaSuccess && ee == cudaSuccess && graph) {
                ie = cudaGraphInstantiate(&g->exec, graph, 0);
                if (ie != cudaSuccess) g->exec = nullptr;
            }
            if (std::getenv("HGA_STEP_TIMING"))
                std::fprintf(stderr, "hga_step_host_bits graph capture: enqueue %s, end %s, instantiate %s\n",
                             cudaGetErrorString(ce), cudaGetErrorString(ee), cudaGetErrorString(ie));
            if (graph) cudaGraphDestroy(graph);
        }
        cudaGetLastError();  // a refused capture leaves the call-by-call path
    }
    if (cache.size() >= 8) {
        step_bits_free(cache.back());
        cache.pop_back();
    }
    cache.insert(cache.begin(), g);
    return g;
}

struct StepUpload {  // callback context of the host pack
    StepBitsGraph* g;
    const StepPieces* P;
    cudaStream_t cs, user;
    int32_t* dflag;
    const int64_t* host_fit;
    const int64_t* st_stage;
    cudaError_t e;
};

// while the workers pack: join the caller's stream, reset the flag, state and
// fitness up, and the select histogram of the uploaded fitness rebuilt
static int step_upload_started(void* ctx) {
    StepUpload& u = *static_cast<StepUpload*>(ctx);
    StepBitsGraph* g = u.g;
    const hga_run_args* a = &g->a;
    const int64_t total = 4 * a->n_pairs;
    cudaError_t e = cudaEventRecord(g->join, u.user);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(g->ks, g->join, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(u.cs, g->join, 0);
    if (e == cudaSuccess) e = cudaMemsetAsync(u.dflag, 0, sizeof(int32_t), g->ks);
    if (e == cudaSuccess) e = cudaMemcpyAsync(a->state, u.st_stage, 8 * sizeof(int64_t), cudaMemcpyHostToDevice, g->ks);
    if (e == cudaSuccess) e = cudaMemcpyAsync(a->fit[0], u.host_fit, total * sizeof(int64_t), cudaMemcpyHostToDevice, u.cs);
    if (e == cudaSuccess) e = cudaEventRecord(g->fitup, u.cs);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(g->ks, g->fitup, 0);
    if (e == cudaSuccess) {
        hga_run_args r = *a;
        r.flags |= HGA_RUN_FORCE | kRunHostCheck;
        const int rc = hga_run_prepare(&r, g->ks);
        if (rc) e = rc >= HGA_E_CUDA_BASE ? (cudaError_t)(rc - HGA_E_CUDA_BASE) : cudaErrorInvalidValue;
    }
    u.e = e;
    return e == cudaSuccess ? 0 : 1;
}

// piece i is packed: upload it, then turn it into column records on ks
static int step_upload_piece(void* ctx, int i) {
    StepUpload& u = *static_cast<StepUpload*>(ctx);
    StepBitsGraph* g = u.g;
    const int m = g->a.m;
    cudaError_t e = cudaMemcpyAsync(g->dev_bits + u.P->wlo[i], g->host_bits + u.P->wlo[i],
                                    (u.P->wlo[i + 1] - u.P->wlo[i]) * 4, cudaMemcpyHostToDevice, u.cs);
    if (e == cudaSuccess) e = cudaEventRecord(g->up[i], u.cs);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(g->ks, g->up[i], 0);
    if (e == cudaSuccess &&
        bits_to_cols(g->dev_bits + u.P->wlo[i], u.P->mlo[i + 1] - u.P->mlo[i], m,
                     g->a.pop[0] + u.P->mlo[i] * m * words_for(m), u.dflag, g->ks))
        e = cudaGetLastError();
    u.e = e;
    return e == cudaSuccess ? 0 : 1;
}

static int step_piece_landed(void* ctx, int i) {
    StepBitsGraph* g = static_cast<StepBitsGraph*>(ctx);
    return cudaEventSynchronize(g->down[i]) == cudaSuccess ? 0 : 1;
}

}  // namespace hga

using namespace hga;

static bool valid_var(uint32_t v) { return v == HGA_VAR_F1 || v == HGA_VAR_F2 || v == HGA_VAR_SQ; }

extern "C" {

int hga_generation_explicit(uint32_t* pop, int64_t* fit, int64_t n_pairs, int32_t m, const int64_t* points,
                            const int64_t* cols, const int64_t* ra, const int64_t* rb, int32_t nc, int32_t nr,
                            uint32_t fit_var, unsigned long long* best_key, void* stream) {
    if (n_pairs < 0 || m < 2 || m > 32 * kMaxRegWords || nc < 1 || nr < 1 || nc > 4096 || nr > 4096 ||
        !valid_var(fit_var))
        return HGA_E_INVALID;
    if (n_pairs == 0) return HGA_OK;
    cudaStream_t st = (cudaStream_t)stream;
    switch (words_for(m)) {
        case 1: return launch_explicit_w<1>(pop, fit, n_pairs, m, points, cols, ra, rb, nc, nr, fit_var, best_key, st);
        case 2: return launch_explicit_w<2>(pop, fit, n_pairs, m, points, cols, ra, rb, nc, nr, fit_var, best_key, st);
        case 3: return launch_explicit_w<3>(pop, fit, n_pairs, m, points, cols, ra, rb, nc, nr, fit_var, best_key, st);
        default: return launch_explicit_w<4>(pop, fit, n_pairs, m, points, cols, ra, rb, nc, nr, fit_var, best_key, st);
    }
}

size_t hga_run_ws_bytes(int64_t n_pairs, int32_t m) {
    (void)m;
    // two-barrier survivor lists (2 x 4N uint64) + one-barrier keys (2 x stride uint16)
    return std::max(run_ws_head() + (size_t)(2 * n_pairs) * 8,
                    run_ws2_head() + (size_t)(8 * n_pairs) * 8 + (size_t)run2_key_stride(n_pairs) * 4);
}


static int run_args_ok(const hga_run_args* a) {
    if (!a || a->n_pairs < 1 || a->m < 4 || a->m > 32 * kMaxRegWords || (a->m & 3) || !valid_var(a->fit_var))
        return 0;
    if (a->strategy < 0 || a->strategy > 2 || a->nc < 1 || a->nc > a->m - 1 || a->nr < 1 || a->nr > a->m / 2) return 0;
    if (4 * a->n_pairs >= ((int64_t)1 << 31)) return 0;  // 32-bit slot ids in the select keys
    if (bit_length(max_fitness(a->m, a->fit_var)) > 24) return 0;
    if (!a->pop[0] || !a->pop[1] || !a->fit[0] || !a->fit[1] || !a->state || !a->best_matrix || !a->ws) return 0;
    if (a->ws_bytes < hga_run_ws_bytes(a->n_pairs, a->m)) return 0;
    return 1;
}

int64_t hga_run_timing_offset(int32_t m) {
    if (m < 4 || m > 64 || (m & 3)) return -1;
    return (int64_t)offsetof(RunWs2, tstamp);
}

int hga_run_prepare(const hga_run_args* a, void* stream) {
    if (!run_args_ok(a)) return HGA_E_INVALID;
    if (!run2_supported(a)) {
        // v1 keeps no cross-generation histogram; only the keys need a reset
        RunWs* ws = (RunWs*)a->ws;
        cudaStream_t st = (cudaStream_t)stream;
        cudaError_t e = cudaMemsetAsync(ws, 0, sizeof(Barrier), st);
        if (e == cudaSuccess) e = cudaMemsetAsync(&ws->best_key[0], 0xFF, 5 * sizeof(unsigned long long), st);
        if (e == cudaSuccess) e = cudaMemsetAsync(&ws->hist1[0], 0, 2 * kHistBins * sizeof(uint32_t), st);
        return to_rc(e);
    }
    return run2_prepare(a, (cudaStream_t)stream);
}

int hga_run_init(const hga_run_args* a, void* stream) {
    if (!run_args_ok(a)) return HGA_E_INVALID;
    cudaStream_t st = (cudaStream_t)stream;
    const int m = a->m, W = words_for(m);
    const int64_t total = 4 * a->n_pairs;
    const int64_t work = total * m;
    const int grid = (int)std::min<int64_t>((work + 255) / 256, (int64_t)sm_count_cached() * 16);
    switch (W) {
        case 1: k_philox_init<1><<<grid, 256, 0, st>>>(a->seed, (uint32_t)kPInit, 0, 0, total, m, a->pop[0]); break;
        case 2: k_philox_init<2><<<grid, 256, 0, st>>>(a->seed, (uint32_t)kPInit, 0, 0, total, m, a->pop[0]); break;
        case 3: k_philox_init<3><<<grid, 256, 0, st>>>(a->seed, (uint32_t)kPInit, 0, 0, total, m, a->pop[0]); break;
        default: k_philox_init<4><<<grid, 256, 0, st>>>(a->seed, (uint32_t)kPInit, 0, 0, total, m, a->pop[0]); break;
    }
    int rc = hga_fitness_packed(a->pop[0], total, m, a->fit_var, a->fit_var == HGA_VAR_F1 ? a->fit[0] : nullptr,
                                a->fit_var == HGA_VAR_F2 ? a->fit[0] : nullptr, nullptr,
                                a->fit_var == HGA_VAR_SQ ? a->fit[0] : nullptr, stream);
    if (rc) return rc;
    RunWs* ws = (RunWs*)a->ws;
    unsigned long long* key = &ws->restart_key;
    cudaError_t e = cudaMemsetAsync(key, 0xFF, 8, st);
    if (e != cudaSuccess) return to_rc(e);
    k_argmin_key2<<<(int)std::min<int64_t>((total + 255) / 256, sm_count_cached() * 8), 256, 0, st>>>(a->fit[0], total, key);
    k_run_finish_init<<<1, 256, 0, st>>>(*a, W, key, ws);
    rc = to_rc(cudaGetLastError());
    if (rc) return rc;
    if (run2_supported(a)) return run2_prepare(a, st);
    return HGA_OK;
}

int hga_step_host(const hga_run_args* a, int8_t* host_pop, int64_t* host_fit, int8_t* dev_i8,
                  const int64_t* state_in, int64_t* state_out, int32_t* flag_out, int32_t chunks, void* stream,
                  void* copy_stream) {
    if (!run_args_ok(a) || !host_pop || !host_fit || !dev_i8 || !state_in || !state_out || !flag_out || chunks < 1)
        return HGA_E_INVALID;
    if (!run2_supported(a)) return HGA_E_UNSUPPORTED;  // orders > 64 keep the torch-side path
    cudaStream_t st = (cudaStream_t)stream, cs = (cudaStream_t)copy_stream;
    const int m = a->m, W = words_for(m);
    const int64_t total = 4 * a->n_pairs, mm = (int64_t)m * m, mw = (int64_t)m * W;
    const int k = (int)std::min<int64_t>(chunks, total);
    int32_t* dflag = &reinterpret_cast<RunWs2*>(a->ws)->host_flag;
    // events: one per download piece plus three stream joins; kept in a per-thread
    // pool (creating ~20 events per call costs tens of microseconds)
    thread_local std::vector<cudaEvent_t> pool;
    while ((int)pool.size() < 2 * k + 3) {
        cudaEvent_t ne;
        const cudaError_t ce = cudaEventCreateWithFlags(&ne, cudaEventDisableTiming);
        if (ce != cudaSuccess) return to_rc(ce);
        pool.push_back(ne);
    }
    cudaEvent_t* ev = pool.data();
    auto done = [](int rc) { return rc; };
    // HGA_STEP_TIMING=1: print the stream timeline of this call (diagnostics)
    const bool tm = std::getenv("HGA_STEP_TIMING") != nullptr;
    cudaEvent_t te[6];
    if (tm)
        for (auto& t : te) cudaEventCreate(&t);
    if (tm) cudaEventRecord(te[0], st);
    cudaError_t e = cudaEventRecord(ev[2 * k], st);  // the staging buffers are free once prior work is done
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ev[2 * k], 0);
    if (e == cudaSuccess) e = cudaMemsetAsync(dflag, 0, sizeof(int32_t), st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(a->fit[0], host_fit, total * sizeof(int64_t), cudaMemcpyHostToDevice, cs);
    // upload in one piece (splitting it costs more than the ~12 us of packing it would hide)
    if (e == cudaSuccess) e = cudaMemcpyAsync(dev_i8, host_pop, total * mm, cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess) e = cudaEventRecord(ev[0], cs);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ev[0], 0);
    if (e == cudaSuccess) {
        const int rc = hga_pack_i8(dev_i8, total, m, a->pop[0], dflag, st);
        if (rc) return done(rc);
    }
    if (e != cudaSuccess) return done(to_rc(e));
    // The pack validated the upload (dflag): the loop's fast paths need the GA
    // invariants (column 0 skipped in the pair chain, fitness >> granule keys).
    // On a violation the generation and the unpack do nothing and the fitness
    // copy-back returns the uploaded values, so the host arrays get their own
    // bytes back; the caller then runs the exact explicit-plan generation.
    // Decided on the device: no host round trip in the middle of the step.
    if (tm) cudaEventRecord(te[1], cs);
    if (tm) cudaEventRecord(te[2], st);
    k_set_state<<<1, 8, 0, st>>>(a->state, state_in[0], state_in[1], state_in[2], state_in[6], state_in[7]);
    hga_run_args r = *a;
    r.gens_this_call = 1;
    r.flags |= HGA_RUN_FORCE | kRunHostCheck;  // exactly one generation: the new population is in buffer 1
    int rc = hga_run_prepare(&r, st);
    if (!rc) rc = hga_run(&r, st);
    if (rc) return done(rc);
    if (tm) cudaEventRecord(te[3], st);
    for (int i = 0; i < k && e == cudaSuccess; ++i) {
        const int64_t lo = total * i / k, hi = total * (i + 1) / k;
        rc = unpack_i8_guarded(a->pop[1] + lo * mw, hi - lo, m, dev_i8 + lo * mm, dflag, st);
        if (rc) return done(rc);
        e = cudaEventRecord(ev[k + i], st);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ev[k + i], 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(host_pop + lo * mm, dev_i8 + lo * mm, (hi - lo) * mm, cudaMemcpyDeviceToHost, cs);
    }
    if (e == cudaSuccess) {
        k_fit_restore_if<<<(unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)sm_count_cached() * 4), 256, 0,
                           st>>>(a->fit[0], a->fit[1], total, dflag);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaEventRecord(ev[2 * k + 1], st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ev[2 * k + 1], 0);
    if (e == cudaSuccess) e = cudaMemcpyAsync(host_fit, a->fit[1], total * sizeof(int64_t), cudaMemcpyDeviceToHost, cs);
    if (e == cudaSuccess) e = cudaMemcpyAsync(state_out, a->state, 8 * sizeof(int64_t), cudaMemcpyDeviceToHost, cs);
    if (e == cudaSuccess) e = cudaMemcpyAsync(flag_out, dflag, sizeof(int32_t), cudaMemcpyDeviceToHost, cs);
    if (tm) cudaEventRecord(te[4], st);
    if (tm) cudaEventRecord(te[5], cs);
    if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
    if (tm) {
        float ms[5];
        for (int i = 1; i < 6; ++i) cudaEventElapsedTime(&ms[i - 1], te[0], te[i]);
        std::fprintf(stderr, "hga_step_host us: h2d_done %.1f packs_done %.1f run_done %.1f unpacks_done %.1f d2h_done %.1f\n",
                     ms[0] * 1e3, ms[1] * 1e3, ms[2] * 1e3, ms[3] * 1e3, ms[4] * 1e3);
        for (auto& t : te) cudaEventDestroy(t);
    }
    return done(to_rc(e));
}

size_t hga_step_host_bits_bytes(int64_t n_pairs, int32_t m) {
    if (n_pairs < 1 || m < 4 || m > 64 || (m & 3)) return 0;
    const int64_t nbytes = 4 * n_pairs * (int64_t)m * m;
    return (size_t)((nbytes + 31) / 32) * 4 + kStepBitsTail;  // + the pinned state block
}

int hga_step_host_bits(const hga_run_args* a, int8_t* host_pop, int64_t* host_fit, uint32_t* host_bits,
                       uint32_t* dev_bits, const int64_t* state_in, int64_t* state_out, int32_t* flag_out,
                       int32_t chunks, void* stream, void* copy_stream) {
    if (!run_args_ok(a) || !host_pop || !host_fit || !host_bits || !dev_bits || !state_in || !state_out || !flag_out ||
        chunks < 1 || !copy_stream)
        return HGA_E_INVALID;
    if (!run2_supported(a) || (a->m & 3)) return HGA_E_UNSUPPORTED;
    const int m = a->m;
    const int64_t total = 4 * a->n_pairs, nbytes = total * (int64_t)m * m, nwords = (nbytes + 31) / 32;
    const StepPieces P(total, m, chunks);
    const bool tm = std::getenv("HGA_STEP_TIMING") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    const auto t0 = now();
    StepBitsGraph* g = step_bits_graph(a, host_bits, dev_bits, state_out, flag_out, P.k);
    if (!g) return HGA_E_CUDA_BASE + (int)cudaErrorUnknown;
    cudaStream_t cs = (cudaStream_t)copy_stream, ks = g->ks;
    int32_t* dflag = &reinterpret_cast<RunWs2*>(a->ws)->host_flag;
    // the previous call on this staging has completed (its end event was synchronised)
    *flag_out = 0;
    int64_t* st_stage = step_state_stage(host_bits, nwords);
    const int64_t sv[8] = {state_in[0], state_in[1], state_in[2], 0, 0, 0, state_in[6], state_in[7]};
    for (int i = 0; i < 8; ++i) st_stage[i] = sv[i];
    // host: validate + pack the pieces on the pool; meanwhile this thread queues the
    // device work that does not need the population (after the work already queued
    // on `stream`), then uploads each packed piece and turns it into column records
    // while the next ones are still being packed
    StepUpload up{g, &P, cs, (cudaStream_t)stream, dflag, host_fit, st_stage, cudaSuccess};
    const int prc = host_pack_pieces(host_pop, nbytes, host_bits, P.wlo, P.k, step_upload_started, step_upload_piece, &up);
    cudaError_t e = cudaSuccess;
    const auto t1 = now();
    if (prc) {
        e = cudaStreamSynchronize(cs);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ks);
        if (prc == 1) {  // an entry is not +-1: nothing that could touch the caller's arrays was enqueued
            *flag_out = HGA_FLAG_NOT_SIGN;
            return to_rc(e);
        }
        return to_rc(up.e != cudaSuccess ? up.e : cudaErrorUnknown);
    }
    e = g->exec ? cudaGraphLaunch(g->exec, ks) : step_bits_tail(g, false);
    if (e == cudaSuccess) e = cudaEventRecord(g->gend, ks);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, g->gend, 0);
    if (e == cudaSuccess) e = cudaMemcpyAsync(host_fit, a->fit[1], total * sizeof(int64_t), cudaMemcpyDeviceToHost, cs);
    if (e == cudaSuccess) e = cudaEventRecord(g->end, cs);
    if (e != cudaSuccess) return to_rc(e);
    const auto t2 = now();
    // host: the validation flag first (on NOT_GA the caller's population stays as it is), then
    // unpack each piece on the pool as soon as it has landed while later pieces are in flight
    e = cudaEventSynchronize(g->flag);
    if (e != cudaSuccess) return to_rc(e);
    const auto t3 = now();
    int urc = 0;
    if (!(*flag_out & (HGA_FLAG_NOT_SIGN | HGA_FLAG_NOT_GA)))
        urc = host_unpack_pieces(host_bits, host_pop, nbytes, P.wlo, P.k, step_piece_landed, g);
    const auto t4 = now();
    e = cudaEventSynchronize(g->end);
    if (e == cudaSuccess && urc) e = cudaErrorUnknown;
    if (tm) {
        auto us = [&](std::chrono::steady_clock::time_point x) {
            return std::chrono::duration<double, std::micro>(x - t0).count();
        };
        std::fprintf(stderr,
                     "hga_step_host_bits us: packed+uploaded %.1f launched %.1f flag %.1f unpacked %.1f done %.1f "
                     "(%d pieces, %d host threads, graph %d)\n",
                     us(t1), us(t2), us(t3), us(t4), us(now()), P.k, host_pool_threads(), g->exec != nullptr);
    }
    return to_rc(e);
}

int hga_philox_init_packed(uint64_t seed, uint64_t purpose, uint64_t generation, int64_t first_slot,
                           int64_t count, int32_t m, uint32_t* cols, void* stream) {
    if (count < 0 || first_slot < 0 || m < 1 || m > 32 * kMaxRegWords) return HGA_E_INVALID;
    if (count == 0) return HGA_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t work = count * m;
    const int grid = (int)std::min<int64_t>((work + 255) / 256, (int64_t)sm_count_cached() * 16);
    // cols points at slot 0 of the population; slots [first_slot, first_slot + count) are written
    switch (words_for(m)) {
        case 1: k_philox_init<1><<<grid, 256, 0, st>>>(seed, (uint32_t)purpose, generation, first_slot, count, m, cols); break;
        case 2: k_philox_init<2><<<grid, 256, 0, st>>>(seed, (uint32_t)purpose, generation, first_slot, count, m, cols); break;
        case 3: k_philox_init<3><<<grid, 256, 0, st>>>(seed, (uint32_t)purpose, generation, first_slot, count, m, cols); break;
        default: k_philox_init<4><<<grid, 256, 0, st>>>(seed, (uint32_t)purpose, generation, first_slot, count, m, cols); break;
    }
    return to_rc(cudaGetLastError());
}

int hga_run(const hga_run_args* a, void* stream) {
    if (!run_args_ok(a)) return HGA_E_INVALID;
    if (a->gens_this_call <= 0) return HGA_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (run2_supported(a)) return launch_run_v2(a, st);
    switch (words_for(a->m)) {
        case 1: return launch_run_w<1>(a, st);
        case 2: return launch_run_w<2>(a, st);
        case 3: return launch_run_w<3>(a, st);
        default: return launch_run_w<4>(a, st);
    }
}

}  // extern "C"
