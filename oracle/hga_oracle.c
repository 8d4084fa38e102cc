/*
 * hga_oracle.c -- CPU restatement of the reference GA inner loop.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity oracle and the CPU
 * baseline ("kind": "port") for bench.py.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product path (paper_2208_14961_b200) never links or calls it.
 *
 * It restates, in plain scalar C over the reference's own int8 row-major
 * (count, m, m) layout, the algorithms of the upstream Python package
 * hadamard_ga (reference: /root/reference/pkg/src/hadamard_ga):
 *
 *   counter streams ........ rand.py:39-77   (splitmix64 finalizer, keys, words)
 *   bounded draws .......... rand.py:116-129 (lo + word % span)
 *   permutation ............ rand.py:131-140 (forward Fisher-Yates)
 *   stream-id packing ...... engine.py:60-90 (4 | 28 | 20 | 12 bits)
 *   balanced init .......... engine.py:154-182
 *   fitness ................ engine.py:200-213, core.py:59-89 (exact integer Gram)
 *   select ................. engine.py:233-248 (stable argsort, permuted gather)
 *   crossover .............. engine.py:251-277
 *   mutation plan / mutate . engine.py:305-373
 *   step ................... engine.py:449-469
 *
 * Pinned against tests/golden/golden.npz, which tests/golden/make_golden.py
 * produced by running the unmodified reference package.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORA_GOLDEN 0x9E3779B97F4A7C15ULL
#define ORA_SEED_SALT 0x5851F42D4C957F2DULL
#define ORA_STREAM_SALT 0x14057B7EF767814FULL

/* ------------------------------------------------------------------ rng */

static inline uint64_t ora_mix(uint64_t x) {
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

uint64_t ora_mix64(uint64_t x) { return ora_mix(x); }

uint64_t ora_stream_key(uint64_t seed, uint64_t sid) {
    uint64_t a = ora_mix(seed ^ ORA_SEED_SALT);
    uint64_t b = ora_mix(sid * ORA_GOLDEN + ORA_STREAM_SALT);
    return ora_mix(a ^ b);
}

static inline uint64_t ora_word(uint64_t key, uint64_t counter) {
    return ora_mix(key + counter * ORA_GOLDEN);
}

void ora_stream_words(uint64_t key, uint64_t c0, int64_t n, uint64_t *out) {
    for (int64_t i = 0; i < n; ++i) out[i] = ora_word(key, c0 + (uint64_t)i);
}

void ora_uniform(uint64_t seed, uint64_t sid, uint64_t c0, int64_t lo, int64_t hi,
                 int64_t n, int64_t *out) {
    uint64_t key = ora_stream_key(seed, sid);
    uint64_t span = (uint64_t)(hi - lo) + 1;
    for (int64_t i = 0; i < n; ++i) out[i] = lo + (int64_t)(ora_word(key, c0 + (uint64_t)i) % span);
}

void ora_permutation(uint64_t seed, uint64_t sid, uint64_t c0, int64_t n, int64_t *out) {
    uint64_t key = ora_stream_key(seed, sid);
    for (int64_t i = 0; i < n; ++i) out[i] = i;
    for (int64_t a = 0; a + 1 < n; ++a) {
        int64_t b = a + (int64_t)(ora_word(key, c0 + (uint64_t)a) % (uint64_t)(n - a));
        int64_t t = out[a];
        out[a] = out[b];
        out[b] = t;
    }
}

/* purpose | generation | matrix | column, widths 4 | 28 | 20 | 12 */
uint64_t ora_sid(uint64_t purpose, uint64_t generation, uint64_t matrix, uint64_t column) {
    return (purpose << 60) | (generation << 32) | (matrix << 12) | column;
}

/* ------------------------------------------------------------------ init */

void ora_random_balanced(int32_t m, int64_t count, uint64_t seed, uint64_t purpose,
                         uint64_t generation, int64_t first_slot, int8_t *out) {
    const int64_t mm = (int64_t)m * m;
    for (int64_t s = 0; s < count; ++s) {
        int8_t *q = out + s * mm;
        for (int r = 0; r < m; ++r)
            for (int c = 0; c < m; ++c) q[r * m + c] = (c > 0 && r < m / 2) ? -1 : 1;
        for (int c = 1; c < m; ++c) {
            uint64_t key = ora_stream_key(seed, ora_sid(purpose, generation,
                                                        (uint64_t)(first_slot + s), (uint64_t)c));
            /* one sequential Fisher-Yates per (slot, column) stream */
            for (int a = 0; a + 1 < m; ++a) {
                int b = a + (int)(ora_word(key, (uint64_t)a) % (uint64_t)(m - a));
                int8_t t = q[a * m + c];
                q[a * m + c] = q[b * m + c];
                q[b * m + c] = t;
            }
        }
    }
}

/* ------------------------------------------------------------------ fitness */

/* Exact off-diagonal penalties of one matrix from its integer Gram.
 * f1 = sum|G| - m^2, f2 = nnz(G) - m, orth = #{i<j : g_ij = 0},
 * sq = sum_{i != j} g_ij^2.  Works for any int8 entries. */
static void ora_one(const int8_t *q, int32_t m, int32_t *colbuf, int64_t *pen) {
    for (int c = 0; c < m; ++c)
        for (int r = 0; r < m; ++r) colbuf[(int64_t)c * m + r] = q[(int64_t)r * m + c];
    int64_t f1 = 0, f2 = 0, orth = 0, sq = 0;
    for (int i = 0; i < m; ++i) {
        const int32_t *ci = colbuf + (int64_t)i * m;
        int64_t d = 0;
        for (int r = 0; r < m; ++r) d += (int64_t)ci[r] * ci[r];
        f1 += (d < 0 ? -d : d);
        f2 += (d != 0);
        for (int j = i + 1; j < m; ++j) {
            const int32_t *cj = colbuf + (int64_t)j * m;
            int64_t g = 0;
            for (int r = 0; r < m; ++r) g += (int64_t)ci[r] * cj[r];
            f1 += 2 * (g < 0 ? -g : g);
            f2 += 2 * (g != 0);
            orth += (g == 0);
            sq += 2 * g * g;
        }
    }
    pen[0] = f1 - (int64_t)m * m;
    pen[1] = f2 - m;
    pen[2] = orth;
    pen[3] = sq;
}

void ora_penalties(const int8_t *pop, int64_t n, int32_t m, int64_t *f1, int64_t *f2,
                   int64_t *orth, int64_t *sq, int32_t threads) {
    const int64_t mm = (int64_t)m * m;
#ifdef _OPENMP
    if (threads < 1) threads = 1;
#pragma omp parallel num_threads(threads)
#endif
    {
        int32_t *colbuf = (int32_t *)malloc(sizeof(int32_t) * (size_t)(mm > 0 ? mm : 1));
        int64_t pen[4];
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
        for (int64_t k = 0; k < n; ++k) {
            ora_one(pop + k * mm, m, colbuf, pen);
            if (f1) f1[k] = pen[0];
            if (f2) f2[k] = pen[1];
            if (orth) orth[k] = pen[2];
            if (sq) sq[k] = pen[3];
        }
        free(colbuf);
    }
}

/* fitness codes: 0 = f1, 1 = f2, 2 = orth, 3 = sq */
void ora_evaluate(const int8_t *pop, int64_t n, int32_t m, int32_t fitness, int64_t *out,
                  int32_t threads) {
    int64_t *slots[4] = {0, 0, 0, 0};
    slots[fitness & 3] = out;
    ora_penalties(pop, n, m, slots[0], slots[1], slots[2], slots[3], threads);
}

/* ------------------------------------------------------------------ select */

typedef struct {
    int64_t f;
    int64_t i;
} ora_key;

static int ora_key_cmp(const void *pa, const void *pb) {
    const ora_key *a = (const ora_key *)pa, *b = (const ora_key *)pb;
    if (a->f != b->f) return a->f < b->f ? -1 : 1;
    return a->i < b->i ? -1 : (a->i > b->i);
}

/* Winners of select in parent-slot order: chosen[s] = order[perm[s]],
 * order = stable argsort(fitness)[:total/2]. */
void ora_select_indices(const int64_t *fit, int64_t total, uint64_t seed, uint64_t sid,
                        uint64_t c0, int64_t *chosen) {
    int64_t half = total / 2;
    ora_key *keys = (ora_key *)malloc(sizeof(ora_key) * (size_t)(total > 0 ? total : 1));
    for (int64_t i = 0; i < total; ++i) {
        keys[i].f = fit[i];
        keys[i].i = i;
    }
    qsort(keys, (size_t)total, sizeof(ora_key), ora_key_cmp); /* (f, index): stable order */
    int64_t *perm = (int64_t *)malloc(sizeof(int64_t) * (size_t)(half > 0 ? half : 1));
    ora_permutation(seed, sid, c0, half, perm);
    for (int64_t s = 0; s < half; ++s) chosen[s] = keys[perm[s]].i;
    free(perm);
    free(keys);
}

void ora_select(int8_t *pop, int64_t *fit, int64_t total, int32_t m, uint64_t seed,
                uint64_t sid, uint64_t c0) {
    int64_t half = total / 2;
    const int64_t mm = (int64_t)m * m;
    int64_t *chosen = (int64_t *)malloc(sizeof(int64_t) * (size_t)(half > 0 ? half : 1));
    ora_select_indices(fit, total, seed, sid, c0, chosen);
    /* out-of-place gather, then copy back: the reference's fancy index copies */
    int8_t *tmp = (int8_t *)malloc((size_t)(half * mm > 0 ? half * mm : 1));
    int64_t *ftmp = (int64_t *)malloc(sizeof(int64_t) * (size_t)(half > 0 ? half : 1));
    for (int64_t s = 0; s < half; ++s) {
        memcpy(tmp + s * mm, pop + chosen[s] * mm, (size_t)mm);
        ftmp[s] = fit[chosen[s]];
    }
    memcpy(pop, tmp, (size_t)(half * mm));
    memcpy(fit, ftmp, sizeof(int64_t) * (size_t)half);
    free(ftmp);
    free(tmp);
    free(chosen);
}

/* ------------------------------------------------------------------ crossover */

/* returns 0, or -1 (bad point) */
int ora_crossover(int8_t *pop, int64_t total, int32_t m, const int64_t *points) {
    int64_t np_ = total / 4;
    const int64_t mm = (int64_t)m * m;
    for (int64_t p = 0; p < np_; ++p)
        if (points[p] < 1 || points[p] > m - 1) return -1;
    for (int64_t p = 0; p < np_; ++p) {
        const int8_t *a = pop + p * mm, *b = pop + (np_ + p) * mm;
        int8_t *o1 = pop + (2 * np_ + p) * mm, *o2 = pop + (3 * np_ + p) * mm;
        int64_t c = points[p];
        for (int r = 0; r < m; ++r)
            for (int j = 0; j < m; ++j) {
                int64_t e = (int64_t)r * m + j;
                o1[e] = j < c ? a[e] : b[e];
                o2[e] = j < c ? b[e] : a[e];
            }
    }
    return 0;
}

/* ------------------------------------------------------------------ mutation */

/* strategy: 0 = shared, 1 = per-matrix, 2 = multi.  Output shapes are
 * (n_off, w) with w = 1 for shared / per-matrix, nc (cols) or nr (rows)
 * for multi. */
void ora_mutation_plan(int32_t m, int64_t n_off, int32_t nc, int32_t nr, int32_t strategy,
                       uint64_t seed, uint64_t generation, int64_t *cols, int64_t *ra,
                       int64_t *rb) {
    uint64_t sc = ora_sid(4, generation, 0, 0), sa = ora_sid(5, generation, 0, 0),
             sb = ora_sid(6, generation, 0, 0);
    if (strategy == 0) {
        int64_t c, a, b;
        ora_uniform(seed, sc, 0, 1, m - 1, 1, &c);
        ora_uniform(seed, sa, 0, 0, m - 1, 1, &a);
        ora_uniform(seed, sb, 0, 0, m - 1, 1, &b);
        for (int64_t o = 0; o < n_off; ++o) {
            cols[o] = c;
            ra[o] = a;
            rb[o] = b;
        }
        return;
    }
    if (strategy == 1) nc = nr = 1;
    ora_uniform(seed, sc, 0, 1, m - 1, n_off * nc, cols);
    ora_uniform(seed, sa, 0, 0, m - 1, n_off * nr, ra);
    ora_uniform(seed, sb, 0, 0, m - 1, n_off * nr, rb);
}

/* returns 0, or -1 (index out of range) */
int ora_mutate(int8_t *pop, int64_t total, int32_t m, const int64_t *cols, const int64_t *ra,
               const int64_t *rb, int32_t nc, int32_t nr) {
    int64_t half = total / 2;
    const int64_t mm = (int64_t)m * m;
    for (int64_t i = 0; i < half * nc; ++i)
        if (cols[i] < 1 || cols[i] > m - 1) return -1;
    for (int64_t i = 0; i < half * nr; ++i)
        if (ra[i] < 0 || ra[i] > m - 1 || rb[i] < 0 || rb[i] > m - 1) return -1;
    for (int64_t o = 0; o < half; ++o) {
        int8_t *q = pop + (half + o) * mm;
        for (int jc = 0; jc < nc; ++jc) {
            int64_t c = cols[o * nc + jc];
            for (int ir = 0; ir < nr; ++ir) {
                int8_t *x = q + ra[o * nr + ir] * m + c, *y = q + rb[o * nr + ir] * m + c;
                if (*x != *y) {
                    int8_t t = *x;
                    *x = *y;
                    *y = t;
                }
            }
        }
    }
    return 0;
}

/* ------------------------------------------------------------------ step */

/* One generation (engine.py:449-469) on (total, m, m) int8 with a current
 * fitness vector.  Returns argmin index of the new fitness (first minimum). */
int64_t ora_step(int8_t *pop, int64_t *fit, int64_t total, int32_t m, uint64_t seed,
                 uint64_t generation, int32_t nc, int32_t nr, int32_t strategy, int32_t fitness,
                 int32_t threads) {
    int64_t np_ = total / 4, half = total / 2;
    ora_select(pop, fit, total, m, seed, ora_sid(2, generation, 0, 0), 0);
    int64_t *pts = (int64_t *)malloc(sizeof(int64_t) * (size_t)(np_ > 0 ? np_ : 1));
    ora_uniform(seed, ora_sid(3, generation, 0, 0), 0, 1, m - 1, np_, pts);
    ora_crossover(pop, total, m, pts);
    free(pts);
    int32_t wc = strategy == 2 ? nc : 1, wr = strategy == 2 ? nr : 1;
    int64_t *cols = (int64_t *)malloc(sizeof(int64_t) * (size_t)(half * wc));
    int64_t *ra = (int64_t *)malloc(sizeof(int64_t) * (size_t)(half * wr));
    int64_t *rb = (int64_t *)malloc(sizeof(int64_t) * (size_t)(half * wr));
    ora_mutation_plan(m, half, nc, nr, strategy, seed, generation, cols, ra, rb);
    ora_mutate(pop, total, m, cols, ra, rb, wc, wr);
    free(cols);
    free(ra);
    free(rb);
    ora_evaluate(pop + half * (int64_t)m * m, half, m, fitness, fit + half, threads);
    int64_t best = 0;
    for (int64_t i = 1; i < total; ++i)
        if (fit[i] < fit[best]) best = i;
    return best;
}

int32_t ora_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
