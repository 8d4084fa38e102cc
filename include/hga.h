/*
 * hga.h -- C ABI of libhga.so, the sm_100a Hadamard-GA inner loop.
 *
 * The reference (hadamard_ga, pure Python/NumPy) has no FFI of its own; its
 * "plugin API" is the Python function surface of engine.py:34-55.  Each entry
 * point below replaces the body of one of those functions (cited per entry),
 * so a maintainer can bind it from hadamard_ga with ctypes.
 *
 * Conventions
 *   - extern "C", plain pointers and sizes, no torch types.
 *   - Every pointer named *pop, *cols, *fit, *out, ... is a DEVICE pointer
 *     (cudaMalloc / torch tensor .data_ptr()).  The library never allocates
 *     device or pinned memory; scratch is passed in after a *_ws_bytes query.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *     asynchronous on that stream and never synchronize the host -- except
 *     the host-state steps (hga_step_host*), which return with the caller's
 *     host arrays updated.  hga_step_host_bits keeps, per calling thread, a
 *     small cache of CUDA graphs / private streams / events keyed by its
 *     buffers, and uses one process-wide host thread pool (calls from
 *     several threads are serialised on it).
 *   - Return 0 (HGA_OK) or an error code; argument errors are detected on the
 *     host before any launch.  Data-dependent errors (a point or plan index
 *     out of range, an entry that is not +-1) are reported through an optional
 *     device int32 flag the caller reads after synchronizing.
 *   - Population layouts: "i8" is the reference's int8 (n, m, m) row-major
 *     array (engine.py:1-21); "packed" is the resident layout of
 *     paper_2208_14961_b200/csrc/hga_common.cuh: m column records of
 *     W = ceil(m/32) uint32 words per matrix, bit r%32 of word r/32 set iff
 *     entry (r, j) is -1.
 */
#ifndef HGA_H
#define HGA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HGA_ABI_VERSION 1

/* return codes */
#define HGA_OK 0
#define HGA_E_INVALID 1      /* bad size / shape / enum argument */
#define HGA_E_UNSUPPORTED 2  /* order or size outside what this build handles */
#define HGA_E_WORKSPACE 3    /* workspace too small */
#define HGA_E_CUDA_BASE 1000 /* HGA_E_CUDA_BASE + cudaError_t */

/* penalty variants (bit mask).  F1 = sum|G| - m^2 (core.py:70-78),
 * F2 = nnz(G) - m (core.py:81-89), ORTH = #{i<j : g_ij = 0},
 * SQ = sum_{i != j} g_ij^2. */
#define HGA_VAR_F1 1u
#define HGA_VAR_F2 2u
#define HGA_VAR_ORTH 4u
#define HGA_VAR_SQ 8u
#define HGA_VAR_ALL 15u

/* device error-flag bits */
#define HGA_FLAG_NOT_SIGN 1     /* an entry is not +1/-1 */
#define HGA_FLAG_POINT_RANGE 2  /* crossover point outside [1, m-1] */
#define HGA_FLAG_PLAN_RANGE 4   /* mutation plan index out of range */
#define HGA_FLAG_FIT_RANGE 8    /* fitness range exceeds the select keys (2^22) */
#define HGA_FLAG_NOT_GA 16      /* hga_pack_i8: column 0 is not all +1 or a column is
                                   unbalanced (the GA invariants, engine.py:440-446) */

/* mutation strategies (engine.py:58) */
#define HGA_MUT_SHARED 0
#define HGA_MUT_PER_MATRIX 1
#define HGA_MUT_MULTI 2

int hga_abi_version(void);
/* pipe-rate microbenchmark: kind 0 = XOR+POPC chains, 1 = LOP3+IADD chains
 * (each thread runs iters * 8 operations); kind 2 / 3 = dense int8
 * tcgen05.mma (s8 x s8 -> s32) of shape 128 x 256 x 32 / 64 x 64 x 32, iters
 * instructions issued back to back by one thread per CTA (one CTA per SM;
 * `threads` ignored; ops = blocks * iters * 2 * M * N * 32). */
int hga_probe(int32_t kind, int64_t iters, int32_t blocks, int32_t threads, uint32_t *out,
              void *stream);
const char *hga_strerror(int rc);
int hga_sm_count(int device);
/* Clears (and returns) the calling thread's sticky-free CUDA error state
 * (cudaGetLastError), e.g. after a failed cudaHostRegister by the host. */
int hga_clear_last_error(void);

/* ---------------------------------------------------------------- fitness */

/* Replaces engine._fitness_batch / engine.evaluate (engine.py:200-230):
 * penalties of n int8 (m, m) sign matrices.  Any of f1/f2/orth/sq may be
 * NULL; `variants` selects which are computed (fused in one pass, the Gram
 * matrix never leaves the SM).  bad_flag (nullable) gets HGA_FLAG_NOT_SIGN
 * OR-ed in when an entry is not +-1.  ws is needed only for m > 128
 * (hga_fitness_i8_ws_bytes).  Orders 48..64 (16-byte aligned pop) run the
 * Gram on the tensor cores (tcgen05.mma.kind::i8, accumulators in TMEM);
 * the others, or HGA_FITNESS_TC=0 in the environment, the XOR+POPC kernels.
 * Results are identical. */
size_t hga_fitness_i8_ws_bytes(int64_t n, int32_t m);
int hga_fitness_i8(const int8_t *pop, int64_t n, int32_t m, uint32_t variants, int64_t *f1,
                   int64_t *f2, int64_t *orth, int64_t *sq, int32_t *bad_flag, void *ws,
                   size_t ws_bytes, void *stream);

/* Same penalties over the packed layout. */
int hga_fitness_packed(const uint32_t *cols, int64_t n, int32_t m, uint32_t variants,
                       int64_t *f1, int64_t *f2, int64_t *orth, int64_t *sq, void *stream);

/* int8 (n, m, m) <-> packed conversion (layout edge of the API).  The pack
 * also ORs HGA_FLAG_NOT_GA into bad_flag when a matrix breaks the GA
 * invariants (column 0 all +1, every other column balanced) -- the Philox
 * generation loop's fast paths rely on them (engine.py:440-446). */
int hga_pack_i8(const int8_t *pop, int64_t n, int32_t m, uint32_t *cols, int32_t *bad_flag,
                void *stream);
int hga_unpack_i8(const uint32_t *cols, int64_t n, int32_t m, int8_t *pop, void *stream);

/* ------------------------------------------------ reference counter streams */

/* Raw stream words, rand.stream_words (rand.py:69-77) at counters c0..c0+n-1. */
int hga_ref_words(uint64_t seed, uint64_t stream_id, uint64_t counter0, int64_t n,
                  uint64_t *out, void *stream);
/* RngStream(seed, stream_id, counter0).uniform_array(lo, hi, n) (rand.py:122-129). */
int hga_ref_uniform(uint64_t seed, uint64_t stream_id, uint64_t counter0, int64_t lo,
                    int64_t hi, int64_t n, int64_t *out, void *stream);
/* RngStream(seed, stream_id, counter0).permutation(n) (rand.py:131-140),
 * bit-identical Fisher-Yates. */
size_t hga_ref_permutation_ws_bytes(int64_t n);
int hga_ref_permutation(uint64_t seed, uint64_t stream_id, uint64_t counter0, int64_t n,
                        int64_t *out, void *ws, size_t ws_bytes, void *stream);
/* engine._random_balanced (engine.py:154-182) into the packed / int8 layout. */
int hga_ref_init_packed(uint64_t seed, uint64_t purpose, uint64_t generation,
                        int64_t first_slot, int64_t count, int32_t m, uint32_t *cols,
                        void *stream);
int hga_ref_init_i8(uint64_t seed, uint64_t purpose, uint64_t generation, int64_t first_slot,
                    int64_t count, int32_t m, int8_t *pop, void *stream);

/* ------------------------------------------------------ operators (int8) */

/* engine.crossover (engine.py:257-277) in place on (4N, m, m) int8. */
int hga_crossover_i8(int8_t *pop, int64_t total, int32_t m, const int64_t *points,
                     int32_t *bad_flag, void *stream);
/* engine.mutate (engine.py:339-373) in place on the offspring half. cols is
 * (total/2, nc), ra/rb are (total/2, nr). */
int hga_mutate_i8(int8_t *pop, int64_t total, int32_t m, const int64_t *cols,
                  const int64_t *ra, const int64_t *rb, int32_t nc, int32_t nr,
                  int32_t *bad_flag, void *stream);

/* select (engine.py:233-248) building blocks.
 * hga_select_order: order[0:total/2] = argsort(fitness, stable)[:total/2].
 * Fitness values may be any int64 whose range (max - min) is below
 * hga_select_max_range(); otherwise HGA_FLAG_FIT_RANGE is raised. */
int64_t hga_select_max_range(void);
/* Any-range variant (stable radix sort of all `total` (fitness, index)
 * pairs; any int64 values): the first k indices of the stable argsort.
 * Used when hga_select_order raised HGA_FLAG_FIT_RANGE.  total < 2^31. */
size_t hga_select_radix_ws_bytes(int64_t total);
int hga_select_smallest_radix(const int64_t *fitness, int64_t total, int64_t k, int64_t *order,
                              void *ws, size_t ws_bytes, void *stream);
size_t hga_select_ws_bytes(int64_t total);
int hga_select_order(const int64_t *fitness, int64_t total, int64_t *order, int32_t *bad_flag,
                     void *ws, size_t ws_bytes, void *stream);
/* order[0:k] = argsort(fitness, stable)[:k] (k <= total): the k best,
 * lowest index first on ties; used for island elites. */
int hga_select_smallest(const int64_t *fitness, int64_t total, int64_t k, int64_t *order,
                        int32_t *bad_flag, void *ws, size_t ws_bytes, void *stream);
/* chosen[s] = order[perm[s]] (s < count); then gathers rows
 * dst[s] = src[chosen[s]] (layout bytes per matrix given) and
 * fit_dst[s] = fit_src[chosen[s]] (either may be NULL). */
int hga_compose_gather(const int64_t *order, const int64_t *perm, int64_t count,
                       const void *src, void *dst, int64_t bytes_per_matrix,
                       const int64_t *fit_src, int64_t *fit_dst, int64_t *chosen,
                       void *stream);

/* -------------------------------------------------- generation (packed) */

/* One generation's crossover + mutation + fitness with EXPLICIT plans
 * (reference-stream mode; engine.py:449-469 minus select).  Reads the 2N
 * parents new_pop[0:2N) (already gathered), writes offspring
 * new_pop[2N:4N) and new_fit[2N:4N) (fitness variant `fit_var`, one bit).
 * points (N,), cols (2N, nc), ra/rb (2N, nr).  best_key (nullable) gets
 * atomicMin((fit << 32) | index) over the offspring. */
int hga_generation_explicit(uint32_t *pop, int64_t *fit, int64_t n_pairs, int32_t m,
                            const int64_t *points, const int64_t *cols, const int64_t *ra,
                            const int64_t *rb, int32_t nc, int32_t nr, uint32_t fit_var,
                            unsigned long long *best_key, void *stream);

/* min over fit[0:n) as (value << 32) | first index, lowest index on ties
 * (numpy argmin, engine.py:417, 432).  Values must lie in [0, 2^31). */
int hga_argmin_key(const int64_t *fit, int64_t n, unsigned long long *key, int init,
                   void *stream);

/* Device mirror of engine._check_state (engine.py:440-446, run when
 * DEBUG_CHECKS is set): over n packed matrices counts[0] = matrices whose
 * column 0 is not all +1, counts[1] = unbalanced columns (popcount != m/2),
 * counts[2] = fitness values that differ from a fresh evaluation (variant
 * fit_var).  ws: hga_check_invariants_ws_bytes(n) bytes. */
size_t hga_check_invariants_ws_bytes(int64_t n);
int hga_check_invariants(const uint32_t *cols, const int64_t *fit, int64_t n, int32_t m,
                         uint32_t fit_var, unsigned long long *counts, void *ws, size_t ws_bytes,
                         void *stream);

/* ------------------------------------------------ production GA (Philox) */

/* Arguments of the persistent, grid-synchronised generation loop. */
typedef struct hga_run_args {
    /* population ping-pong buffers (packed, 4N matrices each) and fitness */
    uint32_t *pop[2];
    int64_t *fit[2];
    int64_t n_pairs;          /* N */
    int32_t m;                /* order */
    int32_t nc, nr;           /* NC, NR */
    int32_t strategy;         /* HGA_MUT_* */
    uint32_t fit_var;         /* one of HGA_VAR_F1 / F2 / SQ */
    int32_t stall_window;     /* 0 = off */
    uint64_t seed;
    int64_t max_generation;   /* stop after this absolute generation */
    int64_t gens_this_call;   /* run at most this many generations now */
    /* device state (int64[8]): [0] iteration, [1] best fitness,
     * [2] last restart, [3] current buffer parity, [4] best index,
     * [5] stop flag, [6..7] reserved */
    int64_t *state;
    int64_t *trace;           /* trace[g] = min fitness after generation g */
    int64_t trace_capacity;
    uint32_t *best_matrix;    /* packed best-so-far (m * W words) */
    void *ws;                 /* hga_run_ws_bytes() */
    size_t ws_bytes;
    uint32_t flags;           /* HGA_RUN_FORCE: run exactly gens_this_call
                                 generations (no stop test, no restart);
                                 HGA_RUN_TIMING: phase timestamps */
} hga_run_args;

#define HGA_RUN_FORCE 1u
#define HGA_RUN_TIMING 2u  /* record per-phase %globaltimer stamps (diagnostics) */
/* Select survivors with the one-barrier generation loop (4N <= 131072):
 * every CTA reads all 16-bit selection keys after the barrier instead of
 * publishing survivor lists behind a second barrier.  Same survivors, same
 * ranks, identical runs; measured slower than the default two-barrier loop
 * on B200 (22.8 vs 17.2 us per generation at order 20, 4N = 40,000), kept for
 * experiments.  Must be the same on hga_run_init / hga_run_prepare and on
 * every hga_run of that state (the loops keep selection state in different
 * slots). */
#define HGA_RUN_ONE_BARRIER 4u

/* Philox balanced matrices into slots [first_slot, first_slot + count) of
 * the packed population `cols` (slot 0 at cols).  The production-mode
 * counterpart of hga_ref_init_packed. */
int hga_philox_init_packed(uint64_t seed, uint64_t purpose, uint64_t generation,
                           int64_t first_slot, int64_t count, int32_t m, uint32_t *cols,
                           void *stream);

size_t hga_run_ws_bytes(int64_t n_pairs, int32_t m);
/* byte offset inside ws of the uint64 [64][20] phase timestamps (HGA_RUN_TIMING),
 * or -1 when the order runs on the fallback loop */
int64_t hga_run_timing_offset(int32_t m);
/* Philox-stream init of all 4N slots of pop[0] + evaluation + state init. */
int hga_run_init(const hga_run_args *args, void *stream);
/* Rebuild the loop's selection state (histogram, keys) from the current
 * population pop/fit[state[3]]; call after replacing the population or the
 * state block from outside (hga_run_init already does it). */
int hga_run_prepare(const hga_run_args *args, void *stream);
int hga_run(const hga_run_args *args, void *stream);

/* One Philox generation on a HOST-resident state: the reference's
 * step(state) (engine.py:449-469) when state.population / state.fitness are
 * host (numpy) arrays that the caller owns and that are updated in place.
 * host_pop (4N x m x m int8) and host_fit (4N int64) should be page-locked
 * (cudaHostRegister) so the copies are DMA.  The population goes up on
 * copy_stream in one piece and is packed on `stream`; the generation runs as
 * hga_run(gens_this_call = 1, HGA_RUN_FORCE)
 * from state_in (8 values: iteration, best, last restart, 0, 0, 0, 1, last
 * trace value); the new population is unpacked and copied back piece by
 * piece (`chunks` pieces, each copied as soon as it is unpacked) on
 * copy_stream.  Orders 4..64 (m % 4 == 0); HGA_E_UNSUPPORTED otherwise.
 * dev_i8 is a device int8 staging buffer of 4N*m*m
 * bytes.  On return (copy_stream synchronised) host_pop/host_fit hold the new
 * population, state_out[0..7] the device state after the generation and
 * *flag_out the HGA_FLAG_* bits.  The pack validates the upload on the
 * device: when HGA_FLAG_NOT_SIGN (an entry is not +-1) or HGA_FLAG_NOT_GA
 * (column 0 not all +1, or an unbalanced column) is set, the generation and
 * the unpack do nothing and host_pop/host_fit get their own values back
 * (no host round trip mid-step); the caller then raises or takes the exact
 * explicit-plan path. */
int hga_step_host(const hga_run_args *args, int8_t *host_pop, int64_t *host_fit, int8_t *dev_i8,
                  const int64_t *state_in, int64_t *state_out, int32_t *flag_out, int32_t chunks,
                  void *stream, void *copy_stream);

/* hga_step_host with the population moved as a BIT STREAM (8x fewer PCIe
 * bytes): the same step (engine.py:449-469) and the same contract as
 * hga_step_host, for orders 4..64 with m % 4 == 0.  The host packs the
 * caller's int8 bytes (validating every byte is +-1; AVX2 on a small host
 * thread pool, HGA_HOST_THREADS) into host_bits -- bit e of the stream set
 * iff byte e of host_pop is -1 -- piece by piece (`chunks` pieces), each
 * piece uploaded as soon as it is packed; the device turns the stream into
 * column records (and checks the GA invariants), runs the generation and
 * turns the new population back into a stream, which is copied down piece
 * by piece and unpacked into host_pop on the host as each piece lands.
 * host_bits: PAGE-LOCKED host buffer, dev_bits: device buffer, each of
 * hga_step_host_bits_bytes(n_pairs, m) bytes (0 = order not supported).
 * A byte that is not +-1 returns with *flag_out = HGA_FLAG_NOT_SIGN before
 * any device work that could touch the caller's arrays; HGA_FLAG_NOT_GA
 * leaves host_pop as it was and host_fit holding its own values. */
/* The host half of hga_step_host_bits as plain host utilities (no GPU):
 * hga_host_pack_bits packs n int8 entries into ceil(n/32) uint32 words of
 * the bit stream (bit e % 32 of word e / 32 set iff src[e] == -1; unused
 * high bits of the last word 0) on libhga's host thread pool and returns
 * HGA_FLAG_NOT_SIGN when some entry is not +-1 (the words are then
 * unspecified), else 0; hga_host_unpack_bits writes n entries of +1 / -1
 * from the stream. */
int hga_host_pack_bits(const int8_t *src, int64_t n, uint32_t *dst);
void hga_host_unpack_bits(const uint32_t *src, int64_t n, int8_t *dst);
/* Bit stream <-> packed column records on the device (orders 4..64,
 * m % 4 == 0; the stream layout of hga_host_pack_bits): hga_bits_to_cols
 * also raises HGA_FLAG_NOT_GA in *flag (if not NULL) when a matrix breaks
 * the GA invariants (column 0 not all +1, an unbalanced column). */
int hga_bits_to_cols(const uint32_t *bits, int64_t n, int32_t m, uint32_t *cols, int32_t *flag,
                     void *stream);
int hga_cols_to_bits(const uint32_t *cols, int64_t n, int32_t m, uint32_t *bits, void *stream);
size_t hga_step_host_bits_bytes(int64_t n_pairs, int32_t m);
int hga_step_host_bits(const hga_run_args *args, int8_t *host_pop, int64_t *host_fit, uint32_t *host_bits,
                       uint32_t *dev_bits, const int64_t *state_in, int64_t *state_out, int32_t *flag_out,
                       int32_t chunks, void *stream, void *copy_stream);

#ifdef __cplusplus
}
#endif

#endif /* HGA_H */
