// fitness.cu -- fused Gram-penalty kernels (replaces engine._fitness_batch,
// reference engine.py:200-213, and core.fitness_f1/f2, core.py:59-89).
//
// One pass per matrix: columns become bit words (bit r set iff entry r is -1),
// every column pair costs W XOR+POPC (g_ij = m - 2 popc(c_i ^ c_j)), and the
// F1 / F2 / ORTH / SQ reductions run in registers, then a warp REDUX and one
// shared-memory atomic per matrix.  The Gram matrix never leaves the SM.
//
// Thread mapping: a 256-thread CTA owns mpb = 256 / m matrices; thread
// (matrix kl, column i) keeps column i in registers and walks the circulant
// pair schedule (i, i + d mod m) over a shared-memory copy of the matrix's
// columns stored twice (so i + d never wraps).  For the int8 input the CTA
// first stages mpb * m * m bytes with 16-byte loads (validating every byte is
// +-1 on the way), then each thread packs its own column from shared memory.
#include "fitness_v2.cuh"

#include <cstdlib>

namespace hga {

HGA_V2_ORDERS(HGA_V2_EXTERN)

// tensor-core int8 path (fitness_tc.cu), orders 36..64
bool fit_tc_order(int m, bool all);
int launch_fit_tc(int m, const int8_t* pop, int64_t n, uint32_t v, int64_t* f1, int64_t* f2, int64_t* orth,
                  int64_t* sq, int32_t* bad, cudaStream_t st);
// round-2 tensor-core kernel (fitness_tc2.cu), orders 36..64
bool fit_tc2_order(int m);
int launch_fit_tc2(int m, const int8_t* pop, int64_t n, uint32_t v, int64_t* f1, int64_t* f2, int64_t* orth,
                   int64_t* sq, int32_t* bad, cudaStream_t st);
// HGA_FITNESS_TC=0 selects the XOR+POPC kernels at every order, =all the
// round-1 tensor-core kernel at every order 4..64, =v1 the round-1 kernel at
// its default orders (48..64), =2 the round-2 kernel at every order 36..64
// (cross-checks, A/B timing); default: the round-2 kernel from order
// HGA_TC2_MIN (default 44) to 64
static int fit_tc_mode() {  // read per call: tests and sweeps switch it at run time
    const char* e = std::getenv("HGA_FITNESS_TC");
    if (e && e[0] == '0') return 0;
    if (e && e[0] == 'a') return 2;
    if (e && e[0] == 'v') return 3;
    if (e && e[0] == '2') return 4;
    return 1;
}
static int tc2_min_order() {
    const char* e = std::getenv("HGA_TC2_MIN");
    return e ? std::atoi(e) : 44;
}

static int launch_fit_v2(int m, bool from_i8, const void* src, int64_t n, uint32_t v, int64_t* f1, int64_t* f2,
                         int64_t* orth, int64_t* sq, int32_t* bad, cudaStream_t st) {
    switch (m) {
#define HGA_V2_CASE(M) \
    case M: return launch_fit_v2_m<M>(from_i8, src, n, v, f1, f2, orth, sq, bad, st);
        HGA_V2_ORDERS(HGA_V2_CASE)
#undef HGA_V2_CASE
        default: return HGA_E_UNSUPPORTED;
    }
}

constexpr int kFitThreads = 256;

template <int W>
__device__ __forceinline__ void pack_column_smem(const int8_t* raw, int m, int i, Col<W>& c) {
#pragma unroll
    for (int w = 0; w < W; ++w) {
        const int r0 = 32 * w;
        const int nr = min(32, m - r0);
        uint32_t word = 0;
        const int8_t* p = raw + (int64_t)r0 * m + i;
#pragma unroll 4
        for (int rr = 0; rr < nr; ++rr) word |= ((uint32_t)(int32_t)p[(int64_t)rr * m] >> 31) << rr;
        c.w[w] = word;
    }
}

__device__ __forceinline__ uint32_t sign_bytes_bad(uint32_t x) {
    // each byte must be 0x01 or 0xFF: bit 0 set and bits 1..7 all equal
    return (~x & 0x01010101u) | ((x ^ (x >> 1)) & 0x7E7E7E7Eu);
}

// Stage `bytes` contiguous bytes global -> shared, validating sign entries.
__device__ __forceinline__ uint32_t stage_bytes(const int8_t* __restrict__ g, int8_t* s,
                                                int64_t bytes) {
    uint32_t bad = 0;
    if ((((uintptr_t)g) & 15) == 0 && (bytes & 15) == 0) {
        const uint4* g4 = reinterpret_cast<const uint4*>(g);
        uint4* s4 = reinterpret_cast<uint4*>(s);
        for (int64_t v = threadIdx.x; v < (bytes >> 4); v += blockDim.x) {
            uint4 x = __ldcs(g4 + v);  // streamed once: evict-first
            bad |= sign_bytes_bad(x.x) | sign_bytes_bad(x.y) | sign_bytes_bad(x.z) |
                   sign_bytes_bad(x.w);
            s4[v] = x;
        }
    } else {
        for (int64_t v = threadIdx.x; v < bytes; v += blockDim.x) {
            int8_t b = g[v];
            bad |= (b != 1 && b != -1);
            s[v] = b;
        }
    }
    return bad;
}

template <int W, int VM, bool FROM_I8>
__global__ void __launch_bounds__(kFitThreads)
    k_fitness(const void* __restrict__ src, int64_t n, int m, int mpb, uint32_t vm_out,
              int64_t* __restrict__ f1, int64_t* __restrict__ f2, int64_t* __restrict__ orth,
              int64_t* __restrict__ sq, int32_t* bad_flag) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* scol = reinterpret_cast<uint32_t*>(smem);
    const int col_words = ((mpb * 2 * m * W) + 3) & ~3;
    uint32_t* sacc = scol + col_words;
    int8_t* sraw = reinterpret_cast<int8_t*>(sacc + ((mpb * 3 + 3) & ~3));

    const int tid = threadIdx.x;
    const int kl = tid / m, i = tid - kl * m;
    const int half = (m & 1) ? -1 : m / 2;
    const int steps = pair_steps(m, i);
    const int64_t mm = (int64_t)m * m;
    const int64_t mw = (int64_t)m * W;
    uint32_t bad = 0;

    for (int64_t k0 = (int64_t)blockIdx.x * mpb; k0 < n; k0 += (int64_t)gridDim.x * mpb) {
        const int cnt = (int)min((int64_t)mpb, n - k0);
        const bool active = kl < cnt;
        Col<W> c;
        if (FROM_I8) {
            bad |= stage_bytes(reinterpret_cast<const int8_t*>(src) + k0 * mm, sraw, cnt * mm);
            for (int z = tid; z < cnt * 3; z += blockDim.x) sacc[z] = 0;
            __syncthreads();
            if (active) pack_column_smem<W>(sraw + kl * mm, m, i, c);
        } else {
            for (int z = tid; z < cnt * 3; z += blockDim.x) sacc[z] = 0;
            if (active) {
                const uint32_t* g = reinterpret_cast<const uint32_t*>(src) + (k0 + kl) * mw + (int64_t)i * W;
#pragma unroll
                for (int w = 0; w < W; ++w) c.w[w] = __ldcs(g + w);
            }
        }
        if (active) {
            uint32_t* dst = scol + ((int64_t)kl * 2 * m + i) * W;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                dst[w] = c.w[w];
                dst[(int64_t)m * W + w] = c.w[w];
            }
        }
        __syncthreads();
        Acc a{0, 0, 0};
        if (active) {
            const uint32_t* base = scol + ((int64_t)kl * 2 * m + i) * W;
            for (int d = 1; d <= steps; ++d) {
                int p = 0;
#pragma unroll
                for (int w = 0; w < W; ++w) p += __popc(c.w[w] ^ base[d * W + w]);
                acc_pair<VM>(a, p, m, half);
            }
        }
        const unsigned peers = __match_any_sync(0xffffffffu, active ? kl : -1);
        const bool leader = (__ffs(peers) - 1) == (int)(tid & 31);
        if (VM & HGA_VAR_F1) {
            uint32_t s = __reduce_add_sync(peers, a.s1);
            if (active && leader) atomicAdd(&sacc[kl * 3 + 0], s);
        }
        if (VM & (HGA_VAR_F2 | HGA_VAR_ORTH)) {
            uint32_t s = __reduce_add_sync(peers, a.s2);
            if (active && leader) atomicAdd(&sacc[kl * 3 + 1], s);
        }
        if (VM & HGA_VAR_SQ) {
            uint32_t s = __reduce_add_sync(peers, a.s4);
            if (active && leader) atomicAdd(&sacc[kl * 3 + 2], s);
        }
        __syncthreads();
        if (tid < cnt)
            write_penalties(vm_out, m, k0 + tid, sacc[tid * 3], sacc[tid * 3 + 1], sacc[tid * 3 + 2],
                            f1, f2, orth, sq);
        __syncthreads();
    }
    if (FROM_I8 && bad_flag) {
        bad = __syncthreads_or(bad != 0);
        if (bad && tid == 0) atomicOr(bad_flag, HGA_FLAG_NOT_SIGN);
    }
}

// ------------------------------------------------------------ generic path
// Any order m (words per column W > 4): pack to a global workspace, then one
// CTA per matrix walks the same circulant schedule with 64-bit accumulators.

__global__ void k_pack_any(const int8_t* __restrict__ pop, int64_t n, int m, int W,
                           uint32_t* __restrict__ cols, int32_t* bad_flag) {
    // thread per (matrix k, column j): neighbouring threads read neighbouring
    // bytes of a row; the column's W words are built (and its popcount taken
    // for the GA-invariant flag) in one walk down the rows
    const int64_t total = n * m;
    uint32_t bad = 0, not_ga = (m & 3) ? 1u : 0u;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(t % m);
        const int8_t* p = pop + (t - j) * (int64_t)m + j;
        int neg = 0;
        for (int w = 0; w < W; ++w) {
            const int nr = min(32, m - 32 * w);
            uint32_t word = 0;
            for (int rr = 0; rr < nr; ++rr) {
                const int8_t b = p[(int64_t)(32 * w + rr) * m];
                bad |= (b != 1 && b != -1);
                word |= ((uint32_t)(int32_t)b >> 31) << rr;
            }
            cols[t * W + w] = word;
            neg += __popc(word);
        }
        not_ga |= (uint32_t)(neg != (j == 0 ? 0 : m / 2));
    }
    const uint32_t f = (bad ? HGA_FLAG_NOT_SIGN : 0u) | (not_ga ? HGA_FLAG_NOT_GA : 0u);
    if (f && bad_flag) atomicOr(bad_flag, (int32_t)f);
}

__global__ void k_fitness_any(const uint32_t* __restrict__ cols, int64_t n, int m, int W,
                              uint32_t vm_out, int64_t idx0, int64_t* f1, int64_t* f2,
                              int64_t* orth, int64_t* sq) {
    __shared__ unsigned long long acc[3];
    const int half = (m & 1) ? -1 : m / 2;
    for (int64_t k = blockIdx.x; k < n; k += gridDim.x) {
        if (threadIdx.x < 3) acc[threadIdx.x] = 0;
        __syncthreads();
        const uint32_t* q = cols + k * m * (int64_t)W;
        unsigned long long s1 = 0, s2 = 0, s4 = 0;
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            const int steps = pair_steps(m, i);
            for (int d = 1; d <= steps; ++d) {
                int j = i + d;
                if (j >= m) j -= m;
                int p = 0;
                for (int w = 0; w < W; ++w) p += __popc(q[(int64_t)i * W + w] ^ q[(int64_t)j * W + w]);
                const long long g = m - 2 * p;
                s1 += (unsigned long long)(g < 0 ? -g : g);
                s2 += (p != half);
                s4 += (unsigned long long)(g * g);
            }
        }
        atomicAdd(&acc[0], s1);
        atomicAdd(&acc[1], s2);
        atomicAdd(&acc[2], s4);
        __syncthreads();
        if (threadIdx.x == 0) write_penalties(vm_out, m, idx0 + k, acc[0], acc[1], acc[2], f1, f2, orth, sq);
        __syncthreads();
    }
}

// ----------------------------------------------------------------- unpack
__global__ void k_unpack(const uint32_t* __restrict__ cols, int64_t n, int m, int W,
                         int8_t* __restrict__ pop) {
    const int64_t mm = (int64_t)m * m;
    const int64_t total = n * mm;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = t / mm;
        const int e = (int)(t - k * mm);
        const int r = e / m, j = e - r * m;
        const uint32_t word = cols[(k * m + j) * W + (r >> 5)];
        pop[t] = ((word >> (r & 31)) & 1u) ? (int8_t)-1 : (int8_t)1;
    }
}

// Pack for m % 4 == 0, m <= 64: thread (matrix k, column quad jq) walks the
// rows with one 4-byte load each (consecutive threads read consecutive
// quads of a row), collects the four columns' sign bits and checks the bytes
// are +-1 (byte ^ 1 has bit 0 clear and bits 1..7 equal) and the columns
// keep the GA invariants (popcount 0 for column 0, m / 2 for the others).
template <int W>
__global__ void k_pack_quads(const int8_t* __restrict__ pop, int64_t n, int m, uint32_t* __restrict__ cols,
                             int32_t* bad_flag) {
    const int q4 = m >> 2;
    const int64_t quads = n * q4;
    uint32_t bad = 0, not_ga = 0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < quads; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = t / q4;
        const int jq = (int)(t - k * q4);
        const uint32_t* p = reinterpret_cast<const uint32_t*>(pop + k * m * (int64_t)m) + jq;
        uint32_t w[4][W];
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int x = 0; x < W; ++x) w[c][x] = 0;
        for (int r = 0; r < m; ++r) {
            const uint32_t v = __ldg(p + r * q4);
            const uint32_t a8 = v ^ 0x01010101u, b8 = a8 & 0xFEFEFEFEu;
            bad |= (a8 & 0x01010101u) | ((b8 ^ (b8 << 1)) & 0xFCFCFCFCu);
#pragma unroll
            for (int x = 0; x < W; ++x) {
                if ((r >> 5) != x) continue;
#pragma unroll
                for (int c = 0; c < 4; ++c) w[c][x] |= ((v >> (8 * c + 7)) & 1u) << (r & 31);
            }
        }
        uint32_t* out = cols + (k * m + 4 * jq) * W;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            int neg = 0;
#pragma unroll
            for (int x = 0; x < W; ++x) {
                out[c * W + x] = w[c][x];
                neg += __popc(w[c][x]);
            }
            not_ga |= (uint32_t)(neg != ((jq | c) == 0 ? 0 : (m >> 1)));
        }
    }
    const uint32_t f = (bad ? HGA_FLAG_NOT_SIGN : 0u) | (not_ga ? HGA_FLAG_NOT_GA : 0u);
    if (f && bad_flag) atomicOr(bad_flag, (int32_t)f);
}

// Row-at-a-time unpack for m % 4 == 0: thread (matrix k, row r) reads row
// r's bit from each column word (neighbouring rows share the words through
// L1) and writes the row as m / 4 four-byte stores.
__global__ void k_unpack_rows(const uint32_t* __restrict__ cols, int64_t n, int m, int W,
                              int8_t* __restrict__ pop, const int32_t* __restrict__ skip_if = nullptr) {
    // skip_if (hga_step_host): a rejected upload leaves the staging bytes (the
    // caller's own population) in place
    if (skip_if && (*skip_if & (HGA_FLAG_NOT_SIGN | HGA_FLAG_NOT_GA))) return;
    const int64_t rows = n * m;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = t / m;
        const int r = (int)(t - k * m);
        const uint32_t* c = cols + k * m * W + (r >> 5);
        const int sh = r & 31;
        uint32_t* out = reinterpret_cast<uint32_t*>(pop + t * m);
        for (int j = 0; j < m; j += 4) {
            uint32_t w = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) w |= (((__ldg(c + (j + q) * W) >> sh) & 1u) ? 0xFFu : 0x01u) << (8 * q);
            out[j >> 2] = w;
        }
    }
}

// -------------------------------------------------------------- host side

static int g_sm_count[16] = {0};

int sm_count_cached() {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 16) dev = 0;
    if (!g_sm_count[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        g_sm_count[dev] = v > 0 ? v : 148;
    }
    return g_sm_count[dev];
}

static size_t fit_smem_bytes(int m, int W, int mpb, bool from_i8) {
    size_t col_words = ((size_t)(mpb * 2 * m * W) + 3) & ~(size_t)3;
    size_t acc_words = ((size_t)(mpb * 3) + 3) & ~(size_t)3;
    size_t raw = from_i8 ? ((size_t)mpb * m * m + 15) & ~(size_t)15 : 0;
    return (col_words + acc_words) * 4 + raw;
}

template <int W, int VM, bool FROM_I8>
static int launch_fitness_t(const void* src, int64_t n, int m, uint32_t vm_out, int64_t* f1,
                            int64_t* f2, int64_t* orth, int64_t* sq, int32_t* bad, cudaStream_t st) {
    const int mpb = kFitThreads / m;
    const size_t smem = fit_smem_bytes(m, W, mpb, FROM_I8);
    auto kern = k_fitness<W, VM, FROM_I8>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return to_rc(e);
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kFitThreads, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t tiles = (n + mpb - 1) / mpb;
    const int64_t grid = std::min<int64_t>(tiles, (int64_t)sm_count_cached() * per_sm);
    kern<<<(unsigned)grid, kFitThreads, smem, st>>>(src, n, m, mpb, vm_out, f1, f2, orth, sq, bad);
    return to_rc(cudaGetLastError());
}

template <int W, bool FROM_I8>
static int launch_fitness_w(const void* src, int64_t n, int m, uint32_t v, int64_t* f1, int64_t* f2,
                            int64_t* orth, int64_t* sq, int32_t* bad, cudaStream_t st) {
    if ((v & ~(HGA_VAR_F2 | HGA_VAR_ORTH)) == 0)
        return launch_fitness_t<W, HGA_VAR_F2 | HGA_VAR_ORTH, FROM_I8>(src, n, m, v, f1, f2, orth, sq, bad, st);
    if (v == HGA_VAR_F1)
        return launch_fitness_t<W, HGA_VAR_F1, FROM_I8>(src, n, m, v, f1, f2, orth, sq, bad, st);
    if (v == HGA_VAR_SQ)
        return launch_fitness_t<W, HGA_VAR_SQ, FROM_I8>(src, n, m, v, f1, f2, orth, sq, bad, st);
    return launch_fitness_t<W, HGA_VAR_ALL, FROM_I8>(src, n, m, v, f1, f2, orth, sq, bad, st);
}

template <bool FROM_I8>
static int launch_fitness(const void* src, int64_t n, int m, uint32_t v, int64_t* f1, int64_t* f2,
                          int64_t* orth, int64_t* sq, int32_t* bad, cudaStream_t st) {
    switch (words_for(m)) {
        case 1: return launch_fitness_w<1, FROM_I8>(src, n, m, v, f1, f2, orth, sq, bad, st);
        case 2: return launch_fitness_w<2, FROM_I8>(src, n, m, v, f1, f2, orth, sq, bad, st);
        case 3: return launch_fitness_w<3, FROM_I8>(src, n, m, v, f1, f2, orth, sq, bad, st);
        case 4: return launch_fitness_w<4, FROM_I8>(src, n, m, v, f1, f2, orth, sq, bad, st);
        default: return HGA_E_UNSUPPORTED;
    }
}

static int64_t generic_chunk(int64_t n, int m) {
    const int64_t per = (int64_t)m * words_for(m) * 4;
    int64_t chunk = std::max<int64_t>(1, (int64_t)(64ll << 20) / per);
    return std::min<int64_t>(n, chunk);
}

static int grid_for(int64_t work, int threads) {
    int64_t g = (work + threads - 1) / threads;
    int64_t cap = (int64_t)sm_count_cached() * 16;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, cap));
}

// hga_step_host's guarded unpack (m % 4 == 0, 4-byte aligned staging): no-op when the
// uploaded population was rejected
int unpack_i8_guarded(const uint32_t* cols, int64_t n, int32_t m, int8_t* pop, const int32_t* flag, cudaStream_t st) {
    if (n <= 0) return HGA_OK;
    k_unpack_rows<<<grid_for(n * (int64_t)m, 256), 256, 0, st>>>(cols, n, m, words_for(m), pop, flag);
    return to_rc(cudaGetLastError());
}

}  // namespace hga

using namespace hga;

extern "C" {

size_t hga_fitness_i8_ws_bytes(int64_t n, int32_t m) {
    if (m <= 32 * kMaxRegWords || n <= 0) return 0;
    return (size_t)generic_chunk(n, m) * m * words_for(m) * 4;
}

int hga_fitness_i8(const int8_t* pop, int64_t n, int32_t m, uint32_t variants, int64_t* f1,
                   int64_t* f2, int64_t* orth, int64_t* sq, int32_t* bad_flag, void* ws,
                   size_t ws_bytes, void* stream) {
    if (n < 0 || m < 1 || m > 4096 || (variants & ~HGA_VAR_ALL) || !variants) return HGA_E_INVALID;
    if (n == 0) return HGA_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int tc_mode = fit_tc_mode();
    const bool al16 = (((uintptr_t)pop) & 15) == 0;
    // several variants at once (or SQ) at orders 36 / 40: the XOR+POPC kernel's
    // all-variant build runs at 0.41-0.54e9 evals/s there, the tensor-core kernel
    // at 1.0e9 (r02_fitness_sweep.csv); F2 or F1 alone stay on XOR+POPC below 44
    const bool multi = (variants & ~(HGA_VAR_F2 | HGA_VAR_ORTH)) != 0 && variants != HGA_VAR_F1;
    if (((tc_mode == 1 && (m >= tc2_min_order() || multi)) || tc_mode == 4) && al16 && fit_tc2_order(m))
        return launch_fit_tc2(m, pop, n, variants, f1, f2, orth, sq, bad_flag, st);
    if ((tc_mode == 2 || tc_mode == 3) && al16 && fit_tc_order(m, tc_mode == 2))
        return launch_fit_tc(m, pop, n, variants, f1, f2, orth, sq, bad_flag, st);
    if (v2_order(m) && (((uintptr_t)pop) & 15) == 0)
        return launch_fit_v2(m, true, pop, n, variants, f1, f2, orth, sq, bad_flag, st);
    if (m <= 32 * kMaxRegWords)
        return launch_fitness<true>(pop, n, m, variants, f1, f2, orth, sq, bad_flag, st);
    const int W = words_for(m);
    const int64_t chunk = generic_chunk(n, m);
    if (!ws || ws_bytes < (size_t)chunk * m * W * 4) return HGA_E_WORKSPACE;
    uint32_t* cols = (uint32_t*)ws;
    for (int64_t k0 = 0; k0 < n; k0 += chunk) {
        const int64_t c = std::min(chunk, n - k0);
        k_pack_any<<<grid_for(c * m, 256), 256, 0, st>>>(pop + k0 * m * (int64_t)m, c, m, W, cols, bad_flag);
        k_fitness_any<<<(unsigned)std::min<int64_t>(c, sm_count_cached() * 8), 128, 0, st>>>(
            cols, c, m, W, variants, k0, f1, f2, orth, sq);
    }
    return to_rc(cudaGetLastError());
}

int hga_fitness_packed(const uint32_t* cols, int64_t n, int32_t m, uint32_t variants, int64_t* f1,
                       int64_t* f2, int64_t* orth, int64_t* sq, void* stream) {
    if (n < 0 || m < 1 || m > 4096 || (variants & ~HGA_VAR_ALL) || !variants) return HGA_E_INVALID;
    if (n == 0) return HGA_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (v2_order(m) && (((uintptr_t)cols) & 15) == 0)
        return launch_fit_v2(m, false, cols, n, variants, f1, f2, orth, sq, nullptr, st);
    if (m <= 32 * kMaxRegWords)
        return launch_fitness<false>(cols, n, m, variants, f1, f2, orth, sq, nullptr, st);
    k_fitness_any<<<(unsigned)std::min<int64_t>(n, sm_count_cached() * 8), 128, 0, st>>>(
        cols, n, m, words_for(m), variants, 0, f1, f2, orth, sq);
    return to_rc(cudaGetLastError());
}

int hga_pack_i8(const int8_t* pop, int64_t n, int32_t m, uint32_t* cols, int32_t* bad_flag,
                void* stream) {
    if (n < 0 || m < 1 || m > 4096) return HGA_E_INVALID;
    if (n == 0) return HGA_OK;
    const int W = words_for(m);
    cudaStream_t st = (cudaStream_t)stream;
    if (m % 4 == 0 && m <= 64 && (((uintptr_t)pop) & 3) == 0) {
        const unsigned g = grid_for(n * (int64_t)(m / 4), 256);
        if (W == 1) k_pack_quads<1><<<g, 256, 0, st>>>(pop, n, m, cols, bad_flag);
        else k_pack_quads<2><<<g, 256, 0, st>>>(pop, n, m, cols, bad_flag);
    } else {
        k_pack_any<<<grid_for(n * m, 256), 256, 0, st>>>(pop, n, m, W, cols, bad_flag);
    }
    return to_rc(cudaGetLastError());
}

int hga_unpack_i8(const uint32_t* cols, int64_t n, int32_t m, int8_t* pop, void* stream) {
    if (n < 0 || m < 1 || m > 4096) return HGA_E_INVALID;
    if (n == 0) return HGA_OK;
    if (m % 4 == 0 && (((uintptr_t)pop) & 3) == 0)
        k_unpack_rows<<<grid_for(n * (int64_t)m, 256), 256, 0, (cudaStream_t)stream>>>(cols, n, m, words_for(m), pop);
    else
        k_unpack<<<grid_for(n * m * (int64_t)m, 256), 256, 0, (cudaStream_t)stream>>>(cols, n, m, words_for(m), pop);
    return to_rc(cudaGetLastError());
}

int hga_abi_version(void) { return HGA_ABI_VERSION; }

int hga_clear_last_error(void) { return (int)cudaGetLastError(); }

int hga_sm_count(int device) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
    return v;
}

const char* hga_strerror(int rc) {
    switch (rc) {
        case HGA_OK: return "ok";
        case HGA_E_INVALID: return "invalid argument";
        case HGA_E_UNSUPPORTED: return "unsupported order or size";
        case HGA_E_WORKSPACE: return "workspace too small";
        default:
            if (rc >= HGA_E_CUDA_BASE) return cudaGetErrorString((cudaError_t)(rc - HGA_E_CUDA_BASE));
            return "unknown error";
    }
}

}  // extern "C"
