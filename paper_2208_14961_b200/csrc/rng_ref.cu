// rng_ref.cu -- the reference's counter-based splitmix64 streams on device
// (reference rand.py:39-140, engine.py:154-182), bit-identical, so the GA can
// replay a reference run exactly ("reference-stream" mode).
//
// Every draw is a pure function of (seed, stream id, counter): one thread per
// draw.  The only sequential piece is Fisher-Yates (rand.py:131-140); its swap
// targets are drawn in parallel, then small permutations run the swap chain in
// one CTA's shared memory and large ones are replayed in parallel (k_pfy_*:
// grouping the steps by target turns the chain into short pointer chases).
#include "hga_common.cuh"

namespace hga {

__global__ void k_ref_words(uint64_t key, uint64_t c0, int64_t n, uint64_t* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = stream_word(key, c0 + (uint64_t)i);
}

__global__ void k_ref_uniform(uint64_t key, uint64_t c0, int64_t lo, uint64_t span, int64_t n,
                              int64_t* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = lo + (int64_t)(stream_word(key, c0 + (uint64_t)i) % span);
}

// b[a] = a + word(a) % (n - a), the partner of step a of the forward shuffle.
__global__ void k_perm_targets(uint64_t key, uint64_t c0, int64_t n, int32_t* b) {
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a + 1 < n;
         a += (int64_t)gridDim.x * blockDim.x)
        b[a] = (int32_t)(a + (int64_t)(stream_word(key, c0 + (uint64_t)a) % (uint64_t)(n - a)));
}

// The swap chain.  Shared-memory copy when n fits, else in global memory.
__global__ void k_perm_chain(const int32_t* __restrict__ b, int64_t n, int64_t* out, int32_t* gperm,
                             int use_smem) {
    extern __shared__ int32_t sperm[];
    int32_t* perm = use_smem ? sperm : gperm;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) perm[i] = (int32_t)i;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int64_t a = 0; a + 1 < n; ++a) {
            const int32_t t = b[a];
            const int32_t x = perm[a];
            perm[a] = perm[t];
            perm[t] = x;
        }
    }
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) out[i] = perm[i];
}

// ---------------------------------------------------------------------
// Parallel replay of the same forward Fisher-Yates (rand.py:131-140) for
// large n.  With b[a] >= a the partner of step a, position a is final after
// step a, so:
//   v[a]     = value at position a just before step a
//            = v[k] for the last k < a with b[k] == a, else a      (a chain)
//   final[a] = v[k] for the last k < a with b[k] == b[a], else b[a]
//   final[n-1] = v[n-1]
// Steps are grouped by target (counting sort, then each small group sorted
// by step index), which gives both "last k" lookups; v follows the chains.
__global__ void k_pfy_targets(uint64_t key, uint64_t c0, int64_t n, int32_t* b, int32_t* cnt) {
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a + 1 < n;
         a += (int64_t)gridDim.x * blockDim.x) {
        const int32_t t = (int32_t)(a + (int64_t)(stream_word(key, c0 + (uint64_t)a) % (uint64_t)(n - a)));
        b[a] = t;
        atomicAdd(&cnt[t], 1);
    }
}

// single CTA: exclusive scan of cnt[0..n) into off[0..n]
__global__ void __launch_bounds__(1024) k_pfy_scan(const int32_t* __restrict__ cnt, int64_t n, int32_t* off) {
    __shared__ int32_t wsum[32];
    __shared__ int32_t carry;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int64_t b0 = 0; b0 < n; b0 += 1024) {
        const int64_t i = b0 + tid;
        const int32_t v = i < n ? cnt[i] : 0;
        int32_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[wid] = x;
        __syncthreads();
        if (wid == 0) {
            int32_t t = wsum[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t y = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += y;
            }
            wsum[lane] = t;
        }
        __syncthreads();
        if (i < n) off[i] = carry + (wid ? wsum[wid - 1] : 0) + x - v;
        __syncthreads();
        if (tid == 0) carry += wsum[31];
        __syncthreads();
    }
    if (tid == 0) off[n] = carry;
}

__global__ void k_pfy_place(const int32_t* __restrict__ b, int64_t n, int32_t* cursor, int32_t* grouped) {
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a + 1 < n;
         a += (int64_t)gridDim.x * blockDim.x)
        grouped[atomicAdd(&cursor[b[a]], 1)] = (int32_t)a;
}

// one thread per target y: sort its (few) steps, emit prev_same and last_hit
__global__ void k_pfy_groups(const int32_t* __restrict__ off, int64_t n, int32_t* grouped, int32_t* prev_same,
                             int32_t* last_hit) {
    for (int64_t y = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; y < n; y += (int64_t)gridDim.x * blockDim.x) {
        const int32_t s0 = off[y], s1 = off[y + 1];
        for (int32_t i = s0 + 1; i < s1; ++i) {  // insertion sort by step index
            const int32_t v = grouped[i];
            int32_t j = i - 1;
            while (j >= s0 && grouped[j] > v) {
                grouped[j + 1] = grouped[j];
                --j;
            }
            grouped[j + 1] = v;
        }
        int32_t lh = -1, prev = -1;
        for (int32_t i = s0; i < s1; ++i) {
            const int32_t k = grouped[i];
            prev_same[k] = prev;
            prev = k;
            if (k < y) lh = k;
        }
        last_hit[y] = lh;
    }
}

__global__ void k_pfy_final(const int32_t* __restrict__ b, const int32_t* __restrict__ prev_same,
                            const int32_t* __restrict__ last_hit, int64_t n, int64_t* out) {
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n; a += (int64_t)gridDim.x * blockDim.x) {
        int32_t src;
        if (a + 1 < n) {
            const int32_t k = prev_same[a];
            if (k < 0) {
                out[a] = b[a];
                continue;
            }
            src = k;
        } else {
            src = (int32_t)a;
        }
        // v[src]: follow last_hit to the chain's root
        int32_t x = src;
        while (last_hit[x] >= 0) x = last_hit[x];
        out[a] = x;
    }
}

// engine._random_balanced: column c of slot s starts with rows [0, m/2) = -1
// (bits set) and gets a Fisher-Yates shuffle from stream
// sid(purpose, generation, first_slot + s, c).  Column 0 stays all +1.
template <int W>
__device__ __forceinline__ void balanced_column(uint64_t seedmix, uint64_t base_sid, int64_t slot,
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
    const uint64_t key = stream_key_from_seedmix(seedmix, base_sid | ((uint64_t)slot << 12) | (uint64_t)c);
    for (int a = 0; a + 1 < m; ++a) {
        const int b = a + (int)mod_u64_u32(stream_word(key, (uint64_t)a), (uint32_t)(m - a));
        swap_rows<W>(col, a, b);
    }
}

template <int W>
__global__ void k_ref_init_packed(uint64_t seedmix, uint64_t base_sid, int64_t first_slot,
                                  int64_t count, int m, uint32_t* __restrict__ cols) {
    const int64_t total = count * m;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = t / m;
        const int c = (int)(t - s * m);
        Col<W> col;
        balanced_column<W>(seedmix, base_sid, first_slot + s, m, c, col);
#pragma unroll
        for (int w = 0; w < W; ++w) cols[t * W + w] = col.w[w];
    }
}

// Any m: the column lives in local memory (orders > 128 only).
__global__ void k_ref_init_packed_any(uint64_t seedmix, uint64_t base_sid, int64_t first_slot,
                                      int64_t count, int m, int W, uint32_t* __restrict__ cols) {
    const int64_t total = count * m;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = t / m;
        const int c = (int)(t - s * m);
        uint32_t* col = cols + t * W;
        for (int w = 0; w < W; ++w) col[w] = 0;
        if (c == 0) continue;
        for (int r = 0; r < m / 2; ++r) col[r >> 5] |= 1u << (r & 31);
        const uint64_t key = stream_key_from_seedmix(seedmix, base_sid | ((uint64_t)(first_slot + s) << 12) | (uint64_t)c);
        for (int a = 0; a + 1 < m; ++a) {
            const int b = a + (int)mod_u64_u32(stream_word(key, (uint64_t)a), (uint32_t)(m - a));
            const uint32_t x = (col[a >> 5] >> (a & 31)) & 1u, y = (col[b >> 5] >> (b & 31)) & 1u;
            if (x != y) {
                col[a >> 5] ^= 1u << (a & 31);
                col[b >> 5] ^= 1u << (b & 31);
            }
        }
    }
}

// Same columns, written straight into the int8 (count, m, m) layout.
template <int W>
__global__ void k_ref_init_i8(uint64_t seedmix, uint64_t base_sid, int64_t first_slot,
                              int64_t count, int m, int8_t* __restrict__ pop) {
    const int64_t total = count * m;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = t / m;
        const int c = (int)(t - s * m);
        Col<W> col;
        balanced_column<W>(seedmix, base_sid, first_slot + s, m, c, col);
        int8_t* q = pop + s * m * (int64_t)m + c;
        for (int r = 0; r < m; ++r) q[(int64_t)r * m] = get_bit<W>(col, r) ? (int8_t)-1 : (int8_t)1;
    }
}

static int grid1d(int64_t work, int threads = 256) {
    int64_t g = (work + threads - 1) / threads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)sm_count_cached() * 16));
}

constexpr int64_t kPermSmemMax = 50 * 1024;  // int32 entries kept in shared memory

}  // namespace hga

using namespace hga;

extern "C" {

int hga_ref_words(uint64_t seed, uint64_t stream_id, uint64_t counter0, int64_t n, uint64_t* out,
                  void* stream) {
    if (n < 0) return HGA_E_INVALID;
    if (n == 0) return HGA_OK;
    k_ref_words<<<grid1d(n), 256, 0, (cudaStream_t)stream>>>(stream_key(seed, stream_id), counter0, n, out);
    return to_rc(cudaGetLastError());
}

int hga_ref_uniform(uint64_t seed, uint64_t stream_id, uint64_t counter0, int64_t lo, int64_t hi,
                    int64_t n, int64_t* out, void* stream) {
    if (n < 0 || hi < lo) return HGA_E_INVALID;
    if (n == 0) return HGA_OK;
    const uint64_t span = (uint64_t)(hi - lo) + 1;
    k_ref_uniform<<<grid1d(n), 256, 0, (cudaStream_t)stream>>>(stream_key(seed, stream_id), counter0, lo, span, n, out);
    return to_rc(cudaGetLastError());
}

constexpr int64_t kPermParallelMin = 8192;  // above this the parallel replay wins

size_t hga_ref_permutation_ws_bytes(int64_t n) {
    if (n <= 0) return 0;
    size_t b = (n >= kPermParallelMin) ? (size_t)(7 * n + 8) * 4 : (size_t)n * 4;
    if (n > kPermSmemMax && n < kPermParallelMin) b += (size_t)n * 4;
    return (b + 255) & ~(size_t)255;
}

int hga_ref_permutation(uint64_t seed, uint64_t stream_id, uint64_t counter0, int64_t n,
                        int64_t* out, void* ws, size_t ws_bytes, void* stream) {
    if (n < 1 || n >= (int64_t)1 << 31) return HGA_E_INVALID;
    if (ws_bytes < hga_ref_permutation_ws_bytes(n) || !ws) return HGA_E_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    int32_t* b = (int32_t*)ws;
    if (n >= kPermParallelMin) {
        int32_t* cnt = b + n;
        int32_t* off = cnt + n;        // n + 1
        int32_t* cursor = off + n + 1;
        int32_t* grouped = cursor + n;
        int32_t* prev_same = grouped + n;
        int32_t* last_hit = prev_same + n;
        cudaError_t e = cudaMemsetAsync(cnt, 0, (size_t)n * 4, st);
        if (e != cudaSuccess) return to_rc(e);
        const uint64_t key = stream_key(seed, stream_id);
        k_pfy_targets<<<grid1d(n), 256, 0, st>>>(key, counter0, n, b, cnt);
        k_pfy_scan<<<1, 1024, 0, st>>>(cnt, n, off);
        e = cudaMemcpyAsync(cursor, off, (size_t)n * 4, cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) return to_rc(e);
        k_pfy_place<<<grid1d(n), 256, 0, st>>>(b, n, cursor, grouped);
        k_pfy_groups<<<grid1d(n), 256, 0, st>>>(off, n, grouped, prev_same, last_hit);
        k_pfy_final<<<grid1d(n), 256, 0, st>>>(b, prev_same, last_hit, n, out);
        return to_rc(cudaGetLastError());
    }
    int32_t* gperm = b + n;
    if (n > 1)
        k_perm_targets<<<grid1d(n), 256, 0, st>>>(stream_key(seed, stream_id), counter0, n, b);
    const int use_smem = n <= kPermSmemMax;
    const size_t smem = use_smem ? (size_t)n * 4 : 0;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_perm_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return to_rc(e);
    }
    k_perm_chain<<<1, 1024, smem, st>>>(b, n, out, gperm, use_smem);
    return to_rc(cudaGetLastError());
}

int hga_ref_init_packed(uint64_t seed, uint64_t purpose, uint64_t generation, int64_t first_slot,
                        int64_t count, int32_t m, uint32_t* cols, void* stream) {
    if (count < 0 || m < 1 || m > 4096 || first_slot < 0) return HGA_E_INVALID;
    if (count == 0) return HGA_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const uint64_t seedmix = mix64(seed ^ kSeedSalt);
    const uint64_t base = sid(purpose, generation, 0, 0);
    const int64_t work = count * m;
    switch (words_for(m)) {
        case 1: k_ref_init_packed<1><<<grid1d(work), 256, 0, st>>>(seedmix, base, first_slot, count, m, cols); break;
        case 2: k_ref_init_packed<2><<<grid1d(work), 256, 0, st>>>(seedmix, base, first_slot, count, m, cols); break;
        case 3: k_ref_init_packed<3><<<grid1d(work), 256, 0, st>>>(seedmix, base, first_slot, count, m, cols); break;
        case 4: k_ref_init_packed<4><<<grid1d(work), 256, 0, st>>>(seedmix, base, first_slot, count, m, cols); break;
        default:
            k_ref_init_packed_any<<<grid1d(work), 256, 0, st>>>(seedmix, base, first_slot, count, m, words_for(m), cols);
    }
    return to_rc(cudaGetLastError());
}

int hga_ref_init_i8(uint64_t seed, uint64_t purpose, uint64_t generation, int64_t first_slot,
                    int64_t count, int32_t m, int8_t* pop, void* stream) {
    if (count < 0 || m < 1 || m > 32 * kMaxRegWords || first_slot < 0) return HGA_E_INVALID;
    if (count == 0) return HGA_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const uint64_t seedmix = mix64(seed ^ kSeedSalt);
    const uint64_t base = sid(purpose, generation, 0, 0);
    const int64_t work = count * m;
    switch (words_for(m)) {
        case 1: k_ref_init_i8<1><<<grid1d(work), 256, 0, st>>>(seedmix, base, first_slot, count, m, pop); break;
        case 2: k_ref_init_i8<2><<<grid1d(work), 256, 0, st>>>(seedmix, base, first_slot, count, m, pop); break;
        case 3: k_ref_init_i8<3><<<grid1d(work), 256, 0, st>>>(seedmix, base, first_slot, count, m, pop); break;
        default: k_ref_init_i8<4><<<grid1d(work), 256, 0, st>>>(seedmix, base, first_slot, count, m, pop); break;
    }
    return to_rc(cudaGetLastError());
}

}  // extern "C"
