// operators.cu -- the reference's select / crossover / mutate on device
// (engine.py:233-373), with the reference's exact semantics.
//
//   crossover_i8   engine.crossover   (engine.py:257-277), int8 layout, in place
//   mutate_i8      engine.mutate      (engine.py:339-373), int8 layout, in place
//   select_order   argsort(F, stable)[:total/2]             (engine.py:245)
//   compose_gather chosen = order[perm]; rows/fitness gather (engine.py:246-248)
//   argmin_key     first-minimum argmin                      (engine.py:417, 432)
#include <cub/device/device_radix_sort.cuh>

#include "hga_common.cuh"

namespace hga {

static int grid_1d(int64_t work, int threads = 256) {
    int64_t g = (work + threads - 1) / threads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)sm_count_cached() * 16));
}

// ------------------------------------------------------------- crossover
// One thread per (pair, row): 4-byte chunks with a byte mask at the split.
__global__ void k_crossover_i8(int8_t* pop, int64_t n_pairs, int m, const int64_t* __restrict__ points,
                               int32_t* bad_flag) {
    const int64_t mm = (int64_t)m * m;
    const int64_t work = n_pairs * m;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < work;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = t / m;
        const int r = (int)(t - p * m);
        const int64_t c = points[p];
        if (c < 1 || c > m - 1) {
            if (r == 0 && bad_flag) atomicOr(bad_flag, HGA_FLAG_POINT_RANGE);
            continue;
        }
        const int64_t row = (int64_t)r * m;
        const int8_t* a = pop + p * mm + row;
        const int8_t* b = pop + (n_pairs + p) * mm + row;
        int8_t* o1 = pop + (2 * n_pairs + p) * mm + row;
        int8_t* o2 = pop + (3 * n_pairs + p) * mm + row;
        if ((m & 3) == 0 && ((((uintptr_t)pop) & 3) == 0)) {
            for (int j0 = 0; j0 < m; j0 += 4) {
                const uint32_t x = *reinterpret_cast<const uint32_t*>(a + j0);
                const uint32_t y = *reinterpret_cast<const uint32_t*>(b + j0);
                const int64_t keep = c - j0;  // leading bytes of this chunk taken from the "left" parent
                const uint32_t mask = keep >= 4 ? 0xFFFFFFFFu : (keep <= 0 ? 0u : ((1u << (8 * keep)) - 1u));
                *reinterpret_cast<uint32_t*>(o1 + j0) = (x & mask) | (y & ~mask);
                *reinterpret_cast<uint32_t*>(o2 + j0) = (y & mask) | (x & ~mask);
            }
        } else {
            for (int j = 0; j < m; ++j) {
                const int8_t x = a[j], y = b[j];
                o1[j] = j < c ? x : y;
                o2[j] = j < c ? y : x;
            }
        }
    }
}

// --------------------------------------------------------------- mutate
// One thread per offspring; columns in plan order, row pairs inner, exactly
// the reference's sequential semantics (duplicates re-apply).
__global__ void k_mutate_i8(int8_t* pop, int64_t half, int m, const int64_t* __restrict__ cols,
                            const int64_t* __restrict__ ra, const int64_t* __restrict__ rb, int nc,
                            int nr, int32_t* bad_flag) {
    const int64_t mm = (int64_t)m * m;
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < half;
         o += (int64_t)gridDim.x * blockDim.x) {
        bool ok = true;
        for (int jc = 0; jc < nc; ++jc) ok &= cols[o * nc + jc] >= 1 && cols[o * nc + jc] <= m - 1;
        for (int ir = 0; ir < nr; ++ir)
            ok &= ra[o * nr + ir] >= 0 && ra[o * nr + ir] <= m - 1 && rb[o * nr + ir] >= 0 && rb[o * nr + ir] <= m - 1;
        if (!ok) {
            if (bad_flag) atomicOr(bad_flag, HGA_FLAG_PLAN_RANGE);
            continue;
        }
        int8_t* q = pop + (half + o) * mm;
        for (int jc = 0; jc < nc; ++jc) {
            const int64_t c = cols[o * nc + jc];
            for (int ir = 0; ir < nr; ++ir) {
                int8_t* x = q + ra[o * nr + ir] * m + c;
                int8_t* y = q + rb[o * nr + ir] * m + c;
                const int8_t u = *x, v = *y;
                if (u != v) {
                    *x = v;
                    *y = u;
                }
            }
        }
    }
}

// ----------------------------------------------------------------- select
// Stable order of the `half` smallest fitness values: the range (min, max)
// of the values, then a stable LSD radix sort (CUB) of the 22-bit keys
// F - min with their indices -- equal values keep index order, the
// stable-argsort tie rule (engine.py:245).  Three digit passes at any
// population size (round 1 scattered the indices from a histogram with one
// warp: 0.78 ms at 4N = 40,000).
constexpr int kSelBits = 22;
constexpr int64_t kSelMaxRange = (int64_t)1 << kSelBits;

struct SelWs {
    long long mn, mx;
};

__global__ void k_sel_minmax(const int64_t* __restrict__ f, int64_t n, SelWs* w) {
    long long mn = LLONG_MAX, mx = LLONG_MIN;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        mn = min(mn, (long long)f[i]);
        mx = max(mx, (long long)f[i]);
    }
    for (int o = 16; o; o >>= 1) {
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&w->mn, mn);
        atomicMax(&w->mx, mx);
    }
}

__global__ void k_sel_init(SelWs* w) {
    w->mn = LLONG_MAX;
    w->mx = LLONG_MIN;
}

// 22-bit sort keys F - min and their indices; a range of 2^22 or more raises
// HGA_FLAG_FIT_RANGE (the keys are then clamped and the order is not valid).
__global__ void k_sel_keys(const int64_t* __restrict__ f, int64_t n, const SelWs* w, uint32_t* __restrict__ keys,
                           int32_t* __restrict__ idx, int32_t* bad_flag) {
    const long long mn = w->mn;
    if ((unsigned long long)(w->mx - mn) >= (unsigned long long)kSelMaxRange && blockIdx.x == 0 && threadIdx.x == 0 &&
        bad_flag)
        atomicOr(bad_flag, HGA_FLAG_FIT_RANGE);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long d = (unsigned long long)((long long)f[i] - mn);
        keys[i] = (uint32_t)min(d, (unsigned long long)(kSelMaxRange - 1));
        idx[i] = (int32_t)i;
    }
}

__global__ void k_sel_order(const int32_t* __restrict__ idx, int64_t k, int64_t* __restrict__ order) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
        order[i] = idx[i];
}

static size_t sel_temp_bytes(int64_t n) {
    size_t t = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, t, (uint32_t*)nullptr, (uint32_t*)nullptr, (int32_t*)nullptr,
                                    (int32_t*)nullptr, (int)n, 0, kSelBits);
    return (t + 255) & ~(size_t)255;
}

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

// Any-range fallback: stable LSD radix sort of (fitness, index) pairs.  int64
// keys become order-preserving uint64 (sign bit flipped); CUB's radix sort is
// stable, so equal values keep index order (the stable-argsort tie rule).
__global__ void k_sel_radix_prep(const int64_t* __restrict__ f, int64_t n, unsigned long long* __restrict__ keys,
                                 int64_t* __restrict__ idx) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        keys[i] = (unsigned long long)f[i] ^ 0x8000000000000000ull;
        idx[i] = i;
    }
}

static size_t radix_temp_bytes(int64_t n) {
    size_t t = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, t, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                    (int64_t*)nullptr, (int64_t*)nullptr, (int)n);
    return (t + 255) & ~(size_t)255;
}

// -------------------------------------------------------- compose + gather
template <typename V>
__global__ void k_compose_gather(const int64_t* __restrict__ order, const int64_t* __restrict__ perm,
                                 int64_t count, const V* __restrict__ src, V* __restrict__ dst,
                                 int64_t vec_per_matrix, const int64_t* __restrict__ fit_src,
                                 int64_t* __restrict__ fit_dst, int64_t* __restrict__ chosen) {
    const int64_t work = count * vec_per_matrix;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < work;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = t / vec_per_matrix;
        const int64_t v = t - s * vec_per_matrix;
        const int64_t c = perm ? order[perm[s]] : order[s];
        if (src) dst[s * vec_per_matrix + v] = src[c * vec_per_matrix + v];
        if (v == 0) {
            if (fit_dst) fit_dst[s] = fit_src[c];
            if (chosen) chosen[s] = c;
        }
    }
}

// ----------------------------------------------------------------- argmin
__global__ void k_argmin_key(const int64_t* __restrict__ f, int64_t n, unsigned long long* key) {
    unsigned long long best = ~0ull;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        best = min(best, ((unsigned long long)f[i] << 32) | (unsigned long long)i);
    for (int o = 16; o; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0) atomicMin(key, best);
}

__global__ void k_set_u64(unsigned long long* p, unsigned long long v) { *p = v; }

}  // namespace hga

using namespace hga;

// _check_state (engine.py:440-446) on the packed resident population: per
// (matrix, column) thread, column 0 must have no -1 bit and every other
// column exactly m/2; per matrix (column-0 thread) the stored fitness must
// equal the freshly recomputed one.  counts[0] = bad first columns,
// counts[1] = unbalanced columns, counts[2] = stale fitness values.
__global__ void k_check_invariants(const uint32_t* __restrict__ cols, const int64_t* __restrict__ fit,
                                   const int64_t* __restrict__ fresh, int64_t n, int m,
                                   unsigned long long* counts) {
    const int W = words_for(m);
    unsigned long long c0 = 0, c1 = 0, c2 = 0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * m; t += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(t % m);
        int neg = 0;
        for (int w = 0; w < W; ++w) neg += __popc(cols[t * W + w]);
        if (j == 0) {
            c0 += neg != 0;
            c2 += fit[t / m] != fresh[t / m];
        } else {
            c1 += neg != m / 2;
        }
    }
    if (c0) atomicAdd(&counts[0], c0);
    if (c1) atomicAdd(&counts[1], c1);
    if (c2) atomicAdd(&counts[2], c2);
}

extern "C" {

int hga_crossover_i8(int8_t* pop, int64_t total, int32_t m, const int64_t* points, int32_t* bad_flag,
                     void* stream) {
    if (total < 0 || total % 4 || m < 1) return HGA_E_INVALID;
    if (total == 0 || m == 1) return HGA_OK;
    const int64_t np_ = total / 4;
    k_crossover_i8<<<grid_1d(np_ * m), 256, 0, (cudaStream_t)stream>>>(pop, np_, m, points, bad_flag);
    return to_rc(cudaGetLastError());
}

int hga_mutate_i8(int8_t* pop, int64_t total, int32_t m, const int64_t* cols, const int64_t* ra,
                  const int64_t* rb, int32_t nc, int32_t nr, int32_t* bad_flag, void* stream) {
    if (total < 0 || total % 2 || m < 1 || nc < 0 || nr < 0) return HGA_E_INVALID;
    const int64_t half = total / 2;
    if (half == 0 || nc == 0 || nr == 0) return HGA_OK;
    k_mutate_i8<<<grid_1d(half, 128), 128, 0, (cudaStream_t)stream>>>(pop, half, m, cols, ra, rb, nc, nr, bad_flag);
    return to_rc(cudaGetLastError());
}

int64_t hga_select_max_range(void) { return kSelMaxRange; }

size_t hga_select_ws_bytes(int64_t total) {
    if (total < 0 || total >= ((int64_t)1 << 31)) return 0;
    const int64_t n = std::max<int64_t>(total, 1);
    return 256 + 4 * align256((size_t)n * 4) + sel_temp_bytes(n);
}

int hga_select_order(const int64_t* fitness, int64_t total, int64_t* order, int32_t* bad_flag, void* ws,
                     size_t ws_bytes, void* stream) {
    if (total < 0) return HGA_E_INVALID;
    return hga_select_smallest(fitness, total, total / 2, order, bad_flag, ws, ws_bytes, stream);
}

size_t hga_select_radix_ws_bytes(int64_t total) {
    if (total <= 0 || total >= ((int64_t)1 << 31)) return 0;
    return (size_t)total * 32 + radix_temp_bytes(total);
}

int hga_select_smallest_radix(const int64_t* fitness, int64_t total, int64_t k, int64_t* order, void* ws,
                              size_t ws_bytes, void* stream) {
    if (total < 0 || total >= ((int64_t)1 << 31) || k < 0 || k > total) return HGA_E_INVALID;
    if (k == 0) return HGA_OK;
    if (!ws || ws_bytes < hga_select_radix_ws_bytes(total)) return HGA_E_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    unsigned long long* keys_in = (unsigned long long*)ws;
    unsigned long long* keys_out = keys_in + total;
    int64_t* idx_in = (int64_t*)(keys_out + total);
    int64_t* idx_out = idx_in + total;
    void* temp = idx_out + total;
    size_t temp_bytes = radix_temp_bytes(total);
    k_sel_radix_prep<<<grid_1d(total), 256, 0, st>>>(fitness, total, keys_in, idx_in);
    cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, idx_in, idx_out, (int)total,
                                                    0, 64, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(order, idx_out, (size_t)k * sizeof(int64_t), cudaMemcpyDeviceToDevice, st);
    return to_rc(e);
}

int hga_select_smallest(const int64_t* fitness, int64_t total, int64_t k, int64_t* order, int32_t* bad_flag,
                        void* ws, size_t ws_bytes, void* stream) {
    if (total < 0 || k < 0 || k > total) return HGA_E_INVALID;
    if (k == 0) return HGA_OK;
    if (total >= ((int64_t)1 << 31)) return HGA_E_UNSUPPORTED;
    if (!ws || ws_bytes < hga_select_ws_bytes(total)) return HGA_E_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    SelWs* w = (SelWs*)ws;
    char* p = (char*)ws + 256;
    const size_t region = align256((size_t)total * 4);
    uint32_t* keys_in = (uint32_t*)p;
    uint32_t* keys_out = (uint32_t*)(p + region);
    int32_t* idx_in = (int32_t*)(p + 2 * region);
    int32_t* idx_out = (int32_t*)(p + 3 * region);
    void* temp = p + 4 * region;
    size_t temp_bytes = sel_temp_bytes(total);
    k_sel_init<<<1, 1, 0, st>>>(w);
    k_sel_minmax<<<grid_1d(total), 256, 0, st>>>(fitness, total, w);
    k_sel_keys<<<grid_1d(total), 256, 0, st>>>(fitness, total, w, keys_in, idx_in, bad_flag);
    cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, idx_in, idx_out, (int)total, 0,
                                                    kSelBits, st);
    if (e != cudaSuccess) return to_rc(e);
    k_sel_order<<<grid_1d(k), 256, 0, st>>>(idx_out, k, order);
    return to_rc(cudaGetLastError());
}

int hga_compose_gather(const int64_t* order, const int64_t* perm, int64_t count, const void* src, void* dst,
                       int64_t bytes_per_matrix, const int64_t* fit_src, int64_t* fit_dst, int64_t* chosen,
                       void* stream) {
    if (count < 0 || bytes_per_matrix < 0) return HGA_E_INVALID;
    if (count == 0) return HGA_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const uintptr_t al = (uintptr_t)src | (uintptr_t)dst | (uintptr_t)bytes_per_matrix;
    if (!src || bytes_per_matrix == 0) {
        k_compose_gather<uint8_t><<<grid_1d(count), 256, 0, st>>>(order, perm, count, nullptr, nullptr, 1,
                                                                   fit_src, fit_dst, chosen);
    } else if ((al & 15) == 0) {
        const int64_t v = bytes_per_matrix / 16;
        k_compose_gather<uint4><<<grid_1d(count * v), 256, 0, st>>>(order, perm, count, (const uint4*)src,
                                                                    (uint4*)dst, v, fit_src, fit_dst, chosen);
    } else if ((al & 3) == 0) {
        const int64_t v = bytes_per_matrix / 4;
        k_compose_gather<uint32_t><<<grid_1d(count * v), 256, 0, st>>>(order, perm, count, (const uint32_t*)src,
                                                                        (uint32_t*)dst, v, fit_src, fit_dst, chosen);
    } else {
        k_compose_gather<uint8_t><<<grid_1d(count * bytes_per_matrix), 256, 0, st>>>(
            order, perm, count, (const uint8_t*)src, (uint8_t*)dst, bytes_per_matrix, fit_src, fit_dst, chosen);
    }
    return to_rc(cudaGetLastError());
}

size_t hga_check_invariants_ws_bytes(int64_t n) { return n > 0 ? (size_t)n * sizeof(int64_t) : 0; }

int hga_check_invariants(const uint32_t* cols, const int64_t* fit, int64_t n, int32_t m, uint32_t fit_var,
                         unsigned long long* counts, void* ws, size_t ws_bytes, void* stream) {
    if (n < 0 || m < 4 || m > 4096 || (m & 3) || !counts ||
        (fit_var != HGA_VAR_F1 && fit_var != HGA_VAR_F2 && fit_var != HGA_VAR_SQ))
        return HGA_E_INVALID;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(counts, 0, 3 * sizeof(unsigned long long), st);
    if (e != cudaSuccess) return to_rc(e);
    if (n == 0) return HGA_OK;
    if (!ws || ws_bytes < hga_check_invariants_ws_bytes(n)) return HGA_E_WORKSPACE;
    int64_t* fresh = (int64_t*)ws;
    const int rc = hga_fitness_packed(cols, n, m, fit_var, fit_var == HGA_VAR_F1 ? fresh : nullptr,
                                      fit_var == HGA_VAR_F2 ? fresh : nullptr, nullptr,
                                      fit_var == HGA_VAR_SQ ? fresh : nullptr, stream);
    if (rc) return rc;
    k_check_invariants<<<grid_1d(n * (int64_t)m), 256, 0, st>>>(cols, fit, fresh, n, m, counts);
    return to_rc(cudaGetLastError());
}

int hga_argmin_key(const int64_t* fit, int64_t n, unsigned long long* key, int init, void* stream) {
    if (n < 0) return HGA_E_INVALID;
    cudaStream_t st = (cudaStream_t)stream;
    if (init) k_set_u64<<<1, 1, 0, st>>>(key, ~0ull);
    if (n > 0) k_argmin_key<<<grid_1d(n), 256, 0, st>>>(fit, n, key);
    return to_rc(cudaGetLastError());
}

}  // extern "C"
