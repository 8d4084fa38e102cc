// Host-side +-1 byte <-> bit packing throughput (AVX2 + OpenMP), 16 MB population
// of the bench config (40,000 order-20 matrices).  Decides whether the drop-in
// host-state step should move bits instead of bytes over PCIe.
//   g++ -O3 -mavx2 -fopenmp scripts/host_pack_probe.cpp -o /tmp/hpp && /tmp/hpp
#include <immintrin.h>
#include <omp.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

static int pack(const int8_t* src, uint32_t* dst, int64_t nwords, int threads) {
    int bad = 0;
#pragma omp parallel for num_threads(threads) schedule(static) reduction(| : bad)
    for (int64_t w = 0; w < nwords; ++w) {
        const __m256i v = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + 32 * w));
        const __m256i ok = _mm256_or_si256(_mm256_cmpeq_epi8(v, _mm256_set1_epi8(1)),
                                           _mm256_cmpeq_epi8(v, _mm256_set1_epi8(-1)));
        bad |= ~_mm256_movemask_epi8(ok) != 0;
        dst[w] = (uint32_t)_mm256_movemask_epi8(v);
    }
    return bad;
}

static void unpack(const uint32_t* src, int8_t* dst, int64_t nwords, int threads) {
    const __m256i shuf = _mm256_setr_epi8(0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 1, 1, 1, 1, 2, 2, 2, 2, 2, 2, 2, 2, 3, 3,
                                          3, 3, 3, 3, 3, 3);
    const __m256i sel = _mm256_set1_epi64x(0x8040201008040201ll);
#pragma omp parallel for num_threads(threads) schedule(static)
    for (int64_t w = 0; w < nwords; ++w) {
        const __m256i b = _mm256_shuffle_epi8(_mm256_set1_epi32((int)src[w]), shuf);
        const __m256i m = _mm256_cmpeq_epi8(_mm256_and_si256(b, sel), sel);  // 0xFF where the bit is set
        _mm256_storeu_si256(reinterpret_cast<__m256i*>(dst + 32 * w), _mm256_or_si256(m, _mm256_set1_epi8(1)));
    }
}

int main() {
    const int64_t bytes = 40000LL * 400, nwords = bytes / 32;
    std::vector<int8_t> a(bytes), b(bytes);
    std::vector<uint32_t> p(nwords);
    srand(1);
    for (auto& x : a) x = (rand() & 1) ? 1 : -1;
    const int maxt = omp_get_num_procs();
    for (int t : {1, 2, 4, 8, 16, 32}) {
        if (t > maxt) break;
        for (int rep = 0; rep < 3; ++rep) pack(a.data(), p.data(), nwords, t), unpack(p.data(), b.data(), nwords, t);
        const int R = 50;
        auto t0 = std::chrono::steady_clock::now();
        int bad = 0;
        for (int r = 0; r < R; ++r) bad |= pack(a.data(), p.data(), nwords, t);
        auto t1 = std::chrono::steady_clock::now();
        for (int r = 0; r < R; ++r) unpack(p.data(), b.data(), nwords, t);
        auto t2 = std::chrono::steady_clock::now();
        const double tp = std::chrono::duration<double>(t1 - t0).count() / R;
        const double tu = std::chrono::duration<double>(t2 - t1).count() / R;
        std::printf("{\"threads\": %d, \"pack_us\": %.1f, \"pack_GBps\": %.1f, \"unpack_us\": %.1f, \"unpack_GBps\": %.1f, "
                    "\"roundtrip_ok\": %d, \"bad\": %d}\n",
                    t, tp * 1e6, bytes / tp / 1e9, tu * 1e6, bytes / tu / 1e9, (int)(memcmp(a.data(), b.data(), bytes) == 0),
                    bad);
    }
    return 0;
}
