// host_bits.cpp -- host half of the bit-stream transfer of hga_step_host_bits.
//
// The drop-in step on a HOST state (reference engine.py:449-469 with numpy
// arrays) must move the caller's int8 (4N, m, m) population to the GPU and
// back every generation.  Over PCIe that is 2 x 16 MB at the bench config
// (~0.3 ms each way at ~55 GB/s); every entry is +-1, i.e. one bit of
// information per byte.  The host therefore moves a flat bit stream instead
// (bit e of the stream = sign of byte e of the population, 8x fewer bytes):
//   pack    byte e -> bit e (AVX2 movemask), validating every byte is +-1
//   unpack  bit e -> byte e (+1 / -1)
// Both run on a small persistent thread pool (std::thread; no OpenMP so the
// library does not bring a second OpenMP runtime into a torch process) at
// host-memory speed (~300 GB/s on the B200 box's 16 cores, L3-resident).
// The device side (bit stream <-> packed column records) is
// csrc/step_bits.cu.
#include <immintrin.h>
#include <pthread.h>
#include <sched.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <new>
#include <thread>
#include <vector>

#include "../../include/hga.h"

namespace hga {
namespace host {

// ------------------------------------------------------------ thread pool
class Pool {
   public:
    static Pool& get() {
        static Pool* p = make();  // never destroyed: workers may outlive static destruction order
        return *p;
    }
    int size() const { return inline_mode() ? 1 : (int)workers_.size() + 1; }
    // start(): runs fn(ctx, t) for t in [0, ntasks) on the worker threads; the
    // calling thread does not take tasks (it drives the CUDA side meanwhile).
    // wait() returns when all tasks are done.  One job at a time: the job lock
    // is held from start() to wait().  A worker only takes a task of the job it
    // sees (compare-exchange on job id | ntasks | next task), so a straggler of
    // the previous job can never run or count a task of this one.
    void start(int ntasks, void (*fn)(void*, int), void* ctx) {
        job_mu_.lock();
        started_ = ntasks;
        if (inline_mode() || ntasks >= (1 << 20)) {
            for (int t = 0; t < ntasks; ++t) fn(ctx, t);  // no workers: run inline (callbacks still see progress)
            started_ = -1;
            return;
        }
        fn_ = fn;
        ctx_ = ctx;
        done_.store(0, std::memory_order_relaxed);
        job_ = (job_ + 1) & 0xFFFFFFull;
        ticket_.store((job_ << 40) | ((uint64_t)ntasks << 20), std::memory_order_release);
        {
            std::lock_guard<std::mutex> lk(mu_);
            gen_.fetch_add(1, std::memory_order_release);
        }
        cv_.notify_all();
    }
    void wait() {
        if (started_ >= 0)
            while (done_.load(std::memory_order_acquire) < started_) _mm_pause();
        job_mu_.unlock();
    }
    // A forked child has none of the parent's worker threads: it runs every
    // job inline on fresh locks (pthread_atfork below).
    bool inline_mode() const { return workers_.empty() || forked_; }

   private:
    static Pool* make() {
        Pool* p = new Pool();
        instance_ = p;
        pthread_atfork(nullptr, nullptr, [] {
            if (Pool* q = instance_) {
                new (&q->job_mu_) std::mutex();
                new (&q->mu_) std::mutex();
                new (&q->cv_) std::condition_variable();
                q->forked_ = true;
            }
        });
        return p;
    }
    static inline Pool* instance_ = nullptr;
    bool forked_ = false;
    int started_ = 0;
    Pool() {
        int n = 0;
        cpu_set_t set;
        if (sched_getaffinity(0, sizeof(set), &set) == 0) n = CPU_COUNT(&set);
        if (n <= 0) n = (int)std::thread::hardware_concurrency();
        if (const char* e = std::getenv("HGA_HOST_THREADS")) n = std::atoi(e);
        n = std::max(1, std::min(n, 32));
        for (int i = 1; i < n; ++i) workers_.emplace_back([this] { loop(); });
        for (auto& t : workers_) t.detach();
    }
    void work() {
        uint64_t cur = ticket_.load(std::memory_order_acquire);
        for (;;) {
            const uint64_t next = cur & 0xFFFFFull, ntasks = (cur >> 20) & 0xFFFFFull;
            if (next >= ntasks) return;
            if (!ticket_.compare_exchange_weak(cur, cur + 1, std::memory_order_acq_rel, std::memory_order_acquire))
                continue;  // cur reloaded
            fn_(ctx_, (int)next);
            done_.fetch_add(1, std::memory_order_release);
            cur = ticket_.load(std::memory_order_acquire);
        }
    }
    void loop() {
        // 0, not the current value: a worker that starts running only after the
        // first job was posted must still see that job (the caller of start() does
        // not take tasks itself, so a job nobody sees would never finish)
        uint64_t seen = 0;
        for (;;) {
            // spin a little (back-to-back steps arrive every few hundred us), then sleep
            int spins = 0;
            while (gen_.load(std::memory_order_acquire) == seen && spins < (1 << 16)) {
                _mm_pause();
                ++spins;
            }
            if (gen_.load(std::memory_order_acquire) == seen) {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_.load(std::memory_order_acquire) != seen; });
            }
            seen = gen_.load(std::memory_order_acquire);
            work();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex job_mu_, mu_;
    std::condition_variable cv_;
    std::atomic<uint64_t> gen_{0};
    std::atomic<uint64_t> ticket_{0};
    std::atomic<int> done_{0};
    uint64_t job_ = 0;
    void (*fn_)(void*, int) = nullptr;
    void* ctx_ = nullptr;
};

// ------------------------------------------------------------ kernels
static bool have_avx2() {
    static const bool v = __builtin_cpu_supports("avx2");
    return v;
}

// bytes [32 w0, 32 w1) of src (clipped to nbytes) -> words [w0, w1) of dst.
// Returns nonzero when some byte is not +-1.
__attribute__((target("avx2"))) static uint32_t pack_avx2(const int8_t* src, int64_t nbytes, uint32_t* dst,
                                                          int64_t w0, int64_t w1) {
    const int64_t full = std::min<int64_t>(w1, nbytes / 32);
    const __m256i one = _mm256_set1_epi8(1), mone = _mm256_set1_epi8(-1);
    uint32_t bad = 0;
    int64_t w = w0;
    for (; w < full; ++w) {
        const __m256i v = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + 32 * w));
        const __m256i ok = _mm256_or_si256(_mm256_cmpeq_epi8(v, one), _mm256_cmpeq_epi8(v, mone));
        bad |= ~(uint32_t)_mm256_movemask_epi8(ok);
        dst[w] = (uint32_t)_mm256_movemask_epi8(v);
    }
    for (; w < w1; ++w) {  // the last, partial word
        uint32_t bits = 0;
        for (int b = 0; b < 32 && 32 * w + b < nbytes; ++b) {
            const int8_t x = src[32 * w + b];
            bad |= (uint32_t)(x != 1 && x != -1);
            bits |= (uint32_t)(x < 0) << b;
        }
        dst[w] = bits;
    }
    return bad;
}

static uint32_t pack_scalar(const int8_t* src, int64_t nbytes, uint32_t* dst, int64_t w0, int64_t w1) {
    uint32_t bad = 0;
    for (int64_t w = w0; w < w1; ++w) {
        uint32_t bits = 0;
        for (int b = 0; b < 32 && 32 * w + b < nbytes; ++b) {
            const int8_t x = src[32 * w + b];
            bad |= (uint32_t)(x != 1 && x != -1);
            bits |= (uint32_t)(x < 0) << b;
        }
        dst[w] = bits;
    }
    return bad;
}

// words [w0, w1) of src -> bytes [32 w0, 32 w1) of dst (clipped to nbytes)
__attribute__((target("avx2"))) static void unpack_avx2(const uint32_t* src, int8_t* dst, int64_t nbytes, int64_t w0,
                                                        int64_t w1) {
    const int64_t full = std::min<int64_t>(w1, nbytes / 32);
    const __m256i shuf = _mm256_setr_epi8(0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 1, 1, 1, 1, 2, 2, 2, 2, 2, 2, 2, 2, 3, 3,
                                          3, 3, 3, 3, 3, 3);
    const __m256i sel = _mm256_set1_epi64x(0x8040201008040201ll);
    const __m256i one = _mm256_set1_epi8(1);
    int64_t w = w0;
    for (; w < full; ++w) {
        const __m256i b = _mm256_shuffle_epi8(_mm256_set1_epi32((int)src[w]), shuf);
        const __m256i m = _mm256_cmpeq_epi8(_mm256_and_si256(b, sel), sel);  // 0xFF where the bit is set
        _mm256_storeu_si256(reinterpret_cast<__m256i*>(dst + 32 * w), _mm256_or_si256(m, one));
    }
    for (; w < w1; ++w)
        for (int b = 0; b < 32 && 32 * w + b < nbytes; ++b) dst[32 * w + b] = ((src[w] >> b) & 1u) ? -1 : 1;
}

static void unpack_scalar(const uint32_t* src, int8_t* dst, int64_t nbytes, int64_t w0, int64_t w1) {
    for (int64_t w = w0; w < w1; ++w)
        for (int b = 0; b < 32 && 32 * w + b < nbytes; ++b) dst[32 * w + b] = ((src[w] >> b) & 1u) ? -1 : 1;
}

static int parts_for(int64_t words) {
    // ~16 KB of int8 per task at least: dispatch costs ~1 us per task
    const int64_t p = std::max<int64_t>(1, words / 512);
    return (int)std::min<int64_t>(p, 4 * (int64_t)Pool::get().size());
}

constexpr int kMaxPieces = 64;

// k pieces x `parts` tasks, piece-major, so pieces complete roughly in order
struct PieceJob {
    const int8_t* src8 = nullptr;
    int8_t* dst8 = nullptr;
    const uint32_t* src32 = nullptr;
    uint32_t* dst32 = nullptr;
    int64_t nbytes = 0;
    const int64_t* wlo = nullptr;
    int k = 0, parts = 1;
    std::atomic<int> piece_done[kMaxPieces];
    std::atomic<int> ready[kMaxPieces];
    std::atomic<int> abort{0};
    std::atomic<uint32_t> bad{0};
    PieceJob() {
        for (auto& x : piece_done) x.store(0, std::memory_order_relaxed);
        for (auto& x : ready) x.store(0, std::memory_order_relaxed);
    }
    void range(int t, int64_t& a, int64_t& b) const {
        const int i = t / parts, q = t % parts;
        const int64_t n = wlo[i + 1] - wlo[i];
        a = wlo[i] + n * q / parts;
        b = wlo[i] + n * (q + 1) / parts;
    }
};

static void pack_piece_task(void* p, int t) {
    PieceJob& j = *static_cast<PieceJob*>(p);
    int64_t a, b;
    j.range(t, a, b);
    const uint32_t bad = have_avx2() ? pack_avx2(j.src8, j.nbytes, j.dst32, a, b) : pack_scalar(j.src8, j.nbytes, j.dst32, a, b);
    if (bad) j.bad.fetch_or(1u, std::memory_order_relaxed);
    j.piece_done[t / j.parts].fetch_add(1, std::memory_order_release);
}

static void unpack_piece_task(void* p, int t) {
    PieceJob& j = *static_cast<PieceJob*>(p);
    const int i = t / j.parts;
    while (!j.ready[i].load(std::memory_order_acquire)) _mm_pause();  // the piece has landed
    if (j.abort.load(std::memory_order_relaxed)) return;
    int64_t a, b;
    j.range(t, a, b);
    if (have_avx2()) unpack_avx2(j.src32, j.dst8, j.nbytes, a, b);
    else unpack_scalar(j.src32, j.dst8, j.nbytes, a, b);
}

}  // namespace host

// Pack the stream words [wlo[0], wlo[k]) in k pieces on the pool; started(ctx)
// (optional) runs on the calling thread while the workers pack, then
// on_piece(ctx, i) as soon as piece i is packed (in order; a nonzero return
// of either stops the calls and is passed back).  Returns 1 when some byte is
// not +-1 (no more pieces are handed out then), else the callbacks' status.
int host_pack_pieces(const int8_t* src, int64_t nbytes, uint32_t* dst, const int64_t* wlo, int k,
                     int (*started)(void*), int (*on_piece)(void*, int), void* ctx) {
    if (k < 1 || k > host::kMaxPieces) return -1;
    host::Pool& pool = host::Pool::get();
    host::PieceJob j;
    j.src8 = src;
    j.dst32 = dst;
    j.nbytes = nbytes;
    j.wlo = wlo;
    j.k = k;
    j.parts = std::max(1, host::parts_for((wlo[k] - wlo[0]) / k));
    pool.start(k * j.parts, host::pack_piece_task, &j);
    int rc = started ? started(ctx) : 0;
    for (int i = 0; i < k && !rc; ++i) {
        while (j.piece_done[i].load(std::memory_order_acquire) < j.parts) _mm_pause();
        if (j.bad.load(std::memory_order_relaxed)) break;
        rc = on_piece(ctx, i);
    }
    pool.wait();
    return j.bad.load() ? 1 : rc;
}

// Unpack the stream words [wlo[0], wlo[k]) in k pieces on the pool: piece i is
// unpacked as soon as landed(ctx, i) -- called on the calling thread, in
// order -- has returned 0; a nonzero return skips the remaining pieces.
int host_unpack_pieces(const uint32_t* src, int8_t* dst, int64_t nbytes, const int64_t* wlo, int k,
                       int (*landed)(void*, int), void* ctx) {
    if (k < 1 || k > host::kMaxPieces) return -1;
    host::Pool& pool = host::Pool::get();
    host::PieceJob j;
    j.src32 = src;
    j.dst8 = dst;
    j.nbytes = nbytes;
    j.wlo = wlo;
    j.k = k;
    j.parts = std::max(1, host::parts_for((wlo[k] - wlo[0]) / k));
    if (pool.inline_mode()) {  // no workers: wait, then unpack inline
        int rc = 0;
        for (int i = 0; i < k && !rc; ++i) {
            rc = landed(ctx, i);
            if (!rc)
                for (int q = 0; q < j.parts; ++q) {
                    j.ready[i].store(1);
                    host::unpack_piece_task(&j, i * j.parts + q);
                }
        }
        return rc;
    }
    pool.start(k * j.parts, host::unpack_piece_task, &j);
    int rc = 0;
    for (int i = 0; i < k; ++i) {
        if (!rc) rc = landed(ctx, i);
        if (rc) j.abort.store(1, std::memory_order_relaxed);
        j.ready[i].store(1, std::memory_order_release);
    }
    pool.wait();
    return rc;
}

int host_pool_threads() { return host::Pool::get().size(); }

}  // namespace hga

static int no_piece_cb(void*, int) { return 0; }

extern "C" int hga_host_pack_bits(const int8_t* src, int64_t n, uint32_t* dst) {
    if (n <= 0) return 0;
    const int64_t wlo[2] = {0, (n + 31) / 32};
    return hga::host_pack_pieces(src, n, dst, wlo, 1, nullptr, no_piece_cb, nullptr) == 1 ? HGA_FLAG_NOT_SIGN : 0;
}

extern "C" void hga_host_unpack_bits(const uint32_t* src, int64_t n, int8_t* dst) {
    if (n <= 0) return;
    const int64_t wlo[2] = {0, (n + 31) / 32};
    hga::host_unpack_pieces(src, dst, n, wlo, 1, no_piece_cb, nullptr);
}
