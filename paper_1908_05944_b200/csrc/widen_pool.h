// widen_pool.h -- host threads that widen int32 rows to the int64 rows of the reference's
// AlphaComplex (pipeline.py:117-130) while later chunks are still crossing PCIe.
//
// The device writes its canonical rows as int32 (ball indices < 2^31), so the D2H copy moves
// half the bytes; the widening runs at host-memory speed on a few threads (non-temporal
// stores) and overlaps the copy stream chunk by chunk.  Pure data-type marshalling of the
// result: no geometry runs on the host.
//
// One producer (the thread inside axb_compute_host_finish) publishes tasks; workers claim them
// with an atomic cursor.  Workers sleep on a condition variable between runs and spin inside one.
#pragma once

#include <stdint.h>

#include <atomic>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <vector>

#if defined(__x86_64__)
#include <immintrin.h>
#endif

namespace axb {

struct WidenTask {
    const int32_t *src;
    int64_t *dst;
    size_t n;
};

#if defined(__x86_64__)
__attribute__((target("avx2"))) inline void widen_avx2(const int32_t *src, int64_t *dst, size_t n) {
    size_t i = 0;
    while (i < n && (reinterpret_cast<uintptr_t>(dst + i) & 31u)) { dst[i] = src[i]; ++i; }
    for (; i + 8 <= n; i += 8) {
        const __m256i v = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(src + i));
        const __m256i a = _mm256_cvtepi32_epi64(_mm256_castsi256_si128(v));
        const __m256i b = _mm256_cvtepi32_epi64(_mm256_extracti128_si256(v, 1));
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i), a);
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i + 4), b);
    }
    for (; i < n; ++i) dst[i] = src[i];
    _mm_sfence();
}
#endif

inline void widen_rows(const int32_t *src, int64_t *dst, size_t n) {
#if defined(__x86_64__)
    static const bool have_avx2 = __builtin_cpu_supports("avx2");
    if (have_avx2) { widen_avx2(src, dst, n); return; }
#endif
    for (size_t i = 0; i < n; ++i) dst[i] = src[i];
}

class WidenPool {
public:
    explicit WidenPool(unsigned workers) {
        for (unsigned w = 0; w < workers; ++w) threads_.emplace_back([this]() { worker(); });
    }
    ~WidenPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto &t : threads_) t.join();
    }
    WidenPool(const WidenPool &) = delete;
    WidenPool &operator=(const WidenPool &) = delete;

    // start a run that will publish at most max_tasks tasks
    void begin(size_t max_tasks) {
        if (tasks_.size() < max_tasks) tasks_.resize(max_tasks);
        closed_.store(false);
        published_.store(0);
        next_.store(0);
        done_.store(0);
        {
            std::lock_guard<std::mutex> lk(mu_);
            ++epoch_;
        }
        cv_.notify_all();
    }
    // split [src, src + n) into pieces and publish them (producer thread only)
    void publish(const int32_t *src, int64_t *dst, size_t n, size_t piece) {
        size_t p = published_.load(std::memory_order_relaxed);
        for (size_t lo = 0; lo < n && p < tasks_.size(); lo += piece) {
            tasks_[p++] = WidenTask{src + lo, dst + lo, n - lo < piece ? n - lo : piece};
            published_.store(p, std::memory_order_release);
        }
    }
    // no more tasks: help with what is left and wait until every task has run
    void finish() {
        closed_.store(true);
        drain();
        while (done_.load(std::memory_order_acquire) < published_.load(std::memory_order_relaxed)) cpu_relax();
    }

private:
    static void cpu_relax() {
#if defined(__x86_64__)
        _mm_pause();
#else
        std::this_thread::yield();
#endif
    }
    bool run_one() {
        size_t i = next_.load(std::memory_order_relaxed);
        while (i < published_.load(std::memory_order_acquire)) {
            if (next_.compare_exchange_weak(i, i + 1, std::memory_order_acq_rel)) {
                const WidenTask t = tasks_[i];
                widen_rows(t.src, t.dst, t.n);
                done_.fetch_add(1, std::memory_order_release);
                return true;
            }
        }
        return false;
    }
    void drain() {
        while (run_one()) {}
    }
    void worker() {
        unsigned long long seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&]() { return stop_ || epoch_ != seen; });
                if (stop_) return;
                seen = epoch_;
            }
            for (;;) {
                if (run_one()) continue;
                if (closed_.load(std::memory_order_acquire) &&
                    next_.load(std::memory_order_relaxed) >= published_.load(std::memory_order_acquire))
                    break;
                cpu_relax();
            }
        }
    }

    std::vector<std::thread> threads_;
    std::vector<WidenTask> tasks_;
    std::mutex mu_;
    std::condition_variable cv_;
    unsigned long long epoch_ = 0;
    bool stop_ = false;
    std::atomic<bool> closed_{true};
    std::atomic<size_t> published_{0}, next_{0}, done_{0};
};

}  // namespace axb
