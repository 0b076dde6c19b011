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
#include <string.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <vector>

#if defined(__x86_64__)
#include <immintrin.h>
#endif

namespace axb {

// What a task produces (dst is always int64):
//   WIDEN     n values copied 1:1
//   EDGE_ROWS rows [row0, row0 + n) of the edge list: (owner, src[r]); owner of row r = the ball a with
//             off[a] <= r < off[a + 1]  (the rows are sorted by their first column, so the device sends
//             only the second column plus the n_index + 1 offsets -- 4 instead of 8 bytes per edge)
//   TRI_ROWS  same for triangles: (owner, src[2r], src[2r + 1]) -- 8 instead of 12 bytes per triangle
//   IOTA      n consecutive values starting at row0 (all vertices kept: nothing crosses PCIe)
//   COPY      n int32 values copied verbatim (pageable input -> pinned staging, in parallel)
//   UNPACK24  n values of a 24-bit chunk: src = chunk base, n_index = values in the chunk (the high bytes start
//             2 * n_index bytes in), row0 = first value of this task inside the chunk
enum WidenKind { WK_WIDEN = 0, WK_EDGE_ROWS = 1, WK_TRI_ROWS = 2, WK_IOTA = 3, WK_COPY = 4, WK_UNPACK24 = 5 };

struct WidenTask {
    const int32_t *src;
    int64_t *dst;
    size_t n;
    int kind;
    const uint32_t *off;      // EDGE_ROWS / TRI_ROWS: row offsets per owner (n_index + 1 entries)
    size_t n_index;
    size_t row0;
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

// 24-bit wire format (ball indices < 2^24): a chunk of m values arrives as m low halves (uint16) followed by
// m high bytes; three bytes per value instead of four cross PCIe
#if defined(__x86_64__)
__attribute__((target("avx2"))) inline void unpack24_avx2(const uint16_t *lo, const uint8_t *hi, int64_t *dst, size_t n) {
    size_t i = 0;
    while (i < n && (reinterpret_cast<uintptr_t>(dst + i) & 31u)) { dst[i] = (int64_t)lo[i] | ((int64_t)hi[i] << 16); ++i; }
    for (; i + 8 <= n; i += 8) {
        const __m256i l = _mm256_cvtepu16_epi32(_mm_loadu_si128(reinterpret_cast<const __m128i *>(lo + i)));
        const __m256i h = _mm256_cvtepu8_epi32(_mm_loadl_epi64(reinterpret_cast<const __m128i *>(hi + i)));
        const __m256i v = _mm256_or_si256(l, _mm256_slli_epi32(h, 16));
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i), _mm256_cvtepi32_epi64(_mm256_castsi256_si128(v)));
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i + 4), _mm256_cvtepi32_epi64(_mm256_extracti128_si256(v, 1)));
    }
    for (; i < n; ++i) dst[i] = (int64_t)lo[i] | ((int64_t)hi[i] << 16);
    _mm_sfence();
}
#endif

inline void unpack24(const uint16_t *lo, const uint8_t *hi, int64_t *dst, size_t n) {
#if defined(__x86_64__)
    static const bool have_avx2 = __builtin_cpu_supports("avx2");
    if (have_avx2) { unpack24_avx2(lo, hi, dst, n); return; }
#endif
    for (size_t i = 0; i < n; ++i) dst[i] = (int64_t)lo[i] | ((int64_t)hi[i] << 16);
}

// copy with non-temporal stores: the destination is a DMA source next, and a copy engine reading lines that
// sit dirty in sixteen cores' caches runs at a quarter of its speed (measured 13 vs 54 GB/s)
#if defined(__x86_64__)
__attribute__((target("avx2"))) inline void copy_stream_avx2(const char *src, char *dst, size_t bytes) {
    size_t i = 0;
    while (i < bytes && (reinterpret_cast<uintptr_t>(dst + i) & 31u)) { dst[i] = src[i]; ++i; }
    for (; i + 64 <= bytes; i += 64) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(src + i));
        const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(src + i + 32));
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i), a);
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i + 32), b);
    }
    for (; i < bytes; ++i) dst[i] = src[i];
    _mm_sfence();
}
#endif

inline void copy_for_dma(const void *src, void *dst, size_t bytes) {
#if defined(__x86_64__)
    static const bool have_avx2 = __builtin_cpu_supports("avx2");
    if (have_avx2) { copy_stream_avx2(static_cast<const char *>(src), static_cast<char *>(dst), bytes); return; }
#endif
    memcpy(dst, src, bytes);
}

inline void stream_i64(int64_t *p, int64_t v) {
#if defined(__x86_64__)
    _mm_stream_si64(reinterpret_cast<long long *>(p), (long long)v);
#else
    *p = v;
#endif
}

// owner of row r: the last a with off[a] <= r (owners without rows share their successor's offset)
inline size_t owner_of_row(const uint32_t *off, size_t n_index, size_t r) {
    size_t lo = 0, hi = n_index;                 // invariant: off[lo] <= r < off[hi]
    while (hi - lo > 1) {
        const size_t mid = (lo + hi) >> 1;
        if (off[mid] <= r) lo = mid; else hi = mid;
    }
    return lo;
}

// owner column of rows [row0, row0 + m) into tmp (runs of equal values: ~4 rows per owner)
inline void fill_owners(const uint32_t *off, size_t n_index, size_t row0, size_t m, int32_t *tmp) {
    size_t a = owner_of_row(off, n_index, row0);
    size_t k = 0;
    while (k < m) {
        const size_t end = std::min<size_t>(off[a + 1], row0 + m) - row0;    // rows of owner a inside the block
        for (; k < end; ++k) tmp[k] = (int32_t)a;
        ++a;
    }
}

#if defined(__x86_64__)
// (owner, b) -> int64 rows, 4 rows per iteration
__attribute__((target("avx2"))) inline void interleave2_avx2(const int32_t *own, const int32_t *b, int64_t *dst, size_t m) {
    size_t k = 0;
    if (reinterpret_cast<uintptr_t>(dst) & 31u) {                 // rows are 16 bytes: at most one scalar row to align
        if (m) { dst[0] = own[0]; dst[1] = b[0]; k = 1; }
    }
    for (; k + 4 <= m; k += 4) {
        const __m256i o = _mm256_cvtepi32_epi64(_mm_loadu_si128(reinterpret_cast<const __m128i *>(own + k)));   // o0 o1 o2 o3
        const __m256i v = _mm256_cvtepi32_epi64(_mm_loadu_si128(reinterpret_cast<const __m128i *>(b + k)));     // b0 b1 b2 b3
        const __m256i lo = _mm256_unpacklo_epi64(o, v);           // o0 b0 o2 b2
        const __m256i hi = _mm256_unpackhi_epi64(o, v);           // o1 b1 o3 b3
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + 2 * k), _mm256_permute2x128_si256(lo, hi, 0x20));       // o0 b0 o1 b1
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + 2 * k + 4), _mm256_permute2x128_si256(lo, hi, 0x31));   // o2 b2 o3 b3
    }
    for (; k < m; ++k) { dst[2 * k] = own[k]; dst[2 * k + 1] = b[k]; }
}

// (owner, b, c) -> int64 rows, 4 rows (12 values, three 32-byte stores) per iteration
__attribute__((target("avx2"))) inline void interleave3_avx2(const int32_t *own, const int32_t *bc, int64_t *dst, size_t m) {
    size_t k = 0;
    while (k < m && (reinterpret_cast<uintptr_t>(dst + 3 * k) & 31u)) {   // 24-byte rows: aligned again after at most 3 rows
        dst[3 * k] = own[k]; dst[3 * k + 1] = bc[2 * k]; dst[3 * k + 2] = bc[2 * k + 1];
        ++k;
    }
    for (; k + 4 <= m; k += 4) {
        const __m256i o = _mm256_cvtepi32_epi64(_mm_loadu_si128(reinterpret_cast<const __m128i *>(own + k)));        // a0 a1 a2 a3
        const __m256i p = _mm256_cvtepi32_epi64(_mm_loadu_si128(reinterpret_cast<const __m128i *>(bc + 2 * k)));     // b0 c0 b1 c1
        const __m256i q = _mm256_cvtepi32_epi64(_mm_loadu_si128(reinterpret_cast<const __m128i *>(bc + 2 * k + 4))); // b2 c2 b3 c3
        // v0 = a0 b0 c0 a1 ; v1 = b1 c1 a2 b2 ; v2 = c2 a3 b3 c3
        const __m256i v0 = _mm256_blend_epi32(_mm256_permute4x64_epi64(o, 0x40 /* a0 a0 a0 a1 */),
                                              _mm256_permute4x64_epi64(p, 0x10 /* b0 b0 c0 b0 */), 0x3c);
        const __m256i v1 = _mm256_blend_epi32(_mm256_blend_epi32(_mm256_permute4x64_epi64(p, 0x0e /* b1 c1 b0 b0 */),
                                                                 _mm256_permute4x64_epi64(o, 0x20 /* a0 a0 a2 a0 */), 0x30),
                                              _mm256_permute4x64_epi64(q, 0x00 /* b2 b2 b2 b2 */), 0xc0);
        const __m256i v2 = _mm256_blend_epi32(_mm256_permute4x64_epi64(q, 0xe5 /* c2 c2 b3 c3 */),
                                              _mm256_permute4x64_epi64(o, 0x0c /* a0 a3 a0 a0 */), 0x0c);
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + 3 * k), v0);
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + 3 * k + 4), v1);
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + 3 * k + 8), v2);
    }
    for (; k < m; ++k) { dst[3 * k] = own[k]; dst[3 * k + 1] = bc[2 * k]; dst[3 * k + 2] = bc[2 * k + 1]; }
}
#endif

inline void interleave_rows(int width, const int32_t *own, const int32_t *src, int64_t *dst, size_t m) {
#if defined(__x86_64__)
    static const bool have_avx2 = __builtin_cpu_supports("avx2");
    if (have_avx2) {
        if (width == 2) interleave2_avx2(own, src, dst, m); else interleave3_avx2(own, src, dst, m);
        return;
    }
#endif
    if (width == 2) {
        for (size_t k = 0; k < m; ++k) { dst[2 * k] = own[k]; dst[2 * k + 1] = src[k]; }
    } else {
        for (size_t k = 0; k < m; ++k) { dst[3 * k] = own[k]; dst[3 * k + 1] = src[2 * k]; dst[3 * k + 2] = src[2 * k + 1]; }
    }
}

inline void run_task(const WidenTask &t) {
    switch (t.kind) {
    case WK_WIDEN:
        widen_rows(t.src, t.dst, t.n);
        break;
    case WK_IOTA:
        for (size_t i = 0; i < t.n; ++i) stream_i64(t.dst + i, (int64_t)(t.row0 + i));
        break;
    case WK_COPY:
        copy_for_dma(t.src, t.dst, t.n * sizeof(int32_t));
        break;
    case WK_UNPACK24:
        unpack24(reinterpret_cast<const uint16_t *>(t.src) + t.row0,
                 reinterpret_cast<const uint8_t *>(t.src) + 2 * t.n_index + t.row0, t.dst, t.n);
        break;
    case WK_EDGE_ROWS:
    case WK_TRI_ROWS: {
        // blocks of 2,048 rows: owner column into a cache-resident buffer, then a vectorised interleave
        constexpr size_t BLOCK = 2048;
        int32_t own[BLOCK];
        const int width = t.kind == WK_EDGE_ROWS ? 2 : 3;
        for (size_t lo = 0; lo < t.n; lo += BLOCK) {
            const size_t m = std::min(BLOCK, t.n - lo);
            fill_owners(t.off, t.n_index, t.row0 + lo, m, own);
            interleave_rows(width, own, t.src + lo * (width - 1), t.dst + lo * width, m);
        }
        break;
    }
    }
#if defined(__x86_64__)
    _mm_sfence();
#endif
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

    // start a run that will publish at most max_tasks tasks.
    // inline_run: a small job (one protein's worth of rows) -- the producer runs every task itself as it
    // publishes it; waking a dozen sleeping threads costs more than widening a few hundred KB
    void begin(size_t max_tasks, bool inline_run = false) {
        inline_ = inline_run;
        if (inline_run) return;
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
    // split n items (values or rows) into pieces and publish them (producer thread only);
    // src_width / dst_width = int32 values per item in src / int64 values per item in dst
    void publish(int kind, const int32_t *src, int64_t *dst, size_t n, size_t piece, int src_width, int dst_width,
                 const uint32_t *off, size_t n_index, size_t row0) {
        if (inline_) {
            for (size_t lo = 0; lo < n; lo += piece)
                run_task(WidenTask{src ? src + lo * src_width : nullptr, dst + lo * dst_width, n - lo < piece ? n - lo : piece,
                                   kind, off, n_index, row0 + lo});
            return;
        }
        size_t p = published_.load(std::memory_order_relaxed);
        for (size_t lo = 0; lo < n; lo += piece) {
            const WidenTask t{src ? src + lo * src_width : nullptr, dst + lo * dst_width, n - lo < piece ? n - lo : piece,
                              kind, off, n_index, row0 + lo};
            if (p < tasks_.size()) {
                tasks_[p++] = t;
                published_.store(p, std::memory_order_release);
            } else {
                run_task(t);      // the task array is full (it cannot grow under the workers): never drop, do it here
            }
        }
    }
    // parallel memcpy of `bytes` (a multiple of 8) from src to dst in pieces of piece_bytes
    void publish_copy(const void *src, void *dst, size_t bytes, size_t piece_bytes) {
        if (inline_) {
            run_task(WidenTask{static_cast<const int32_t *>(src), static_cast<int64_t *>(dst), bytes / sizeof(int32_t), WK_COPY,
                               nullptr, 0, 0});
            return;
        }
        size_t p = published_.load(std::memory_order_relaxed);
        for (size_t lo = 0; lo < bytes; lo += piece_bytes) {
            const size_t m = bytes - lo < piece_bytes ? bytes - lo : piece_bytes;
            const WidenTask t{reinterpret_cast<const int32_t *>(static_cast<const char *>(src) + lo),
                              reinterpret_cast<int64_t *>(static_cast<char *>(dst) + lo), m / sizeof(int32_t), WK_COPY,
                              nullptr, 0, 0};
            if (p < tasks_.size()) {
                tasks_[p++] = t;
                published_.store(p, std::memory_order_release);
            } else {
                run_task(t);
            }
        }
    }
    // no more tasks: help with what is left and wait until every task has run
    void finish() {
        if (inline_) { inline_ = false; return; }
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
                run_task(t);
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
    bool inline_ = false;              // producer-only state of the current run
    std::atomic<bool> closed_{true};
    std::atomic<size_t> published_{0}, next_{0}, done_{0};
};

}  // namespace axb
