// fsld_hostcast.cu -- host-side casts for the numpy (reference-signature) calls (host code only).
//
// optim.loss_and_grad is called with numpy complex128 volumes (optim.py:165-190); the device works in
// complex64.  A cast written with ordinary stores leaves the page-locked staging buffer dirty in the
// CPU caches, and the copy engine then reads it at a fraction of the PCIe rate (measured on the B200
// box: the pipelined host step takes 2.3 ms after a cached cast vs 0.8 ms from a clean buffer).
// These casts use non-temporal (streaming) stores, so the staged data goes straight to DRAM.  One
// call casts one contiguous range; callers split a volume over host threads (the Python side calls
// it from a thread pool -- ctypes releases the GIL -- rather than linking a second OpenMP runtime
// into a process that already carries torch's).  SSE2 only (baseline x86-64).
#include <emmintrin.h>
#include <stdint.h>
#include <xmmintrin.h>

#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "fsld_b200.h"
#include "fsld_hostpool.h"

// dst[i] = (float) src[i] over n doubles (n = 2 x complex count); dst 16-byte aligned for the stream.
extern "C" int fsld_host_cast_f64_to_f32(const double* src, float* dst, int64_t n) {
    if (n < 0 || (n > 0 && (!src || !dst))) return FSLD_EINVAL;
    if (reinterpret_cast<uintptr_t>(dst) & 15) {
        for (int64_t i = 0; i < n; ++i) dst[i] = (float)src[i];
        return FSLD_OK;
    }
    const int64_t n4 = n & ~int64_t(3);
    for (int64_t i = 0; i < n4; i += 4) {
        const __m128 lo = _mm_cvtpd_ps(_mm_loadu_pd(src + i));
        const __m128 hi = _mm_cvtpd_ps(_mm_loadu_pd(src + i + 2));
        _mm_stream_ps(dst + i, _mm_movelh_ps(lo, hi));
    }
    for (int64_t i = n4; i < n; ++i) dst[i] = (float)src[i];
    _mm_sfence();
    return FSLD_OK;
}

// dst[i] = (double) src[i] over n floats; dst 16-byte aligned for the stream.
extern "C" int fsld_host_cast_f32_to_f64(const float* src, double* dst, int64_t n) {
    if (n < 0 || (n > 0 && (!src || !dst))) return FSLD_EINVAL;
    if (reinterpret_cast<uintptr_t>(dst) & 15) {
        for (int64_t i = 0; i < n; ++i) dst[i] = (double)src[i];
        return FSLD_OK;
    }
    const int64_t n4 = n & ~int64_t(3);
    for (int64_t i = 0; i < n4; i += 4) {
        const __m128 x = _mm_loadu_ps(src + i);
        _mm_stream_pd(dst + i, _mm_cvtps_pd(x));
        _mm_stream_pd(dst + i + 2, _mm_cvtps_pd(_mm_movehl_ps(x, x)));
    }
    for (int64_t i = n4; i < n; ++i) dst[i] = (double)src[i];
    _mm_sfence();
    return FSLD_OK;
}

// The two row loops of the touched-ball host step (fsld_loss_grad_host_np_ball): both return the sum of
// squares of the n doubles they read (the ||v||^2 term of the loss, accumulated in fp64 in a fixed
// order) and write with streaming stores (dst 16-byte aligned, n a multiple of 2).
namespace fsld_host {
// dst = (float) src
double cast_f64_to_f32_sumsq(const double* src, float* dst, int64_t n) {
    __m128d acc0 = _mm_setzero_pd(), acc1 = _mm_setzero_pd();
    double s = 0.0;
    int64_t i = 0;
    for (; i < n && (reinterpret_cast<uintptr_t>(dst + i) & 15); ++i) {  // (odd M: rows start 8 bytes off)
        dst[i] = (float)src[i];
        s += src[i] * src[i];
    }
    for (; i + 4 <= n; i += 4) {
        const __m128d a = _mm_loadu_pd(src + i), b = _mm_loadu_pd(src + i + 2);
        acc0 = _mm_add_pd(acc0, _mm_mul_pd(a, a));
        acc1 = _mm_add_pd(acc1, _mm_mul_pd(b, b));
        _mm_stream_ps(dst + i, _mm_movelh_ps(_mm_cvtpd_ps(a), _mm_cvtpd_ps(b)));
    }
    double t[2];
    _mm_storeu_pd(t, _mm_add_pd(acc0, acc1));
    s += t[0] + t[1];
    for (; i < n; ++i) {
        dst[i] = (float)src[i];
        s += src[i] * src[i];
    }
    return s;
}
// dst = lam * src
double scale_f64_sumsq(const double* src, double* dst, int64_t n, double lam) {
    __m128d acc = _mm_setzero_pd();
    const __m128d l2 = _mm_set1_pd(lam);
    const int64_t n2 = n & ~int64_t(1);
    for (int64_t i = 0; i < n2; i += 2) {
        const __m128d a = _mm_loadu_pd(src + i);
        acc = _mm_add_pd(acc, _mm_mul_pd(a, a));
        _mm_stream_pd(dst + i, _mm_mul_pd(a, l2));
    }
    double t[2];
    _mm_storeu_pd(t, acc);
    double s = t[0] + t[1];
    for (int64_t i = n2; i < n; ++i) {
        dst[i] = lam * src[i];
        s += src[i] * src[i];
    }
    return s;
}
void store_fence() { _mm_sfence(); }
void cpu_pause() { _mm_pause(); }
}  // namespace fsld_host

// ---------------------------------------------------------------- host thread pool
// A persistent pool for the numpy-signature host step (fsld_loss_grad_host_np): the casts of one
// z-slab are split over the workers and the calling thread, which waits for all of them.  Plain
// std::thread (no second OpenMP runtime next to torch's).  One parallel_for at a time (the host
// step holds its pipe mutex while it casts).
namespace fsld_host {
namespace {
struct Pool {
    std::vector<std::thread> workers;
    std::mutex m;
    std::condition_variable cv, done_cv;
    const std::function<void(int64_t, int64_t)>* fn = nullptr;
    int64_t n = 0, grain = 1;
    std::atomic<int64_t> next{0};
    int active = 0;
    std::atomic<unsigned long long> gen{0};
    bool stop = false;

    void run_chunks() {
        for (;;) {
            const int64_t i0 = next.fetch_add(grain);
            if (i0 >= n) return;
            (*fn)(i0, std::min(n, i0 + grain));
        }
    }
    // A worker that has just finished a job spins for a short while before it blocks: the host step
    // issues a dozen small jobs per call (one per z-slab), a few tens of microseconds apart, and a
    // condition-variable wake-up of 15 sleeping threads costs about as much as one of those jobs.
    static constexpr long long kSpinNs = 400000;
    void loop() {
        unsigned long long seen = 0;
        for (;;) {
            const auto t0 = std::chrono::steady_clock::now();
            for (unsigned it = 0; gen.load(std::memory_order_acquire) == seen; ++it) {
                _mm_pause();
                if ((it & 63) == 63 &&
                    std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count() >
                        kSpinNs)
                    break;
            }
            {
                std::unique_lock<std::mutex> lk(m);
                cv.wait(lk, [&] { return stop || gen.load(std::memory_order_relaxed) != seen; });
                if (stop) return;
                seen = gen.load(std::memory_order_relaxed);
            }
            run_chunks();
            std::lock_guard<std::mutex> lk(m);
            if (--active == 0) done_cv.notify_one();
        }
    }
    Pool() {
        const unsigned hc = std::thread::hardware_concurrency();
        unsigned want = std::min(16u, hc ? hc : 1u);
        if (const char* e = std::getenv("FSLD_HOST_THREADS")) {  // (A/B: threads of the host casts)
            const int v = std::atoi(e);
            if (v >= 1 && v <= 256) want = (unsigned)v;
        }
        const int nw = (int)std::max(1u, want) - 1;  // + the calling thread
        for (int i = 0; i < nw; ++i) workers.emplace_back([this] { loop(); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> lk(m);
            stop = true;
        }
        cv.notify_all();
        for (auto& t : workers) t.join();
    }
};
Pool& pool() {
    static Pool p;
    return p;
}
std::mutex g_pf_mu;
}  // namespace

void parallel_for(int64_t n, int64_t grain, const std::function<void(int64_t, int64_t)>& f) {
    if (n <= 0) return;
    Pool& P = pool();
    if (P.workers.empty() || n <= grain) {
        f(0, n);
        return;
    }
    std::lock_guard<std::mutex> one(g_pf_mu);
    {
        std::lock_guard<std::mutex> lk(P.m);
        P.fn = &f;
        P.n = n;
        P.grain = grain;
        P.next.store(0);
        P.active = (int)P.workers.size();
        P.gen.fetch_add(1, std::memory_order_release);
    }
    P.cv.notify_all();
    P.run_chunks();
    std::unique_lock<std::mutex> lk(P.m);
    P.done_cv.wait(lk, [&] { return P.active == 0; });
    P.fn = nullptr;
}

int workers() { return (int)pool().workers.size() + 1; }
}  // namespace fsld_host
