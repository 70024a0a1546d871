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

#include "fsld_b200.h"

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
