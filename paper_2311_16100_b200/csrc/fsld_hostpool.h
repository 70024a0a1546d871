// fsld_hostpool.h -- the library's host thread pool (fsld_hostcast.cu), used by the numpy-signature
// host step to cast volume slabs in parallel while the device works on earlier slabs.
#pragma once

#include <stdint.h>

#include <functional>

namespace fsld_host {
// f(i0, i1) over [0, n) in chunks of `grain` on the pool's workers and the calling thread; returns
// when every chunk is done.
void parallel_for(int64_t n, int64_t grain, const std::function<void(int64_t, int64_t)>& f);
int workers();
// row loops of the touched-ball host step (streaming stores; return the sum of squares of src)
double cast_f64_to_f32_sumsq(const double* src, float* dst, int64_t n);
double scale_f64_sumsq(const double* src, double* dst, int64_t n, double lam);
void store_fence();
void cpu_pause();
}  // namespace fsld_host
