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
}  // namespace fsld_host
