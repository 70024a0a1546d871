// fsld_kernels.cuh -- launch interface between the C ABI (fsld_capi.cu) and the kernels.
#pragma once

#include "fsld_common.cuh"

namespace fsld {

enum Op { OP_PROJECT = 0, OP_LOSS, OP_LOSS_GRAD, OP_BACKPROJECT, OP_HVP, OP_DIAG };

struct SliceArgs {
    int M, c2, n_mask;
    int tiles;  // CTAs per image
    int ppt;    // pixels per thread
    double bnd;
    const short2* pix;
    const fsld_image_rec* recs;
    const int32_t* idx;
    const float2* v;       // volume / probe (complex64)
    const float2* x;       // image rows (complex64)
    int x_by_idx;          // x row = idx[b] (dataset) or b (batch-local)
    float2* out;           // projection output (B, n_mask)
    void* acc;             // scatter accumulator
    double* partials;      // per-CTA loss partials
    const double* fx;      // fixed-point scale (deterministic)
    const float2* ftab;    // optional (B, n_mask) factor table f = phase*ctf (numba-style calls)
};

cudaError_t launch_slice(int op, int mode, bool det, const SliceArgs& a, int nblocks, cudaStream_t s);
cudaError_t launch_reduce(const double* part, int n, double* out, cudaStream_t s);
cudaError_t launch_assign_nn(const SliceArgs& a, int nblocks, int32_t* out, cudaStream_t s);
cudaError_t launch_hutch(int mode, bool det, const SliceArgs& a, int nblocks, const uint32_t* zbits,
                         int words, int k, cudaStream_t s);
cudaError_t launch_pack_probes(int64_t n, int k, const double* z, uint32_t* zbits, int* bad, cudaStream_t s);
cudaError_t launch_gen_probes(int64_t n, int k, uint64_t seed, uint32_t* zbits, cudaStream_t s);
cudaError_t launch_fixed_scale(const float2* data, int64_t n, double mult, double add, double* fx,
                               cudaStream_t s);
cudaError_t launch_grad_finalize(int64_t nvox, const void* acc, bool det, const double* fx,
                                 const float2* v, double scale, double lam, float2* out, cudaStream_t s);
cudaError_t launch_real_finalize(int64_t nvox, const void* acc, bool det, const double* fx, double scale,
                                 double add, float* out, cudaStream_t s);
cudaError_t launch_norm2(int64_t n, const float2* v, double* out, double* part, int nparts, cudaStream_t s);

}  // namespace fsld
