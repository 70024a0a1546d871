// fsld_aux.cu -- volume-sized elementwise / reduction kernels (HBM-streaming).
//
//  - fixed-point scale for the deterministic int64 accumulators;
//  - accumulator finalize: grad = scale*acc + lam*v (optim.py:186-189,
//    forward.py:570), real variant for Hutchinson / exact diagonal;
//  - ||v||^2 in a fixed order (optim.py:187).
#include "fsld_kernels.cuh"

namespace fsld {

// max |data| over complex64, via atomicMax on the (non-negative) float bits:
// order-independent, hence deterministic.
__global__ void maxabs_kernel(const float2* __restrict__ d, int64_t n, unsigned* out) {
    float m = 0.f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float2 z = d[i];
        m = fmaxf(m, fmaxf(fabsf(z.x), fabsf(z.y)));
    }
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(out, __float_as_uint(m));
}

// fx = 2^floor(61 - log2(bound)), bound = mult * (2*max|component| + add).
// 2*max|component| bounds |z|.  Accumulated totals then stay below 2^62 in
// magnitude as long as sum_contributions |value| <= bound.
__global__ void fixed_scale_kernel(const unsigned* mx, double mult, double add, double* fx) {
    const double m = mx ? (double)__uint_as_float(*mx) : 0.0;
    double bound = mult * (2.0 * m + add);
    if (!(bound > 0.0)) bound = 1.0;
    int e;
    frexp(bound, &e);  // bound < 2^e
    *fx = ldexp(1.0, 61 - e);
}

cudaError_t launch_fixed_scale(const float2* data, int64_t n, double mult, double add, double* fx,
                               cudaStream_t s) {
    // scratch for the max: the fx slot itself is reused as a 4-byte counter
    unsigned* mx = nullptr;
    if (data && n > 0) {
        mx = reinterpret_cast<unsigned*>(fx);
        cudaError_t e = cudaMemsetAsync(mx, 0, sizeof(double), s);
        if (e != cudaSuccess) return e;
        int blocks = (int)((n + 255) / 256);
        blocks = blocks > 1184 ? 1184 : blocks;
        maxabs_kernel<<<blocks, 256, 0, s>>>(data, n, mx);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    fixed_scale_kernel<<<1, 1, 0, s>>>(mx, mult, add, fx);
    return cudaGetLastError();
}

template <bool DET>
__global__ void grad_finalize_kernel(int64_t n, const void* __restrict__ acc, const double* fxp,
                                     const float2* __restrict__ v, double scale, double lam, float2* out) {
    const double inv = DET ? 1.0 / *fxp : 1.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double re, im;
        if (DET) {
            const longlong2 q = reinterpret_cast<const longlong2*>(acc)[i];
            re = (double)q.x * inv;
            im = (double)q.y * inv;
        } else {
            const float2 q = reinterpret_cast<const float2*>(acc)[i];
            re = q.x;
            im = q.y;
        }
        re *= scale;
        im *= scale;
        if (v) {
            const float2 w = v[i];
            re += lam * (double)w.x;
            im += lam * (double)w.y;
        }
        out[i] = make_float2((float)re, (float)im);
    }
}

cudaError_t launch_grad_finalize(int64_t nvox, const void* acc, bool det, const double* fx, const float2* v,
                                 double scale, double lam, float2* out, cudaStream_t s) {
    int blocks = (int)((nvox + 255) / 256);
    blocks = blocks > 148 * 16 ? 148 * 16 : blocks;
    if (det) grad_finalize_kernel<true><<<blocks, 256, 0, s>>>(nvox, acc, fx, v, scale, lam, out);
    else grad_finalize_kernel<false><<<blocks, 256, 0, s>>>(nvox, acc, fx, v, scale, lam, out);
    return cudaGetLastError();
}

template <bool DET>
__global__ void real_finalize_kernel(int64_t n, const void* __restrict__ acc, const double* fxp, double scale,
                                     double add, float* out) {
    const double inv = DET ? 1.0 / *fxp : 1.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double a = DET ? (double)reinterpret_cast<const long long*>(acc)[i] * inv
                       : (double)reinterpret_cast<const float*>(acc)[i];
        out[i] = (float)(scale * a + add);
    }
}

cudaError_t launch_real_finalize(int64_t nvox, const void* acc, bool det, const double* fx, double scale,
                                 double add, float* out, cudaStream_t s) {
    int blocks = (int)((nvox + 255) / 256);
    blocks = blocks > 148 * 16 ? 148 * 16 : blocks;
    if (det) real_finalize_kernel<true><<<blocks, 256, 0, s>>>(nvox, acc, fx, scale, add, out);
    else real_finalize_kernel<false><<<blocks, 256, 0, s>>>(nvox, acc, fx, scale, add, out);
    return cudaGetLastError();
}

__global__ void norm2_kernel(int64_t n, const float2* __restrict__ v, double* part) {
    __shared__ double smem[32];
    double s = 0.0;
    const int64_t n2 = n / 2, stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if ((reinterpret_cast<uintptr_t>(v) & 15) == 0) {
        for (int64_t i = t0; i < n2; i += stride) {  // two complex per 16-byte load
            const float4 z = __ldg(reinterpret_cast<const float4*>(v) + i);
            s += (double)fmaf(z.x, z.x, z.y * z.y) + (double)fmaf(z.z, z.z, z.w * z.w);
        }
    } else {
        for (int64_t i = t0; i < 2 * n2; i += stride) {
            const float2 z = v[i];
            s += (double)z.x * z.x + (double)z.y * z.y;
        }
    }
    for (int64_t i = 2 * n2 + t0; i < n; i += stride) {
        const float2 z = v[i];
        s += (double)z.x * z.x + (double)z.y * z.y;
    }
    s = block_sum(s, smem);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

cudaError_t launch_norm2(int64_t n, const float2* v, double* out, double* part, int nparts, cudaStream_t s) {
    norm2_kernel<<<nparts, 256, 0, s>>>(n, v, part);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_reduce(part, nparts, out, s);
}

}  // namespace fsld

namespace fsld {

// Fused loss_and_grad epilogue (optim.py:186-189) in one pass over the volume:
//   grad = scale * acc + lam * v;  acc <- 0 (ready for the next step);
//   per-block partials of ||v||^2 (fixed order) -> loss kernel.
__global__ void __launch_bounds__(256) grad_epilogue_kernel(int64_t n, float2* __restrict__ acc,
                                                            const float2* __restrict__ v, float scale, float lam,
                                                            float2* __restrict__ grad, double* part) {
    __shared__ double smem[32];
    double s = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool vec = ((reinterpret_cast<uintptr_t>(acc) | reinterpret_cast<uintptr_t>(v) |
                       reinterpret_cast<uintptr_t>(grad)) & 15) == 0;
    const int64_t n2 = vec ? n / 2 : 0;
    for (int64_t i = t0; i < n2; i += stride) {  // two voxels per 16-byte access
        const float4 a = reinterpret_cast<const float4*>(acc)[i];
        const float4 w = __ldg(reinterpret_cast<const float4*>(v) + i);
        reinterpret_cast<float4*>(grad)[i] = make_float4(fmaf(scale, a.x, lam * w.x), fmaf(scale, a.y, lam * w.y),
                                                         fmaf(scale, a.z, lam * w.z), fmaf(scale, a.w, lam * w.w));
        reinterpret_cast<float4*>(acc)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        s += (double)fmaf(w.x, w.x, w.y * w.y) + (double)fmaf(w.z, w.z, w.w * w.w);
    }
    for (int64_t i = 2 * n2 + t0; i < n; i += stride) {
        const float2 a = acc[i];
        const float2 w = v[i];
        grad[i] = make_float2(fmaf(scale, a.x, lam * w.x), fmaf(scale, a.y, lam * w.y));
        acc[i] = make_float2(0.f, 0.f);
        s += (double)w.x * w.x + (double)w.y * w.y;
    }
    s = block_sum(s, smem);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// loss = 0.5 * scale * sq + 0.5 * lam * sum(part)   (fixed reduction order)
__global__ void __launch_bounds__(1024) loss_kernel(const double* __restrict__ part, int nparts, const double* sq,
                                                    double scale, double lam, double* loss, double* norm2) {
    __shared__ double smem[32];
    double s = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += part[i];
    s = block_sum(s, smem);
    if (threadIdx.x == 0) {
        if (norm2) *norm2 = s;
        if (loss) *loss = 0.5 * scale * (*sq) + 0.5 * lam * s;
    }
}

cudaError_t launch_grad_epilogue(int64_t nvox, float2* acc, const float2* v, double scale, double lam, float2* grad,
                                 const double* sq, double* loss, double* norm2, double* part, int nparts,
                                 cudaStream_t s) {
    grad_epilogue_kernel<<<nparts, 256, 0, s>>>(nvox, acc, v, (float)scale, (float)lam, grad, part);
    loss_kernel<<<1, 1024, 0, s>>>(part, nparts, sq, scale, lam, loss, norm2);
    return cudaGetLastError();
}

// Fused-epilogue form of the loss+grad step: grad = lam v written BEFORE the brick pass, whose flush
// then adds scale * (its contributions) straight into grad (no accumulator read-back, no zeroing pass);
// per-block partials of ||v||^2 for the loss.
__global__ void __launch_bounds__(256) grad_init_kernel(int64_t n, const float2* __restrict__ v, float lam,
                                                        float2* __restrict__ grad, double* part) {
    __shared__ double smem[32];
    double s = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool vec = ((reinterpret_cast<uintptr_t>(v) | reinterpret_cast<uintptr_t>(grad)) & 15) == 0;
    const int64_t n2 = vec ? n / 2 : 0;
    for (int64_t i = t0; i < n2; i += 4 * stride) {  // four independent 16-byte loads in flight
        float4 w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            w[u] = i + u * stride < n2 ? __ldg(reinterpret_cast<const float4*>(v) + i + u * stride)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (i + u * stride >= n2) break;
            reinterpret_cast<float4*>(grad)[i + u * stride] =
                make_float4(lam * w[u].x, lam * w[u].y, lam * w[u].z, lam * w[u].w);
            s += (double)fmaf(w[u].x, w[u].x, w[u].y * w[u].y) + (double)fmaf(w[u].z, w[u].z, w[u].w * w[u].w);
        }
    }
    for (int64_t i = 2 * n2 + t0; i < n; i += stride) {
        const float2 w = v[i];
        grad[i] = make_float2(lam * w.x, lam * w.y);
        s += (double)w.x * w.x + (double)w.y * w.y;
    }
    s = block_sum(s, smem);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// sq = sum(part_sq) (the brick pass's per-CTA |r|^2), loss = 0.5 scale sq + 0.5 lam sum(part_norm)
__global__ void __launch_bounds__(1024) loss_finalize_kernel(const double* __restrict__ part_sq, int n_sq,
                                                             const double* __restrict__ part_norm, int n_norm,
                                                             double scale, double lam, double* sq_out, double* loss) {
    __shared__ double smem[32];
    double a = 0.0, b = 0.0;
    for (int i = threadIdx.x; i < n_sq; i += blockDim.x) a += part_sq[i];
    a = block_sum(a, smem);
    __syncthreads();
    for (int i = threadIdx.x; i < n_norm; i += blockDim.x) b += part_norm[i];
    b = block_sum(b, smem);
    if (threadIdx.x == 0) {
        *sq_out = a;
        *loss = 0.5 * scale * a + 0.5 * lam * b;
    }
}

cudaError_t launch_grad_init(int64_t nvox, const float2* v, double lam, float2* grad, double* part, int nparts,
                             cudaStream_t s) {
    grad_init_kernel<<<nparts, 256, 0, s>>>(nvox, v, (float)lam, grad, part);
    return cudaGetLastError();
}

cudaError_t launch_loss_finalize(const double* part_sq, int n_sq, const double* part_norm, int n_norm, double scale,
                                 double lam, double* sq_out, double* loss, cudaStream_t s) {
    loss_finalize_kernel<<<1, 1024, 0, s>>>(part_sq, n_sq, part_norm, n_norm, scale, lam, sq_out, loss);
    return cudaGetLastError();
}

// Touched-ball compaction for the data-parallel all-reduce: only voxels within
// radius R + 1/2 + sqrt(3) can receive scatter contributions (Appendix A item 7), ~54 % of the
// cube at M=128, so the all-reduce moves the compacted vector.  Element-generic (4 or 8 bytes).
template <typename T>
__global__ void ball_gather_kernel(int64_t n, const int32_t* __restrict__ idx, const T* __restrict__ src,
                                   T* __restrict__ dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[idx[i]];
}

template <typename T>
__global__ void ball_scatter_kernel(int64_t n, const int32_t* __restrict__ idx, const T* __restrict__ src,
                                    T* __restrict__ dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[idx[i]] = src[i];
}

cudaError_t launch_ball(bool gather, int64_t n, const int32_t* idx, const void* src, void* dst, int elem_bytes,
                        cudaStream_t s) {
    int blocks = (int)((n + 255) / 256);
    blocks = blocks > 148 * 16 ? 148 * 16 : (blocks < 1 ? 1 : blocks);
    if (elem_bytes == 8) {
        if (gather) ball_gather_kernel<float2><<<blocks, 256, 0, s>>>(n, idx, (const float2*)src, (float2*)dst);
        else ball_scatter_kernel<float2><<<blocks, 256, 0, s>>>(n, idx, (const float2*)src, (float2*)dst);
    } else {
        if (gather) ball_gather_kernel<float><<<blocks, 256, 0, s>>>(n, idx, (const float*)src, (float*)dst);
        else ball_scatter_kernel<float><<<blocks, 256, 0, s>>>(n, idx, (const float*)src, (float*)dst);
    }
    return cudaGetLastError();
}

// Rows of the touched ball between the M^3 volume and its packed form (the numpy-signature host step:
// fsld_loss_grad_host_np_ball moves only the ball over PCIe, as one contiguous range per z-slab).
// rows[r] = (voxel offset, length, packed offset, -); one warp per row, 8-byte voxels (complex64).
template <bool PACK>
__global__ void __launch_bounds__(256) ball_rows_kernel(const int4* __restrict__ rows, int nrows,
                                                        const float2* __restrict__ src, float2* __restrict__ dst) {
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nrows; r += nw) {
        const int4 q = rows[r];
        const float2* a = src + (PACK ? q.x : q.z);
        float2* b = dst + (PACK ? q.z : q.x);
        for (int i = lane; i < q.y; i += 32) b[i] = a[i];
    }
}

cudaError_t launch_ball_rows(bool pack, const int4* rows, int nrows, const void* src, void* dst, cudaStream_t s) {
    if (nrows <= 0) return cudaSuccess;
    int blocks = (nrows + 7) / 8;
    blocks = blocks > 148 * 8 ? 148 * 8 : blocks;
    if (pack) ball_rows_kernel<true><<<blocks, 256, 0, s>>>(rows, nrows, (const float2*)src, (float2*)dst);
    else ball_rows_kernel<false><<<blocks, 256, 0, s>>>(rows, nrows, (const float2*)src, (float2*)dst);
    return cudaGetLastError();
}

}  // namespace fsld
