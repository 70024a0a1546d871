// fsld_slice.cu -- fused Fourier-slice kernels for sm_100a.
//
// One CTA = one image x one tile of its masked pixels (kThreads threads,
// `ppt` pixels per thread).  Per pixel: rotate the frequency (fp64, no FMA,
// kernels.py:42-60) -> gather 8 corners / nearest voxel from the L2-resident
// complex64 volume (kernels.py:138-190) -> multiply by the in-kernel CTF x
// shift factor (forward.py:93-111, 299-312) -> op-specific epilogue:
//   OP_PROJECT     out = f * P v                       (Projector.project_batch)
//   OP_LOSS        sum |f P v - x|^2                   (optim._resid_pass, no grad)
//   OP_LOSS_GRAD   ... + scatter conj(f) r             (optim._resid_pass + backproject)
//   OP_BACKPROJECT scatter conj(f) img                 (Projector.backproject_batch)
//   OP_HVP         scatter C^2 P z                     (DatasetOperator.hvp body)
//   OP_DIAG        scatter C^2 w^2 (tri) / C^2 (nn)    (scatter_sq_tri / nn bincount)
//   OP_ARMIJO      sum |r|^2, sum Re(conj(r) q), sum |q|^2 with r = f P v - x,
//                  q = f P d: the closed-form line-search terms
// The residual never touches HBM; loss partials are per-CTA fp64 slots
// reduced in a fixed order; the adjoint scatter uses red.global.add.v2.f32
// (or int64 fixed point in deterministic mode).
#include "fsld_kernels.cuh"

namespace fsld {

template <int MODE, int OP, bool DET>
__global__ void __launch_bounds__(kThreads) slice_kernel(SliceArgs a) {
    __shared__ fsld_image_rec rec;
    __shared__ double red_smem[32];
    const int b = blockIdx.x / a.tiles;
    const int tile = blockIdx.x - b * a.tiles;
    const int row = a.idx ? a.idx[b] : b;
    load_record(a.recs, row, &rec);
    __syncthreads();
    const float2* __restrict__ frow = a.ftab ? a.ftab + (size_t)b * a.n_mask : nullptr;

    const int M = a.M, c2 = a.c2, n = a.n_mask;
    const double bnd = a.bnd;
    const double fx = DET ? *a.fx : 0.0;
    const float2* __restrict__ xrow = nullptr;
    if (OP == OP_LOSS || OP == OP_LOSS_GRAD || OP == OP_BACKPROJECT || OP == OP_ARMIJO)
        xrow = a.x + (size_t)(a.x_by_idx ? row : b) * n;
    float sq = 0.0f, rq = 0.0f, qq = 0.0f;
    // brick-sorted dataset layout: per-(row, p) coordinates instead of the shared mask table
    const char2* __restrict__ pcrow = a.pc ? a.pc + (size_t)(a.x_by_idx ? row : b) * n : nullptr;

    const int p0 = tile * a.ppt * kThreads + threadIdx.x;
    for (int k = 0; k < a.ppt; ++k) {
        const int p = p0 + k * kThreads;
        if (p >= n) break;
        short2 kk;
        if (pcrow) {
            const char2 q = pcrow[p];
            kk = make_short2(q.x, q.y);
        } else {
            kk = __ldg(a.pix + p);
        }
        const int kx = kk.x, ky = kk.y;
        double cx, cy, cz;
        rotate_pixel(rec.rot, (double)kx, (double)ky, bnd, cx, cy, cz);

        Tri t;
        int jn = 0;
        if (MODE == FSLD_MODE_TRI) tri_setup(cx, cy, cz, M, c2, t);
        else jn = nn_index(cx, cy, cz, M, c2);

        if constexpr (OP == OP_DIAG) {
            const float c2v = frow ? __ldg(frow + p).x : ctf_sq(rec, kx, ky);
            if (MODE == FSLD_MODE_TRI) {
                float w[8];
                tri_weights(t, w);
#pragma unroll
                for (int c = 0; c < 8; ++c) scatter_r<DET>(a.acc, t.j[c], w[c] * w[c] * c2v, fx);
            } else {
                scatter_r<DET>(a.acc, jn, c2v, fx);
            }
            continue;
        }

        float2 val = make_float2(0.f, 0.f);  // value to scatter (complex)
        if constexpr (OP == OP_BACKPROJECT) {
            const float2 f = frow ? __ldg(frow + p) : pixel_factor(rec, kx, ky);
            val = cmulconj(f, __ldg(xrow + p));
        } else {
            const float2 pv = (MODE == FSLD_MODE_TRI) ? tri_gather(a.v, t) : __ldg(a.v + jn);
            if constexpr (OP == OP_ARMIJO) {
                const float2 pd = (MODE == FSLD_MODE_TRI) ? tri_gather(a.v2, t) : __ldg(a.v2 + jn);
                const float2 f = frow ? __ldg(frow + p) : pixel_factor(rec, kx, ky);
                const float2 pr = cmul(pv, f), q = cmul(pd, f);
                const float2 xv = __ldg(xrow + p);
                const float2 r = make_float2(pr.x - xv.x, pr.y - xv.y);
                sq = fmaf(r.x, r.x, fmaf(r.y, r.y, sq));
                rq = fmaf(r.x, q.x, fmaf(r.y, q.y, rq));
                qq = fmaf(q.x, q.x, fmaf(q.y, q.y, qq));
                continue;
            } else if constexpr (OP == OP_HVP) {
                const float c2v = ctf_sq(rec, kx, ky);
                val = make_float2(c2v * pv.x, c2v * pv.y);
            } else {
                const float2 f = frow ? __ldg(frow + p) : pixel_factor(rec, kx, ky);
                const float2 pr = cmul(pv, f);
                if constexpr (OP == OP_PROJECT) {
                    a.out[(size_t)b * n + p] = pr;
                    continue;
                } else {
                    const float2 xv = __ldg(xrow + p);
                    const float2 r = make_float2(pr.x - xv.x, pr.y - xv.y);
                    sq = fmaf(r.x, r.x, fmaf(r.y, r.y, sq));
                    if constexpr (OP == OP_LOSS) continue;
                    val = cmulconj(f, r);
                }
            }
        }
        // adjoint scatter (kernels.py:193-248)
        if (MODE == FSLD_MODE_TRI) {
            float w[8];
            tri_weights(t, w);
#pragma unroll
            for (int c = 0; c < 8; ++c) scatter_c<DET>(a.acc, t.j[c], w[c] * val.x, w[c] * val.y, fx);
        } else {
            scatter_c<DET>(a.acc, jn, val.x, val.y, fx);
        }
    }

    if constexpr (OP == OP_LOSS || OP == OP_LOSS_GRAD) {
        const double s = block_sum((double)sq, red_smem);
        if (threadIdx.x == 0) a.partials[blockIdx.x] = s;
    }
    if constexpr (OP == OP_ARMIJO) {
        const double s0 = block_sum((double)sq, red_smem);
        __syncthreads();
        const double s1 = block_sum((double)rq, red_smem);
        __syncthreads();
        const double s2 = block_sum((double)qq, red_smem);
        if (threadIdx.x == 0) {
            a.partials[blockIdx.x] = s0;
            a.partials[a.nparts + blockIdx.x] = s1;
            a.partials[2 * a.nparts + blockIdx.x] = s2;
        }
    }
}

// Fixed-order reduction of per-CTA partials (one CTA) -> *out.
__global__ void __launch_bounds__(1024) reduce_partials_kernel(const double* __restrict__ part, int n,
                                                               double* out) {
    __shared__ double smem[32];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
    s = block_sum(s, smem);
    if (threadIdx.x == 0) *out = s;
}

__global__ void __launch_bounds__(kThreads) assign_nn_kernel(SliceArgs a, int32_t* out) {
    __shared__ fsld_image_rec rec;
    const int b = blockIdx.x / a.tiles;
    const int tile = blockIdx.x - b * a.tiles;
    load_record(a.recs, a.idx ? a.idx[b] : b, &rec);
    __syncthreads();
    const int p0 = tile * a.ppt * kThreads + threadIdx.x;
    for (int k = 0; k < a.ppt; ++k) {
        const int p = p0 + k * kThreads;
        if (p >= a.n_mask) break;
        const short2 kk = __ldg(a.pix + p);
        double cx, cy, cz;
        rotate_pixel(rec.rot, (double)kk.x, (double)kk.y, a.bnd, cx, cy, cz);
        out[(size_t)b * a.n_mask + p] = nn_index(cx, cy, cz, a.M, a.c2);
    }
}

template <int MODE, int OP, bool DET>
static cudaError_t launch_t(const SliceArgs& a, int nblocks, cudaStream_t s) {
    slice_kernel<MODE, OP, DET><<<nblocks, kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

template <int OP, bool DET>
static cudaError_t launch_m(int mode, const SliceArgs& a, int nblocks, cudaStream_t s) {
    return mode == FSLD_MODE_TRI ? launch_t<FSLD_MODE_TRI, OP, DET>(a, nblocks, s)
                                 : launch_t<FSLD_MODE_NN, OP, DET>(a, nblocks, s);
}

cudaError_t launch_slice(int op, int mode, bool det, const SliceArgs& a, int nblocks, cudaStream_t s) {
    switch (op) {
        case OP_ARMIJO: return launch_m<OP_ARMIJO, false>(mode, a, nblocks, s);
        case OP_PROJECT: return launch_m<OP_PROJECT, false>(mode, a, nblocks, s);
        case OP_LOSS: return launch_m<OP_LOSS, false>(mode, a, nblocks, s);
        case OP_LOSS_GRAD:
            return det ? launch_m<OP_LOSS_GRAD, true>(mode, a, nblocks, s)
                       : launch_m<OP_LOSS_GRAD, false>(mode, a, nblocks, s);
        case OP_BACKPROJECT:
            return det ? launch_m<OP_BACKPROJECT, true>(mode, a, nblocks, s)
                       : launch_m<OP_BACKPROJECT, false>(mode, a, nblocks, s);
        case OP_HVP:
            return det ? launch_m<OP_HVP, true>(mode, a, nblocks, s)
                       : launch_m<OP_HVP, false>(mode, a, nblocks, s);
        case OP_DIAG:
            return det ? launch_m<OP_DIAG, true>(mode, a, nblocks, s)
                       : launch_m<OP_DIAG, false>(mode, a, nblocks, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_reduce(const double* part, int n, double* out, cudaStream_t s) {
    reduce_partials_kernel<<<1, 1024, 0, s>>>(part, n, out);
    return cudaGetLastError();
}

// One CTA per column of a (ncols, n) partial table: out[q] = sum_i part[q*n + i], fixed order.
__global__ void __launch_bounds__(1024) reduce_cols_kernel(const double* __restrict__ part, int n, double* out) {
    __shared__ double smem[32];
    const double* col = part + (size_t)blockIdx.x * n;
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += col[i];
    s = block_sum(s, smem);
    if (threadIdx.x == 0) out[blockIdx.x] = s;
}

cudaError_t launch_reduce_cols(const double* part, int n, int ncols, double* out, cudaStream_t s) {
    reduce_cols_kernel<<<ncols, 1024, 0, s>>>(part, n, out);
    return cudaGetLastError();
}

cudaError_t launch_assign_nn(const SliceArgs& a, int nblocks, int32_t* out, cudaStream_t s) {
    assign_nn_kernel<<<nblocks, kThreads, 0, s>>>(a, out);
    return cudaGetLastError();
}

}  // namespace fsld
