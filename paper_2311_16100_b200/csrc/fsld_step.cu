// fsld_step.cu -- the rest of one Algorithm-1 step on the device.
//
// After the fused loss+grad pass (and the Hutchinson probe pass) have filled
// the gradient accumulator and the probe fold, the reference's per-step host
// work is (optim.py:362-382, 186-189, 210-247, 269-306):
//   grad = s acc + lam v;  d_avg / d updates;  dhat = max(|d|, alpha);
//   direction = grad / dhat;  decrease = ||grad||^2_{dhat^-1};
//   (1 + backtracks) batch_loss passes;  v <- v - eta direction.
// Here that is three M^3 streaming passes (precond_step, apply_step, and the
// projection of the direction) plus a one-thread select: the loss is quadratic
// in v, so every trial loss of the backtracking comes from five scalars.
#include "fsld_kernels.cuh"

namespace fsld {

constexpr int kStepThreads = 256;

// Per voxel (optim.py:186-189, 226-229, 244-247, 292-293); fp32 state, fp64 sums.
__global__ void __launch_bounds__(kStepThreads) precond_step_kernel(int64_t n, float2* __restrict__ acc,
                                                                    const float2* __restrict__ v,
                                                                    float* __restrict__ fold,
                                                                    float* __restrict__ d_avg, float* __restrict__ d,
                                                                    const float* __restrict__ dhat_fixed,
                                                                    fsld_step_params p, float2* __restrict__ dir,
                                                                    float2* __restrict__ grad_out,
                                                                    float* __restrict__ dhat_out, double* part,
                                                                    int nparts) {
    __shared__ double smem[32];
    double s_dec = 0.0, s_vv = 0.0, s_vd = 0.0, s_dd = 0.0;
    const float scale = (float)p.scale, lam = (float)p.lam;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float2 a = acc[i];
        const float2 w = v[i];
        const float2 g = make_float2(fmaf(scale, a.x, lam * w.x), fmaf(scale, a.y, lam * w.y));
        acc[i] = make_float2(0.f, 0.f);
        float dh;
        if (p.estimating) {
            const float sample = (float)(p.hutch_scale * (double)fold[i] + p.lam);
            fold[i] = 0.f;
            const float da = (float)(p.w_old * (double)d_avg[i] + p.w_new * (double)sample);
            d_avg[i] = da;
            const float dd = (float)(p.beta * (double)d[i] + (1.0 - p.beta) * (double)da);
            d[i] = dd;
            dh = fmaxf(fabsf(dd), (float)p.floor);
        } else {
            dh = dhat_fixed ? dhat_fixed[i] : 1.0f;
        }
        const float2 q = make_float2(g.x / dh, g.y / dh);
        dir[i] = q;
        if (grad_out) grad_out[i] = g;
        if (dhat_out) dhat_out[i] = dh;
        s_dec += ((double)g.x * g.x + (double)g.y * g.y) / (double)dh;
        s_vv += (double)w.x * w.x + (double)w.y * w.y;
        s_vd += (double)w.x * q.x + (double)w.y * q.y;
        s_dd += (double)q.x * q.x + (double)q.y * q.y;
    }
    double t = block_sum(s_dec, smem);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
    __syncthreads();
    t = block_sum(s_vv, smem);
    if (threadIdx.x == 0) part[nparts + blockIdx.x] = t;
    __syncthreads();
    t = block_sum(s_vd, smem);
    if (threadIdx.x == 0) part[2 * nparts + blockIdx.x] = t;
    __syncthreads();
    t = block_sum(s_dd, smem);
    if (threadIdx.x == 0) part[3 * nparts + blockIdx.x] = t;
}

cudaError_t launch_precond_step(int64_t nvox, float2* acc, const float2* v, float* fold, float* d_avg, float* d,
                                const float* dhat_fixed, const fsld_step_params& p, float2* dir, float2* grad_out,
                                float* dhat_out, double* out4, double* part, int nparts, cudaStream_t s) {
    precond_step_kernel<<<nparts, kStepThreads, 0, s>>>(nvox, acc, v, fold, d_avg, d, dhat_fixed, p, dir, grad_out,
                                                        dhat_out, part, nparts);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_reduce_cols(part, nparts, 4, out4, s);
}

// optim.armijo_search (optim.py:269-306) with the trial losses in closed form:
//   f(eta) - f0 = 1/2 s (eta^2 qq - 2 eta rq) + 1/2 lam (eta^2 dd - 2 eta vd).
// The sufficient-decrease test f(eta) <= f0 - c eta dec is evaluated on the
// difference (no cancellation against f0).
__global__ void armijo_select_kernel(const double* __restrict__ sq, const double* __restrict__ t3,
                                     const double* __restrict__ vol4, double scale, double lam, double c,
                                     int max_halvings, fsld_armijo_state* st, double* hist, int hist_cap) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const double dec = vol4[0], vv = vol4[1], vd = vol4[2], dd = vol4[3];
    const double rq = t3[1], qq = t3[2];
    const double f0 = 0.5 * scale * (*sq) + 0.5 * lam * vv;
    double eta = st->eta;
    st->f0 = f0;
    st->decrease = dec;
    st->status = 0;
    int bt = 0;
    double f_next = f0, applied = 0.0;
    if (dec != 0.0) {
        bool ok = false;
        for (bt = 0; bt <= max_halvings; ++bt) {
            const double delta = 0.5 * scale * (eta * eta * qq - 2.0 * eta * rq) +
                                 0.5 * lam * (eta * eta * dd - 2.0 * eta * vd);
            if (delta <= -c * eta * dec) {
                f_next = f0 + delta;
                applied = eta;
                ok = true;
                break;
            }
            eta *= 0.5;
        }
        if (!ok) {
            st->status = 1;
            bt = max_halvings + 1;
        }
    }
    st->eta = eta;
    st->f_next = f_next;
    st->eta_applied = applied;
    st->backtracks = bt;
    const int k = st->n_steps;
    if (hist && k < hist_cap) {
        hist[5 * k + 0] = f0;
        hist[5 * k + 1] = eta;
        hist[5 * k + 2] = f_next;
        hist[5 * k + 3] = (double)bt;
        hist[5 * k + 4] = dec;
    }
    st->n_steps = k + 1;
}

cudaError_t launch_armijo_select(const double* sq, const double* t3, const double* vol4, double scale, double lam,
                                 double c, int max_halvings, fsld_armijo_state* st, double* hist, int hist_cap,
                                 cudaStream_t s) {
    armijo_select_kernel<<<1, 32, 0, s>>>(sq, t3, vol4, scale, lam, c, max_halvings, st, hist, hist_cap);
    return cudaGetLastError();
}

__global__ void __launch_bounds__(kStepThreads) apply_step_kernel(int64_t n, float2* __restrict__ v,
                                                                  const float2* __restrict__ dir,
                                                                  const fsld_armijo_state* __restrict__ st) {
    const float eta = (float)st->eta_applied;
    if (eta == 0.0f) return;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float2 w = v[i], q = dir[i];
        v[i] = make_float2(fmaf(-eta, q.x, w.x), fmaf(-eta, q.y, w.y));
    }
}

cudaError_t launch_apply_step(int64_t nvox, float2* v, const float2* dir, const fsld_armijo_state* st,
                              cudaStream_t s) {
    int blocks = (int)((nvox + kStepThreads - 1) / kStepThreads);
    blocks = blocks > 148 * 8 ? 148 * 8 : blocks;
    apply_step_kernel<<<blocks, kStepThreads, 0, s>>>(nvox, v, dir, st);
    return cudaGetLastError();
}

}  // namespace fsld
