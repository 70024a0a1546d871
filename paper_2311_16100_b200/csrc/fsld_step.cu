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
constexpr int kStepBlocks = 148 * 16;  // one sweep covers 2.4M voxels at 4 voxels per thread

struct StepSums {
    double dec, vv, vd, dd, ad;
};

// One voxel (optim.py:186-189, 226-229, 244-247, 292-293): fp32 state and arithmetic.
__device__ __forceinline__ void precond_voxel(const fsld_step_params& p, float scale, float lam, float2 a, float2 w,
                                              float* fo, float* da, float* dd, float dfix, float2& g, float2& q,
                                              float& dh, StepSums& S) {
    g = make_float2(fmaf(scale, a.x, lam * w.x), fmaf(scale, a.y, lam * w.y));
    if (p.estimating) {
        const float sample = fmaf((float)p.hutch_scale, *fo, lam);
        *fo = 0.f;
        *da = fmaf((float)p.w_old, *da, (float)p.w_new * sample);
        *dd = fmaf((float)p.beta, *dd, (float)(1.0 - p.beta) * *da);
        dh = fmaxf(fabsf(*dd), (float)p.floor);
    } else {
        dh = dfix;
    }
    const float r = __frcp_rn(dh);
    q = make_float2(g.x * r, g.y * r);
    S.dec += (double)(fmaf(g.x, g.x, g.y * g.y) * r);
    S.vv += (double)fmaf(w.x, w.x, w.y * w.y);
    S.vd += (double)fmaf(w.x, q.x, w.y * q.y);
    S.dd += (double)fmaf(q.x, q.x, q.y * q.y);
    S.ad += (double)fmaf(a.x, q.x, a.y * q.y);  // Re<A^* r, d> = Re<r, A d>
}

// Two voxels per thread (16-byte volume / accumulator accesses, 8-byte state accesses), 4 CTAs / SM;
// fp64 per-thread sums, fixed-order block and grid reductions.
__global__ void __launch_bounds__(kStepThreads, 4) precond_step_kernel(int64_t n, float2* __restrict__ acc,
                                                                    const float2* __restrict__ v,
                                                                    float* __restrict__ fold,
                                                                    float* __restrict__ d_avg, float* __restrict__ d,
                                                                    const float* __restrict__ dhat_fixed,
                                                                    fsld_step_params p, float2* __restrict__ dir,
                                                                    float2* __restrict__ grad_out,
                                                                    float* __restrict__ dhat_out, double* part,
                                                                    int nparts) {
    __shared__ double smem[5][kStepThreads / 32];
    StepSums S{0.0, 0.0, 0.0, 0.0, 0.0};
    const float scale = (float)p.scale, lam = (float)p.lam;
    const int64_t n4 = n / 2, stride = (int64_t)gridDim.x * blockDim.x;  // voxel pairs
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t q4 = t0; q4 < n4; q4 += stride) {
        const float4 a01 = reinterpret_cast<const float4*>(acc)[q4];
        const float4 w01 = __ldg(reinterpret_cast<const float4*>(v) + q4);
        float2 fo = make_float2(0.f, 0.f), da = fo, dd = fo, df = make_float2(1.f, 1.f);
        if (p.estimating) {
            fo = reinterpret_cast<const float2*>(fold)[q4];
            da = reinterpret_cast<const float2*>(d_avg)[q4];
            dd = reinterpret_cast<const float2*>(d)[q4];
        } else if (dhat_fixed) {
            df = __ldg(reinterpret_cast<const float2*>(dhat_fixed) + q4);
        }
        float2 g[2], q[2];
        float dh[2];
        precond_voxel(p, scale, lam, make_float2(a01.x, a01.y), make_float2(w01.x, w01.y), &fo.x, &da.x, &dd.x, df.x,
                      g[0], q[0], dh[0], S);
        precond_voxel(p, scale, lam, make_float2(a01.z, a01.w), make_float2(w01.z, w01.w), &fo.y, &da.y, &dd.y, df.y,
                      g[1], q[1], dh[1], S);
        reinterpret_cast<float4*>(acc)[q4] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (p.estimating) {
            reinterpret_cast<float2*>(fold)[q4] = make_float2(0.f, 0.f);
            reinterpret_cast<float2*>(d_avg)[q4] = da;
            reinterpret_cast<float2*>(d)[q4] = dd;
        }
        reinterpret_cast<float4*>(dir)[q4] = make_float4(q[0].x, q[0].y, q[1].x, q[1].y);
        if (grad_out) reinterpret_cast<float4*>(grad_out)[q4] = make_float4(g[0].x, g[0].y, g[1].x, g[1].y);
        if (dhat_out) reinterpret_cast<float2*>(dhat_out)[q4] = make_float2(dh[0], dh[1]);
    }
    for (int64_t i = 2 * n4 + t0; i < n; i += stride) {  // tail (n odd)
        float fo = p.estimating ? fold[i] : 0.f, da = p.estimating ? d_avg[i] : 0.f, dd = p.estimating ? d[i] : 0.f;
        float2 g, q;
        float dh;
        precond_voxel(p, scale, lam, acc[i], v[i], &fo, &da, &dd, dhat_fixed ? dhat_fixed[i] : 1.f, g, q, dh, S);
        acc[i] = make_float2(0.f, 0.f);
        if (p.estimating) {
            fold[i] = 0.f;
            d_avg[i] = da;
            d[i] = dd;
        }
        dir[i] = q;
        if (grad_out) grad_out[i] = g;
        if (dhat_out) dhat_out[i] = dh;
    }
    // the five block sums with one barrier: warp shuffles, then warp 0 adds the per-warp partials in order
    double x[5] = {S.dec, S.vv, S.vd, S.dd, S.ad};
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        for (int o = 16; o > 0; o >>= 1) x[k] += __shfl_xor_sync(0xffffffffu, x[k], o);
        if (lane == 0) smem[k][wid] = x[k];
    }
    __syncthreads();
    if (threadIdx.x < 5) {
        double t = 0.0;
        for (int w = 0; w < kStepThreads / 32; ++w) t += smem[threadIdx.x][w];
        part[threadIdx.x * nparts + blockIdx.x] = t;
    }
}

cudaError_t launch_precond_step(int64_t nvox, float2* acc, const float2* v, float* fold, float* d_avg, float* d,
                                const float* dhat_fixed, const fsld_step_params& p, float2* dir, float2* grad_out,
                                float* dhat_out, double* out4, double* part, int nparts, cudaStream_t s) {
    precond_step_kernel<<<nparts, kStepThreads, 0, s>>>(nvox, acc, v, fold, d_avg, d, dhat_fixed, p, dir, grad_out,
                                                        dhat_out, part, nparts);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_reduce_cols(part, nparts, 5, out4, s);
}

// optim.armijo_search (optim.py:269-306) with the trial losses in closed form:
//   f(eta) - f0 = 1/2 s (eta^2 qq - 2 eta rq) + 1/2 lam (eta^2 dd - 2 eta vd).
// The sufficient-decrease test f(eta) <= f0 - c eta dec is evaluated on the
// difference (no cancellation against f0).
__global__ void armijo_select_kernel(const double* __restrict__ sq, const double* __restrict__ rqp,
                                     const double* __restrict__ qqp, const double* __restrict__ vol4, double scale,
                                     double lam, double c, int max_halvings, fsld_armijo_state* st, double* hist,
                                     int hist_cap) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const double dec = vol4[0], vv = vol4[1], vd = vol4[2], dd = vol4[3];
    const double rq = *rqp, qq = *qqp;
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

cudaError_t launch_armijo_select(const double* sq, const double* rq, const double* qq, const double* vol,
                                 double scale, double lam, double c, int max_halvings, fsld_armijo_state* st,
                                 double* hist, int hist_cap, cudaStream_t s) {
    armijo_select_kernel<<<1, 32, 0, s>>>(sq, rq, qq, vol, scale, lam, c, max_halvings, st, hist, hist_cap);
    return cudaGetLastError();
}

__global__ void __launch_bounds__(kStepThreads) apply_step_kernel(int64_t n, float2* __restrict__ v,
                                                                  const float2* __restrict__ dir,
                                                                  const fsld_armijo_state* __restrict__ st) {
    const float eta = (float)st->eta_applied;
    if (eta == 0.0f) return;
    const int64_t n2 = n / 2, stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t i = t0; i < n2; i += stride) {  // two voxels (16 B) per access
        const float4 w = reinterpret_cast<const float4*>(v)[i];
        const float4 q = __ldg(reinterpret_cast<const float4*>(dir) + i);
        reinterpret_cast<float4*>(v)[i] =
            make_float4(fmaf(-eta, q.x, w.x), fmaf(-eta, q.y, w.y), fmaf(-eta, q.z, w.z), fmaf(-eta, q.w, w.w));
    }
    for (int64_t i = 2 * n2 + t0; i < n; i += stride) {
        const float2 w = v[i], q = dir[i];
        v[i] = make_float2(fmaf(-eta, q.x, w.x), fmaf(-eta, q.y, w.y));
    }
}

cudaError_t launch_apply_step(int64_t nvox, float2* v, const float2* dir, const fsld_armijo_state* st,
                              cudaStream_t s) {
    int blocks = (int)((nvox / 2 + kStepThreads - 1) / kStepThreads);
    blocks = blocks < 1 ? 1 : (blocks > kStepBlocks ? kStepBlocks : blocks);
    apply_step_kernel<<<blocks, kStepThreads, 0, s>>>(nvox, v, dir, st);
    return cudaGetLastError();
}

}  // namespace fsld
