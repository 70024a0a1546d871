// fsld_common.cuh -- device helpers shared by the sm_100a slice/adjoint kernels.
//
// Geometry and index math restate the reference's numba kernels
// (/root/reference/pkg/src/fsld/kernels.py); the per-pixel phase/CTF factor
// restates forward.py:93-111 / 299-312 evaluated in-kernel from the 128-byte
// per-image record (include/fsld_b200.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "fsld_b200.h"

namespace fsld {

constexpr int kThreads = 256;

struct Geo {
    int M;
    int c2;      // (M+1)//2, kernels.py:127
    double bnd;  // M//2 - 1, kernels.py:128
};

// kernels.py:63-66
__device__ __forceinline__ int lin_index(int ix, int iy, int iz, int M, int c2) {
    int zi = iz < 0 ? iz + M : iz;
    return (zi * M + iy + c2) * M + ix + c2;
}

// kernels.py:42-60.  fp64 with every product and sum separately rounded
// (the numba kernels contain no FMA), so clamps, floors and nn indices are
// bit-identical to the reference.
__device__ __forceinline__ void rotate_pixel(const double* __restrict__ r, double px, double py,
                                             double bnd, double& cx, double& cy, double& cz) {
    cx = __dadd_rn(__dmul_rn(r[0], px), __dmul_rn(r[3], py));
    cy = __dadd_rn(__dmul_rn(r[1], px), __dmul_rn(r[4], py));
    cz = __dadd_rn(__dmul_rn(r[2], px), __dmul_rn(r[5], py));
    cx = cx > bnd ? bnd : (cx < -bnd ? -bnd : cx);
    cy = cy > bnd ? bnd : (cy < -bnd ? -bnd : cy);
    cz = cz > bnd ? bnd : (cz < -bnd ? -bnd : cz);
}

// kernels.py:69-120: nearest lattice point; exact 0.5 ties on any axis take
// the candidate with the smallest linear index (z wraps, so compare indices).
__device__ __forceinline__ int nn_index(double cx, double cy, double cz, int M, int c2) {
    double fx = floor(cx), fy = floor(cy), fz = floor(cz);
    double wx = cx - fx, wy = cy - fy, wz = cz - fz;
    int ix0 = (int)fx, iy0 = (int)fy, iz0 = (int)fz;
    bool tx = wx == 0.5, ty = wy == 0.5, tz = wz == 0.5;
    int ix = ix0 + (wx > 0.5), iy = iy0 + (wy > 0.5), iz = iz0 + (wz > 0.5);
    if (!(tx || ty || tz)) return lin_index(ix, iy, iz, M, c2);
    int best = 0x7fffffff;
    for (int dx = 0; dx <= (int)tx; ++dx)
        for (int dy = 0; dy <= (int)ty; ++dy)
            for (int dz = 0; dz <= (int)tz; ++dz) {
                int j = lin_index(tx ? ix0 + dx : ix, ty ? iy0 + dy : iy, tz ? iz0 + dz : iz, M, c2);
                best = j < best ? j : best;
            }
    return best;
}

// Trilinear footprint (kernels.py:147-170): corner indices and fp32 weights.
// Degenerate axes (w == 0, incl. every clamped component) keep the low corner.
struct Tri {
    int j[8];  // 000,100,010,110,001,101,011,111 (x fastest)
    float wx, wy, wz, ax, ay, az;
};

__device__ __forceinline__ void tri_setup(double cx, double cy, double cz, int M, int c2, Tri& t) {
    double fx = floor(cx), fy = floor(cy), fz = floor(cz);
    double dx = cx - fx, dy = cy - fy, dz = cz - fz;
    int ix0 = (int)fx, iy0 = (int)fy, iz0 = (int)fz;
    int ix1 = dx > 0.0 ? ix0 + 1 : ix0;
    int iy1 = dy > 0.0 ? iy0 + 1 : iy0;
    int iz1 = dz > 0.0 ? iz0 + 1 : iz0;
    t.wx = (float)dx; t.wy = (float)dy; t.wz = (float)dz;
    t.ax = (float)(1.0 - dx); t.ay = (float)(1.0 - dy); t.az = (float)(1.0 - dz);
    int b00 = lin_index(0, iy0, iz0, M, c2), b10 = lin_index(0, iy1, iz0, M, c2);
    int b01 = lin_index(0, iy0, iz1, M, c2), b11 = lin_index(0, iy1, iz1, M, c2);
    t.j[0] = b00 + ix0; t.j[1] = b00 + ix1;
    t.j[2] = b10 + ix0; t.j[3] = b10 + ix1;
    t.j[4] = b01 + ix0; t.j[5] = b01 + ix1;
    t.j[6] = b11 + ix0; t.j[7] = b11 + ix1;
}

__device__ __forceinline__ void tri_weights(const Tri& t, float w[8]) {
    float zy00 = t.az * t.ay, zy10 = t.az * t.wy, zy01 = t.wz * t.ay, zy11 = t.wz * t.wy;
    w[0] = zy00 * t.ax; w[1] = zy00 * t.wx;
    w[2] = zy10 * t.ax; w[3] = zy10 * t.wx;
    w[4] = zy01 * t.ax; w[5] = zy01 * t.wx;
    w[6] = zy11 * t.ax; w[7] = zy11 * t.wx;
}

// Nested blend in the reference's order (kernels.py:171-176).
__device__ __forceinline__ float2 tri_gather(const float2* __restrict__ v, const Tri& t) {
    float2 v0 = __ldg(v + t.j[0]), v1 = __ldg(v + t.j[1]), v2 = __ldg(v + t.j[2]), v3 = __ldg(v + t.j[3]);
    float2 v4 = __ldg(v + t.j[4]), v5 = __ldg(v + t.j[5]), v6 = __ldg(v + t.j[6]), v7 = __ldg(v + t.j[7]);
    float2 a, b, c, d;
    a.x = t.ax * v0.x + t.wx * v1.x; a.y = t.ax * v0.y + t.wx * v1.y;
    b.x = t.ax * v2.x + t.wx * v3.x; b.y = t.ax * v2.y + t.wx * v3.y;
    c.x = t.ax * v4.x + t.wx * v5.x; c.y = t.ax * v4.y + t.wx * v5.y;
    d.x = t.ax * v6.x + t.wx * v7.x; d.y = t.ax * v6.y + t.wx * v7.y;
    float2 lo, hi, r;
    lo.x = t.ay * a.x + t.wy * b.x; lo.y = t.ay * a.y + t.wy * b.y;
    hi.x = t.ay * c.x + t.wy * d.x; hi.y = t.ay * c.y + t.wy * d.y;
    r.x = t.az * lo.x + t.wz * hi.x; r.y = t.az * lo.y + t.wz * hi.y;
    return r;
}

constexpr double kTwoPiHi = 6.283185307179586232;     // fl(2 pi)
constexpr double kTwoPiLo = 2.449293598294706e-16;    // 2 pi - fl(2 pi)
constexpr double kInvTwoPi = 0.15915494309189535;

// CTF value at the unrotated pixel (forward.py:93-111 generalised; see
// fsld_image_rec).  gamma is evaluated in fp64 (it reaches ~470 rad at the
// mask edge for the physical CTF) and range-reduced before the fp32 sincos.
template <class Rec>
__device__ __forceinline__ float ctf_value(const Rec& R, int kx, int ky) {
    double k2 = (double)(kx * kx + ky * ky);
    double c2 = (double)(kx * kx - ky * ky);
    double s2 = (double)(2 * kx * ky);
    double g = fma(R.gamma[0], k2, fma(R.gamma[1], c2, fma(R.gamma[2], s2, R.gamma[3] * (k2 * k2))));
    double n = rint(g * kInvTwoPi);
    double r = fma(-n, kTwoPiHi, g);
    r = fma(-n, kTwoPiLo, r);
    float s, c;
    __sincosf((float)r, &s, &c);
    float ctf = -(R.wsin * s + R.wcos * c);
    if (R.env != 0.0) ctf *= __expf(-(float)(R.env * k2));
    return ctf;
}

// exp(i*pi*(shift . k)) (forward.py:299-303), argument reduced mod 2 in fp64.
template <class Rec>
__device__ __forceinline__ float2 shift_phase(const Rec& R, int kx, int ky) {
    double t = fma(R.shift[0], (double)kx, R.shift[1] * (double)ky);
    t -= 2.0 * rint(0.5 * t);
    float s, c;
    __sincosf((float)t * 3.14159265358979f, &s, &c);
    return make_float2(c, s);
}

// Full per-pixel factor f = C * phase (complex).
template <class Rec>
__device__ __forceinline__ float2 pixel_factor(const Rec& R, int kx, int ky) {
    float ctf = (R.flags & FSLD_REC_CTF) ? ctf_value(R, kx, ky) : 1.0f;
    if (R.flags & FSLD_REC_SHIFT) {
        float2 p = shift_phase(R, kx, ky);
        return make_float2(ctf * p.x, ctf * p.y);
    }
    return make_float2(ctf, 0.0f);
}

template <class Rec>
__device__ __forceinline__ float ctf_sq(const Rec& R, int kx, int ky) {
    if (!(R.flags & FSLD_REC_CTF)) return 1.0f;
    float c = ctf_value(R, kx, ky);
    return c * c;
}

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmulconj(float2 a, float2 b) {  // conj(a) * b
    return make_float2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}

// ---- accumulation ---------------------------------------------------------

__device__ __forceinline__ void red_f32x2(float* addr, float x, float y) {
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(addr), "f"(x), "f"(y) : "memory");
}

// the same on a multicast address (fsld_nvls_bind): NVSwitch adds into every rank's copy
__device__ __forceinline__ void red_mc_f32x2(float* addr, float x, float y) {
    asm volatile("multimem.red.relaxed.sys.global.add.v2.f32 [%0], {%1, %2};" ::"l"(addr), "f"(x), "f"(y) : "memory");
}

__device__ __forceinline__ void red_fixed(long long* addr, double val, double fx) {
    atomicAdd(reinterpret_cast<unsigned long long*>(addr),
              static_cast<unsigned long long>(__double2ll_rn(val * fx)));
}

template <bool DET>
__device__ __forceinline__ void scatter_c(void* acc, int j, float re, float im, double fx) {
    if constexpr (DET) {
        long long* a = reinterpret_cast<long long*>(acc) + 2 * (size_t)j;
        red_fixed(a, (double)re, fx);
        red_fixed(a + 1, (double)im, fx);
    } else {
        red_f32x2(reinterpret_cast<float*>(acc) + 2 * (size_t)j, re, im);
    }
}

template <bool DET>
__device__ __forceinline__ void scatter_r(void* acc, int j, float val, double fx) {
    if constexpr (DET) {
        red_fixed(reinterpret_cast<long long*>(acc) + j, (double)val, fx);
    } else {
        atomicAdd(reinterpret_cast<float*>(acc) + j, val);
    }
}

// Block-wide fp64 sum in a fixed order; result valid in thread 0.
__device__ __forceinline__ double block_sum(double x, double* smem /* >= 32 */) {
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) smem[wid] = x;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) {
        int nw = (blockDim.x + 31) >> 5;
        for (int w = 0; w < nw; ++w) s += smem[w];
    }
    return s;
}

// Load the 128-byte record of batch entry b into shared memory (32 x 4 B, coalesced).
__device__ __forceinline__ void load_record(const fsld_image_rec* __restrict__ recs, int row,
                                            fsld_image_rec* dst) {
    if (threadIdx.x < 32) {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(recs + row);
        reinterpret_cast<uint32_t*>(dst)[threadIdx.x] = __ldg(src + threadIdx.x);
    }
}

}  // namespace fsld
