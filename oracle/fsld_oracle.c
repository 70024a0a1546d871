/*
 * fsld_oracle.c -- CPU restatement of the reference slice/adjoint kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port") for the B200 path; the product never links or calls it.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs load the shared object built from it.
 *
 * It restates, in plain C99 + OpenMP, the numba kernels of the reference:
 *   /root/reference/pkg/src/fsld/kernels.py
 *     _rotate_pixel   kernels.py:42-60    (c = R^T (px,py,0), clamp +-(M//2-1))
 *     _lin_index      kernels.py:63-66    (z in FFT order, x/y centred)
 *     _nn_index       kernels.py:69-120   (exact 0.5 ties -> smallest linear index)
 *     assign_nn       kernels.py:123-135
 *     project_tri     kernels.py:138-177
 *     project_nn      kernels.py:180-190
 *     backproject_tri kernels.py:193-230  (per-64-image private partial volumes)
 *     backproject_nn  kernels.py:233-248
 *     scatter_sq_tri  kernels.py:251-294
 *     fold_chunks     kernels.py:297-302  (fixed chunk-order fold)
 *
 * Arithmetic contract: fp64, every product and sum separately rounded (build
 * with -ffp-contract=off; the numba kernels contain no FMA), and complex
 * arithmetic done the way numba lowers it: a real operand is promoted to a
 * complex with zero imaginary part and multiplied with the schoolbook
 * formula (ac - bd, ad + bc).  With that, outputs are bit-identical to the
 * reference (pinned by tests/test_oracle_golden.py against fixtures the
 * reference itself produced, tests/golden/make_golden.py).
 *
 * Complex arrays are interleaved (re, im) doubles; real arrays are doubles.
 * Rotation matrices are (B,3,3) row-major; pixel coordinates (n,2) doubles.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_SCATTER_CHUNK 64 /* kernels.py:35 */

typedef struct { double re, im; } cplx;

static inline cplx cmk(double re, double im) { cplx z; z.re = re; z.im = im; return z; }
static inline cplx cmul(cplx a, cplx b) {
    return cmk(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re);
}
/* real * complex, numba-style promotion of the real operand */
static inline cplx rmul(double r, cplx b) { return cmul(cmk(r, 0.0), b); }
static inline cplx cadd(cplx a, cplx b) { return cmk(a.re + b.re, a.im + b.im); }
static inline cplx cconj(cplx a) { return cmk(a.re, -a.im); }
static inline cplx cload(const double* p, int64_t i) { return cmk(p[2 * i], p[2 * i + 1]); }

/* kernels.py:42-60 -- only rows 0 and 1 of R are read */
static inline void rotate_pixel(const double* R, double px, double py, double bnd,
                                double* cx, double* cy, double* cz) {
    double x = R[0] * px + R[3] * py;
    double y = R[1] * px + R[4] * py;
    double z = R[2] * px + R[5] * py;
    if (x > bnd) x = bnd; else if (x < -bnd) x = -bnd;
    if (y > bnd) y = bnd; else if (y < -bnd) y = -bnd;
    if (z > bnd) z = bnd; else if (z < -bnd) z = -bnd;
    *cx = x; *cy = y; *cz = z;
}

/* kernels.py:63-66 */
static inline int64_t lin_index(int64_t ix, int64_t iy, int64_t iz, int64_t M, int64_t c2) {
    int64_t zi = iz < 0 ? iz + M : iz;
    return (zi * M + iy + c2) * M + ix + c2;
}

/* kernels.py:69-120: nearest lattice point, exact-0.5 ties -> min linear index */
static inline int64_t nn_index(double cx, double cy, double cz, int64_t M, int64_t c2) {
    double fx = floor(cx), fy = floor(cy), fz = floor(cz);
    double wx = cx - fx, wy = cy - fy, wz = cz - fz;
    int64_t ix0 = (int64_t)fx, iy0 = (int64_t)fy, iz0 = (int64_t)fz;
    int tx = (wx == 0.5), ty = (wy == 0.5), tz = (wz == 0.5);
    if (!(tx || ty || tz)) {
        return lin_index(ix0 + (wx > 0.5), iy0 + (wy > 0.5), iz0 + (wz > 0.5), M, c2);
    }
    int64_t best = -1;
    for (int dx = 0; dx < (tx ? 2 : 1); ++dx) {
        int64_t ix = tx ? ix0 + dx : ix0 + (wx > 0.5);
        for (int dy = 0; dy < (ty ? 2 : 1); ++dy) {
            int64_t iy = ty ? iy0 + dy : iy0 + (wy > 0.5);
            for (int dz = 0; dz < (tz ? 2 : 1); ++dz) {
                int64_t iz = tz ? iz0 + dz : iz0 + (wz > 0.5);
                int64_t j = lin_index(ix, iy, iz, M, c2);
                if (best < 0 || j < best) best = j;
            }
        }
    }
    return best;
}

typedef struct {
    int64_t j[8];   /* corner order 000,100,010,110,001,101,011,111 (x fastest) */
    double wx, wy, wz, ax, ay, az;
} tri_corners;

/* kernels.py:147-170 (shared by project_tri, backproject_tri, scatter_sq_tri) */
static inline void tri_setup(double cx, double cy, double cz, int64_t M, int64_t c2, tri_corners* t) {
    double fx = floor(cx), fy = floor(cy), fz = floor(cz);
    t->wx = cx - fx; t->wy = cy - fy; t->wz = cz - fz;
    int64_t ix0 = (int64_t)fx, iy0 = (int64_t)fy, iz0 = (int64_t)fz;
    int64_t ix1 = t->wx > 0.0 ? ix0 + 1 : ix0;
    int64_t iy1 = t->wy > 0.0 ? iy0 + 1 : iy0;
    int64_t iz1 = t->wz > 0.0 ? iz0 + 1 : iz0;
    t->ax = 1.0 - t->wx; t->ay = 1.0 - t->wy; t->az = 1.0 - t->wz;
    t->j[0] = lin_index(ix0, iy0, iz0, M, c2);
    t->j[1] = lin_index(ix1, iy0, iz0, M, c2);
    t->j[2] = lin_index(ix0, iy1, iz0, M, c2);
    t->j[3] = lin_index(ix1, iy1, iz0, M, c2);
    t->j[4] = lin_index(ix0, iy0, iz1, M, c2);
    t->j[5] = lin_index(ix1, iy0, iz1, M, c2);
    t->j[6] = lin_index(ix0, iy1, iz1, M, c2);
    t->j[7] = lin_index(ix1, iy1, iz1, M, c2);
}

static void set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

int64_t orc_n_chunks(int64_t B) { return (B + ORC_SCATTER_CHUNK - 1) / ORC_SCATTER_CHUNK; }

/* kernels.py:123-135 */
void orc_assign_nn(const double* rt, int64_t B, const double* pix, int64_t n, int64_t M,
                   int64_t* out, int nthreads) {
    int64_t c2 = (M + 1) / 2;
    double bnd = (double)(M / 2 - 1);
    set_threads(nthreads);
#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < B; ++b) {
        const double* R = rt + 9 * b;
        for (int64_t p = 0; p < n; ++p) {
            double cx, cy, cz;
            rotate_pixel(R, pix[2 * p], pix[2 * p + 1], bnd, &cx, &cy, &cz);
            out[b * n + p] = nn_index(cx, cy, cz, M, c2);
        }
    }
}

/* kernels.py:138-177 (tri) and 180-190 (nn); phase complex (B,n), ctf real (B,n) */
void orc_project(int tri, const double* v, const double* rt, int64_t B, const double* pix,
                 int64_t n, const double* phase, const double* ctf, int64_t M, double* out,
                 int nthreads) {
    int64_t c2 = (M + 1) / 2;
    double bnd = (double)(M / 2 - 1);
    set_threads(nthreads);
#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < B; ++b) {
        const double* R = rt + 9 * b;
        for (int64_t p = 0; p < n; ++p) {
            double cx, cy, cz;
            rotate_pixel(R, pix[2 * p], pix[2 * p + 1], bnd, &cx, &cy, &cz);
            cplx acc;
            if (tri) {
                tri_corners t;
                tri_setup(cx, cy, cz, M, c2, &t);
                cplx lo = cadd(rmul(t.ay, cadd(rmul(t.ax, cload(v, t.j[0])), rmul(t.wx, cload(v, t.j[1])))),
                               rmul(t.wy, cadd(rmul(t.ax, cload(v, t.j[2])), rmul(t.wx, cload(v, t.j[3])))));
                cplx hi = cadd(rmul(t.ay, cadd(rmul(t.ax, cload(v, t.j[4])), rmul(t.wx, cload(v, t.j[5])))),
                               rmul(t.wy, cadd(rmul(t.ax, cload(v, t.j[6])), rmul(t.wx, cload(v, t.j[7])))));
                acc = cadd(rmul(t.az, lo), rmul(t.wz, hi));
            } else {
                acc = cload(v, nn_index(cx, cy, cz, M, c2));
            }
            /* numba evaluates (acc * phase) * ctf: complex * real(promoted) */
            cplx o = cmul(cmul(acc, cload(phase, b * n + p)), cmk(ctf[b * n + p], 0.0));
            out[2 * (b * n + p)] = o.re;
            out[2 * (b * n + p) + 1] = o.im;
        }
    }
}

/* kernels.py:297-302: fold partials in chunk order */
void orc_fold_chunks(const double* vols, int64_t nch, int64_t len, double* out) {
    memcpy(out, vols, (size_t)len * sizeof(double));
    for (int64_t c = 1; c < nch; ++c) {
        const double* src = vols + c * len;
        for (int64_t i = 0; i < len; ++i) out[i] += src[i];
    }
}

/* kernels.py:193-248: adjoint, per-chunk private volumes then fixed fold.
 * vols_scratch: nch * M^3 complex (caller-provided, any content) -> out M^3 complex. */
void orc_backproject(int tri, const double* img, const double* rt, int64_t B, const double* pix,
                     int64_t n, const double* phase, const double* ctf, int64_t M,
                     double* vols_scratch, double* out, int nthreads) {
    int64_t c2 = (M + 1) / 2;
    double bnd = (double)(M / 2 - 1);
    int64_t nvox = M * M * M;
    int64_t nch = orc_n_chunks(B);
    memset(vols_scratch, 0, (size_t)(nch * nvox * 2) * sizeof(double));
    set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t c = 0; c < nch; ++c) {
        double* vol = vols_scratch + c * nvox * 2;
        int64_t lo = c * ORC_SCATTER_CHUNK;
        int64_t hi = lo + ORC_SCATTER_CHUNK < B ? lo + ORC_SCATTER_CHUNK : B;
        for (int64_t b = lo; b < hi; ++b) {
            const double* R = rt + 9 * b;
            for (int64_t p = 0; p < n; ++p) {
                double cx, cy, cz;
                rotate_pixel(R, pix[2 * p], pix[2 * p + 1], bnd, &cx, &cy, &cz);
                cplx val = cmul(cmul(cload(img, b * n + p), cconj(cload(phase, b * n + p))),
                                cmk(ctf[b * n + p], 0.0));
                if (tri) {
                    tri_corners t;
                    tri_setup(cx, cy, cz, M, c2, &t);
                    double w[8];
                    w[0] = t.az * t.ay * t.ax; w[1] = t.az * t.ay * t.wx;
                    w[2] = t.az * t.wy * t.ax; w[3] = t.az * t.wy * t.wx;
                    w[4] = t.wz * t.ay * t.ax; w[5] = t.wz * t.ay * t.wx;
                    w[6] = t.wz * t.wy * t.ax; w[7] = t.wz * t.wy * t.wx;
                    for (int k = 0; k < 8; ++k) {
                        cplx d = rmul(w[k], val);
                        vol[2 * t.j[k]] += d.re;
                        vol[2 * t.j[k] + 1] += d.im;
                    }
                } else {
                    int64_t j = nn_index(cx, cy, cz, M, c2);
                    vol[2 * j] += val.re;
                    vol[2 * j + 1] += val.im;
                }
            }
        }
    }
    orc_fold_chunks(vols_scratch, nch, nvox * 2, out);
}

/* kernels.py:251-294: sum of squared trilinear weights times weights[b,p] */
void orc_scatter_sq_tri(const double* weights, const double* rt, int64_t B, const double* pix,
                        int64_t n, int64_t M, double* vols_scratch, double* out, int nthreads) {
    int64_t c2 = (M + 1) / 2;
    double bnd = (double)(M / 2 - 1);
    int64_t nvox = M * M * M;
    int64_t nch = orc_n_chunks(B);
    memset(vols_scratch, 0, (size_t)(nch * nvox) * sizeof(double));
    set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t c = 0; c < nch; ++c) {
        double* vol = vols_scratch + c * nvox;
        int64_t lo = c * ORC_SCATTER_CHUNK;
        int64_t hi = lo + ORC_SCATTER_CHUNK < B ? lo + ORC_SCATTER_CHUNK : B;
        for (int64_t b = lo; b < hi; ++b) {
            const double* R = rt + 9 * b;
            for (int64_t p = 0; p < n; ++p) {
                double cx, cy, cz;
                rotate_pixel(R, pix[2 * p], pix[2 * p + 1], bnd, &cx, &cy, &cz);
                tri_corners t;
                tri_setup(cx, cy, cz, M, c2, &t);
                double s = weights[b * n + p];
                double w[8];
                w[0] = t.az * t.ay * t.ax; w[1] = t.az * t.ay * t.wx;
                w[2] = t.az * t.wy * t.ax; w[3] = t.az * t.wy * t.wx;
                w[4] = t.wz * t.ay * t.ax; w[5] = t.wz * t.ay * t.wx;
                w[6] = t.wz * t.wy * t.ax; w[7] = t.wz * t.wy * t.wx;
                for (int k = 0; k < 8; ++k) vol[t.j[k]] += (w[k] * w[k]) * s;
            }
        }
    }
    orc_fold_chunks(vols_scratch, nch, nvox, out);
}
