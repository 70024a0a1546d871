/*
 * capi_demo.c -- the C ABI (include/fsld_b200.h) driven from plain C, no Python:
 * what a non-Python host (or the cgo/ctypes binding in INTEGRATION.md) does.
 *
 *  1. adjointness of the slice operator: <y, P v> == <P^* y, v>  (fsld_project / fsld_backproject);
 *  2. brick-sorted fused loss+grad (fsld_sorted_count/fill + fsld_loss_grad_sorted) against the
 *     per-pixel tile kernel (fsld_loss_grad) on the same batch, on both brick kernels: the
 *     compute path (ptab = NULL) and the table-driven one (fsld_sorted_tables).
 * Prints one line and exits 0 on success.  Built and run by tests/test_gpu_capi_c.py.
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "fsld_b200.h"

#define CK(x)                                                                            \
    do {                                                                                 \
        int st_ = (x);                                                                   \
        if (st_ != 0) {                                                                  \
            fprintf(stderr, "%s:%d %s -> %d (%s)\n", __FILE__, __LINE__, #x, st_,       \
                    st_ < 0 ? fsld_status_string(st_) : cudaGetErrorString((cudaError_t)st_)); \
            return 2;                                                                    \
        }                                                                                \
    } while (0)

static unsigned long long rng_state = 88172645463325252ull;
static double urand(void) { /* xorshift64*, uniform in [0, 1) */
    rng_state ^= rng_state >> 12;
    rng_state ^= rng_state << 25;
    rng_state ^= rng_state >> 27;
    return (double)((rng_state * 2685821657736338717ull) >> 11) / 9007199254740992.0;
}
static double nrand(void) { return sqrt(-2.0 * log(1.0 - urand())) * cos(6.283185307179586 * urand()); }

int main(void) {
    const int M = 32, R = M / 2 - 1, B = 24;
    const int c = (M + 1) / 2;
    int n = 0;
    int16_t* pix = malloc(sizeof(int16_t) * 2 * M * M);
    for (int y = 0; y < M; ++y)
        for (int x = 0; x < M; ++x) { /* disk mask, ascending pixel index (grid.py:185-189) */
            const int kx = x - c, ky = y - c;
            if (lround(sqrt((double)(kx * kx + ky * ky))) <= R) {
                pix[2 * n] = (int16_t)kx;
                pix[2 * n + 1] = (int16_t)ky;
                ++n;
            }
        }
    fsld_image_rec* recs = calloc(B, sizeof(fsld_image_rec));
    for (int b = 0; b < B; ++b) { /* random rotation (rows 0, 1 of R from a unit quaternion) */
        double w = nrand(), qx = nrand(), qy = nrand(), qz = nrand();
        const double s = 1.0 / sqrt(w * w + qx * qx + qy * qy + qz * qz);
        w *= s, qx *= s, qy *= s, qz *= s;
        const double r[6] = {1 - 2 * (qy * qy + qz * qz), 2 * (qx * qy - qz * w), 2 * (qx * qz + qy * w),
                             2 * (qx * qy + qz * w),     1 - 2 * (qx * qx + qz * qz), 2 * (qy * qz - qx * w)};
        memcpy(recs[b].rot, r, sizeof(r));
        recs[b].shift[0] = 0.05 * nrand(); /* shift phase only; no CTF */
        recs[b].shift[1] = 0.05 * nrand();
        recs[b].flags = FSLD_REC_SHIFT;
    }
    const size_t nv = (size_t)M * M * M, ni = (size_t)B * n;
    float* v = malloc(8 * nv);
    float* y = malloc(8 * ni);
    for (size_t i = 0; i < 2 * nv; ++i) v[i] = (float)nrand();
    for (size_t i = 0; i < 2 * ni; ++i) y[i] = (float)nrand();

    int ndev = 0;
    if (fsld_device_count(&ndev) != FSLD_OK) {
        fprintf(stderr, "no sm_100 device\n");
        return 3;
    }
    void *d_pix, *d_recs, *d_v, *d_y, *d_py, *d_acc, *d_acc2, *d_scr, *d_sq, *d_seg_off, *d_segs, *d_pc, *d_xs;
    CK(cudaMalloc(&d_pix, sizeof(int16_t) * 2 * n));
    CK(cudaMalloc(&d_recs, sizeof(fsld_image_rec) * B));
    CK(cudaMalloc(&d_v, 8 * nv));
    CK(cudaMalloc(&d_y, 8 * ni));
    CK(cudaMalloc(&d_py, 8 * ni));
    CK(cudaMalloc(&d_acc, 8 * nv));
    CK(cudaMalloc(&d_acc2, 8 * nv));
    CK(cudaMalloc(&d_sq, 3 * sizeof(double)));
    CK(cudaMemcpy(d_pix, pix, sizeof(int16_t) * 2 * n, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_recs, recs, sizeof(fsld_image_rec) * B, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_v, v, 8 * nv, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_y, y, 8 * ni, cudaMemcpyHostToDevice));
    const size_t scr_bytes = fsld_scratch_bytes(M, n, B);
    CK(cudaMalloc(&d_scr, scr_bytes));
    CK(fsld_prepare(M, n, d_pix, d_scr, scr_bytes, NULL));

    /* 1. adjointness */
    CK(cudaMemset(d_acc, 0, 8 * nv));
    CK(fsld_project(M, FSLD_MODE_TRI, n, d_pix, d_recs, NULL, B, d_v, d_py, NULL));
    CK(fsld_backproject(M, FSLD_MODE_TRI, n, d_pix, d_recs, NULL, B, d_y, d_acc, 0u, NULL, NULL));
    float* py = malloc(8 * ni);
    float* pty = malloc(8 * nv);
    CK(cudaMemcpy(py, d_py, 8 * ni, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(pty, d_acc, 8 * nv, cudaMemcpyDeviceToHost));
    double lr = 0, li = 0, rr = 0, ri = 0; /* <y, Pv> and <P^* y, v> */
    for (size_t i = 0; i < ni; ++i) {
        lr += (double)y[2 * i] * py[2 * i] + (double)y[2 * i + 1] * py[2 * i + 1];
        li += (double)y[2 * i] * py[2 * i + 1] - (double)y[2 * i + 1] * py[2 * i];
    }
    for (size_t i = 0; i < nv; ++i) {
        rr += (double)pty[2 * i] * v[2 * i] + (double)pty[2 * i + 1] * v[2 * i + 1];
        ri += (double)pty[2 * i] * v[2 * i + 1] - (double)pty[2 * i + 1] * v[2 * i];
    }
    const double adj = hypot(lr - rr, li - ri) / hypot(lr, li);

    /* 2. brick-sorted dataset layout (images = y) and the fused loss+grad vs the tile kernel */
    CK(cudaMalloc(&d_seg_off, sizeof(int32_t) * (B + 1)));
    CK(fsld_sorted_count(M, n, d_pix, d_recs, B, d_seg_off, NULL));
    int32_t nseg = 0;
    CK(cudaMemcpy(&nseg, (int32_t*)d_seg_off + B, sizeof(int32_t), cudaMemcpyDeviceToHost));
    CK(cudaMalloc(&d_segs, sizeof(int32_t) * 2 * (nseg > 0 ? nseg : 1)));
    CK(cudaMalloc(&d_pc, 2 * ni));
    CK(cudaMalloc(&d_xs, 8 * ni));
    CK(fsld_sorted_fill(M, n, d_pix, d_recs, B, d_y, d_xs, d_pc, d_seg_off, d_segs, NULL));
    CK(cudaMemset(d_acc, 0, 8 * nv));
    CK(cudaMemset(d_acc2, 0, 8 * nv));
    CK(fsld_loss_grad(M, FSLD_MODE_TRI, n, d_pix, d_recs, NULL, B, d_v, d_y, d_acc, (double*)d_sq, 0u, NULL, d_scr,
                      scr_bytes, NULL));
    CK(fsld_loss_grad_sorted(M, FSLD_MODE_TRI, n, d_recs, NULL, B, d_v, d_xs, d_pc, NULL, d_seg_off, d_segs, d_acc2,
                             (double*)d_sq + 1, 0u, NULL, d_scr, scr_bytes, NULL));
    void* d_ptab = NULL;
    void* d_acc3 = NULL;
    CK(cudaMalloc(&d_ptab, fsld_sorted_tables_bytes(B, n)));
    CK(cudaMalloc(&d_acc3, 8 * nv));
    CK(cudaMemset(d_acc3, 0, 8 * nv));
    CK(fsld_sorted_tables(M, FSLD_MODE_TRI, n, d_recs, B, d_pc, d_seg_off, d_segs, d_ptab, NULL));
    CK(fsld_loss_grad_sorted(M, FSLD_MODE_TRI, n, d_recs, NULL, B, d_v, d_xs, d_pc, d_ptab, d_seg_off, d_segs,
                             d_acc3, (double*)d_sq + 2, 0u, NULL, d_scr, scr_bytes, NULL));
    double sq[3];
    float* g1 = malloc(8 * nv);
    float* g2 = malloc(8 * nv);
    float* g3 = malloc(8 * nv);
    CK(cudaMemcpy(sq, d_sq, sizeof(sq), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(g1, d_acc, 8 * nv, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(g2, d_acc2, 8 * nv, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(g3, d_acc3, 8 * nv, cudaMemcpyDeviceToHost));
    double num = 0, num3 = 0, den = 0;
    for (size_t i = 0; i < 2 * nv; ++i) {
        num += ((double)g1[i] - g2[i]) * ((double)g1[i] - g2[i]);
        num3 += ((double)g1[i] - g3[i]) * ((double)g1[i] - g3[i]);
        den += (double)g1[i] * g1[i];
    }
    const double grel = fmax(sqrt(num / den), sqrt(num3 / den));
    const double srel = fmax(fabs(sq[0] - sq[1]), fabs(sq[0] - sq[2])) / sq[0];
    const int bad = fsld_loss_grad(M, 7, n, d_pix, d_recs, NULL, B, d_v, d_y, d_acc, (double*)d_sq, 0u, NULL, d_scr,
                                   scr_bytes, NULL) != FSLD_EINVAL;
    printf("capi_demo M=%d n_mask=%d B=%d segments=%d adjointness=%.3e sq_rel=%.3e grad_rel=%.3e\n", M, n, B, nseg,
           adj, srel, grel);
    const int ok = adj < 1e-5 && srel < 1e-6 && grel < 5e-6 && !bad;
    return ok ? 0 : 1;
}
