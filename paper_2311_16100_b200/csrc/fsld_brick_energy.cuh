// fsld_brick_energy.cuh -- projection energy sum_b sum_p C^2 |P d|^2 on the brick-sorted layout
// (included by fsld_brick.cu after fsld_brick_main.cuh).
//
// The closed-form line search (fsld_step.cu) needs ||A d||^2 for the search
// direction d: |f P d|^2 = C^2 |P d|^2 (the shift phase has modulus one), so
// this is a gather-only pass: no images, no residual, no scatter.  Same work
// items as the loss+grad kernel (brick, <= BC segments); the brick of d is
// staged in shared memory and each pixel's 8 corners are read from there.
#pragma once

#ifndef FSLD_RB_ENERGY  // pixels per round (the pixel -> segment table)
#define FSLD_RB_ENERGY 4096
#endif

struct EnergySmem {
    float2 vb[BH3];
    int4 segw[BC * SEG_W];  // segment records, SEG_W words apart (fsld_kernels.cuh)
    __device__ __forceinline__ SegRec& seg(int k) { return *reinterpret_cast<SegRec*>(segw + k * SEG_W); }
    int pref[BC + 1];
    int wtot[BC / 32];
    unsigned char bk[FSLD_RB_ENERGY];
    int4 item_desc;
    double red[BW];
};

__device__ __forceinline__ float seg_ctf(const SegRec& R, int kx, int ky) {
    const int kx2 = kx * kx, ky2 = ky * ky;
    const uint32_t k2 = (uint32_t)(kx2 + ky2);
    const uint32_t c2 = (uint32_t)(kx2 - ky2 + 32768);
    const uint32_t s2 = (uint32_t)(2 * kx * ky + 65536);
    const uint32_t tg = R.gc + turns_term(R.glo[0], R.ghi[0], k2) + turns_term(R.glo[1], R.ghi[1], c2) +
                        turns_term(R.glo[2], R.ghi[2], s2) + turns_term(R.glo[3], R.ghi[3], k2 * k2);
    constexpr float kTurn = 1.4629180792671596e-09f;  // 2 pi / 2^32
    float sg, cg;
    __sincosf((float)(int)tg * kTurn, &sg, &cg);
    return -(R.wsin * sg + R.wcos * cg) * exp2f(-R.envl * (float)k2);
}

__global__ void __launch_bounds__(BTHREADS) sorted_energy_kernel(SortedArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    EnergySmem& S = *reinterpret_cast<EnergySmem*>(smem_raw);
    a.pairs += a.ctl[3];  // this batch's pairs / items (non-zero offsets in a multi-batch plan)
    a.items += a.ctl[4];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int M = a.M, c = a.c, nb = a.nb;
    const float bnd = a.bnd;
    const int n_items = a.ctl[0];
    double lsum = 0.0;
    for (;;) {
        if (threadIdx.x == 0) {
            const int it = atomicAdd(a.ctl + 1, 1);
            S.item_desc = it < n_items ? a.items[it] : make_int4(-1, 0, 0, 0);
        }
        __syncthreads();
        const int4 item = S.item_desc;
        if (item.x < 0) break;
        const int bid = item.x, pstart = item.y, nseg = item.z;
        const int ox = -c + BT * (bid % nb), oy = -c + BT * ((bid / nb) % nb), oz = -c + BT * (bid / (nb * nb));
        {
            for (int w = threadIdx.x; w < nseg * 8; w += BTHREADS)
                S.segw[(w >> 3) * SEG_W + (w & 7)] = seg_chunk(a, pstart + (w >> 3), w & 7);
        }
        if (warp < BC / 32) {
            const int k = threadIdx.x;
            const int len = k < nseg ? __ldg(&a.pairs[pstart + k].count) : 0;
            int incl = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            S.pref[k] = incl - len;
            if (lane == 31) S.wtot[warp] = incl;
        }
        for (int l = threadIdx.x; l < BH3; l += BTHREADS) {
            const int kx = ox + l % BH, ky = oy + (l / BH) % BH, kz = oz + l / (BH * BH);
            S.vb[l] = (kx < M - c && ky < M - c && kz < M - c) ? __ldg(a.v + lin_index(kx, ky, kz, M, c))
                                                               : make_float2(0.f, 0.f);
        }
        __syncthreads();
        if (threadIdx.x < nseg) {
            const int k = threadIdx.x;
            int p = S.pref[k];
            for (int w = 0; w < (k >> 5); ++w) p += S.wtot[w];
            S.pref[k] = p;
            S.seg(k).gofs -= p;
        }
        if (threadIdx.x == 0) {
            int t = 0;
            for (int w = 0; w < BC / 32; ++w) t += S.wtot[w];
            S.pref[nseg] = t;
        }
        __syncthreads();
        const int total = S.pref[nseg];
        for (int r0 = 0; r0 < total; r0 += FSLD_RB_ENERGY) {
            const int rn = min(FSLD_RB_ENERGY, total - r0);
            {
                const int k = threadIdx.x / SEG_T, q = threadIdx.x % SEG_T;
                if (k < nseg) {
                    const int e1 = min(S.pref[k + 1], r0 + rn) - r0;
                    for (int e = max(S.pref[k], r0) - r0 + q; e < e1; e += SEG_T) S.bk[e] = (unsigned char)k;
                }
            }
            __syncthreads();
            float en = 0.f;
            for (int e = threadIdx.x; e < rn; e += BTHREADS) {
                const SegRec& R = S.seg(S.bk[e]);
                const char2 kk = a.pc[R.gofs + (r0 + e)];
                const int px = kk.x, py = kk.y;
                float cx, cy, cz, fx, fy, fz;
                floor_corner((float)px, (float)py, R.frame, bnd, cx, cy, cz, fx, fy, fz);
                const int l0 = (((int)fz - oz) * BH + ((int)fy - oy)) * BH + ((int)fx - ox);
                const float wx = cx - fx, wy = cy - fy, wz = cz - fz;
                const float ax = 1.f - wx, ay = 1.f - wy, az = 1.f - wz;
                const float2* vb = S.vb + l0;
                const float2 WX = make_float2(wx, wx), AX = make_float2(ax, ax);
                const float2 e0 = __ffma2_rn(WX, vb[1], __fmul2_rn(AX, vb[0]));
                const float2 e1 = __ffma2_rn(WX, vb[BH + 1], __fmul2_rn(AX, vb[BH]));
                const float2 e2 = __ffma2_rn(WX, vb[BH * BH + 1], __fmul2_rn(AX, vb[BH * BH]));
                const float2 e3 = __ffma2_rn(WX, vb[BH * BH + BH + 1], __fmul2_rn(AX, vb[BH * BH + BH]));
                const float2 q0 = __ffma2_rn(make_float2(wy, wy), e1, __fmul2_rn(make_float2(ay, ay), e0));
                const float2 q1 = __ffma2_rn(make_float2(wy, wy), e3, __fmul2_rn(make_float2(ay, ay), e2));
                const float2 pv = __ffma2_rn(make_float2(wz, wz), q1, __fmul2_rn(make_float2(az, az), q0));
                const float ct = seg_ctf(R, px, py);
                en = fmaf(ct * ct, fmaf(pv.x, pv.x, pv.y * pv.y), en);
            }
            lsum += (double)en;
            __syncthreads();
        }
    }
    for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
    if (lane == 0) S.red[warp] = lsum;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < BW; ++w) s += S.red[w];
        a.part[blockIdx.x] = s;
    }
}
