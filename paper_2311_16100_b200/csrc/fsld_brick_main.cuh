// fsld_brick_main.cuh -- the work-item kernel of the brick-sorted loss+gradient path
// (included by fsld_brick.cu; see the design note there).
#pragma once

// float -> int32 round-to-nearest for |x| < 2^22 via the 1.5*2^23 magic (FFMA + IADD, no F2I).
constexpr float kMagic = 12582912.0f;
constexpr int kMagicBits = 0x4B400000;

// Optional per-phase cycle accounting of the item loop (thread 0 of each CTA), enabled by
// fsld_debug_phase_profile(); costs one clock64 read per phase when on.
__device__ unsigned long long* g_phase_prof = nullptr;
#define PHASE_INIT() \
    unsigned long long ph_t = clock64(), ph_acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}; \
    const bool ph_on = g_phase_prof != nullptr && threadIdx.x == 0
#define PHASE_MARK(i) \
    if (ph_on) { const unsigned long long t = clock64(); ph_acc[i] += t - ph_t; ph_t = t; ph_acc[8] += (i) == 7; }
#define PHASE_FLUSH() \
    if (ph_on) for (int q = 0; q < 9; ++q) atomicAdd(g_phase_prof + q, ph_acc[q])

// Upper bound on the pixels one image owns in one brick: lattice points of a
// plane section of a BT^3 cube (area <= BT^2 sqrt 2, perimeter <= 2 BT (1 + sqrt 2)).
constexpr int BOWN_MAX = 112;
constexpr int BBUF = BC * BOWN_MAX;

// The record fields pixel_factor reads (bytes 48..119 of fsld_image_rec, same layout).
struct FactorRec {
    double shift[2];
    double gamma[4];
    double env;
    float wsin, wcos;
    uint32_t flags;
    float xmax;
};
static_assert(sizeof(FactorRec) == 72, "FactorRec mirrors fsld_image_rec bytes 48..119");

struct SortedSmem {
    float2 vb[BH3];                 // v brick + halo
    int accr[BH3];                  // fixed-point adjoint accumulator (re)
    int acci[BH3];                  // (im)
    float2 bval[BBUF];              // pass 1 -> 2: conj(f) r per pixel of the item
    unsigned char bk[BBUF];         // segment (image) of each pixel of the item
    char2 bpc[BBUF];                // its (kx, ky), kept for pass 2
    FactorRec fac[BC];              // CTF / shift parameters of the item's images
    float frame[BC][6];             // fp32 rows 0,1 of R
    int seg_row[BC];                // dataset row of segment k
    int seg_pos[BC];                // start of segment k in its row (sorted order)
    int pref[BC + 1];               // exclusive prefix of segment lengths
    int4 item_desc;
    int item;
    int vmax_bits;
    double red[BW];
};

// Per work item (brick, <= BC image segments):
//   A  claim the item (thread 0);
//   B  warp 0: segment table + prefix of lengths; warps 1-7: the brick's 9^3
//      voxels of v (+halo, zero off the grid) -> smem;
//   C  frames, CTF/shift records (straight from the global records) and the
//      pixel -> segment table;
//   1. per pixel (flattened over the item's segments, all lanes busy):
//      gather 8 corners from the smem brick, f = C * phase, r = f P v - x,
//      |r|^2 -> loss, val = conj(f) r -> smem buffer;
//   2. with the item's max |val| known, quantise val * w to int32 with a
//      power-of-two scale (|val w s| <= 2^22; <= BC*12 contributions per voxel
//      -> |sum| < 2^31) and add with native ATOMS.ADD (order-free, no CAS);
//   3. flush: one red.global.add.v2.f32 per touched brick voxel.
// The scale follows the residual, not |Pv| or |x|: quantum ~2^-22 of the
// item's largest contribution.
__global__ void __launch_bounds__(BTHREADS, 4) sorted_loss_grad_kernel(SortedArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SortedSmem& S = *reinterpret_cast<SortedSmem*>(smem_raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int M = a.M, c = a.c, nb = a.nb, n = a.n_mask;
    const float bnd = a.bnd;
    double lsum = 0.0;
    // Work claiming runs ahead on one thread of the last warp (off warp 0's critical path):
    // its atomicAdd for item i+2 and descriptor load for item i+1 are issued during item i
    // and only consumed one iteration later.
    constexpr int kClaimer = BTHREADS - 32;
    const int n_items = a.ctl[0];
    int next_it = 0, claimed = 0;
    int4 next_item = make_int4(0, 0, 0, 0);
    if (threadIdx.x == kClaimer) {
        next_it = atomicAdd(a.ctl + 1, 1);
        if (next_it < n_items) next_item = a.items[next_it];
        claimed = atomicAdd(a.ctl + 1, 1);
    }
    PHASE_INIT();

    for (;;) {
        // ---------------- A
        if (threadIdx.x == kClaimer) {
            S.item_desc = next_item;
            S.item = next_it;
        }
        if (threadIdx.x == 0) S.vmax_bits = 0;
        __syncthreads();
        const int it = S.item;
        if (it >= n_items) break;
        const int4 item = S.item_desc;
        if (threadIdx.x == kClaimer) {  // consumed next iteration / the one after
            next_it = claimed;
            if (next_it < n_items) next_item = a.items[next_it];
            if (next_it < n_items) claimed = atomicAdd(a.ctl + 1, 1);
        }
        const int bid = item.x, pstart = item.y, nseg = item.z;
        const int ox = -c + BT * (bid % nb), oy = -c + BT * ((bid / nb) % nb), oz = -c + BT * (bid / (nb * nb));
        PHASE_MARK(0);
        // ---------------- B
        if (warp == 0) {
            int len = 0;
            if (lane < nseg) {
                const int4 pr = a.pairs[pstart + lane];  // (row, start, count)
                S.seg_row[lane] = pr.x;
                S.seg_pos[lane] = pr.y;
                len = pr.z;
            }
            int incl = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            if (lane < nseg) S.pref[lane] = incl - len;
            if (lane == 31) S.pref[nseg] = incl;
        } else {
            constexpr int U = (BH3 + BTHREADS - 32 - 1) / (BTHREADS - 32);
            float2 vv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int l = threadIdx.x - 32 + u * (BTHREADS - 32);
                const int lx = l % BH, ly = (l / BH) % BH, lz = l / (BH * BH);
                const int kx = ox + lx, ky = oy + ly, kz = oz + lz;
                vv[u] = make_float2(0.f, 0.f);
                if (l < BH3 && kx < M - c && ky < M - c && kz < M - c) vv[u] = __ldg(a.v + lin_index(kx, ky, kz, M, c));
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int l = threadIdx.x - 32 + u * (BTHREADS - 32);
                if (l < BH3) {
                    S.vb[l] = vv[u];
                    S.accr[l] = 0;
                    S.acci[l] = 0;
                }
            }
        }
        __syncthreads();
        PHASE_MARK(1);
        // ---------------- C
        for (int w = threadIdx.x; w < nseg * 24; w += BTHREADS) {
            const int k = w / 24, q = w - 24 * (w / 24);
            const uint32_t* rec = reinterpret_cast<const uint32_t*>(a.recs + S.seg_row[k]);
            if (q < 18) {
                reinterpret_cast<uint32_t*>(S.fac + k)[q] = __ldg(rec + 12 + q);
            } else {
                S.frame[k][q - 18] = (float)__ldg(reinterpret_cast<const double*>(rec) + (q - 18));
            }
        }
        const int total = min(S.pref[nseg], BBUF);
        for (int k = warp; k < nseg; k += BW)
            for (int e = S.pref[k] + lane; e < min(S.pref[k + 1], BBUF); e += 32) S.bk[e] = (unsigned char)k;
        __syncthreads();
        PHASE_MARK(2);

        // ---------------- pass 1 (loads of the next pixel issued before the current one is computed)
        float sq = 0.f, vmax = 0.f;
        int kn = 0;
        char2 kkn = make_char2(0, 0);
        float2 xvn = make_float2(0.f, 0.f);
        if ((int)threadIdx.x < total) {
            kn = S.bk[threadIdx.x];
            const size_t g = (size_t)S.seg_row[kn] * n + S.seg_pos[kn] + (threadIdx.x - S.pref[kn]);
            kkn = a.pc[g];
            xvn = __ldg(a.xs + g);
        }
        for (int e = threadIdx.x; e < total; e += BTHREADS) {
            const int k = kn;
            const char2 kk = kkn;
            const float2 xv = xvn;
            if (e + BTHREADS < total) {
                kn = S.bk[e + BTHREADS];
                const size_t g = (size_t)S.seg_row[kn] * n + S.seg_pos[kn] + (e + BTHREADS - S.pref[kn]);
                kkn = a.pc[g];
                xvn = __ldg(a.xs + g);
            }
            S.bpc[e] = kk;
            const float* fr = S.frame[k];
            const int px = kk.x, py = kk.y;
            float cx, cy, cz, fx, fy, fz;
            floor_corner((float)px, (float)py, fr, bnd, cx, cy, cz, fx, fy, fz);
            const int l0 = (((int)fz - oz) * BH + ((int)fy - oy)) * BH + ((int)fx - ox);
            const float wx = cx - fx, wy = cy - fy, wz = cz - fz;
            const float ax = 1.f - wx, ay = 1.f - wy, az = 1.f - wz;
            const float2 f = pixel_factor(S.fac[k], px, py);
            const float2* vb = S.vb + l0;
            // trilinear gather (kernels.py:171-176) from the smem brick
            const float2 WX = make_float2(wx, wx), AX = make_float2(ax, ax);
            const float2 e0 = __ffma2_rn(WX, vb[1], __fmul2_rn(AX, vb[0]));
            const float2 e1 = __ffma2_rn(WX, vb[BH + 1], __fmul2_rn(AX, vb[BH]));
            const float2 e2 = __ffma2_rn(WX, vb[BH * BH + 1], __fmul2_rn(AX, vb[BH * BH]));
            const float2 e3 = __ffma2_rn(WX, vb[BH * BH + BH + 1], __fmul2_rn(AX, vb[BH * BH + BH]));
            const float2 q0 = __ffma2_rn(make_float2(wy, wy), e1, __fmul2_rn(make_float2(ay, ay), e0));
            const float2 q1 = __ffma2_rn(make_float2(wy, wy), e3, __fmul2_rn(make_float2(ay, ay), e2));
            const float2 pv = __ffma2_rn(make_float2(wz, wz), q1, __fmul2_rn(make_float2(az, az), q0));
            const float2 prj = cmul(pv, f);
            const float2 rr = make_float2(prj.x - xv.x, prj.y - xv.y);
            sq = fmaf(rr.x, rr.x, fmaf(rr.y, rr.y, sq));
            const float2 val = cmulconj(f, rr);
            vmax = fmaxf(vmax, fmaxf(fabsf(val.x), fabsf(val.y)));
            S.bval[e] = val;
        }
        for (int o = 16; o > 0; o >>= 1) {
            sq += __shfl_xor_sync(0xffffffffu, sq, o);
            vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
        }
        if (lane == 0) {
            lsum += (double)sq;
            atomicMax(&S.vmax_bits, __float_as_int(vmax));
        }
        __syncthreads();
        PHASE_MARK(3);

        // ---------------- pass 2: fixed-point adjoint scatter (kernels.py:221-230)
        const float vm = __int_as_float(S.vmax_bits);
        const float sc = vm > 0.f ? exp2f(floorf(log2f(4194303.0f / vm))) : 1.0f;
        const float inv_sc = 1.0f / sc;
        for (int e = threadIdx.x; e < total; e += BTHREADS) {
            const int k = S.bk[e];
            const char2 kk = S.bpc[e];
            float cx, cy, cz, fx, fy, fz;
            floor_corner((float)kk.x, (float)kk.y, S.frame[k], bnd, cx, cy, cz, fx, fy, fz);
            const int l0 = (((int)fz - oz) * BH + ((int)fy - oy)) * BH + ((int)fx - ox);
            const float wx = cx - fx, wy = cy - fy, wz = cz - fz;
            const float ax = 1.f - wx, ay = 1.f - wy, az = 1.f - wz;
            const float2 val = __fmul2_rn(S.bval[e], make_float2(sc, sc));
            const float zy00 = az * ay, zy10 = az * wy, zy01 = wz * ay, zy11 = wz * wy;
            const float w8[8] = {zy00 * ax, zy00 * wx, zy10 * ax, zy10 * wx, zy01 * ax, zy01 * wx, zy11 * ax, zy11 * wx};
            const int off8[8] = {0, 1, BH, BH + 1, BH * BH, BH * BH + 1, BH * BH + BH, BH * BH + BH + 1};
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const float2 y = __ffma2_rn(make_float2(w8[q], w8[q]), val, make_float2(kMagic, kMagic));
                atomicAdd(S.accr + l0 + off8[q], __float_as_int(y.x) - kMagicBits);
                atomicAdd(S.acci + l0 + off8[q], __float_as_int(y.y) - kMagicBits);
            }
        }
        __syncthreads();
        PHASE_MARK(4);
        // ---------------- flush: one vector reduction per touched brick voxel
        for (int l = threadIdx.x; l < BH3; l += BTHREADS) {
            const int qr = S.accr[l], qi = S.acci[l];
            if ((qr | qi) == 0) continue;
            const int lx = l % BH, ly = (l / BH) % BH, lz = l / (BH * BH);
            const int kx = ox + lx, ky = oy + ly, kz = oz + lz;
            if (kx >= M - c || ky >= M - c || kz >= M - c) continue;
            red_f32x2(reinterpret_cast<float*>(a.acc) + 2 * (size_t)lin_index(kx, ky, kz, M, c),
                      (float)qr * inv_sc, (float)qi * inv_sc);
        }
        __syncthreads();
        PHASE_MARK(7);
    }
    PHASE_FLUSH();
    if (lane == 0) S.red[warp] = lsum;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < BW; ++w) s += S.red[w];
        a.part[blockIdx.x] = s;
    }
}
