// fsld_brick_v3.cuh -- the table-driven brick kernel of the fused loss+gradient (included by fsld_brick.cu).
//
// Same work items, shared-memory brick and fixed-point adjoint as sorted_loss_grad_kernel
// (fsld_brick_main.cuh), with pass 1 rebuilt around the dataset's per-pixel tables
// (fsld_brick_tables.cuh):
//   * no per-pixel segment record, no geometry / CTF / phase arithmetic: f = C * phase (8 B) and
//     the trilinear footprint (16 B) come from the dataset tables next to the 8-byte image value,
//     so pass 1 is the 8-corner gather, the residual and conj(f) r;
//   * the pixel -> segment byte table is built once per work item (not per round), so a thread
//     can address any pixel of the item: each thread's next pixel is loaded while the current
//     one is computed, and the first pixel of the next round is loaded before the round's
//     barrier, so it arrives during pass 2 (the per-pixel HBM latency was the top stall of
//     the compute path);
//   * pass 2 (fixed-point scatter, kernels.py:221-230) is unchanged.
#pragma once

#ifndef FSLD_RB3
#if FSLD_V3_FULLW
#define FSLD_RB3 768
#else
#define FSLD_RB3 1024
#endif
#endif
constexpr int RB3 = FSLD_RB3;
#ifndef FSLD_V3_MINB  // CTAs per SM the registers are budgeted for: 4 (64 registers).  5 (48) fits
#define FSLD_V3_MINB 4   // without spills since the work-item state lives in shared memory, but measured
#endif                   // 141 vs 130.5 us (the 48-register schedule loses the loads' overlap)
constexpr int BK3 = BC * kSegMax;  // pixels per work item (<= BC segments of <= kSegMax pixels)

template <bool HUTCH>
struct BrickSmem3T {
    float2 vb[BH3];         // v brick + halo
    int accr[BH3];          // fixed-point adjoint accumulator (re)
    int acci[BH3];          // (im)
#if FSLD_V3_FULLW
    float2 bval[RB3];       // pass 1 -> 2: conj(f) r
    float4 bgeo[RB3];       // pass 1 -> 2: the footprint as read from the table (fp32 weights, corner index)
#else
    uint4 brec[RB3];        // pass 1 -> 2: conj(f) r (2 x fp32) + the packed footprint (geo_pack)
#endif
    int acch[HUTCH ? BH3 : 1];            // fixed-point Hutchinson accumulator
    float hval[HUTCH ? RB3 : 1];          // pass 1 -> 2: h = |f|^2 P z
    unsigned char zs[HUTCH ? BH3 : 1];    // the probe's sign bit per brick voxel (staged)
    unsigned char zc[HUTCH ? BH3 : 1];    // corner sign masks (bit c = z at corner c of floor voxel l)
    int hmax2[HUTCH ? 2 : 1];
    unsigned char bk[BK3];  // item pixel -> segment
    PairRec prec[BC];       // the item's pair records (gofs, count)
    long long sg[BC];       // segment start rebased to the item's flat pixel index: gofs - pref
    int pref[BC + 1];       // exclusive prefix of segment lengths
    // work items: the current one, the next, and the one after (claimed one item ahead) -- in shared
    // memory rather than registers (uniform per CTA, read a few times per item); ring_geo = (ox, oy,
    // oz, lim bits) of the brick, computed once by the claimer
    int4 ring_desc[3], ring_geo[3];
    int vmax2[2];           // round maximum |conj(f) r| bits, by round parity
    int wtot[BC / 32];
    double red[BW];
};
using BrickSmem3 = BrickSmem3T<false>;

// The footprint in 8 bytes for the pass-1 -> pass-2 buffer: corner index (10 bits) and the three
// weights as 18-bit fixed point (round to nearest; |error| <= 2^-19 on the adjoint's weights).
__device__ __forceinline__ uint32_t q18(float w) {
    const uint32_t q = (uint32_t)(__float_as_int(fmaf(w, 262144.0f, kMagic)) - kMagicBits);
    return min(q, 262143u);
}
__device__ __forceinline__ uint2 geo_pack(float4 g) {
    const uint32_t qx = q18(g.x), qy = q18(g.y), qz = q18(g.z);
    return make_uint2((uint32_t)__float_as_int(g.w) | (qx << 10) | (qy << 28), (qy >> 4) | (qz << 14));
}
__device__ __forceinline__ float w18(uint32_t q) { return __int_as_float(0x3F800000u | (q << 5)) - 1.0f; }

// L2 prefetch of [p, p + bytes) (TMA bulk prefetch: 16-byte granules, rounded outwards; the
// callers' arrays carry >= 16 bytes of slack past their end).
__device__ __forceinline__ void l2_prefetch(const void* p, size_t bytes) {
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
    const uintptr_t a1 = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((uint32_t)(a1 - a0)) : "memory");
}

struct Pix3 {  // one pixel's inputs in registers
    float2 x, f;
    float4 geo;  // wx, wy, wz, l0 (int bits)
};

__device__ __forceinline__ void load_pix3(const SortedArgs& a, const float2* tf, const float4* tg, long long g,
                                          bool has_x, Pix3& p) {
#ifdef FSLD_EXP_NO_LOADS  // ablation (results wrong by construction): no pixel stream from HBM
    const float t = (float)(g & 1023) * 1e-3f;
    p.f = make_float2(t, 1.f - t);
    p.geo = make_float4(t, 0.5f * t, 1.f - t, __int_as_float((int)(g & 511)));
    p.x = make_float2(t, t);
#elif defined(FSLD_EXP_NO_GEO2)  // ablation (results wrong): footprint not loaded, the real corner index
    // from f.x's bits (copied there once by exp_l0_into_f_kernel): realistic bank patterns, 16 B / pixel
    p.f = __ldg(tf + g);
    const float t = (float)(g & 1023) * 1e-3f;
    p.geo = make_float4(t, 0.5f * t, 1.f - t, p.f.x);
    p.x = has_x ? __ldg(a.xs + g) : make_float2(0.f, 0.f);
#elif defined(FSLD_EXP_NO_F)  // ablation (results wrong): f not loaded
    const float t = (float)(g & 1023) * 1e-3f;
    p.f = make_float2(t, 1.f - t);
    p.geo = __ldg(tg + g);
    p.x = has_x ? __ldg(a.xs + g) : make_float2(0.f, 0.f);
#else
    p.f = __ldg(tf + g);
    p.geo = __ldg(tg + g);
    p.x = has_x ? __ldg(a.xs + g) : make_float2(0.f, 0.f);
#endif
}

// Per work item (brick, <= BC image segments), as sorted_loss_grad_kernel; per round of RB3 pixels:
//   pass 1: image value + PixTab, 8-corner gather from the smem brick, r = f P v - x, |r|^2,
//           conj(f) r and the packed footprint -> brec (the next pixel's loads in flight);
//   pass 2: fixed-point scatter of val * w (item scale, power of two, non-increasing).
// NN: nearest-neighbour slicing (kernels.py:180-190, 233-248): one gather and one complex scatter
// (two ATOMS) per pixel at the nn voxel the table holds.
// HUTCH (trilinear): the k = 1 Rademacher probe rides along (optim.py:210-229 numerator): P z from
// the corner signs of the staged probe bits, h = |f|^2 P z, 8 more fixed-point shared adds, and
// fold_j += z_j (sum P^* C^2 P z)_j at the flush.
// DET (deterministic mode, trilinear, no probe): the item's int32 sums go to the int64 fixed-point
// accumulator at the caller's scale *a.fxp (exact power-of-two shifts, order-free RED.ADD.64), and
// the loss is summed per item (a.part[item index], the items in brick order) -- bitwise the same
// for any grid, any claim order and any batch order.
// GATHER: the projection pass alone -- sum |f P v - x|^2 over the work items (optim.py:193-207, the
// batch_loss data term; the full-dataset loss of each optim.run epoch), no round buffer, no scatter,
// no flush; an item's pixels in one sweep.
// DIAG: the exact Hessian diagonal's data term, fold_j += sum_p C_p^2 w_pj^2 (kernels.py:251-294,
// hessian.py:62-107): no volume, no gathers, no images -- |f|^2 from the table and the squared
// footprint weights scattered into the real fixed-point accumulator: a.fold (fp32), or with DET
// int64 at the scale *a.fxp like the deterministic gradient.
template <bool NN, bool HUTCH, bool DET, bool GATHER = false, bool DIAG = false>
__global__ void __launch_bounds__(BTHREADS, (HUTCH || DIAG) ? 4 : FSLD_V3_MINB) brick_loss_grad_kernel(SortedArgs a) {
    static_assert(!(NN && HUTCH), "the fused probe is trilinear only");
    static_assert(!(DET && (NN || HUTCH)), "deterministic mode: trilinear loss+grad");
    static_assert(!(GATHER && (HUTCH || DET)), "the gather-only pass carries no probe and no fixed point");
    static_assert(!(DIAG && (NN || HUTCH || GATHER)), "the exact diagonal is its own trilinear pass");
    constexpr bool RACC = HUTCH || DIAG;  // the real accumulator (probe fold / diagonal)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BrickSmem3T<RACC>& S = *reinterpret_cast<BrickSmem3T<RACC>*>(smem_raw);
    a.pairs += a.ctl[3];
    a.items += a.ctl[4];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int M = a.M, c = a.c, nb = a.nb;
    const bool has_x = !DIAG && a.xs != nullptr;
    const float2* tf = tab_f(a.ptab);
    const float4* tg = tab_geo(a.ptab, reinterpret_cast<const TabHeader*>(a.ptab)->npx);
    double lsum = 0.0;
    int rpar = 0;  // round parity counter (continues across items)
    // brick voxel l = threadIdx.x + u * BTHREADS as (lx | ly << 4 | lz << 8), or -1 past the brick
    // (recomputed where used: no long-lived registers)
    auto lxyz = [](int u) -> int {
        const int l = (int)threadIdx.x + u * BTHREADS;
        return l < BH3 ? (l % BH) | (((l / BH) % BH) << 4) | ((l / (BH * BH)) << 8) : -1;
    };
#pragma unroll
    for (int u = 0; u < BU; ++u) {
        const int l = threadIdx.x + u * BTHREADS;
        if (l < BH3) {
            S.accr[l] = 0;
            S.acci[l] = 0;
            if (RACC) S.acch[l] = 0;
        }
    }
    constexpr int kClaimer = BTHREADS - 32;
    const int n_items = a.ctl[0];
    auto claim = [&](int4& geo) -> int4 {  // (w = the item's index; geo = brick origin and fixed-point bound)
        const int it = atomicAdd(a.ctl + 1, 1);
        if (it >= n_items) return make_int4(-1, 0, 0, 0);
        int4 r = a.items[it];
        r.w = it;
        const int bid = r.x;
        geo = make_int4(-c + BT * (bid % nb), -c + BT * ((bid / nb) % nb), -c + BT * (bid / (nb * nb)),
                        __float_as_int(fixed_lim<NN>(r.z)));
        return r;
    };
    // lin_index(ox + lx, oy + ly, oz + lz) (kernels.py:63-66), or -1 off the grid
    auto voxel_j = [&](const int4& geo, int u) -> int {
        const int lx = lxyz(u) & 15, ly = (lxyz(u) >> 4) & 15, lz = lxyz(u) >> 8;
        if (lx >= M - c - geo.x || ly >= M - c - geo.y || lz >= M - c - geo.z) return -1;
        const int kz = geo.z + lz;
        return ((kz < 0 ? kz + M : kz) * M + geo.y + ly + c) * M + geo.x + lx + c;
    };
    // deterministic mode: exponent of the int64 fixed-point scale (a power of two)
    const int efx = DET ? (int)((__double_as_longlong(*a.fxp) >> 52) & 0x7ff) - 1023 : 0;
    auto stage_item3 = [&](int slot) {  // pair records + v brick (+ halo, zero off the grid), async
        const int4 item = S.ring_desc[slot], geo = S.ring_geo[slot];
        for (int k = threadIdx.x; k < item.z; k += BTHREADS) cp_async16(S.prec + k, a.pairs + item.y + k);
#pragma unroll
        for (int u = 0; u < BU; ++u) {
            if (lxyz(u) < 0) continue;
            const int l = threadIdx.x + u * BTHREADS;
            const int jv = voxel_j(geo, u);
            const bool in = jv >= 0;
            const int j = in ? jv : 0;
            if (!DIAG) cp_async8_zfill(S.vb + l, a.v + j, in);
            if (HUTCH) S.zs[l] = in ? (unsigned char)(__ldg(a.zbits + j) & 1u) : 0;
        }
    };
    if (threadIdx.x == kClaimer) {
        S.ring_desc[0] = claim(S.ring_geo[0]);
        S.ring_desc[1] = claim(S.ring_geo[1]);
    }
    if (threadIdx.x < 2) {
        S.vmax2[threadIdx.x] = 0;
        if (RACC) S.hmax2[threadIdx.x] = 0;
    }
    __syncthreads();
    int cur = 0;  // ring slot of the current item
    if (S.ring_desc[0].x >= 0) stage_item3(0);
    bool init_seen = !a.fuse;  // (fused step) every CTA's slice of acc = lam v is written
    bool init_done = !a.fuse;  // this CTA's slice is written
    // this CTA's slice of acc = lam v, ||v||^2 partial; then count the slice as written -- before the
    // first item (writing it just before the CTA's first flush instead, overlapped with the other
    // CTAs' first items, measured 0.1445 vs 0.136 ms per step: the first flushes then wait longer)
    auto fused_init = [&]() {
        const int64_t n = (int64_t)M * M * M;
        const int64_t lo = n * blockIdx.x / gridDim.x, hi = n * (blockIdx.x + 1) / gridDim.x;
        double s2 = 0.0;
        for (int64_t j = lo + threadIdx.x; j < hi; j += BTHREADS) {
            const float2 w = __ldg(a.v + j);
            a.acc[j] = make_float2(a.flam * w.x, a.flam * w.y);
            s2 += (double)fmaf(w.x, w.x, w.y * w.y);
        }
        for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        if (lane == 0) S.red[warp] = s2;
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < BW; ++w) t += S.red[w];
            a.fnorm[blockIdx.x] = t;
            atomicAdd(a.ctl + 6, 1);
        }
        __syncthreads();  // (S.red is free again)
        init_done = true;
    };
    if (!init_done) fused_init();

    for (;;) {
        if (S.ring_desc[cur].x < 0) break;
        cp_async_wait_all();
        __syncthreads();  // (A) this item's pair records and v brick are in shared memory
        const int nxs = cur == 2 ? 0 : cur + 1;  // ring slot of the next item
        const int nseg = S.ring_desc[cur].z;
        if (warp < BC / 32) {  // segment-length prefix
            const int k = threadIdx.x;
            const int len = k < nseg ? S.prec[k].count : 0;
            int incl = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            S.pref[k] = incl - len;
            if (lane == 31) S.wtot[warp] = incl;
        }
        if (HUTCH) {  // corner sign masks (x fastest: 000,100,010,110,001,101,011,111) of the floor voxels
#pragma unroll
            for (int u = 0; u < BU; ++u) {
                if (lxyz(u) < 0) continue;
                const int l = threadIdx.x + u * BTHREADS;
                unsigned m = S.zs[l];
                if ((lxyz(u) & 15) < BT && ((lxyz(u) >> 4) & 15) < BT && (lxyz(u) >> 8) < BT)
                    m |= (unsigned)S.zs[l + 1] << 1 | (unsigned)S.zs[l + BH] << 2 | (unsigned)S.zs[l + BH + 1] << 3 |
                         (unsigned)S.zs[l + BH * BH] << 4 | (unsigned)S.zs[l + BH * BH + 1] << 5 |
                         (unsigned)S.zs[l + BH * BH + BH] << 6 | (unsigned)S.zs[l + BH * BH + BH + 1] << 7;
                S.zc[l] = (unsigned char)m;
            }
        }
        __syncthreads();  // (B)
        if (threadIdx.x == kClaimer) {  // the item after the next one, into the finished item's slot
            const int s2 = nxs == 2 ? 0 : nxs + 1;
            S.ring_desc[s2] = claim(S.ring_geo[s2]);
        }
        if (threadIdx.x < nseg) {
            const int k = threadIdx.x;
            int p = S.pref[k];
            for (int w = 0; w < (k >> 5); ++w) p += S.wtot[w];
            S.pref[k] = p;
            S.sg[k] = S.prec[k].gofs - p;
        }
        if (threadIdx.x == 0) {
            int t = 0;
            for (int w = 0; w < BC / 32; ++w) t += S.wtot[w];
            S.pref[nseg] = t;
        }
        __syncthreads();
        {  // item pixel -> segment table: SEG_T threads per segment
            const int k = threadIdx.x / SEG_T, q = threadIdx.x % SEG_T;
            if (k < nseg)
                for (int e = S.pref[k] + q; e < S.pref[k + 1]; e += SEG_T) S.bk[e] = (unsigned char)k;
        }
        __syncthreads();
        const int total = S.pref[nseg];
#ifdef FSLD_EXP_LIM_DIV  // experiment: a looser fixed-point scale (precision headroom of an a-priori bound)
        const float lim = __int_as_float(S.ring_geo[cur].w) * (1.0f / FSLD_EXP_LIM_DIV);
#else
        const float lim = __int_as_float(S.ring_geo[cur].w);
#endif
        double item_lsum = 0.0;  // (DET: the item's loss partial)
        float item_sc = 0.f, item_inv_sc = 1.f, item_sch = 0.f, item_inv_sch = 1.f;
        // this thread's first pixel of the item (register buffers A / B alternate: no moves of
        // in-flight load destinations, so a load is waited for only where its pixel is computed)
        Pix3 pa, pb;
        bool next_in_b = false;  // the next round's first pixel was loaded into pb
        if ((int)threadIdx.x < total) load_pix3(a, tf, tg, S.sg[S.bk[threadIdx.x]] + threadIdx.x, has_x, pa);
        for (int r0 = 0; r0 < total; r0 += (GATHER ? total : RB3), ++rpar) {
            const int r1 = GATHER ? total : min(r0 + RB3, total);
            const int par = rpar & 1;
            // ---------------- pass 1 (flattened over the round; the next pixel's loads in flight)
            float vmax = 0.f, hmax = 0.f, sq = 0.f;
            auto compute = [&](const Pix3& cur, int e) {
                const float wx = cur.geo.x, wy = cur.geo.y, wz = cur.geo.z;
                const int l0 = __float_as_int(cur.geo.w);
                const float ax = 1.f - wx, ay = 1.f - wy, az = 1.f - wz;
                const float2 f = cur.f;
                if constexpr (DIAG) {  // |f|^2 = C^2 (the phase has modulus 1) and the footprint
                    const float h = fmaf(f.x, f.x, f.y * f.y);
                    S.hval[e - r0] = h;
                    hmax = fmaxf(hmax, h);
#if FSLD_V3_FULLW
                    S.bgeo[e - r0] = cur.geo;
#else
                    const uint2 gp = geo_pack(cur.geo);
                    S.brec[e - r0] = make_uint4(0u, 0u, gp.x, gp.y);
#endif
                    return;
                }
                const float2* vb = S.vb + l0;
                float2 pv;
                if (NN) {
                    pv = vb[0];
                } else {
                    const float2 WX = make_float2(wx, wx), AX = make_float2(ax, ax);
#ifdef FSLD_EXP_ONE_GATHER  // ablation (results wrong by construction): one corner gather per pixel
                    const float2 g0 = vb[0];
                    const float2 e0 = __ffma2_rn(WX, g0, __fmul2_rn(AX, g0));
                    const float2 e1 = __fmul2_rn(AX, e0), e2 = __fmul2_rn(WX, e0), e3 = __fmul2_rn(WX, e1);
#else
                    const float2 e0 = __ffma2_rn(WX, vb[1], __fmul2_rn(AX, vb[0]));
                    const float2 e1 = __ffma2_rn(WX, vb[BH + 1], __fmul2_rn(AX, vb[BH]));
                    const float2 e2 = __ffma2_rn(WX, vb[BH * BH + 1], __fmul2_rn(AX, vb[BH * BH]));
                    const float2 e3 = __ffma2_rn(WX, vb[BH * BH + BH + 1], __fmul2_rn(AX, vb[BH * BH + BH]));
#endif
                    const float2 q0 = __ffma2_rn(make_float2(wy, wy), e1, __fmul2_rn(make_float2(ay, ay), e0));
                    const float2 q1 = __ffma2_rn(make_float2(wy, wy), e3, __fmul2_rn(make_float2(ay, ay), e2));
                    pv = __ffma2_rn(make_float2(wz, wz), q1, __fmul2_rn(make_float2(az, az), q0));
                }
                const float2 prj = cmul(pv, f);
                const float2 rr = make_float2(prj.x - cur.x.x, prj.y - cur.x.y);
                sq = fmaf(rr.x, rr.x, fmaf(rr.y, rr.y, sq));
                if constexpr (GATHER) return;
                const float2 val = cmulconj(f, rr);
                vmax = fmaxf(vmax, fmaxf(fabsf(val.x), fabsf(val.y)));
#if FSLD_V3_FULLW
                S.bval[e - r0] = val;
                S.bgeo[e - r0] = cur.geo;
#else
                const uint2 gp = geo_pack(cur.geo);
                S.brec[e - r0] = make_uint4(__float_as_uint(val.x), __float_as_uint(val.y), gp.x, gp.y);
#endif
                if (HUTCH) {  // P z in the same nested order, z = +-1 from the corner sign bits
                    const unsigned m = S.zc[l0];
                    auto zf = [m](int b) { return __int_as_float(0xBF800000u ^ (((m >> b) & 1u) << 31)); };
                    const float z0 = ax * zf(0) + wx * zf(1), z1 = ax * zf(2) + wx * zf(3);
                    const float z2 = ax * zf(4) + wx * zf(5), z3 = ax * zf(6) + wx * zf(7);
                    const float pz = az * (ay * z0 + wy * z1) + wz * (ay * z2 + wy * z3);
                    const float h = fmaf(f.x, f.x, f.y * f.y) * pz;
                    S.hval[e - r0] = h;
                    hmax = fmaxf(hmax, fabsf(h));
                }
            };
            // target of the load issued before computing pixel e: the thread's next pixel of this
            // round, else its first pixel of the next round
            auto next_of = [&](int e) { return e + BTHREADS < r1 ? e + BTHREADS : (r1 < total ? r1 + (int)threadIdx.x : total); };
            if (next_in_b) pa = pb;  // (arrived during the previous round's pass 2)
            for (int e = r0 + threadIdx.x; e < r1;) {
                const int n1 = next_of(e);
                if (n1 < total) load_pix3(a, tf, tg, S.sg[S.bk[n1]] + n1, has_x, pb);
                compute(pa, e);
                if (e + BTHREADS >= r1) {
                    next_in_b = true;
                    break;
                }
                e += BTHREADS;
                const int n2 = next_of(e);
                if (n2 < total) load_pix3(a, tf, tg, S.sg[S.bk[n2]] + n2, has_x, pa);
                compute(pb, e);
                next_in_b = false;
                e += BTHREADS;
            }
            if (DET) item_lsum += (double)sq;
            else lsum += (double)sq;
            {
                const int vb_max = __reduce_max_sync(0xffffffffu, __float_as_int(vmax));
                if (lane == 0) atomicMax(&S.vmax2[par], vb_max);
                if (RACC) {
                    const int hb_max = __reduce_max_sync(0xffffffffu, __float_as_int(hmax));
                    if (lane == 0) atomicMax(&S.hmax2[par], hb_max);
                }
            }
            __syncthreads();
            if (r1 >= total && S.ring_desc[nxs].x >= 0) stage_item3(nxs);  // overlaps pass 2 + flush
            if constexpr (GATHER) continue;
            // ---------------- pass 2: fixed-point adjoint scatter (kernels.py:221-230)
            {
                // one power-of-two scale per item and accumulator, non-increasing over its rounds: a
                // round that needs a smaller one first shifts the partial sums down (rounded)
                auto shift_down = [&](int sh, int* acc_a, int* acc_b) {
#pragma unroll
                    for (int u = 0; u < BU; ++u) {
                        if (lxyz(u) < 0) continue;
                        const int l = threadIdx.x + u * BTHREADS;
                        if (sh >= 31) {
                            acc_a[l] = 0;
                            if (acc_b) acc_b[l] = 0;
                        } else {
                            const long long half = 1ll << (sh - 1);
                            acc_a[l] = (int)(((long long)acc_a[l] + half) >> sh);
                            if (acc_b) acc_b[l] = (int)(((long long)acc_b[l] + half) >> sh);
                        }
                    }
                };
                bool sync = false;
                float inv_r;
                const float sc_r = pow2_scale(lim, __int_as_float(S.vmax2[par]), inv_r);
                if (r0 == 0) {
                    item_sc = sc_r;
                    item_inv_sc = inv_r;
                } else if (sc_r < item_sc) {
                    shift_down((__float_as_int(item_sc) - __float_as_int(sc_r)) >> 23, S.accr, S.acci);
                    item_sc = sc_r;
                    item_inv_sc = inv_r;
                    sync = true;
                }
                if (RACC) {
                    float inv_h;
                    const float sh_r = pow2_scale(lim, __int_as_float(S.hmax2[par]), inv_h);
                    if (r0 == 0) {
                        item_sch = sh_r;
                        item_inv_sch = inv_h;
                    } else if (sh_r < item_sch) {
                        shift_down((__float_as_int(item_sch) - __float_as_int(sh_r)) >> 23, S.acch, nullptr);
                        item_sch = sh_r;
                        item_inv_sch = inv_h;
                        sync = true;
                    }
                }
                if (sync) __syncthreads();  // (uniform: every thread read the same maxima)
            }
            const float sc = item_sc;
#ifdef FSLD_EXP_NO_PASS2  // ablation (results wrong by construction): no pass 2
            const int rn = 0;
#else
            const int rn = r1 - r0;
#endif
            for (int e = threadIdx.x; e < rn; e += BTHREADS) {
#if FSLD_V3_FULLW
                const float4 gq = S.bgeo[e];
                const int l0 = __float_as_int(gq.w);
                const float2 val = __fmul2_rn(S.bval[e], make_float2(sc, sc));
                const float wx = gq.x, wy = gq.y, wz = gq.z;
#else
                const uint4 rec = S.brec[e];
                const int l0 = (int)(rec.z & 1023u);
                const float wx = w18((rec.z >> 10) & 262143u);
                const float wy = w18(__funnelshift_r(rec.z, rec.w, 28) & 262143u);
                const float wz = w18(rec.w >> 14);
                const float2 val = __fmul2_rn(make_float2(__uint_as_float(rec.x), __uint_as_float(rec.y)), make_float2(sc, sc));
#endif
                if (NN) {  // one complex contribution at the nn voxel
#if FSLD_V3_F2I
                    atomicAdd(S.accr + l0, __float2int_rn(val.x));
                    atomicAdd(S.acci + l0, __float2int_rn(val.y));
#else
                    const float2 y = __fadd2_rn(val, make_float2(kMagic, kMagic));
                    atomicAdd(S.accr + l0, __float_as_int(y.x) - kMagicBits);
                    atomicAdd(S.acci + l0, __float_as_int(y.y) - kMagicBits);
#endif
                    continue;
                }
                const float ax = 1.f - wx, ay = 1.f - wy, az = 1.f - wz;
                // the 8 corner weights as packed products (bitwise the scalar ones)
                const float2 AW = make_float2(ax, wx), YW = make_float2(ay, wy);
                const float2 z0 = __fmul2_rn(make_float2(az, az), YW), z1 = __fmul2_rn(make_float2(wz, wz), YW);
                const float2 w01 = __fmul2_rn(make_float2(z0.x, z0.x), AW), w23 = __fmul2_rn(make_float2(z0.y, z0.y), AW);
                const float2 w45 = __fmul2_rn(make_float2(z1.x, z1.x), AW), w67 = __fmul2_rn(make_float2(z1.y, z1.y), AW);
                const float w8[8] = {w01.x, w01.y, w23.x, w23.y, w45.x, w45.y, w67.x, w67.y};
                const int off8[8] = {0, 1, BH, BH + 1, BH * BH, BH * BH + 1, BH * BH + BH, BH * BH + BH + 1};
                if constexpr (DIAG) {  // C^2 w^2 per corner
                    const float h = S.hval[e] * item_sch;
#pragma unroll
                    for (int q = 0; q < 8; ++q) atomicAdd(S.acch + l0 + off8[q], __float2int_rn(w8[q] * w8[q] * h));
                }
#pragma unroll
                for (int q = 0; q < (DIAG ? 0 : 8); ++q) {
#if FSLD_V3_F2I
                    const float2 y = __fmul2_rn(make_float2(w8[q], w8[q]), val);
                    const int qr = __float2int_rn(y.x), qi = __float2int_rn(y.y);
#else
                    const float2 y = __ffma2_rn(make_float2(w8[q], w8[q]), val, make_float2(kMagic, kMagic));
                    const int qr = __float_as_int(y.x) - kMagicBits, qi = __float_as_int(y.y) - kMagicBits;
#endif
#ifdef FSLD_EXP_NO_ATOMS  // ablation (results wrong by construction): one shared add per pixel
                    if (q == 0) atomicAdd(S.accr + l0, qr ^ qi);
#else
                    atomicAdd(S.accr + l0 + off8[q], qr);
                    atomicAdd(S.acci + l0 + off8[q], qi);
#endif
                }
                if (HUTCH) {
                    const float h = S.hval[e] * item_sch;
#pragma unroll
                    for (int q = 0; q < 8; ++q)
#if FSLD_V3_F2I
                        atomicAdd(S.acch + l0 + off8[q], __float2int_rn(w8[q] * h));
#else
                        atomicAdd(S.acch + l0 + off8[q], __float_as_int(fmaf(w8[q], h, kMagic)) - kMagicBits);
#endif
                }
            }
            if (threadIdx.x == 0) {  // the next round's slots (unused since this round's barrier)
                S.vmax2[par ^ 1] = 0;
                if (RACC) S.hmax2[par ^ 1] = 0;
            }
            __syncthreads();
        }
        if (!init_seen) {  // (fused step) every CTA's slice of acc = lam v is in place before the first add
            if (!init_done) fused_init();
            if (threadIdx.x == 0)
                while (*reinterpret_cast<volatile int*>(a.ctl + 6) < (int)gridDim.x) __nanosleep(64);
            __syncthreads();
            __threadfence();
            init_seen = true;
        }
        if (DET) {  // the item's loss partial, in a fixed order
            for (int o = 16; o > 0; o >>= 1) item_lsum += __shfl_xor_sync(0xffffffffu, item_lsum, o);
            if (lane == 0) S.red[warp] = item_lsum;
            __syncthreads();
            if (threadIdx.x == 0) {
                double t = 0.0;
                for (int w = 0; w < BW; ++w) t += S.red[w];
                a.part[S.ring_desc[cur].w] = t;
            }
        }
        // item value q at scale 2^esc -> q * 2^(efx - esc) at the deterministic scale (exact left
        // shift; a right shift rounds, for items whose values are below the scale's resolution)
        const int dsh = DET ? efx - (((__float_as_int(DIAG ? item_sch : item_sc) >> 23) & 0xff) - 127) : 0;
        auto to_fixed = [dsh](int q) -> unsigned long long {
            long long r;
            if (dsh >= 0) r = (long long)q << min(dsh, 62);
            else if (dsh > -63) r = ((long long)q + (1ll << ((-dsh - 1) & 63))) >> ((-dsh) & 63);
            else r = 0;
            return (unsigned long long)r;
        };
        // flush of the item: one reduction per touched voxel, accumulators re-zeroed
        const int4 igeo = S.ring_geo[cur];
#pragma unroll
        for (int u = 0; u < (GATHER ? 0 : BU); ++u) {
            if (lxyz(u) < 0) continue;
            const int l = threadIdx.x + u * BTHREADS;
            const int qr = S.accr[l], qi = S.acci[l];
            const int qh = RACC ? S.acch[l] : 0;
            if ((qr | qi | qh) == 0) continue;
            S.accr[l] = 0;
            S.acci[l] = 0;
            if (RACC) S.acch[l] = 0;
            const int jv = voxel_j(igeo, u);
            if (jv < 0) continue;
            const size_t j = (size_t)jv;
            if (DET) {
                unsigned long long* q64 = reinterpret_cast<unsigned long long*>(a.acc) + 2 * j;
                if (qr) atomicAdd(q64, to_fixed(qr));
                if (qi) atomicAdd(q64 + 1, to_fixed(qi));
            } else if ((qr | qi) != 0) {
                const float fs = item_inv_sc * a.out_scale;
                if (a.mc) red_mc_f32x2(reinterpret_cast<float*>(a.acc) + 2 * j, (float)qr * fs, (float)qi * fs);
                else red_f32x2(reinterpret_cast<float*>(a.acc) + 2 * j, (float)qr * fs, (float)qi * fs);
            }
            if (DIAG && DET) atomicAdd(reinterpret_cast<unsigned long long*>(a.fold) + j, to_fixed(qh));
            else if (DIAG) atomicAdd(a.fold + j, (float)qh * item_inv_sch);  // diag_j += sum C^2 w^2
            if (HUTCH && qh != 0) {  // fold_j += z_j h_j
                const float hz = (S.zc[l] & 1u) ? (float)qh * item_inv_sch : -(float)qh * item_inv_sch;
                atomicAdd(a.fold + j, hz);
            }
        }
        cur = nxs;
    }
    if (!init_done) fused_init();  // (fused step, a CTA that got no item)
    if constexpr (!DET) {  // (deterministic mode: the loss partials are per item, a.part[item index])
        for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
        if (lane == 0) S.red[warp] = lsum;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
            for (int w = 0; w < BW; ++w) s += S.red[w];
            a.part[blockIdx.x] = s;
        }
        if (a.fuse) {  // the last CTA: sq and the loss in a fixed order, counters re-armed for the next step
            __shared__ bool last;
            if (threadIdx.x == 0) {
                __threadfence();
                last = atomicAdd(a.ctl + 7, 1) == (int)gridDim.x - 1;
            }
            __syncthreads();
            if (last && warp == 0) {
                __threadfence();
                double q = 0.0, v2 = 0.0;
                for (int b = lane; b < (int)gridDim.x; b += 32) {
                    q += reinterpret_cast<volatile double*>(a.part)[b];
                    v2 += reinterpret_cast<volatile double*>(a.fnorm)[b];
                }
                for (int o = 16; o > 0; o >>= 1) {
                    q += __shfl_xor_sync(0xffffffffu, q, o);
                    v2 += __shfl_xor_sync(0xffffffffu, v2, o);
                }
                if (lane == 0) {
                    *a.fsq = q;
                    *a.floss = 0.5 * a.fscale * q + 0.5 * (double)a.flam * v2;
                    a.ctl[6] = 0;
                    a.ctl[7] = 0;
                }
            }
        }
    }
}
