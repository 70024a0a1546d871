// fsld_brick_main.cuh -- the work-item kernel of the brick-sorted loss+gradient path
// (included by fsld_brick.cu; see the design note there).
#pragma once

// float -> int32 round-to-nearest for |x| < 2^22 via the 1.5*2^23 magic (FFMA + IADD, no F2I).
constexpr float kMagic = 12582912.0f;
constexpr int kMagicBits = 0x4B400000;

// FSLD_V3_FULLW (default): the pass-1 -> pass-2 buffer of the table-driven kernel keeps the fp32
// footprint as read from the table, and both brick kernels round their scatter with cvt.rni (F2I) at
// a scale bounded by the per-voxel weight sum (fixed_lim) -- 6.6x lower gradient error at cfg3
// (tools/prec_probe.py); 0: the round-1 18-bit packed weights and the 1.5 * 2^23 magic-number
// rounding (|q| < 2^22).
#ifndef FSLD_V3_FULLW
#define FSLD_V3_FULLW 1
#endif
#ifndef FSLD_V3_F2I  // the cvt.rni rounding and the weight-sum bound (independent of the buffer layout;
#define FSLD_V3_F2I 1  // measured: either change alone already needs > 48 registers, i.e. 4 CTAs/SM)
#endif
// Fixed-point bound of an item of nseg segments: the largest |contribution| after scaling.  FULLW:
// one image's pixels put a trilinear weight sum of at most 1.28 on any voxel (measured over 2e5 random
// poses and offsets; bound 2 used) and at most 3 pixels share an nn voxel (bound 4), so a voxel's
// item total stays below 2^31 with lim = 2^31 / (bound * nseg), capped at 2^30 for cvt.rni.
// Round 1: |q| < 2^22 for the magic-number rounding and 12 contributions per voxel and segment.
template <bool NN>
__device__ __forceinline__ float fixed_lim(int nseg) {
#if FSLD_V3_F2I
    return __fdiv_rn(NN ? 536870912.0f : 1073741824.0f, (float)nseg);
#else
    return (float)min(4194303, 178956970 / nseg);
#endif
}

// Ablation builds (tools/build_exp.sh <name> -DFSLD_EXP_...; never defined in the product build)
// remove one part of the work at a time to measure its share: FSLD_EXP_NO_ATOMS (pass-2 shared
// atomics), FSLD_EXP_ONE_GATHER (7 of the 8 corner gathers), FSLD_EXP_NO_XLOAD (image loads),
// FSLD_EXP_NO_PASS1, FSLD_EXP_NO_PASS2.  Results are wrong by construction.

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

constexpr int RB = 1024;                               // pixels per round (hutch / energy kernels)
// Pixels per round of the loss+grad kernel (pass 1 -> pass 2 buffer): 1,280 fills the shared memory
// of 4 CTAs/SM (fewer rounds per item: +1.3 % over 1,024); the probe-carrying variant keeps 1,024
// (its extra buffers would drop it to 3 CTAs/SM).
#ifndef FSLD_RB_MAIN
#define FSLD_RB_MAIN 1280
#endif
template <bool HUTCH>
constexpr int rb_main() { return HUTCH ? 1024 : FSLD_RB_MAIN; }
constexpr int BU = (BH3 + BTHREADS - 1) / BTHREADS;    // brick voxels per thread (3)
constexpr int SEG_T = BTHREADS / BC;                   // threads per segment in the bk build (4)
static_assert(BTHREADS % BC == 0 && BC % 32 == 0 && BC <= BTHREADS, "segment table: one scan warp per 32 segments");

template <bool HUTCH>
struct SortedSmemT {
    float2 vb[BH3];                 // v brick + halo
    int accr[BH3];                  // fixed-point adjoint accumulator of the current round (re)
    int acci[BH3];                  // (im)
    int acch[HUTCH ? BH3 : 1];      // fixed-point Hutchinson accumulator (real)
    unsigned char zc[HUTCH ? BH3 : 1];  // z signs: bit c = z at corner c of floor voxel l (bit 0 = z_l)
    float2 bval[rb_main<HUTCH>()];             // pass 1 -> 2: conj(f) r
    float4 bgeo[rb_main<HUTCH>()];             // pass 1 -> 2: (wx, wy, wz, local corner index)
    float hval[HUTCH ? rb_main<HUTCH>() : 1];  // pass 1 -> 2: C^2 P z (also z staging during setup)
    int4 segw[BC * SEG_W];          // the item's segment records (gofs rebased to the flat index), SEG_W words apart
    __device__ __forceinline__ SegRec& seg(int k) { return *reinterpret_cast<SegRec*>(segw + k * SEG_W); }
    PairRec prec[BC];               // the next item's pair records (staged first: their tslots address the templates)
    int pref[BC + 1];               // exclusive prefix of segment lengths
    unsigned char bk[rb_main<HUTCH>()];  // round pixel -> segment
    int4 item_desc;                 // first item of this CTA (prologue)
    int4 next_desc;                 // the item after the current one ((-1, ..) = none)
    int vmax_bits, hmax_bits;
    int wtot[BC / 32];                    // per-warp segment-length totals
    double red[BW];
};

// 64-bit shared load (ptxas pairs adjacent ones into LDS.128, which measured
// fewer smem wavefronts per warp than separate broadcast LDS.64: ~3.4 vs ~2.7 each).
__device__ __forceinline__ uint2 lds64(const void* p) {
    uint2 r;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];"
                 : "=r"(r.x), "=r"(r.y)
                 : "r"((uint32_t)__cvta_generic_to_shared(p)));
    return r;
}

// The per-pixel fields of a SegRec, in registers.
struct SegRegs {
    long long gofs;
    float fr[6];
    float wsin, wcos, envl;
    uint32_t gc, sc, glo[4], ghi[4], slo[2], shi[2];
};

__device__ __forceinline__ void load_seg(const SegRec& R, SegRegs& Q) {
    uint2 t = lds64(&R.gofs);
    Q.gofs = (long long)(((unsigned long long)t.y << 32) | t.x);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        t = lds64(R.frame + 2 * q);
        Q.fr[2 * q] = __uint_as_float(t.x);
        Q.fr[2 * q + 1] = __uint_as_float(t.y);
    }
    t = lds64(&R.wsin);
    Q.wsin = __uint_as_float(t.x);
    Q.wcos = __uint_as_float(t.y);
    t = lds64(&R.envl);
    Q.envl = __uint_as_float(t.x);
    Q.gc = t.y;
    Q.sc = lds64(&R.sc).x;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        t = lds64(R.glo + 2 * q);
        Q.glo[2 * q] = t.x;
        Q.glo[2 * q + 1] = t.y;
        t = lds64(R.ghi + 2 * q);
        Q.ghi[2 * q] = t.x;
        Q.ghi[2 * q + 1] = t.y;
    }
    t = lds64(R.slo);
    Q.slo[0] = t.x;
    Q.slo[1] = t.y;
    t = lds64(R.shi);
    Q.shi[0] = t.x;
    Q.shi[1] = t.y;
}

// Fixed-point scale 2^k with k = floor(log2(lim / vm)) exactly (integer exponent / mantissa
// comparison: no log2 / exp2 / division on the per-round path); inv = 2^-k.  vm = 0 -> 1.
__device__ __forceinline__ float pow2_scale(float lim, float vm, float& inv) {
    const int bl = __float_as_int(lim), bv = __float_as_int(vm);
    const int el = (bl >> 23) & 0xff, ev = (bv >> 23) & 0xff;
    if (ev == 0 || el == 0) {  // zero or denormal maximum: the slow formula
        const float sc = vm > 0.f ? exp2f(floorf(log2f(lim / vm))) : 1.0f;
        inv = 1.0f / sc;
        return sc;
    }
    int k = el - ev - ((bl & 0x7fffff) < (bv & 0x7fffff) ? 1 : 0);
    k = max(-126, min(126, k));
    inv = __int_as_float((127 - k) << 23);
    return __int_as_float((127 + k) << 23);
}

// hi32(F * u mod 2^64) for F = hi:lo (64-bit fixed-point turns), u < 2^32, wrapping
__device__ __forceinline__ uint32_t turns_term(uint32_t lo, uint32_t hi, uint32_t u) {
    return hi * u + __umulhi(lo, u);
}

// f = CTF(k) * exp(i pi shift.k) for a segment's image (fsld_common.cuh pixel_factor,
// forward.py:93-111, 299-303): both phases mod 1 turn, exactly, in 32-bit integer
// arithmetic (error < 6 * 2^-32 turn), then the fp32 sin/cos.
__device__ __forceinline__ float2 seg_factor(const SegRegs& R, int kx, int ky) {
    const int kx2 = kx * kx, ky2 = ky * ky;
    const uint32_t k2 = (uint32_t)(kx2 + ky2);
    const uint32_t c2 = (uint32_t)(kx2 - ky2 + 32768);
    const uint32_t s2 = (uint32_t)(2 * kx * ky + 65536);
    const uint32_t tg = R.gc + turns_term(R.glo[0], R.ghi[0], k2) + turns_term(R.glo[1], R.ghi[1], c2) +
                        turns_term(R.glo[2], R.ghi[2], s2) + turns_term(R.glo[3], R.ghi[3], k2 * k2);
    const uint32_t ts = R.sc + turns_term(R.slo[0], R.shi[0], (uint32_t)(kx + 128)) +
                        turns_term(R.slo[1], R.shi[1], (uint32_t)(ky + 128));
    constexpr float kTurn = 1.4629180792671596e-09f;  // 2 pi / 2^32
    float sg, cg, ss, cs;
    __sincosf((float)(int)tg * kTurn, &sg, &cg);
    __sincosf((float)(int)ts * kTurn, &ss, &cs);
    const float ctf = -(R.wsin * sg + R.wcos * cg) * exp2f(-R.envl * (float)k2);
    return make_float2(ctf * cs, ctf * ss);
}


// cp.async helpers (sm_80+ LDGSTS): 16-byte copy, and 8-byte copy with zero fill when !valid.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async8_zfill(void* dst, const void* src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(valid ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// 16-byte chunk q of the SegRec of pair p: chunk 0 from the PairRec (gofs, count), the rest from
// the image's template (synchronous version, for the kernels that stage an item in place).
__device__ __forceinline__ int4 seg_chunk(const SortedArgs& a, int p, int q) {
    const int4 pr = __ldg(reinterpret_cast<const int4*>(a.pairs + p));  // (gofs lo, gofs hi, count, tslot)
    if (q == 0) return make_int4(pr.x, pr.y, pr.z, 0);
    return __ldg(reinterpret_cast<const int4*>(a.tmpl + pr.w) + q);
}

// Stage a work item's inputs in shared memory without waiting: its segment records, the brick of
// v (+halo, zero off the grid) and, for HUTCH, the probe sign of each brick voxel (into S.bk).
// Issued for the NEXT item right after the current item's last pass 1, so the loads overlap that
// item's pass 2 and flush (none of S.seg / S.vb / S.bk is read after pass 1).
template <bool HUTCH>
__device__ __forceinline__ void stage_pairs(SortedSmemT<HUTCH>& S, const SortedArgs& a, int4 item) {
    for (int k = threadIdx.x; k < item.z; k += BTHREADS) cp_async16(S.prec + k, a.pairs + item.y + k);
}

// second stage (S.prec of `item` complete and visible): segment records = PairRec + template,
// the v brick, and for HUTCH the probe sign of each brick voxel (into S.bk)
template <bool HUTCH>
__device__ __forceinline__ void stage_item(SortedSmemT<HUTCH>& S, const SortedArgs& a, int4 item, const int* lxyz) {
    const int M = a.M, c = a.c, nb = a.nb;
    const int bid = item.x, nseg = item.z;
    const int ox = -c + BT * (bid % nb), oy = -c + BT * ((bid / nb) % nb), oz = -c + BT * (bid / (nb * nb));
    int4* dst = S.segw;
    for (int w = threadIdx.x; w < nseg * 8; w += BTHREADS) {
        const int j = w >> 3, q = w & 7;
        const PairRec& pr = S.prec[j];
        if (q == 0) dst[j * SEG_W] = make_int4((int)(unsigned)pr.gofs, (int)(pr.gofs >> 32), pr.count, 0);
        else cp_async16(dst + j * SEG_W + q, reinterpret_cast<const int4*>(a.tmpl + pr.tslot) + q);
    }
#pragma unroll
    for (int u = 0; u < BU; ++u) {
        if (lxyz[u] < 0) continue;
        const int l = threadIdx.x + u * BTHREADS;
        const int kx = ox + (lxyz[u] & 15), ky = oy + ((lxyz[u] >> 4) & 15), kz = oz + (lxyz[u] >> 8);
        const bool in = kx < M - c && ky < M - c && kz < M - c;
        const int j = in ? lin_index(kx, ky, kz, M, c) : 0;
        cp_async8_zfill(S.vb + l, a.v + j, in);
        if (HUTCH) S.bk[l] = in ? (unsigned char)(__ldg(a.zbits + j) & 1u) : 0;
    }
}

// Per work item (brick, <= BC image segments):
//   setup: claim (run ahead on one thread), the segment records (one 128-B
//          SegRec each, written by the fill pass), their prefix, the brick's
//          9^3 voxels of v (+halo, zero off the grid) [and the probe's signs];
//   rounds of <= RB pixels (flattened over the item's segments):
//     0. round pixel -> segment byte table (SEG_T threads per segment);
//     1. gather 8 corners from the smem brick, f = C * phase, r = f P v - x,
//        |r|^2 -> loss; conj(f) r and the corner geometry -> smem buffers
//        [HUTCH: h = |f|^2 P z from the corner signs -> smem buffer];
//     2. with the round's max |val| known, quantise val * w to int32 with the
//        item's power-of-two scale (|val w s| <= min(2^22, 2^31 / (12 nseg)):
//        <= 12 contributions per voxel per image; a round that needs a smaller
//        scale first shifts the partial sums down to it) and add with native
//        ATOMS.ADD [HUTCH: the same for h w into a real accumulator];
//   flush, once per item: one red.global.add.v2.f32 per touched brick voxel
//        [HUTCH: fold_j += z_j h_j, one red.global.add.f32], accumulators zeroed.
template <bool HUTCH>
__global__ void __launch_bounds__(BTHREADS, 4) sorted_loss_grad_kernel(SortedArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SortedSmemT<HUTCH>& S = *reinterpret_cast<SortedSmemT<HUTCH>*>(smem_raw);
    a.pairs += a.ctl[3];  // this batch's pairs / items (non-zero offsets in a multi-batch plan)
    a.items += a.ctl[4];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int M = a.M, c = a.c, nb = a.nb;
    const float bnd = a.bnd;
    double lsum = 0.0;  // this thread's sum of |r|^2 (fp32 within a round)
    int lxyz[BU];  // this thread's brick voxels: lx | ly << 4 | lz << 8 (or -1)
#pragma unroll
    for (int u = 0; u < BU; ++u) {
        const int l = threadIdx.x + u * BTHREADS;
        lxyz[u] = l < BH3 ? (l % BH) | (((l / BH) % BH) << 4) | ((l / (BH * BH)) << 8) : -1;
        if (l < BH3) {  // accumulators start at zero; every round's flush re-zeroes what it reads
            S.accr[l] = 0;
            S.acci[l] = 0;
            if (HUTCH) S.acch[l] = 0;
        }
    }
    // work items are claimed one ahead: the claimer thread publishes the item after the current
    // one in S.next_desc, whose inputs are staged (asynchronously) during the current item
    constexpr int kClaimer = BTHREADS - 32;
    const int n_items = a.ctl[0];
    auto claim = [&]() -> int4 {
        const int it = atomicAdd(a.ctl + 1, 1);
        return it < n_items ? a.items[it] : make_int4(-1, 0, 0, 0);
    };
    if (threadIdx.x == kClaimer) {
        S.item_desc = claim();
        S.next_desc = claim();
    }
    __syncthreads();
    int4 item = S.item_desc;
    if (item.x >= 0) {
        stage_pairs(S, a, item);
        cp_async_wait_all();
        __syncthreads();
        stage_item(S, a, item, lxyz);
    }
    PHASE_INIT();

    for (;;) {
        if (item.x < 0) break;
        cp_async_wait_all();
        __syncthreads();  // (A) this item's inputs are in shared memory
        const int4 nxt = S.next_desc;
        const int bid = item.x, nseg = item.z;
        const int ox = -c + BT * (bid % nb), oy = -c + BT * ((bid / nb) % nb), oz = -c + BT * (bid / (nb * nb));
        // ---------------- setup: segment-length prefix (warps 0, 1) [corner sign masks]
        if (warp < BC / 32) {
            const int k = threadIdx.x;
            const int len = k < nseg ? S.seg(k).count : 0;
            int incl = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            S.pref[k] = incl - len;  // warp 1 adds warp 0's total below
            if (lane == 31) S.wtot[warp] = incl;
        }
        if (HUTCH) {  // corner sign masks (x fastest: 000,100,010,110,001,101,011,111) from the staged signs
            const unsigned char* zs = S.bk;
#pragma unroll
            for (int u = 0; u < BU; ++u) {
                if (lxyz[u] < 0) continue;
                const int l = threadIdx.x + u * BTHREADS;
                unsigned m = zs[l];
                if ((lxyz[u] & 15) < BT && ((lxyz[u] >> 4) & 15) < BT && (lxyz[u] >> 8) < BT) {
                    m |= (unsigned)zs[l + 1] << 1 | (unsigned)zs[l + BH] << 2 | (unsigned)zs[l + BH + 1] << 3 |
                         (unsigned)zs[l + BH * BH] << 4 | (unsigned)zs[l + BH * BH + 1] << 5 |
                         (unsigned)zs[l + BH * BH + BH] << 6 | (unsigned)zs[l + BH * BH + BH + 1] << 7;
                }
                S.zc[l] = (unsigned char)m;
            }
        }
        __syncthreads();  // (B)
        if (threadIdx.x == kClaimer) S.next_desc = claim();  // everyone has read nxt
        if (nxt.x >= 0) stage_pairs(S, a, nxt);  // S.prec is free: this item's were consumed before (A)
        if (threadIdx.x < nseg) {  // final prefix; rebase gofs to the flat pixel index
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
        PHASE_MARK(0);
        const int total = S.pref[nseg];
        // fixed-point budget: a voxel's item total stays below 2^31 (fixed_lim)
        const float lim = fixed_lim<false>(nseg);

        // flush of a completed item: one reduction per touched voxel, accumulators re-zeroed
        auto flush_round = [&](float f_inv_sc, float f_inv_sch) {
#pragma unroll
            for (int u = 0; u < BU; ++u) {
                if (lxyz[u] < 0) continue;
                const int l = threadIdx.x + u * BTHREADS;
                const int qr = S.accr[l], qi = S.acci[l];
                const int qh = HUTCH ? S.acch[l] : 0;
                if ((qr | qi | qh) == 0) continue;
                S.accr[l] = 0;
                S.acci[l] = 0;
                if (HUTCH) S.acch[l] = 0;
                const int kx = ox + (lxyz[u] & 15), ky = oy + ((lxyz[u] >> 4) & 15), kz = oz + (lxyz[u] >> 8);
                if (kx >= M - c || ky >= M - c || kz >= M - c) continue;
                const size_t j = (size_t)lin_index(kx, ky, kz, M, c);
                if ((qr | qi) != 0) {
                    const float fs = f_inv_sc * a.out_scale;  // exact for out_scale = 1
                    red_f32x2(reinterpret_cast<float*>(a.acc) + 2 * j, (float)qr * fs, (float)qi * fs);
                }
                if (HUTCH && qh != 0) {
                    const float hz = (S.zc[l] & 1u) ? (float)qh * f_inv_sch : -(float)qh * f_inv_sch;
                    atomicAdd(a.fold + j, hz);
                }
            }
        };
        // One fixed-point scale per item, power of two and non-increasing over its rounds: a round
        // whose maximum needs a smaller scale first shifts the partial sums down (rounded) to it, so
        // the accumulators carry the whole item and are flushed once.  The overflow budget holds
        // for the whole item: <= 12 contributions per voxel per image over all of its rounds.
        float item_sc = 0.f, item_inv_sc = 1.f, item_sch = 0.f, item_inv_sch = 1.f;
        auto rescale = [&](int sh, int* acc_a, int* acc_b) {
#pragma unroll
            for (int u = 0; u < BU; ++u) {
                if (lxyz[u] < 0) continue;
                const int l = threadIdx.x + u * BTHREADS;
                if (sh >= 31) {
                    acc_a[l] = 0;
                    if (acc_b) acc_b[l] = 0;
                } else {
                    const long long half = 1ll << (sh - 1);  // rounded (64-bit: no overflow near 2^31)
                    acc_a[l] = (int)(((long long)acc_a[l] + half) >> sh);
                    if (acc_b) acc_b[l] = (int)(((long long)acc_b[l] + half) >> sh);
                }
            }
        };

        constexpr int RBK = rb_main<HUTCH>();
        for (int r0 = 0; r0 < total; r0 += RBK) {
            const int rn = min(RBK, total - r0);
            {  // round pixel -> segment table: SEG_T threads per segment
                const int k = threadIdx.x / SEG_T, q = threadIdx.x % SEG_T;
                if (k < nseg) {
                    const int e1 = min(S.pref[k + 1], r0 + rn) - r0;
                    for (int e = max(S.pref[k], r0) - r0 + q; e < e1; e += SEG_T) S.bk[e] = (unsigned char)k;
                }
            }
            if (threadIdx.x == 0) {
                S.vmax_bits = 0;
                S.hmax_bits = 0;
            }
            __syncthreads();
            PHASE_MARK(1);
            // ---------------- pass 1
            float vmax = 0.f, hmax = 0.f, sq = 0.f;
#if defined(FSLD_EXP_NO_PASS1)
            for (int e = threadIdx.x; e < rn; e += BTHREADS) {
                S.bval[e] = make_float2(1.f, 1.f);
                S.bgeo[e] = make_float4(0.5f, 0.5f, 0.5f, __int_as_float((e * 37) % 500));
                vmax = 1.f;
            }
            for (int e = threadIdx.x; e < 0; e += BTHREADS) {
#else
#pragma unroll 1
            for (int e = threadIdx.x; e < rn; e += BTHREADS) {
#endif
                SegRegs R;
#if defined(FSLD_EXP_NO_SEGREC)
                load_seg(S.seg(0), R);
                R.gofs = S.seg(S.bk[e]).gofs;
#else
                load_seg(S.seg(S.bk[e]), R);
#endif
                const long long g = R.gofs + (r0 + e);
                const char2 kk = a.pc[g];
#if defined(FSLD_EXP_NO_XLOAD)
                const float2 xv = make_float2((float)(g & 7), 0.f);
#else
                const float2 xv = a.xs ? __ldg(a.xs + g) : make_float2(0.f, 0.f);  // NULL: Hessian product
#endif
                const int px = kk.x, py = kk.y;
                float cx, cy, cz, fx, fy, fz;
                floor_corner((float)px, (float)py, R.fr, bnd, cx, cy, cz, fx, fy, fz);
                const int l0 = (((int)fz - oz) * BH + ((int)fy - oy)) * BH + ((int)fx - ox);
                const float wx = cx - fx, wy = cy - fy, wz = cz - fz;
                const float ax = 1.f - wx, ay = 1.f - wy, az = 1.f - wz;
#if defined(FSLD_EXP_NO_FACTOR)
                const float2 f = __ldg(a.xs + g + 7);
#else
                const float2 f = seg_factor(R, px, py);
#endif
                const float2* vb = S.vb + l0;
                // trilinear gather (kernels.py:171-176) from the smem brick
                const float2 WX = make_float2(wx, wx), AX = make_float2(ax, ax);
#if defined(FSLD_EXP_ONE_GATHER)
                const float2 g0 = vb[0];
                const float2 e0 = __ffma2_rn(WX, g0, __fmul2_rn(AX, g0)), e1 = __ffma2_rn(AX, g0, __fmul2_rn(WX, g0));
                const float2 e2 = __ffma2_rn(WX, e0, __fmul2_rn(AX, g0)), e3 = __ffma2_rn(AX, e1, __fmul2_rn(WX, g0));
#else
                const float2 e0 = __ffma2_rn(WX, vb[1], __fmul2_rn(AX, vb[0]));
                const float2 e1 = __ffma2_rn(WX, vb[BH + 1], __fmul2_rn(AX, vb[BH]));
                const float2 e2 = __ffma2_rn(WX, vb[BH * BH + 1], __fmul2_rn(AX, vb[BH * BH]));
                const float2 e3 = __ffma2_rn(WX, vb[BH * BH + BH + 1], __fmul2_rn(AX, vb[BH * BH + BH]));
#endif
                const float2 q0 = __ffma2_rn(make_float2(wy, wy), e1, __fmul2_rn(make_float2(ay, ay), e0));
                const float2 q1 = __ffma2_rn(make_float2(wy, wy), e3, __fmul2_rn(make_float2(ay, ay), e2));
                const float2 pv = __ffma2_rn(make_float2(wz, wz), q1, __fmul2_rn(make_float2(az, az), q0));
                const float2 prj = cmul(pv, f);
                const float2 rr = make_float2(prj.x - xv.x, prj.y - xv.y);
                sq = fmaf(rr.x, rr.x, fmaf(rr.y, rr.y, sq));
                const float2 val = cmulconj(f, rr);
                vmax = fmaxf(vmax, fmaxf(fabsf(val.x), fabsf(val.y)));
                S.bval[e] = val;
                S.bgeo[e] = make_float4(wx, wy, wz, __int_as_float(l0));
                if (HUTCH) {  // P z in the same nested order, z = +-1 from the corner sign bits
                    const unsigned m = S.zc[l0];
                    auto zf = [m](int b) { return __int_as_float(0xBF800000u ^ (((m >> b) & 1u) << 31)); };
                    const float z0 = ax * zf(0) + wx * zf(1), z1 = ax * zf(2) + wx * zf(3);
                    const float z2 = ax * zf(4) + wx * zf(5), z3 = ax * zf(6) + wx * zf(7);
                    const float pz = az * (ay * z0 + wy * z1) + wz * (ay * z2 + wy * z3);
                    const float h = fmaf(f.x, f.x, f.y * f.y) * pz;
                    S.hval[e] = h;
                    hmax = fmaxf(hmax, fabsf(h));
                }
            }
            lsum += (double)sq;
            if (r0 + RBK >= total && nxt.x >= 0) cp_async_wait_all();  // nxt's pair records (stage_pairs)
            {  // maxima >= 0, so their bit patterns order like ints
                const int vb_max = __reduce_max_sync(0xffffffffu, __float_as_int(vmax));
                if (lane == 0) atomicMax(&S.vmax_bits, vb_max);
                if (HUTCH) {
                    const int hb_max = __reduce_max_sync(0xffffffffu, __float_as_int(hmax));
                    if (lane == 0) atomicMax(&S.hmax_bits, hb_max);
                }
            }
            __syncthreads();
            PHASE_MARK(2);
            if (r0 + RBK >= total && nxt.x >= 0) stage_item(S, a, nxt, lxyz);  // overlaps pass 2 + flush
            // ---------------- pass 2: fixed-point adjoint scatter (kernels.py:221-230)
            {
                const float vm = __int_as_float(S.vmax_bits);
                float inv_r;
                const float sc_r = pow2_scale(lim, vm, inv_r);
                bool sync = false;
                if (r0 == 0 || sc_r >= item_sc) {
                    if (r0 == 0) { item_sc = sc_r; item_inv_sc = inv_r; }
                } else {  // exponent difference of two powers of two
                    rescale((__float_as_int(item_sc) - __float_as_int(sc_r)) >> 23, S.accr, S.acci);
                    item_sc = sc_r;
                    item_inv_sc = inv_r;
                    sync = true;
                }
                if (HUTCH) {
                    const float hm = __int_as_float(S.hmax_bits);
                    float inv_h;
                    const float sh_r = pow2_scale(lim, hm, inv_h);
                    if (r0 == 0) {
                        item_sch = sh_r;
                        item_inv_sch = inv_h;
                    } else if (sh_r < item_sch) {
                        rescale((__float_as_int(item_sch) - __float_as_int(sh_r)) >> 23, S.acch, nullptr);
                        item_sch = sh_r;
                        item_inv_sch = inv_h;
                        sync = true;
                    }
                }
                if (sync) __syncthreads();  // uniform: every thread read the same maxima
            }
            const float sc = item_sc, sch = item_sch;
#if defined(FSLD_EXP_NO_PASS2)
            for (int e = threadIdx.x; e < 0; e += BTHREADS) {
#else
            for (int e = threadIdx.x; e < rn; e += BTHREADS) {
#endif
                const float4 geo = S.bgeo[e];
                const int l0 = __float_as_int(geo.w);
                const float wx = geo.x, wy = geo.y, wz = geo.z;
                const float ax = 1.f - wx, ay = 1.f - wy, az = 1.f - wz;
                const float2 val = __fmul2_rn(S.bval[e], make_float2(sc, sc));
                const float zy00 = az * ay, zy10 = az * wy, zy01 = wz * ay, zy11 = wz * wy;
                const float w8[8] = {zy00 * ax, zy00 * wx, zy10 * ax, zy10 * wx, zy01 * ax, zy01 * wx, zy11 * ax, zy11 * wx};
                const int off8[8] = {0, 1, BH, BH + 1, BH * BH, BH * BH + 1, BH * BH + BH, BH * BH + BH + 1};
#if defined(FSLD_EXP_NO_ATOMS)
                int sink = 0;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float2 y = __ffma2_rn(make_float2(w8[q], w8[q]), val, make_float2(kMagic, kMagic));
                    sink += (__float_as_int(y.x) - kMagicBits) ^ (__float_as_int(y.y) - kMagicBits) ^ (l0 + off8[q]);
                }
                if (sink == 0x7fffffff) S.accr[0] = sink;
#else
#pragma unroll
                for (int q = 0; q < 8; ++q) {
#if FSLD_V3_F2I
                    const float2 y = __fmul2_rn(make_float2(w8[q], w8[q]), val);
                    atomicAdd(S.accr + l0 + off8[q], __float2int_rn(y.x));
                    atomicAdd(S.acci + l0 + off8[q], __float2int_rn(y.y));
#else
                    const float2 y = __ffma2_rn(make_float2(w8[q], w8[q]), val, make_float2(kMagic, kMagic));
                    atomicAdd(S.accr + l0 + off8[q], __float_as_int(y.x) - kMagicBits);
                    atomicAdd(S.acci + l0 + off8[q], __float_as_int(y.y) - kMagicBits);
#endif
                }
#endif
                if (HUTCH) {
                    const float h = S.hval[e] * sch;
#pragma unroll
                    for (int q = 0; q < 8; ++q)
#if FSLD_V3_F2I
                        atomicAdd(S.acch + l0 + off8[q], __float2int_rn(w8[q] * h));
#else
                        atomicAdd(S.acch + l0 + off8[q], __float_as_int(fmaf(w8[q], h, kMagic)) - kMagicBits);
#endif
                }
            }
            __syncthreads();
            PHASE_MARK(3);
        }
        flush_round(item_inv_sc, item_inv_sch);  // once per item (the next item's (A) barrier follows)
        PHASE_MARK(7);
        item = nxt;
    }
    PHASE_FLUSH();
    for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
    if (lane == 0) S.red[warp] = lsum;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < BW; ++w) s += S.red[w];
        a.part[blockIdx.x] = s;
    }
}
