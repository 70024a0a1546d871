// fsld_brick.cu -- brick-sorted fused loss+gradient path (tri mode) for sm_100a.
//
// Why: the reference's adjoint (kernels.py:193-230) scatters 8 complex corner
// contributions per pixel.  As global red.add that is 8 L2 atomics per pixel
// and the per-pixel tile kernel is L2-atomic bound (profiles/r01_v1_*).
//
// Refinement has KNOWN, FIXED poses (optim.run never changes them), so the
// pixel -> voxel footprint of every image is fixed for the whole run.  The
// dataset is therefore laid out once in HBM grouped by owner brick: for image
// i, its masked pixels are reordered so that pixels whose floor corner
// (floor(clamp(R^T k)), kernels.py:42-60, 147-170) falls in the same 8^3 brick
// are contiguous; per pixel we keep (kx, ky) as int8 (2 B) and per image a
// segment list (brick, start, count).
//
// Per step (all on device, stream-ordered; or for K batches at once in a plan):
// the batch's segments are counted per brick, scanned into work items (brick,
// <= BC segments) and filled (a 16-byte pair record per segment, a segment-
// record template per image).  A persistent CTA takes an item, stages the
// brick's 9^3 voxels of v and the item's segment records in shared memory
// (the next item's with cp.async while the current one finishes), and walks
// the item's pixels in rounds: pass 1 gathers 8 corners from shared memory,
// f = CTF * shift phase, r = f P v - x, |r|^2, and buffers conj(f) r with the
// corner geometry; pass 2 adds val * w to a shared int32 fixed-point
// accumulator (scale from the round's max, native ATOMS.ADD); each round is
// flushed with one red.global.add.v2.f32 per touched brick voxel.  Every pixel
// belongs to exactly one segment, so it is processed exactly once.
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "fsld_kernels.cuh"

namespace fsld {

ScratchLayout scratch_layout(int M, int n_mask, int B) {
    ScratchLayout L{};
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    L.nb = (M + BT - 1) / BT;
    L.nbr = L.nb * L.nb * L.nb;
    // a slice plane crosses at most ~3 nb^2 bricks; 4 nb^2 is a safe per-image bound
    long long pp = (long long)B * (long long)(L.nbr < 4 * L.nb * L.nb ? L.nbr : 4 * L.nb * L.nb);
    L.cap_pairs = (int)(pp > 0 ? pp : 1);
    L.cap_items = L.nbr + L.cap_pairs / BC + 1;
    int tiles = (n_mask + kThreads * 4 - 1) / (kThreads * 4);
    long long v1parts = (long long)(B > 0 ? B : 1) * (tiles > 0 ? tiles : 1);
    L.cap_part = (int)(3 * v1parts > 8192 ? 3 * v1parts : 8192);  // 3 columns (OP_ARMIJO)
    if (L.cap_part < L.cap_items) L.cap_part = L.cap_items;         // per-item loss partials (deterministic)
    size_t o = 0;
    L.hdr = o; o = al(o + 256);
    L.cnt = o; o = al(o + sizeof(int) * (size_t)L.nbr);
    L.off = o; o = al(o + sizeof(int) * (size_t)(L.nbr + 1));
    L.fill = o; o = al(o + sizeof(int) * (size_t)L.nbr);
    L.pairs = o; o = al(o + sizeof(PairRec) * (size_t)L.cap_pairs);
    L.tmpl = o; o = al(o + sizeof(SegRec) * (size_t)(B > 0 ? B : 1));
    L.items = o; o = al(o + sizeof(int4) * (size_t)L.cap_items);
    L.ctl = o; o = al(o + 64);
    L.part = o; o = al(o + sizeof(double) * (size_t)L.cap_part);
    L.gitems = o; o = al(o + sizeof(int4) * (size_t)L.cap_items);
    L.gctl = o; o = al(o + sizeof(int) * 16 * (size_t)kMaxSlabs);
    L.gpart = o; o = al(o + sizeof(double) * (size_t)kMaxSlabs * kSlabCtas);
    L.npart = o; o = al(o + sizeof(double) * (size_t)kMaxSlabs * 2 * kInitParts);
    L.hout = o; o = al(o + sizeof(double) * 2);
    L.bidx = o; o = al(o + sizeof(int32_t) * (size_t)(B > 0 ? B : 1));
    L.gate = o; o = al(o + sizeof(int));
    L.total = o;
    return L;
}

// ---------------------------------------------------------------- dataset layout (once per dataset)

// Floor corner of the clamped rotated pixel, fp32 -- the exact formula of the main kernel.
__device__ __forceinline__ void floor_corner(float px, float py, const float* fr, float bnd, float& cx, float& cy,
                                             float& cz, float& fx, float& fy, float& fz) {
    cx = fminf(fmaxf(fmaf(px, fr[0], py * fr[3]), -bnd), bnd);
    cy = fminf(fmaxf(fmaf(px, fr[1], py * fr[4]), -bnd), bnd);
    cz = fminf(fmaxf(fmaf(px, fr[2], py * fr[5]), -bnd), bnd);
    fx = floorf(cx);
    fy = floorf(cy);
    fz = floorf(cz);
}

__device__ __forceinline__ int owner_brick(short2 k, const float* fr, float bnd, int c, int nb) {
    float cx, cy, cz, fx, fy, fz;
    floor_corner((float)k.x, (float)k.y, fr, bnd, cx, cy, cz, fx, fy, fz);
    const int bx = ((int)fx + c) / BT, by = ((int)fy + c) / BT, bz = ((int)fz + c) / BT;
    return (bz * nb + by) * nb + bx;
}

// Per image: number of distinct owner bricks -> seg_off[i + 1] (scanned afterwards).
__global__ void __launch_bounds__(256) sorted_count_kernel(int M, int n_mask, const short2* __restrict__ pix,
                                                           const fsld_image_rec* __restrict__ recs, int32_t* seg_off) {
    extern __shared__ int hist[];
    __shared__ float fr[6];
    __shared__ int nseg;
    const int i = blockIdx.x;
    const int c = (M + 1) / 2, nb = (M + BT - 1) / BT, nbr = nb * nb * nb;
    const float bnd = (float)(M / 2 - 1);
    if (threadIdx.x < 6) fr[threadIdx.x] = (float)recs[i].rot[threadIdx.x];
    if (threadIdx.x == 0) nseg = 0;
    for (int b = threadIdx.x; b < nbr; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    for (int p = threadIdx.x; p < n_mask; p += blockDim.x) atomicAdd(hist + owner_brick(pix[p], fr, bnd, c, nb), 1);
    __syncthreads();
    int cnt = 0;  // segments: a brick's pixels in runs of at most kSegMax
    for (int b = threadIdx.x; b < nbr; b += blockDim.x) cnt += (hist[b] + kSegMax - 1) / kSegMax;
    atomicAdd(&nseg, cnt);
    __syncthreads();
    if (threadIdx.x == 0) seg_off[i + 1] = nseg;
}

// In-place inclusive scan of seg_off[1..N] (one CTA), seg_off[0] = 0.
__global__ void __launch_bounds__(1024) scan_offsets_kernel(int32_t* seg_off, int N) {
    __shared__ int part[1024];
    const int per = (N + 1023) / 1024;
    const int lo = 1 + threadIdx.x * per, hi = min(lo + per, N + 1);
    int s = 0;
    for (int i = lo; i < hi; ++i) s += seg_off[i];
    part[threadIdx.x] = s;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        const int v = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    int run = part[threadIdx.x] - s;
    for (int i = lo; i < hi; ++i) {
        run += seg_off[i];
        seg_off[i] = run;
    }
    if (threadIdx.x == 0) seg_off[0] = 0;
}

// Per image: counting sort of the masked pixels by owner brick -> sorted x,
// per-pixel (kx, ky) and the segment list in ascending brick order.
__global__ void __launch_bounds__(256) sorted_fill_kernel(int M, int n_mask, const short2* __restrict__ pix,
                                                          const fsld_image_rec* __restrict__ recs,
                                                          const float2* __restrict__ x_in, float2* __restrict__ x_out,
                                                          char2* __restrict__ pc_out, const int32_t* __restrict__ seg_off,
                                                          int2* __restrict__ segs) {
    extern __shared__ int word[];  // per brick: count, then (start | count << 16) running position
    __shared__ float fr[6];
    __shared__ int tsum[256], tseg[256];
    const int i = blockIdx.x;
    const int c = (M + 1) / 2, nb = (M + BT - 1) / BT, nbr = nb * nb * nb;
    const float bnd = (float)(M / 2 - 1);
    if (threadIdx.x < 6) fr[threadIdx.x] = (float)recs[i].rot[threadIdx.x];
    for (int b = threadIdx.x; b < nbr; b += blockDim.x) word[b] = 0;
    __syncthreads();
    for (int p = threadIdx.x; p < n_mask; p += blockDim.x) atomicAdd(word + owner_brick(pix[p], fr, bnd, c, nb), 1);
    __syncthreads();
    // exclusive scans of counts and of non-empty flags over contiguous brick chunks
    const int per = (nbr + blockDim.x - 1) / blockDim.x;
    const int lo = threadIdx.x * per, hi = min(lo + per, nbr);
    int s = 0, g = 0;
    for (int b = lo; b < hi; ++b) {
        s += word[b];
        g += (word[b] + kSegMax - 1) / kSegMax;
    }
    tsum[threadIdx.x] = s;
    tseg[threadIdx.x] = g;
    __syncthreads();
    for (int o = 1; o < (int)blockDim.x; o <<= 1) {
        const int v1 = (int)threadIdx.x >= o ? tsum[threadIdx.x - o] : 0;
        const int v2 = (int)threadIdx.x >= o ? tseg[threadIdx.x - o] : 0;
        __syncthreads();
        tsum[threadIdx.x] += v1;
        tseg[threadIdx.x] += v2;
        __syncthreads();
    }
    int start = tsum[threadIdx.x] - s, ord = tseg[threadIdx.x] - g;
    const int sbase = seg_off[i];
    for (int b = lo; b < hi; ++b) {
        const int cnt = word[b];
        word[b] = start | (cnt << 16);
        for (int q = 0; q < cnt; q += kSegMax)  // runs of <= kSegMax pixels (the brick kernels' bound)
            segs[sbase + ord++] = make_int2(b, (start + q) | (min(kSegMax, cnt - q) << 16));
        start += cnt;
    }
    __syncthreads();
    const size_t row = (size_t)i * n_mask;
    for (int p = threadIdx.x; p < n_mask; p += blockDim.x) {
        const short2 k = pix[p];
        const int b = owner_brick(k, fr, bnd, c, nb);
        const int pos = atomicAdd(word + b, 1) & 0xFFFF;
        pc_out[row + pos] = make_char2((signed char)k.x, (signed char)k.y);
        if (x_in) x_out[row + pos] = x_in[row + p];
    }
}

#include "fsld_brick_wave.cuh"
#include "fsld_brick_tables.cuh"

static int smem_optin(const void* fn, size_t bytes) {
    if (bytes <= 48 * 1024) return 0;
    return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) == cudaSuccess ? 0 : -1;
}

cudaError_t launch_sorted_count(int M, int n_mask, const short2* pix, const fsld_image_rec* recs, int N,
                                int32_t* seg_off, cudaStream_t s) {
    const int nb = (M + BT - 1) / BT;
    const size_t smem = sizeof(int) * (size_t)nb * nb * nb;
    if (smem_optin((const void*)sorted_count_kernel, smem)) return cudaErrorInvalidValue;
    sorted_count_kernel<<<N, 256, smem, s>>>(M, n_mask, pix, recs, seg_off);
    scan_offsets_kernel<<<1, 1024, 0, s>>>(seg_off, N);
    return cudaGetLastError();
}

cudaError_t launch_sorted_fill(int M, int n_mask, const short2* pix, const fsld_image_rec* recs, int N,
                               const float2* x_in, float2* x_out, char2* pc_out, const int32_t* seg_off, int2* segs,
                               cudaStream_t s) {
    const int nb = (M + BT - 1) / BT;
    const size_t smem = sizeof(int) * (size_t)nb * nb * nb;
    if (smem_optin((const void*)sorted_fill_kernel, smem)) return cudaErrorInvalidValue;
    sorted_fill_kernel<<<N, 256, smem, s>>>(M, n_mask, pix, recs, x_in, x_out, pc_out, seg_off, segs);
    wave_order_kernel<<<N, 256, 0, s>>>(M, n_mask, recs, x_in ? x_out : nullptr, pc_out, seg_off, segs);
    return cudaGetLastError();
}

size_t sorted_tables_bytes(long long npx) { return tables_bytes(npx); }

cudaError_t launch_sorted_tables(int M, int n_mask, int mode, const fsld_image_rec* recs, int N, const char2* pc,
                                 const int32_t* seg_off, const int2* segs, void* ptab, cudaStream_t s) {
    if (N < 1) return cudaSuccess;
    sorted_tables_kernel<<<N, 256, 0, s>>>(M, n_mask, mode == FSLD_MODE_NN, recs, pc, seg_off, segs, ptab,
                                           (long long)N * n_mask);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- per-step binning

// frac(hi + lo) * 2^64 as a wrapping 64-bit fixed-point "turns" value
// (double-double input, |hi| < 2^40).  Every step but the last rounding is exact.
__device__ __forceinline__ unsigned long long frac_fixed64(double hi, double lo) {
    const double f = hi - rint(hi);               // exact, |f| <= 1/2
    const double a = f * 4294967296.0;            // exact
    const double ah = floor(a);                   // exact
    const double r = (a - ah) + lo * 4294967296.0;  // a - ah exact, in [0, 1)
    const long long l = __double2ll_rn(r * 4294967296.0);
    return ((unsigned long long)(long long)ah << 32) + (unsigned long long)l;
}

// x / (2 pi) in turns, fixed point: double-double product with 1/(2 pi).
__device__ __forceinline__ unsigned long long turns_of_radians(double x) {
    constexpr double kInv2PiHi = 0.15915494309189535;     // fl(1 / 2pi)
    constexpr double kInv2PiLo = -9.839338337591243e-18;  // 1/2pi - fl(1/2pi)
    const double hi = x * kInv2PiHi;
    const double lo = fma(x, kInv2PiHi, -hi) + x * kInv2PiLo;
    return frac_fixed64(hi, lo);
}

// The per-image part of a SegRec (everything except gofs / count / start / row),
// from the 128-byte record (fsld_common.cuh ctf_value / shift_phase restated):
//   gamma = g0 k2 + g1 c2 + g2 s2 + g3 k2^2 with c2 = kx^2 - ky^2, s2 = 2 kx ky;
//   the kernel multiplies non-negative monomials (k2, c2 + 2^15, s2 + 2^16, k2^2),
//   so the offsets go into the constant term.  Shift: t = (s0 kx + s1 ky) / 2 turns,
//   with kx + 128, ky + 128.
// Computed by one warp, one fixed-point conversion per lane (the conversions are fp64 chains).
__device__ void seg_template_warp(const fsld_image_rec* __restrict__ rp, SegRec& T) {
    const int lane = threadIdx.x & 31;
    const uint32_t flags = rp->flags;
    const bool ctf = (flags & FSLD_REC_CTF) != 0, shift = (flags & FSLD_REC_SHIFT) != 0;
    unsigned long long u = 0;
    if (lane < 6) T.frame[lane] = (float)rp->rot[lane];
    else if (lane < 10) u = ctf ? turns_of_radians(rp->gamma[lane - 6]) : 0ull;
    else if (lane == 10) u = ctf ? turns_of_radians(-32768.0 * rp->gamma[1]) : 0ull;
    else if (lane == 11) u = ctf ? turns_of_radians(-65536.0 * rp->gamma[2]) : 0ull;
    else if (lane < 14) u = shift ? frac_fixed64(0.5 * rp->shift[lane - 12], 0.0) : 0ull;
    else if (lane < 16) u = shift ? frac_fixed64(-64.0 * rp->shift[lane - 14], 0.0) : 0ull;
    const unsigned long long g11 = __shfl_sync(0xffffffffu, u, 11);
    const unsigned long long s15 = __shfl_sync(0xffffffffu, u, 15);
    if (lane >= 6 && lane < 10) {
        T.glo[lane - 6] = (uint32_t)u;
        T.ghi[lane - 6] = (uint32_t)(u >> 32);
    } else if (lane == 10) {
        T.gc = (uint32_t)((u + g11 + 0x80000000ull) >> 32);  // constants: nearest 2^-32 turn
    } else if (lane == 12 || lane == 13) {
        T.slo[lane - 12] = (uint32_t)u;
        T.shi[lane - 12] = (uint32_t)(u >> 32);
    } else if (lane == 14) {
        T.sc = (uint32_t)((u + s15 + 0x80000000ull) >> 32);
    } else if (lane == 16) {
        T.wsin = ctf ? rp->wsin : 0.f;
        T.wcos = ctf ? rp->wcos : -1.f;  // no CTF: -(0 sin 0 + (-1) cos 0) = 1
        T.envl = ctf ? (float)(rp->env * 1.4426950408889634) : 0.f;
    } else if (lane >= 20 && lane < 24) {
        T.pad[lane - 20] = 0;
    }
}

// Fill for one batch image (block-cooperative): its SegRec template -> tmpl[tslot] (written by
// warp 0), and one 16-byte PairRec per segment at its brick's next slot.
__device__ __forceinline__ void fill_image(const SortedArgs& a, int row, int tslot, int* fill, const int* off,
                                           PairRec* pairs, SegRec& T) {
    const int s0 = a.seg_off[row], s1 = a.seg_off[row + 1];
    if (threadIdx.x < 32) {
        seg_template_warp(a.recs + row, T);
        __syncwarp();
        if (threadIdx.x < 8)
            reinterpret_cast<int4*>(a.tmpl + tslot)[threadIdx.x] = reinterpret_cast<const int4*>(&T)[threadIdx.x];
    }
    for (int sidx = s0 + threadIdx.x; sidx < s1; sidx += blockDim.x) {
        const int2 seg = a.segs[sidx];
        const int slot = atomicAdd(fill + seg.x, 1);
        PairRec r;
        r.gofs = (long long)row * a.n_mask + (seg.y & 0xFFFF);
        r.count = seg.y >> 16;
        r.tslot = tslot;
        pairs[off[seg.x] + slot] = r;
    }
}

template <bool FILL>
__global__ void __launch_bounds__(128) bin_sorted_kernel(SortedArgs a) {
    if (a.gate && *a.gate == 0) return;  // reuse: the items in scratch are this batch's already
    const int b = blockIdx.x;
    const int row = a.idx ? a.idx[b] : b;
    if (!FILL && threadIdx.x == 0 && a.bidx) a.bidx[b] = row;  // what these work items were binned for
    if (FILL) {
        __shared__ SegRec T;
        fill_image(a, row, b, a.fill, a.off, a.pairs, T);
    } else {
        const int s0 = a.seg_off[row], s1 = a.seg_off[row + 1];
        for (int sidx = s0 + threadIdx.x; sidx < s1; sidx += blockDim.x) atomicAdd(a.cnt + a.segs[sidx].x, 1);
    }
}

// Exclusive scan of per-brick pair counts and expansion into work items
// (brick, first pair, n pairs <= BC).  Full items (BC pairs) are listed first
// and the partial remainders after them in descending segment count (largest
// first: the persistent kernel's last claims are the smallest items, so the CTAs
// finish together -- measured +6.6 % on the cfg3 step over brick order).  One CTA of 1024 threads,
// warp-shuffle scans.  Leaves cnt[] zeroed for the next call (fsld_prepare
// zeroes it once).  ctl = {n_items, claim counter, overflow, pairs base, items base}: the
// work-item kernels read their pairs at pairs + ctl[3] and their items at items + ctl[4]
// (both 0 for a single batch; per-batch offsets in a multi-batch plan).
__device__ void scan_batch(int* cnt, int* off, int* fill, int4* items, int* ctl, int nbr, int cap_items,
                           int cap_pairs, int pairs_base, int items_base, bool det = false) {
    __shared__ int wp[32], wf[32], wr[32];
    __shared__ int rh[BC];  // partial items per segment count, then the descending-size cursor
    if (threadIdx.x < BC) rh[threadIdx.x] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int per = (nbr + 1023) / 1024;
    const int lo = threadIdx.x * per;
    const int hi = min(lo + per, nbr);
    int np = 0, nf = 0, nr = 0;
    for (int i = lo; i < hi; ++i) {
        const int c = cnt[i];
        np += c;
        nf += c / BC;
        nr += (c % BC) != 0;
        if (c % BC) atomicAdd(rh + c % BC, 1);
    }
    int ip = np, jf = nf, jr = nr;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int tp = __shfl_up_sync(0xffffffffu, ip, o), tf = __shfl_up_sync(0xffffffffu, jf, o),
                  tr = __shfl_up_sync(0xffffffffu, jr, o);
        if (lane >= o) {
            ip += tp;
            jf += tf;
            jr += tr;
        }
    }
    if (lane == 31) {
        wp[warp] = ip;
        wf[warp] = jf;
        wr[warp] = jr;
    }
    __syncthreads();
    if (warp == 0) {
        int vp = wp[lane], vf = wf[lane], vr = wr[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int tp = __shfl_up_sync(0xffffffffu, vp, o), tf = __shfl_up_sync(0xffffffffu, vf, o),
                      tr = __shfl_up_sync(0xffffffffu, vr, o);
            if (lane >= o) {
                vp += tp;
                vf += tf;
                vr += tr;
            }
        }
        wp[lane] = vp;
        wf[lane] = vf;
        wr[lane] = vr;
    }
    __syncthreads();
    const int n_full = wf[31];
    if (threadIdx.x == 0) {  // partial items in descending segment count: cursor of size r = sum of larger bins
        int run = 0;
        for (int r = BC - 1; r >= 1; --r) {
            const int h = rh[r];
            rh[r] = n_full + run;
            run += h;
        }
    }
    __syncthreads();
    int pbase = (warp > 0 ? wp[warp - 1] : 0) + ip - np;
    int fbase = (warp > 0 ? wf[warp - 1] : 0) + jf - nf;
    int rbase = n_full + (warp > 0 ? wr[warp - 1] : 0) + jr - nr;  // (det: partial items in brick order)
    int4* it = items + items_base;
    for (int i = lo; i < hi; ++i) {
        const int c = cnt[i];
        cnt[i] = 0;
        off[i] = pbase;
        fill[i] = 0;
        int k = 0;
        for (; k + BC <= c; k += BC, ++fbase)
            if (fbase < cap_items) it[fbase] = make_int4(i, pbase + k, BC, 0);
        if (k < c) {
            const int slot = det ? rbase++ : atomicAdd(rh + (c - k), 1);
            if (slot < cap_items) it[slot] = make_int4(i, pbase + k, c - k, 0);
        }
        pbase += c;
    }
    if (threadIdx.x == 1023) {
        off[nbr] = wp[31];
        ctl[0] = min(n_full + wr[31], cap_items);
        ctl[1] = 0;
        ctl[2] = wp[31] > cap_pairs;  // overflow flag (cannot happen for the 4 nb^2 bound)
        ctl[3] = pairs_base;
        ctl[4] = items_base;
    }
}

__global__ void __launch_bounds__(1024) brick_scan_kernel(SortedArgs a) {
    if (a.gate && *a.gate == 0) return;
    scan_batch(a.cnt, a.off, a.fill, a.items, a.ctl, a.nbr, a.cap_items, a.cap_pairs, 0, 0, a.det != 0);
}

// Deterministic mode: each brick's pair records sorted by dataset offset (the fill pass places them
// in atomic order), one CTA per brick, bitonic in shared memory (<= 2 x kDetMaxBatch records).
__global__ void __launch_bounds__(256) sort_pairs_kernel(const int* __restrict__ off, PairRec* pairs, int* ctl) {
    __shared__ long long key[2 * kDetMaxBatch];
    __shared__ int2 val[2 * kDetMaxBatch];
    const int i = blockIdx.x, lo = off[i], n = off[i + 1] - lo;
    if (n <= 1) return;
    if (n > 2 * kDetMaxBatch) {  // cannot happen for <= 2 segments per image and brick; flagged, left unsorted
        if (threadIdx.x == 0) atomicOr(ctl + 2, 2);
        return;
    }
    int P = 1;
    while (P < n) P <<= 1;
    for (int t = threadIdx.x; t < P; t += blockDim.x) {
        if (t < n) {
            const PairRec r = pairs[lo + t];
            key[t] = r.gofs;
            val[t] = make_int2(r.count, r.tslot);
        } else {
            key[t] = 0x7fffffffffffffffll;
        }
    }
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int t = threadIdx.x; t < P; t += blockDim.x) {
                const int u = t ^ j;
                if (u > t) {
                    const bool up = (t & k) == 0;
                    if ((key[t] > key[u]) == up) {
                        const long long kk = key[t];
                        key[t] = key[u];
                        key[u] = kk;
                        const int2 vv = val[t];
                        val[t] = val[u];
                        val[u] = vv;
                    }
                }
            }
            __syncthreads();
        }
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
        PairRec r;
        r.gofs = key[t];
        r.count = val[t].x;
        r.tslot = val[t].y;
        pairs[lo + t] = r;
    }
}

// Deterministic mode: the loss partials of the work items (one per item, in item order) -> *out.
__global__ void __launch_bounds__(1024) reduce_items_kernel(const double* __restrict__ part, const int* __restrict__ ctl,
                                                            double* out) {
    __shared__ double red[32];
    const int n = ctl[0];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
    const double t = block_sum(s, red);
    if (threadIdx.x == 0) *out = t;
}

// ---------------------------------------------------------------- multi-batch plans
// The batches of an epoch are known in advance (optim.py:133-139), so their binning can be
// done for K batches at once: three launches per plan instead of three per step.  Plan layout
// (PlanLayout): per batch k its own cnt / off / fill / ctl, and shared items / pairs arrays in
// which batch k starts at ctl_k[4] / ctl_k[3].

__global__ void __launch_bounds__(128) plan_count_kernel(SortedArgs a, int K, int* seg_tot) {
    const int k = blockIdx.x / a.B, b = blockIdx.x - k * a.B;
    const int row = a.idx[(size_t)k * a.B + b];
    const int s0 = a.seg_off[row], s1 = a.seg_off[row + 1];
    int* cnt = a.cnt + (size_t)k * a.nbr;
    for (int sidx = s0 + threadIdx.x; sidx < s1; sidx += blockDim.x) atomicAdd(cnt + a.segs[sidx].x, 1);
    if (threadIdx.x == 0) atomicAdd(seg_tot + k, s1 - s0);
}

__global__ void __launch_bounds__(1024) plan_scan_kernel(SortedArgs a, int K, const int* seg_tot,
                                                         int items_cap_total) {
    __shared__ int base_s;
    const int k = blockIdx.x;
    if (threadIdx.x < 32) {  // pairs before batch k
        int s = 0;
        for (int q = threadIdx.x; q < k; q += 32) s += seg_tot[q];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) base_s = s;
    }
    __syncthreads();
    const int pairs_base = base_s;
    // items of batch k <= nbr + pairs_k / BC: a non-overlapping upper-bound layout
    const int items_base = k * (a.nbr + 2) + (pairs_base + BC - 1) / BC;
    const int cap = min(a.nbr + seg_tot[k] / BC + 2, items_cap_total - items_base);
    scan_batch(a.cnt + (size_t)k * a.nbr, a.off + (size_t)k * (a.nbr + 1), a.fill + (size_t)k * a.nbr, a.items,
               a.ctl + 16 * k, a.nbr, cap, seg_tot[k], pairs_base, items_base);
}

__global__ void __launch_bounds__(128) plan_fill_kernel(SortedArgs a, int K) {
    __shared__ SegRec T;
    const int k = blockIdx.x / a.B, b = blockIdx.x - k * a.B;
    const int row = a.idx[(size_t)k * a.B + b];
    const int* ctl = a.ctl + 16 * k;
    fill_image(a, row, k * a.B + b, a.fill + (size_t)k * a.nbr, a.off + (size_t)k * (a.nbr + 1), a.pairs + ctl[3], T);
}

PlanLayout plan_layout(int M, int B, int K, long long total_pairs) {
    PlanLayout P{};
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    const int nb = (M + BT - 1) / BT;
    P.nbr = nb * nb * nb;
    P.K = K;
    P.B = B;
    P.total_pairs = total_pairs;
    P.cap_items = (long long)K * (P.nbr + 2) + (total_pairs + BC - 1) / BC + K;
    size_t o = 0;
    P.hdr = o; o = al(o + 256);
    P.cnt = o; o = al(o + sizeof(int) * (size_t)K * P.nbr);
    P.off = o; o = al(o + sizeof(int) * (size_t)K * (P.nbr + 1));
    P.fill = o; o = al(o + sizeof(int) * (size_t)K * P.nbr);
    P.ctl = o; o = al(o + sizeof(int) * 16 * (size_t)K);
    P.seg_tot = o; o = al(o + sizeof(int) * (size_t)K);
    P.items = o; o = al(o + sizeof(int4) * (size_t)P.cap_items);
    P.pairs = o; o = al(o + sizeof(PairRec) * (size_t)(total_pairs > 0 ? total_pairs : 1));
    P.tmpl = o; o = al(o + sizeof(SegRec) * (size_t)K * B);
    P.total = o;
    return P;
}

cudaError_t launch_plan_build(SortedArgs a, const PlanLayout& P, char* plan, cudaStream_t s) {
    // zero the per-batch counters and pair totals (scan leaves cnt / fill zeroed, but a plan
    // buffer is fresh memory)
    cudaError_t e = cudaMemsetAsync(plan + P.cnt, 0, P.off - P.cnt, s);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(plan + P.fill, 0, P.items - P.fill, s);
    if (e != cudaSuccess) return e;
    a.cnt = reinterpret_cast<int*>(plan + P.cnt);
    a.off = reinterpret_cast<int*>(plan + P.off);
    a.fill = reinterpret_cast<int*>(plan + P.fill);
    a.ctl = reinterpret_cast<int*>(plan + P.ctl);
    a.items = reinterpret_cast<int4*>(plan + P.items);
    a.pairs = reinterpret_cast<PairRec*>(plan + P.pairs);
    a.tmpl = reinterpret_cast<SegRec*>(plan + P.tmpl);
    int* seg_tot = reinterpret_cast<int*>(plan + P.seg_tot);
    plan_count_kernel<<<P.K * a.B, 128, 0, s>>>(a, P.K, seg_tot);
    plan_scan_kernel<<<P.K, 1024, 0, s>>>(a, P.K, seg_tot, (int)P.cap_items);
    plan_fill_kernel<<<P.K * a.B, 128, 0, s>>>(a, P.K);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- main kernel

#include "fsld_brick_main.cuh"  // the work-item kernel (kept separate: it is the tuning target)
#include "fsld_brick_energy.cuh"
#include "fsld_brick_hutch.cuh"
#include "fsld_brick_v3.cuh"

cudaError_t set_phase_profile(unsigned long long* buf) {
    return cudaMemcpyToSymbol(g_phase_prof, &buf, sizeof(buf));
}

// Persistent grid (SMs x resident CTAs) of a brick kernel and its >48 KB dynamic shared-memory
// opt-in, per device: the attribute belongs to a device context, so every device a process uses
// is set up on its own first launch (std::call_once per device and kernel).
constexpr int kMaxDevices = 16;
struct GridCache {
    std::once_flag once[kMaxDevices];
    int grid[kMaxDevices] = {};
    cudaError_t err[kMaxDevices] = {};
};

template <typename Kern>
static cudaError_t persistent_grid(GridCache& C, Kern kern, size_t smem, int& out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    std::call_once(C.once[dev], [&] {
        cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int sms = 0, occ = 0;
        if (r == cudaSuccess) r = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (r == cudaSuccess) r = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, BTHREADS, smem);
        C.grid[dev] = sms * (occ > 0 ? occ : 1);
        C.err[dev] = r;
    });
    out = C.grid[dev];
    return C.err[dev];
}

template <bool HUTCH>
static cudaError_t main_grid(int& out) {
    static GridCache cache;
    return persistent_grid(cache, sorted_loss_grad_kernel<HUTCH>, sizeof(SortedSmemT<HUTCH>), out);
}

template <bool NN, bool HUTCH>
static cudaError_t v3_grid(int& out) {
    static GridCache cache;
    return persistent_grid(cache, brick_loss_grad_kernel<NN, HUTCH, false>, sizeof(BrickSmem3T<HUTCH>), out);
}

template <bool HUTCH>
static cudaError_t launch_sorted_main(const SortedArgs& a, double* sq_out, cudaStream_t s, int* grid_out = nullptr) {
    int grid = 0;
    if (a.ptab && (!HUTCH || !a.nn)) {  // the table-driven kernel (per-pixel f and footprint from the tables)
        cudaError_t e0 = HUTCH ? v3_grid<false, true>(grid) : a.nn ? v3_grid<true, false>(grid)
                                                                  : v3_grid<false, false>(grid);
        if (e0 != cudaSuccess) return e0;
        if (HUTCH) brick_loss_grad_kernel<false, true, false><<<grid, BTHREADS, sizeof(BrickSmem3T<true>), s>>>(a);
        else if (a.nn) brick_loss_grad_kernel<true, false, false><<<grid, BTHREADS, sizeof(BrickSmem3), s>>>(a);
        else brick_loss_grad_kernel<false, false, false><<<grid, BTHREADS, sizeof(BrickSmem3), s>>>(a);
    } else {
        const size_t smem = sizeof(SortedSmemT<HUTCH>);
        cudaError_t e0 = main_grid<HUTCH>(grid);
        if (e0 != cudaSuccess) return e0;
        sorted_loss_grad_kernel<HUTCH><<<grid, BTHREADS, smem, s>>>(a);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (grid_out) {  // the caller reduces the per-CTA partials
        *grid_out = grid;
        return cudaSuccess;
    }
    return launch_reduce(a.part, grid, sq_out, s);
}

cudaError_t launch_sorted_bin(const SortedArgs& a, cudaStream_t s) {
    // cnt[] is zero on entry: zeroed by fsld_prepare, and re-zeroed by every scan
    bin_sorted_kernel<false><<<a.B, 128, 0, s>>>(a);
    brick_scan_kernel<<<1, 1024, 0, s>>>(a);
    bin_sorted_kernel<true><<<a.B, 128, 0, s>>>(a);
    if (a.det) sort_pairs_kernel<<<a.nbr, 256, 0, s>>>(a.off, a.pairs, a.ctl);
    return cudaGetLastError();
}

// sum |f P v - x|^2 over a batch of a table-built dataset (trilinear): binning + the table-driven
// kernel's projection pass alone (GATHER) + the fixed-order reduce.
cudaError_t launch_sorted_loss_tab(const SortedArgs& a, double* sq_out, cudaStream_t s) {
    cudaError_t e = launch_sorted_bin(a, s);
    if (e != cudaSuccess) return e;
    static GridCache cache;
    int grid = 0;
    e = persistent_grid(cache, brick_loss_grad_kernel<false, false, false, true>, sizeof(BrickSmem3), grid);
    if (e != cudaSuccess) return e;
    brick_loss_grad_kernel<false, false, false, true><<<grid, BTHREADS, sizeof(BrickSmem3), s>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_reduce(a.part, grid, sq_out, s);
}

// Exact Hessian diagonal (data term) of a batch of a table-built dataset, trilinear: binning + the
// table-driven kernel's DIAG pass (a.fold += sum C^2 w^2; DET: int64 at *a.fxp, bitwise the same for
// any grid and batch order, B <= kDetMaxBatch).
cudaError_t launch_sorted_diag(const SortedArgs& a0, cudaStream_t s) {
    SortedArgs a = a0;
    cudaError_t e = launch_sorted_bin(a, s);
    if (e != cudaSuccess) return e;
    int grid = 0;
    if (a.det) {
        static GridCache cache;
        e = persistent_grid(cache, brick_loss_grad_kernel<false, false, true, false, true>, sizeof(BrickSmem3T<true>), grid);
        if (e != cudaSuccess) return e;
        if (const char* g = getenv("FSLD_DET_GRID")) {
            const int want = atoi(g);
            if (want > 0 && want < grid) grid = want;
        }
        brick_loss_grad_kernel<false, false, true, false, true><<<grid, BTHREADS, sizeof(BrickSmem3T<true>), s>>>(a);
    } else {
        static GridCache cache;
        e = persistent_grid(cache, brick_loss_grad_kernel<false, false, false, false, true>, sizeof(BrickSmem3T<true>), grid);
        if (e != cudaSuccess) return e;
        brick_loss_grad_kernel<false, false, false, false, true><<<grid, BTHREADS, sizeof(BrickSmem3T<true>), s>>>(a);
    }
    return cudaGetLastError();
}

// Deterministic loss+grad on the table-driven kernel: bitwise the same gradient (int64 pairs at
// scale *a.fxp, accumulated in a.acc) and loss for any launch grid and any order of the batch.
cudaError_t launch_sorted_loss_grad_det(const SortedArgs& a0, double* sq_out, cudaStream_t s) {
    SortedArgs a = a0;
    a.det = 1;
    cudaError_t e = launch_sorted_bin(a, s);
    if (e != cudaSuccess) return e;
    static GridCache cache;
    int grid = 0;
    e = persistent_grid(cache, brick_loss_grad_kernel<false, false, true>, sizeof(BrickSmem3), grid);
    if (e != cudaSuccess) return e;
    if (const char* g = getenv("FSLD_DET_GRID")) {  // (tests: the result must not depend on the grid)
        const int want = atoi(g);
        if (want > 0 && want < grid) grid = want;
    }
    brick_loss_grad_kernel<false, false, true><<<grid, BTHREADS, sizeof(BrickSmem3), s>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    reduce_items_kernel<<<1, 1024, 0, s>>>(a.part, a.ctl, sq_out);
    return cudaGetLastError();
}

cudaError_t launch_sorted_loss_grad(const SortedArgs& a, double* sq_out, cudaStream_t s) {
    cudaError_t e = launch_sorted_bin(a, s);
    if (e != cudaSuccess) return e;
    return a.zbits ? launch_sorted_main<true>(a, sq_out, s) : launch_sorted_main<false>(a, sq_out, s);
}

// The loss+grad brick pass over the items a.ctl describes, per-CTA |r|^2 partials left in
// a.part[0 .. *grid) for the caller to reduce.
cudaError_t launch_sorted_pass(const SortedArgs& a, cudaStream_t s, int* grid) {
    return launch_sorted_main<false>(a, nullptr, s, grid);
}

// Work items of one binned batch regrouped by z-slab (brick z-layer -> slab from `map`) for the
// slab-pipelined host step (fsld_loss_grad_host): a stable partition, so every slab keeps the
// full-first / largest-first order of scan_batch.  Slab g's items are gitems[gctl_g[4] ..
// + gctl_g[0]), gctl_g = gctl + 16 g = {n, claim counter 0, 0, pairs base, items base}.
// One CTA of 32 warps; warp w owns a contiguous run of items: per-(warp, slab) counts with
// match.any, a (slab-major, warp-minor) scan, then each item's rank among its chunk's equal-slab
// lanes gives its position.
__global__ void __launch_bounds__(1024) slab_items_kernel(const int4* __restrict__ items, const int* __restrict__ ctl,
                                                          int nb, SlabMap map, int G, int4* __restrict__ gitems,
                                                          int* __restrict__ gctl) {
    __shared__ int cnt[32][kMaxSlabs];  // per warp and slab: count, then the running output position
    items += ctl[4];
    const int n = ctl[0], nb2 = nb * nb;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int per = ((n + 31) / 32 + 31) & ~31;  // items per warp, whole chunks of 32
    const int lo = min(warp * per, n), hi = min(lo + per, n);
    for (int t = threadIdx.x; t < 32 * kMaxSlabs; t += blockDim.x) cnt[t / kMaxSlabs][t % kMaxSlabs] = 0;
    __syncthreads();
    for (int b = lo; b < hi; b += 32) {
        const int i = b + lane;
        const int g = i < hi ? (int)map.of_layer[__ldg(&items[i].x) / nb2] : -1;
        const unsigned m = __match_any_sync(0xffffffffu, g);
        if (g >= 0 && lane == __ffs(m) - 1) cnt[warp][g] += __popc(m);
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan over (slab, warp), slab-major; lane handles one warp column
        int base = 0;
        for (int g = 0; g < G; ++g) {
            const int c = cnt[lane][g];
            int incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            cnt[lane][g] = base + incl - c;
            const int sum = __shfl_sync(0xffffffffu, incl, 31);
            if (lane == 0) {
                int* q = gctl + 16 * g;
                q[0] = sum;
                q[1] = 0;
                q[2] = 0;
                q[3] = ctl[3];
                q[4] = base;
            }
            base += sum;
        }
    }
    __syncthreads();
    for (int b = lo; b < hi; b += 32) {
        const int i = b + lane;
        int4 it = make_int4(0, 0, 0, 0);
        int g = -1;
        if (i < hi) {
            it = items[i];
            g = map.of_layer[it.x / nb2];
        }
        const unsigned m = __match_any_sync(0xffffffffu, g);
        if (g >= 0) gitems[cnt[warp][g] + __popc(m & ((1u << lane) - 1u))] = it;
        __syncwarp();
        if (g >= 0 && lane == __ffs(m) - 1) cnt[warp][g] += __popc(m);
        __syncwarp();
    }
}

// Function attributes / grid size of the host-step kernel on the current device (outside any
// stream capture); also the grid the slab passes will use (<= kSlabCtas, checked before launch).
cudaError_t prepare_host_step(int* grid_out) {
    int grid = 0, grid3 = 0;
    cudaError_t e = main_grid<false>(grid);
    if (e == cudaSuccess) e = v3_grid<false, false>(grid3);
    if (grid3 > grid) grid = grid3;
    if (grid_out) *grid_out = grid;
    return e;
}

cudaError_t launch_slab_items(const SortedArgs& a, const SlabMap& map, int G, int4* gitems, int* gctl, cudaStream_t s) {
    cudaError_t e = prepare_host_step(nullptr);
    if (e != cudaSuccess) return e;
    slab_items_kernel<<<1, 1024, 0, s>>>(a.items, a.ctl, a.nb, map, G, gitems, gctl);
    return cudaGetLastError();
}

// One batch of a plan: its work items are ready; re-arm its claim counter and run.
#ifdef FSLD_EXP_NO_GEO2
static void exp_l0_once(const SortedArgs& a, cudaStream_t s);
#endif
cudaError_t launch_planned_loss_grad(const SortedArgs& a, double* sq_out, cudaStream_t s) {
#ifdef FSLD_EXP_NO_GEO2
    exp_l0_once(a, s);
#endif
    cudaError_t e = cudaMemsetAsync(a.ctl + 1, 0, sizeof(int), s);
    if (e != cudaSuccess) return e;
    return a.zbits ? launch_sorted_main<true>(a, sq_out, s) : launch_sorted_main<false>(a, sq_out, s);
}

// The whole loss+grad step of batch k of a plan with the epilogue fused around the brick pass:
// grad = lam v (+ ||v||^2 partials), the brick pass adding scale * contributions into grad, and one
// finalize of sq and the loss.  a.acc = grad, a.v = v.
#ifdef FSLD_EXP_NO_GEO2
__global__ void exp_l0_into_f_kernel(void* ptab) {
    const long long npx = reinterpret_cast<const TabHeader*>(ptab)->npx;
    float2* tf = const_cast<float2*>(tab_f(ptab));
    const float4* tg = tab_geo(ptab, npx);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < npx; i += (long long)gridDim.x * blockDim.x)
        tf[i].x = tg[i].w;
}
static void exp_l0_once(const SortedArgs& a, cudaStream_t s) {
    static const void* done = nullptr;
    if (a.ptab && done != a.ptab) {
        exp_l0_into_f_kernel<<<1184, 256, 0, s>>>(const_cast<void*>(a.ptab));
        done = a.ptab;
    }
}
#endif

cudaError_t launch_planned_loss_grad_step(SortedArgs a, int64_t nvox, double scale, double lam, double* sq_out,
                                          double* loss, double* norm_part, int n_norm, cudaStream_t s) {
#ifdef FSLD_EXP_NO_GEO2
    exp_l0_once(a, s);
#endif
    if (a.ptab && !a.nn) {  // the table-driven kernels do the whole step in one launch
        int grid = 0;
        cudaError_t e = v3_grid<false, false>(grid);
        if (e != cudaSuccess) return e;
        if (grid > n_norm) return cudaErrorInvalidValue;
        e = cudaMemsetAsync(a.ctl + 1, 0, sizeof(int), s);  // re-arm the claim counter (any earlier use)
        if (e != cudaSuccess) return e;
        a.out_scale = (float)scale;
        a.fuse = 1;
        a.flam = (float)lam;
        a.fscale = scale;
        a.fnorm = norm_part;
        a.fsq = sq_out;
        a.floss = loss;
        brick_loss_grad_kernel<false, false, false><<<grid, BTHREADS, sizeof(BrickSmem3), s>>>(a);
        return cudaGetLastError();
    }
    cudaError_t e = launch_grad_init(nvox, a.v, lam, a.acc, norm_part, n_norm, s);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(a.ctl + 1, 0, sizeof(int), s);
    if (e != cudaSuccess) return e;
    a.out_scale = (float)scale;
    int grid = 0;
    e = launch_sorted_main<false>(a, nullptr, s, &grid);
    if (e != cudaSuccess) return e;
    return launch_loss_finalize(a.part, grid, norm_part, n_norm, scale, lam, sq_out, loss, s);
}

// FSLD_REUSE_BINS: the work items left in scratch are reused only if they were binned for this very
// batch -- the rows are compared on the device with the copy the count pass stored (bidx); any
// difference (or another batch size) opens the gate and the three binning kernels run again.
__global__ void __launch_bounds__(1024) bins_check_kernel(const int32_t* __restrict__ idx, const int32_t* __restrict__ bidx,
                                                          int B, int* gate) {
    int diff = 0;
    for (int b = threadIdx.x; b < B; b += blockDim.x) diff |= (idx ? idx[b] : b) != bidx[b];
    diff = __syncthreads_or(diff);
    if (threadIdx.x == 0) *gate = diff;
}

cudaError_t launch_sorted_energy(const SortedArgs& a, double* out, bool rebin, cudaStream_t s) {
    static GridCache cache;
    const size_t smem = sizeof(EnergySmem);
    int grid = 0;
    cudaError_t e0 = persistent_grid(cache, sorted_energy_kernel, smem, grid);
    if (e0 != cudaSuccess) return e0;
    if (rebin) {
        bin_sorted_kernel<false><<<a.B, 128, 0, s>>>(a);
        brick_scan_kernel<<<1, 1024, 0, s>>>(a);
        bin_sorted_kernel<true><<<a.B, 128, 0, s>>>(a);
    } else {  // the work items of the previous sorted call on this scratch, if its rows are these
        cudaError_t e = cudaMemsetAsync(a.ctl + 1, 0, sizeof(int), s);  // re-arm the claim counter
        if (e != cudaSuccess) return e;
        if (a.gate) {  // (binning plans carry their own work items: nothing to check)
            bins_check_kernel<<<1, 1024, 0, s>>>(a.idx, a.bidx, a.B, a.gate);
            bin_sorted_kernel<false><<<a.B, 128, 0, s>>>(a);  // (gated: no-ops unless the rows differ)
            brick_scan_kernel<<<1, 1024, 0, s>>>(a);
            bin_sorted_kernel<true><<<a.B, 128, 0, s>>>(a);
        }
    }
    // (the gather-only pass stays on the compute path: the table-driven variant measured 70 vs 66 us
    // per planned call at cfg3 -- without a scatter to feed, the lean energy kernel's occupancy wins)
    sorted_energy_kernel<<<grid, BTHREADS, smem, s>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_reduce(a.part, grid, out, s);
}

cudaError_t launch_sorted_hutch(const SortedArgs& a, int k, cudaStream_t s) {
    static GridCache cache;
    const size_t smem = sizeof(HutchSmem);
    int grid = 0;
    cudaError_t e0 = persistent_grid(cache, sorted_hutch_kernel, smem, grid);
    if (e0 != cudaSuccess) return e0;
    bin_sorted_kernel<false><<<a.B, 128, 0, s>>>(a);
    brick_scan_kernel<<<1, 1024, 0, s>>>(a);
    bin_sorted_kernel<true><<<a.B, 128, 0, s>>>(a);
    sorted_hutch_kernel<<<grid, BTHREADS, smem, s>>>(a, k, (k + 31) / 32);
    return cudaGetLastError();
}

}  // namespace fsld
