// fsld_brick.cu -- brick-binned fused loss+gradient kernel (tri mode) for sm_100a.
//
// Why: the reference's adjoint (kernels.py:193-230) scatters 8 complex
// corner contributions per pixel.  As global red.add that is 8 L2 atomics
// per pixel and the v1 tile kernel is L2-atomic bound (profiles/r01_v1_*).
// Here the M^3 volume is cut into 8^3-voxel bricks in frequency space.  For
// a batch, every (brick, image) pair whose slice plane can own a pixel of
// the brick is binned (count -> scan -> fill, all on device).  A persistent
// CTA takes a work item (brick, <= 32 images), stages the brick's 9^3
// voxels of v in shared memory, and for every owned pixel (floor corner in
// the brick) gathers 8 corners from smem, forms f*Pv - x, accumulates
// |r|^2 and scatters conj(f) r w into a 9^3 int32 fixed-point accumulator in
// smem (native ATOMS.ADD; the fixed-point scale is a power of two chosen
// per item from a bound on its contributions).  The item ends with one
// red.global.add.v2.f32 per touched brick voxel.
//
// Exactness contract: each pixel is owned by exactly one brick (the one
// containing floor(clamp(c)), c = R^T (kx,ky,0) in fp32, kernels.py:42-60,
// 147-170); binning and per-row candidate intervals are conservative and
// the ownership test is exact, so every pixel is processed exactly once.
#include "fsld_kernels.cuh"

namespace fsld {

ScratchLayout scratch_layout(int M, int n_mask, int B) {
    ScratchLayout L{};
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    L.nb = (M + BT - 1) / BT;
    L.nbr = L.nb * L.nb * L.nb;
    long long pp = (long long)B * (long long)(L.nbr < 4 * L.nb * L.nb ? L.nbr : 4 * L.nb * L.nb);
    L.cap_pairs = (int)(pp > 0 ? pp : 1);
    L.cap_items = L.nbr + L.cap_pairs / BC + 1;
    int tiles = (n_mask + kThreads * 4 - 1) / (kThreads * 4);
    long long v1parts = (long long)(B > 0 ? B : 1) * (tiles > 0 ? tiles : 1);
    L.cap_part = (int)(v1parts > 4096 ? v1parts : 4096);
    size_t o = 0;
    L.hdr = o; o = al(o + 256);
    L.pix2p = o; o = al(o + sizeof(int) * (size_t)M * M);
    L.rowmin = o; o = al(o + sizeof(int) * (size_t)M);
    L.rowmax = o; o = al(o + sizeof(int) * (size_t)M);
    L.cnt = o; o = al(o + sizeof(int) * (size_t)L.nbr);
    L.off = o; o = al(o + sizeof(int) * (size_t)(L.nbr + 1));
    L.fill = o; o = al(o + sizeof(int) * (size_t)L.nbr);
    L.pairs = o; o = al(o + sizeof(int) * (size_t)L.cap_pairs);
    L.items = o; o = al(o + sizeof(int4) * (size_t)L.cap_items);
    L.ctl = o; o = al(o + 64);
    L.part = o; o = al(o + sizeof(double) * (size_t)L.cap_part);
    L.total = o;
    return L;
}

// ---------------------------------------------------------------- geometry

__global__ void geom_prepare_kernel(int M, int n_mask, const short2* __restrict__ pix, GeomHeader* hdr,
                                    int* pix2p, int* rowmin, int* rowmax) {
    const int c = (M + 1) / 2;
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n_mask; p += gridDim.x * blockDim.x) {
        const short2 k = pix[p];
        pix2p[(k.y + c) * M + (k.x + c)] = p;
        atomicMin(rowmin + k.y + c, (int)k.x);
        atomicMax(rowmax + k.y + c, (int)k.x);
        atomicMax(&hdr->rmax2, (unsigned)(k.x * k.x + k.y * k.y));
    }
}

__global__ void geom_header_kernel(int M, int n_mask, const void* pix, GeomHeader* hdr) {
    hdr->magic = kGeomMagic;
    hdr->M = M;
    hdr->n_mask = n_mask;
    hdr->pix = pix;
}

__global__ void fill_int_kernel(int* p, int n, int v) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = v;
}

cudaError_t launch_geom_prepare(int M, int n_mask, const short2* pix, const ScratchLayout& L, char* scratch,
                                cudaStream_t s) {
    GeomHeader* hdr = reinterpret_cast<GeomHeader*>(scratch + L.hdr);
    int* pix2p = reinterpret_cast<int*>(scratch + L.pix2p);
    int* rmin = reinterpret_cast<int*>(scratch + L.rowmin);
    int* rmax = reinterpret_cast<int*>(scratch + L.rowmax);
    cudaError_t e = cudaMemsetAsync(hdr, 0, 256, s);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(pix2p, 0xFF, sizeof(int) * (size_t)M * M, s);
    if (e != cudaSuccess) return e;
    fill_int_kernel<<<(M + 255) / 256, 256, 0, s>>>(rmin, M, 0x3fffffff);
    fill_int_kernel<<<(M + 255) / 256, 256, 0, s>>>(rmax, M, -0x3fffffff);
    geom_prepare_kernel<<<(n_mask + 255) / 256, 256, 0, s>>>(M, n_mask, pix, hdr, pix2p, rmin, rmax);
    geom_header_kernel<<<1, 1, 0, s>>>(M, n_mask, pix, hdr);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- binning

struct Frame {
    float r0x, r0y, r0z, r1x, r1y, r1z;
};

__device__ __forceinline__ Frame frame_of(const fsld_image_rec& R) {
    Frame f;
    f.r0x = (float)R.rot[0]; f.r0y = (float)R.rot[1]; f.r0z = (float)R.rot[2];
    f.r1x = (float)R.rot[3]; f.r1y = (float)R.rot[4]; f.r1z = (float)R.rot[5];
    return f;
}

// Can the slice plane of frame F own a pixel of brick (bx,by,bz)?  Plane-box
// and ball-box tests on the brick box grown by a safety margin.
__device__ __forceinline__ bool brick_hit(const Frame& F, int bx, int by, int bz, int c, float rball) {
    const float m = 0.05f;
    const float ox = (float)(-c + BT * bx), oy = (float)(-c + BT * by), oz = (float)(-c + BT * bz);
    const float h = 0.5f * BT;
    const float cx = ox + h, cy = oy + h, cz = oz + h;
    const float nx = F.r0y * F.r1z - F.r0z * F.r1y;
    const float ny = F.r0z * F.r1x - F.r0x * F.r1z;
    const float nz = F.r0x * F.r1y - F.r0y * F.r1x;
    const float d = fabsf(nx * cx + ny * cy + nz * cz);
    if (d > (h + m) * (fabsf(nx) + fabsf(ny) + fabsf(nz)) + m) return false;
    const float dx = fmaxf(fmaxf(ox - m, 0.f), -(ox + BT + m));
    const float dy = fmaxf(fmaxf(oy - m, 0.f), -(oy + BT + m));
    const float dz = fmaxf(fmaxf(oz - m, 0.f), -(oz + BT + m));
    return dx * dx + dy * dy + dz * dz <= rball * rball;
}

template <bool FILL>
__global__ void __launch_bounds__(256) brick_bin_kernel(BrickArgs a) {
    __shared__ fsld_image_rec rec;
    const int b = blockIdx.x;
    load_record(a.recs, a.idx ? a.idx[b] : b, &rec);
    __syncthreads();
    const Frame F = frame_of(rec);
    const float rball = sqrtf((float)a.hdr->rmax2) + 0.51f;
    for (int id = threadIdx.x; id < a.nbr; id += blockDim.x) {
        const int bx = id % a.nb, by = (id / a.nb) % a.nb, bz = id / (a.nb * a.nb);
        if (!brick_hit(F, bx, by, bz, a.c, rball)) continue;
        if (FILL) {
            const int slot = atomicAdd(a.fill + id, 1);
            a.pairs[a.off[id] + slot] = b;
        } else {
            atomicAdd(a.cnt + id, 1);
        }
    }
}

// Exclusive scan of per-brick pair counts and expansion into work items
// (brick, first pair, n pairs <= BC).  One CTA of 1024 threads.
__global__ void __launch_bounds__(1024) brick_scan_kernel(BrickArgs a) {
    __shared__ int s_pairs[1024];
    __shared__ int s_items[1024];
    const int per = (a.nbr + 1023) / 1024;
    const int lo = threadIdx.x * per;
    const int hi = min(lo + per, a.nbr);
    int np = 0, ni = 0;
    for (int i = lo; i < hi; ++i) {
        const int c = a.cnt[i];
        np += c;
        ni += (c + BC - 1) / BC;
    }
    s_pairs[threadIdx.x] = np;
    s_items[threadIdx.x] = ni;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {  // Hillis-Steele inclusive scan
        int vp = threadIdx.x >= o ? s_pairs[threadIdx.x - o] : 0;
        int vi = threadIdx.x >= o ? s_items[threadIdx.x - o] : 0;
        __syncthreads();
        s_pairs[threadIdx.x] += vp;
        s_items[threadIdx.x] += vi;
        __syncthreads();
    }
    int pbase = s_pairs[threadIdx.x] - np;
    int ibase = s_items[threadIdx.x] - ni;
    for (int i = lo; i < hi; ++i) {
        const int c = a.cnt[i];
        a.off[i] = pbase;
        a.fill[i] = 0;
        for (int k = 0; k < c; k += BC) {
            if (ibase < a.cap_items) a.items[ibase] = make_int4(i, pbase + k, min(BC, c - k), 0);
            ++ibase;
        }
        pbase += c;
    }
    if (threadIdx.x == 1023) {
        a.off[a.nbr] = s_pairs[1023];
        a.ctl[0] = min(s_items[1023], a.cap_items);
        a.ctl[1] = 0;
        a.ctl[2] = s_pairs[1023] > a.cap_pairs;  // overflow flag (never expected)
    }
}

// ---------------------------------------------------------------- main kernel

constexpr float kMagic = 12582912.0f;   // 1.5 * 2^23: float -> int32 round-to-nearest
constexpr int kMagicBits = 0x4B400000;

__device__ __forceinline__ int to_fixed(float x) {  // |x| < 2^22
    return __float_as_int(x + kMagic) - kMagicBits;
}

struct BrickSmem {
    float2 vb[BH3];
    int accr[BH3];
    int acci[BH3];
    fsld_image_rec recs[BC];
    unsigned char rowof[BW][BMAXCAND];
    int item;
    float vmax;
    float xmax;
    double red[BW];
};

__global__ void __launch_bounds__(BTHREADS, 3) brick_loss_grad_kernel(BrickArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BrickSmem& S = *reinterpret_cast<BrickSmem*>(smem_raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int M = a.M, c = a.c, nb = a.nb, n = a.n_mask;
    const float bnd = a.bnd;
    double lsum = 0.0;
    const bool bad_geom = a.hdr->magic != kGeomMagic || a.hdr->M != M || a.hdr->n_mask != n;

    for (;;) {
        if (threadIdx.x == 0) {
            S.item = atomicAdd(a.ctl + 1, 1);
            S.vmax = 0.f;
            S.xmax = 0.f;
        }
        __syncthreads();
        const int it = S.item;
        if (it >= a.ctl[0] || bad_geom) break;
        const int4 item = a.items[it];
        const int bid = item.x, pstart = item.y, nimg = item.z;
        const int bx = bid % nb, by = (bid / nb) % nb, bz = bid / (nb * nb);
        const int ox = -c + BT * bx, oy = -c + BT * by, oz = -c + BT * bz;

        // records of this item's images (32 x 4 B per record, coalesced)
        for (int w = threadIdx.x; w < nimg * 32; w += BTHREADS) {
            const int k = w >> 5, q = w & 31;
            const int bimg = a.pairs[pstart + k];
            const int row = a.idx ? a.idx[bimg] : bimg;
            const uint32_t word = __ldg(reinterpret_cast<const uint32_t*>(a.recs + row) + q);
            reinterpret_cast<uint32_t*>(S.recs + k)[q] = word;
            if (q == 29) atomicMax(reinterpret_cast<int*>(&S.xmax), (int)word);  // pad[0] = max|x| (>= 0)
        }
        // v brick (+halo) and zeroed accumulators
        float vm = 0.f;
        for (int l = threadIdx.x; l < BH3; l += BTHREADS) {
            const int lx = l % BH, ly = (l / BH) % BH, lz = l / (BH * BH);
            const int kx = ox + lx, ky = oy + ly, kz = oz + lz;
            float2 val = make_float2(0.f, 0.f);
            if (kx < M - c && ky < M - c && kz < M - c && kx >= -c && ky >= -c && kz >= -c)
                val = __ldg(a.v + lin_index(kx, ky, kz, M, c));
            S.vb[l] = val;
            S.accr[l] = 0;
            S.acci[l] = 0;
            vm = fmaxf(vm, fmaxf(fabsf(val.x), fabsf(val.y)));
        }
        for (int o = 16; o > 0; o >>= 1) vm = fmaxf(vm, __shfl_xor_sync(0xffffffffu, vm, o));
        if (lane == 0) atomicMax(reinterpret_cast<int*>(&S.vmax), __float_as_int(vm));
        __syncthreads();
        // fixed-point scale: |contribution| <= |val| <= U = 2 max|v comp| + max|x|  ->  |U s| <= 2^21;
        // per voxel and item <= BC * 12 contributions  ->  < 2^30.
        const float U = 2.0f * S.vmax + S.xmax;
        const float sc = U > 0.f ? exp2f(floorf(log2f(2097152.0f / U))) : 1.0f;
        const float inv_sc = 1.0f / sc;

        for (int k = warp; k < nimg; k += BW) {
            const fsld_image_rec& R = S.recs[k];
            const int bimg = a.pairs[pstart + k];
            const int row = a.idx ? a.idx[bimg] : bimg;
            const float2* __restrict__ xrow = a.x + (size_t)row * n;
            const Frame F = frame_of(R);
            // candidate rows: py = c . r1 over the brick box, +-1
            const float h = 0.5f * BT;
            const float cyc = (ox + h) * F.r1x + (oy + h) * F.r1y + (oz + h) * F.r1z;
            const float ext = h * (fabsf(F.r1x) + fabsf(F.r1y) + fabsf(F.r1z)) + 1.0f;
            const int rlim = (int)sqrtf((float)a.hdr->rmax2) + 1;
            const int pylo = max((int)floorf(cyc - ext), -rlim);
            const int pyhi = min((int)ceilf(cyc + ext), rlim);
            const int nrows = pyhi - pylo + 1;  // <= 2*(BT*sqrt(3)/2 + 1) + 2 < 32
            int lo = 0, cntr = 0;
            if (lane < nrows) {
                const int py = pylo + lane;
                float flo = -1e30f, fhi = 1e30f;
                bool empty = (py + c) < 0 || (py + c) >= M;
                const float r0[3] = {F.r0x, F.r0y, F.r0z};
                const float r1[3] = {F.r1x, F.r1y, F.r1z};
                const float o3[3] = {(float)ox, (float)oy, (float)oz};
#pragma unroll
                for (int ax = 0; ax < 3; ++ax) {
                    const float base = (float)py * r1[ax];
                    if (fabsf(r0[ax]) > 1e-4f) {
                        const float inv = 1.0f / r0[ax];
                        const float t0 = (o3[ax] - base) * inv, t1 = (o3[ax] + BT - base) * inv;
                        flo = fmaxf(flo, fminf(t0, t1));
                        fhi = fminf(fhi, fmaxf(t0, t1));
                    } else if (base < o3[ax] - 0.02f || base > o3[ax] + BT + 0.02f) {
                        empty = true;
                    }
                }
                if (!empty && flo <= fhi + 2.0f) {
                    int ilo = (int)floorf(flo) - 1, ihi = (int)ceilf(fhi) + 1;
                    ilo = max(ilo, a.rowmin[py + c]);
                    ihi = min(ihi, a.rowmax[py + c]);
                    if (ihi >= ilo) {
                        lo = ilo;
                        cntr = ihi - ilo + 1;
                    }
                }
            }
            // exclusive scan of row counts
            int incl = cntr;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const int total = min(__shfl_sync(0xffffffffu, incl, 31), BMAXCAND);
            const int start = incl - cntr;
            for (int i = 0; i < cntr && start + i < BMAXCAND; ++i) S.rowof[warp][start + i] = (unsigned char)lane;
            __syncwarp();

            float sq = 0.f;
            for (int base = 0; base < total; base += 32) {
                const int i = base + lane;
                const bool valid = i < total;
                const int r = valid ? (int)S.rowof[warp][i] : 0;
                const int rlo = __shfl_sync(0xffffffffu, lo, r);
                const int rst = __shfl_sync(0xffffffffu, start, r);
                if (!valid) continue;
                const int py = pylo + r;
                const int px = rlo + (i - rst);
                const int p = __ldg(a.pix2p + (py + c) * M + (px + c));
                if (p < 0) continue;
                const float fpx = (float)px, fpy = (float)py;
                float cx = fmaf(fpx, F.r0x, fpy * F.r1x);
                float cy = fmaf(fpx, F.r0y, fpy * F.r1y);
                float cz = fmaf(fpx, F.r0z, fpy * F.r1z);
                cx = fminf(fmaxf(cx, -bnd), bnd);
                cy = fminf(fmaxf(cy, -bnd), bnd);
                cz = fminf(fmaxf(cz, -bnd), bnd);
                const float fx = floorf(cx), fy = floorf(cy), fz = floorf(cz);
                const int lx = (int)fx - ox, ly = (int)fy - oy, lz = (int)fz - oz;
                if ((unsigned)lx >= (unsigned)BT || (unsigned)ly >= (unsigned)BT || (unsigned)lz >= (unsigned)BT)
                    continue;  // owned by another brick
                const float wx = cx - fx, wy = cy - fy, wz = cz - fz;
                const float ax = 1.f - wx, ay = 1.f - wy, az = 1.f - wz;
                const float2 xv = __ldg(xrow + p);
                const float2 f = pixel_factor(R, px, py);
                const int l0 = (lz * BH + ly) * BH + lx;
                const float2* vb = S.vb + l0;
                // trilinear gather (kernels.py:171-176) from the smem brick
                float2 e0 = __ffma2_rn(make_float2(wx, wx), vb[1], __fmul2_rn(make_float2(ax, ax), vb[0]));
                float2 e1 = __ffma2_rn(make_float2(wx, wx), vb[BH + 1], __fmul2_rn(make_float2(ax, ax), vb[BH]));
                float2 e2 = __ffma2_rn(make_float2(wx, wx), vb[BH * BH + 1], __fmul2_rn(make_float2(ax, ax), vb[BH * BH]));
                float2 e3 = __ffma2_rn(make_float2(wx, wx), vb[BH * BH + BH + 1],
                                       __fmul2_rn(make_float2(ax, ax), vb[BH * BH + BH]));
                const float2 q0 = __ffma2_rn(make_float2(wy, wy), e1, __fmul2_rn(make_float2(ay, ay), e0));
                const float2 q1 = __ffma2_rn(make_float2(wy, wy), e3, __fmul2_rn(make_float2(ay, ay), e2));
                const float2 pv = __ffma2_rn(make_float2(wz, wz), q1, __fmul2_rn(make_float2(az, az), q0));
                const float2 pr = cmul(pv, f);
                const float2 rr = make_float2(pr.x - xv.x, pr.y - xv.y);
                sq = fmaf(rr.x, rr.x, fmaf(rr.y, rr.y, sq));
                float2 val = cmulconj(f, rr);
                val = __fmul2_rn(val, make_float2(sc, sc));
                // adjoint scatter into the smem brick (kernels.py:221-230), fixed point
                const float zy00 = az * ay, zy10 = az * wy, zy01 = wz * ay, zy11 = wz * wy;
                const float w8[8] = {zy00 * ax, zy00 * wx, zy10 * ax, zy10 * wx,
                                     zy01 * ax, zy01 * wx, zy11 * ax, zy11 * wx};
                const int off8[8] = {0, 1, BH, BH + 1, BH * BH, BH * BH + 1, BH * BH + BH, BH * BH + BH + 1};
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    atomicAdd(S.accr + l0 + off8[q], to_fixed(w8[q] * val.x));
                    atomicAdd(S.acci + l0 + off8[q], to_fixed(w8[q] * val.y));
                }
            }
            for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
            if (lane == 0) lsum += (double)sq;
            __syncwarp();
        }
        __syncthreads();
        // flush: one vector reduction per touched brick voxel
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
    }
    // per-CTA loss partial (fixed slot)
    if (lane == 0) S.red[warp] = lsum;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < BW; ++w) s += S.red[w];
        a.part[blockIdx.x] = bad_geom ? __longlong_as_double(0x7ff8000000000000ll) : s;
    }
}

static int g_brick_grid = 0;

cudaError_t launch_brick_loss_grad(const BrickArgs& a, double* sq_out, cudaStream_t s) {
    const size_t smem = sizeof(BrickSmem);
    if (g_brick_grid == 0) {
        cudaError_t e = cudaFuncSetAttribute(brick_loss_grad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        int dev = 0, sms = 0, occ = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, brick_loss_grad_kernel, BTHREADS, smem);
        g_brick_grid = sms * (occ > 0 ? occ : 1);
    }
    cudaError_t e = cudaMemsetAsync(a.cnt, 0, sizeof(int) * (size_t)a.nbr, s);
    if (e != cudaSuccess) return e;
    brick_bin_kernel<false><<<a.B, 256, 0, s>>>(a);
    brick_scan_kernel<<<1, 1024, 0, s>>>(a);
    brick_bin_kernel<true><<<a.B, 256, 0, s>>>(a);
    const int grid = g_brick_grid;
    brick_loss_grad_kernel<<<grid, BTHREADS, smem, s>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_reduce(a.part, grid, sq_out, s);
}

}  // namespace fsld
