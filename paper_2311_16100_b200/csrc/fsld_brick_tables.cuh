// fsld_brick_tables.cuh -- per-pixel invariants of a brick-sorted dataset (included by fsld_brick.cu).
//
// Poses, shifts and CTFs are fixed for a refinement run (optim.run never changes them), so
// everything a pixel contributes besides its observed value and the volume is a constant of
// the dataset -- the reference itself keeps per-(image, pixel) phase and CTF tables for the whole
// dataset (forward.py:524-527, 24 B per pixel in fp64).  fsld_sorted_tables evaluates them once,
// in fp64, in the brick-sorted pixel order, as two arrays (structure of arrays, so a warp's
// loads are dense: 8 + 16 bytes per pixel):
//   f   : C(k) * exp(i pi shift.k) as fp32 complex (forward.py:93-111, 299-312)
//   geo : float4 -- the trilinear footprint of the clamped rotated pixel (kernels.py:42-60,
//         147-170) in the frame of the brick that owns it: the fractional weights (wx, wy, wz)
//         = c - floor(c) rounded from fp64 to fp32, and the floor-corner index
//         l0 = lx + 9 ly + 81 lz in the 9^3 (+halo) shared-memory brick (int bits).
// Layout of the table buffer: a 256-byte header {magic, N * n_mask}, then f[N * n_mask], then
// geo[N * n_mask] (tables_bytes).
// The rotated coordinates use the reference's arithmetic (fp64, separately rounded products,
// clamp), so floors and weights are the reference's up to the final fp32 rounding (the compute
// path's fp32 coordinates carry up to ~4e-6 voxel at |c| = 64).  The owning brick comes from the
// sort (fsld_sorted_fill, fp32 floors); where the fp32 and fp64 floors straddle a brick face (a
// coordinate within ~1e-6 of a multiple of 8) the corner is clamped into the owning brick and the
// weight saturates at 0 or 1 -- the same point up to < 1e-6 voxel.
#pragma once

constexpr uint32_t kTabMagic = 0xF51D7AB5u;
struct TabHeader {
    uint32_t magic, pad;
    long long npx;  // N * n_mask
};

// f[] is padded to an even count so that geo[] starts 16-byte aligned; 256 bytes of slack at the end
// (L2 prefetches round their ranges out to 16-byte granules)
__host__ __device__ inline size_t tables_bytes(long long npx) {
    return 256 + (size_t)((npx + 1) & ~1ll) * 8 + (size_t)npx * 16 + 256;
}
__device__ __forceinline__ const float2* tab_f(const void* ptab) {
    return reinterpret_cast<const float2*>(reinterpret_cast<const char*>(ptab) + 256);
}
__device__ __forceinline__ const float4* tab_geo(const void* ptab, long long npx) {
    return reinterpret_cast<const float4*>(reinterpret_cast<const char*>(ptab) + 256 + 8 * ((npx + 1) & ~1ll));
}

__device__ __forceinline__ float geo_weight(double w) {
    const float f = (float)w;
    return f < 0.f ? 0.f : (f > 1.f ? 1.f : f);
}

// One CTA per image, one warp per segment (lanes over its pixels).
__global__ void __launch_bounds__(256) sorted_tables_kernel(int M, int n_mask, int nn,
                                                            const fsld_image_rec* __restrict__ recs,
                                                            const char2* __restrict__ pc,
                                                            const int32_t* __restrict__ seg_off,
                                                            const int2* __restrict__ segs, void* __restrict__ ptab,
                                                            long long npx) {
    __shared__ fsld_image_rec R;
    const int i = blockIdx.x;
    float2* tf = const_cast<float2*>(tab_f(ptab));
    float4* tg = const_cast<float4*>(tab_geo(ptab, npx));
    if (i == 0 && threadIdx.x == 0) {
        TabHeader* h = reinterpret_cast<TabHeader*>(ptab);
        h->magic = kTabMagic;
        h->pad = 0;
        h->npx = npx;
    }
    load_record(recs, i, &R);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c = (M + 1) / 2, nb = (M + BT - 1) / BT;
    const double bnd = (double)(M / 2 - 1);
    const size_t row = (size_t)i * n_mask;
    for (int s = seg_off[i] + warp; s < seg_off[i + 1]; s += BW) {
        const int2 sg = segs[s];
        const int start = sg.y & 0xFFFF, len = sg.y >> 16, bid = sg.x;
        const int ox = -c + BT * (bid % nb), oy = -c + BT * ((bid / nb) % nb), oz = -c + BT * (bid / (nb * nb));
        for (int e = lane; e < len; e += 32) {
            const char2 k = pc[row + start + e];
            double cx, cy, cz;
            rotate_pixel(R.rot, (double)k.x, (double)k.y, bnd, cx, cy, cz);
            const int lx = min(max((int)floor(cx) - ox, 0), BT - 1);
            const int ly = min(max((int)floor(cy) - oy, 0), BT - 1);
            const int lz = min(max((int)floor(cz) - oz, 0), BT - 1);
            const size_t g = row + start + e;
            tf[g] = pixel_factor(R, (int)k.x, (int)k.y);
            if (nn) {  // the nn voxel j -> (kx, ky, kz) -> the brick frame
                const int j = nn_index(cx, cy, cz, M, c);
                const int x = j % M, y = (j / M) % M, zi = j / (M * M);
                const int nx = min(max(x - c - ox, 0), BH - 1), ny = min(max(y - c - oy, 0), BH - 1);
                const int nz = min(max((zi < M - c ? zi : zi - M) - oz, 0), BH - 1);
                tg[g] = make_float4(0.f, 0.f, 0.f, __int_as_float((nz * BH + ny) * BH + nx));
            } else {
                tg[g] = make_float4(geo_weight(cx - (double)(ox + lx)), geo_weight(cy - (double)(oy + ly)),
                                    geo_weight(cz - (double)(oz + lz)), __int_as_float((lz * BH + ly) * BH + lx));
            }
        }
    }
}
