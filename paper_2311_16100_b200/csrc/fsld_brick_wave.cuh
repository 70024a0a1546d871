// fsld_brick_wave.cuh -- one-time "wave" ordering of each brick segment (included by fsld_brick.cu).
//
// Within one image, several pixels can share a floor voxel (their 2x2x2
// footprints coincide).  If two such pixels sit in the same warp when the
// brick kernel adds their contributions to shared memory, the two lanes hit
// the same addresses and their shared atomics serialise.  Reordering every
// segment by "wave" -- the rank of a pixel among the pixels of its image with
// the same floor voxel -- puts pixels with distinct floor voxels next to each
// other.  Order is irrelevant to the result (an order-free integer sum), only
// to speed.
#pragma once

__global__ void __launch_bounds__(256) wave_order_kernel(int M, int n_mask, const fsld_image_rec* __restrict__ recs,
                                                         float2* xs, char2* pc, const int32_t* __restrict__ seg_off,
                                                         const int2* __restrict__ segs) {
    __shared__ int cnt[BW][BT * BT * BT];
    __shared__ float frs[6];
    const int i = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c = (M + 1) / 2, nb = (M + BT - 1) / BT;
    const float bnd = (float)(M / 2 - 1);
    if (threadIdx.x < 6) frs[threadIdx.x] = (float)recs[i].rot[threadIdx.x];
    for (int q = lane; q < BT * BT * BT; q += 32) cnt[warp][q] = 0;
    __syncthreads();
    float fr[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) fr[q] = frs[q];
    const size_t row = (size_t)i * n_mask;
    constexpr int U = 4;  // 4 x 32 >= BOWN_MAX pixels per segment
    for (int s = seg_off[i] + warp; s < seg_off[i + 1]; s += BW) {
        const int2 seg = segs[s];
        const int start = seg.y & 0xFFFF, len = seg.y >> 16;
        const int bid = seg.x;
        const int ox = -c + BT * (bid % nb), oy = -c + BT * ((bid / nb) % nb), oz = -c + BT * (bid / (nb * nb));
        char2 kk[U];
        float2 xv[U];
        int lv[U], wv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = lane + 32 * u;
            wv[u] = -1;
            lv[u] = 0;
            if (e < len) {
                kk[u] = pc[row + start + e];
                if (xs) xv[u] = xs[row + start + e];
                float cx, cy, cz, fx, fy, fz;
                floor_corner((float)kk[u].x, (float)kk[u].y, fr, bnd, cx, cy, cz, fx, fy, fz);
                lv[u] = (((int)fz - oz) * BT + ((int)fy - oy)) * BT + ((int)fx - ox);
                wv[u] = min(atomicAdd(&cnt[warp][lv[u]], 1), 3);
            }
        }
        __syncwarp();
        // counting sort of the segment by wave, stable in (u, lane) order
        int base[4];
        int run = 0;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            base[w] = run;
#pragma unroll
            for (int u = 0; u < U; ++u) run += __popc(__ballot_sync(0xffffffffu, wv[u] == w));
        }
        int seen[4] = {0, 0, 0, 0};
#pragma unroll
        for (int u = 0; u < U; ++u) {
            int pos = -1;
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const unsigned bw = __ballot_sync(0xffffffffu, wv[u] == w);
                if (wv[u] == w) pos = base[w] + seen[w] + __popc(bw & ((1u << lane) - 1u));
                seen[w] += __popc(bw);
            }
            if (pos >= 0) {
                pc[row + start + pos] = kk[u];
                if (xs) xs[row + start + pos] = xv[u];
                cnt[warp][lv[u]] = 0;
            }
        }
        __syncwarp();
    }
}
