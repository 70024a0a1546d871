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

#ifndef FSLD_BANK_LEVELS  // rank levels of the bank order (ranks beyond the last share it)
#define FSLD_BANK_LEVELS 8
#endif
#ifndef FSLD_BANK_ORDER  // 1: order segments by (rank within bank, bank); 0: by wave (same floor voxel rank)
#define FSLD_BANK_ORDER 1
#endif

__global__ void __launch_bounds__(256) wave_order_kernel(int M, int n_mask, const fsld_image_rec* __restrict__ recs,
                                                         float2* xs, char2* pc, const int32_t* __restrict__ seg_off,
                                                         const int2* __restrict__ segs) {
    __shared__ int cnt[BW][BT * BT * BT];
#if FSLD_BANK_ORDER
    __shared__ int hist[BW][32 * FSLD_BANK_LEVELS];
    __shared__ int bank_cnt[BW][32];  // per-bank rank counters (own array: cnt still holds voxel counts)
#endif
    __shared__ float frs[6];
    const int i = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c = (M + 1) / 2, nb = (M + BT - 1) / BT;
    const float bnd = (float)(M / 2 - 1);
    if (threadIdx.x < 6) frs[threadIdx.x] = (float)recs[i].rot[threadIdx.x];
    for (int q = lane; q < BT * BT * BT; q += 32) cnt[warp][q] = 0;
#if FSLD_BANK_ORDER
    bank_cnt[warp][lane] = 0;
#endif
    __syncthreads();
    float fr[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) fr[q] = frs[q];
    const size_t row = (size_t)i * n_mask;
    constexpr int U = kSegMax / 32;  // segments hold <= kSegMax pixels (fsld_sorted_fill splits longer runs)
    for (int s = seg_off[i] + warp; s < seg_off[i + 1]; s += BW) {
        const int2 seg = segs[s];
        const int start = seg.y & 0xFFFF, len = seg.y >> 16;
        const int bid = seg.x;
        const int ox = -c + BT * (bid % nb), oy = -c + BT * ((bid / nb) % nb), oz = -c + BT * (bid / (nb * nb));
        char2 kk[U];
        float2 xv[U];
        int lv[U], wv[U], l9[U];
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
                l9[u] = (((int)fz - oz) * BH + ((int)fy - oy)) * BH + ((int)fx - ox);
                wv[u] = min(atomicAdd(&cnt[warp][lv[u]], 1), 3);
            }
        }
        __syncwarp();
#if FSLD_BANK_ORDER
        // counting sort of the segment by (rank among the segment's pixels in the same shared-memory
        // bank, bank): bank = 9-stride brick index of the floor voxel mod 32.  Every run of 32
        // consecutive pixels then takes at most one pixel per bank from each rank level, so a
        // warp's corner gathers (LDS.64) and scatters (ATOMS) see few bank conflicts; pixels with
        // the same floor voxel share a bank and land on different rank levels (the wave order's
        // property is kept).
        for (int q = lane; q < 32 * FSLD_BANK_LEVELS; q += 32) hist[warp][q] = 0;
        __syncwarp();
        int key[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {  // rank within the bank
            key[u] = -1;
            if (wv[u] >= 0) {
                const int bank = l9[u] & 31;
                key[u] = min(atomicAdd(&bank_cnt[warp][bank], 1), FSLD_BANK_LEVELS - 1) * 32 + bank;
            }
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (key[u] >= 0) atomicAdd(&hist[warp][key[u]], 1);
        __syncwarp();
        {  // exclusive scan of the 32 * FSLD_BANK_LEVELS counters, FSLD_BANK_LEVELS per lane
            constexpr int NL = FSLD_BANK_LEVELS;
            int h[NL], t = 0;
#pragma unroll
            for (int j = 0; j < NL; ++j) {
                h[j] = hist[warp][NL * lane + j];
                t += h[j];
            }
            int incl = t;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            int b = incl - t;
#pragma unroll
            for (int j = 0; j < NL; ++j) {
                hist[warp][NL * lane + j] = b;
                b += h[j];
            }
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (key[u] < 0) continue;
            const int pos = atomicAdd(&hist[warp][key[u]], 1);
            pc[row + start + pos] = kk[u];
            if (xs) xs[row + start + pos] = xv[u];
            cnt[warp][lv[u]] = 0;
        }
        __syncwarp();
        bank_cnt[warp][lane] = 0;
#else
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
#endif
        __syncwarp();
    }
}
