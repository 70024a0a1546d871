// fsld_hutch.cu -- Hutchinson probe batcher for sm_100a.
//
// The reference estimates diag(H) one probe per batch: hvp(z) =
// (N/|B|) sum_i P_i^* C_i^2 P_i z + lam z, then z * Re(hvp(z)) is folded into
// a running mean (optim.py:210-229, forward.py:554-570).  Here k probes are
// bit-packed (1 bit per voxel per probe) and folded inside one pass:
//
//   acc[j] += sum_p z_p[j] (A^*A z_p)[j]
//          = sum_pixels C^2 w_j sum_c' w_c' Q(j, c'),   Q(c, c') = sum_p z_p[c] z_p[c']
//
// and Q(c, c') = k - 2 popc(bits[c] ^ bits[c']) for +-1 probes.  So a pass
// costs 8 corner-word loads per pixel and ONE scatter per corner regardless
// of k (the volume is streamed once per batch of probes).  nn mode collapses
// to acc[j] += k C^2 (the estimator is exact).
#include "fsld_kernels.cuh"

namespace fsld {

template <int MODE, bool DET>
__global__ void __launch_bounds__(kThreads) hutch_kernel(SliceArgs a, const uint32_t* __restrict__ zbits,
                                                         int words, int k) {
    __shared__ fsld_image_rec rec;
    const int b = blockIdx.x / a.tiles;
    const int tile = blockIdx.x - b * a.tiles;
    load_record(a.recs, a.idx ? a.idx[b] : b, &rec);
    __syncthreads();
    const double fx = DET ? *a.fx : 0.0;
    const float kf = (float)k;
    const int p0 = tile * a.ppt * kThreads + threadIdx.x;
    for (int it = 0; it < a.ppt; ++it) {
        const int p = p0 + it * kThreads;
        if (p >= a.n_mask) break;
        const short2 kk = __ldg(a.pix + p);
        double cx, cy, cz;
        rotate_pixel(rec.rot, (double)kk.x, (double)kk.y, a.bnd, cx, cy, cz);
        const float c2v = ctf_sq(rec, kk.x, kk.y);
        if (MODE == FSLD_MODE_NN) {
            scatter_r<DET>(a.acc, nn_index(cx, cy, cz, a.M, a.c2), kf * c2v, fx);
            continue;
        }
        Tri t;
        tri_setup(cx, cy, cz, a.M, a.c2, t);
        float w[8];
        tri_weights(t, w);
        // d[c][c'] = popc over words of bits[c] ^ bits[c'], c < c'
        int d[8][8];
#pragma unroll
        for (int c = 0; c < 8; ++c)
#pragma unroll
            for (int e = 0; e < 8; ++e) d[c][e] = 0;
        for (int wd = 0; wd < words; ++wd) {
            uint32_t z[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) z[c] = __ldg(zbits + (size_t)t.j[c] * words + wd);
#pragma unroll
            for (int c = 0; c < 8; ++c)
#pragma unroll
                for (int e = c + 1; e < 8; ++e) d[c][e] += __popc(z[c] ^ z[e]);
        }
        float wsum = 0.f;
#pragma unroll
        for (int c = 0; c < 8; ++c) wsum += w[c];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            float s = 0.f;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                if (e == c) continue;
                const int dd = c < e ? d[c][e] : d[e][c];
                s = fmaf(w[e], (float)dd, s);
            }
            // sum_c' w_c' Q(c,c') = k * sum w - 2 * sum_c' w_c' d(c,c')
            const float S = kf * wsum - 2.0f * s;
            scatter_r<DET>(a.acc, t.j[c], c2v * w[c] * S, fx);
        }
    }
}

cudaError_t launch_hutch(int mode, bool det, const SliceArgs& a, int nblocks, const uint32_t* zbits, int words,
                         int k, cudaStream_t s) {
    if (mode == FSLD_MODE_TRI) {
        if (det) hutch_kernel<FSLD_MODE_TRI, true><<<nblocks, kThreads, 0, s>>>(a, zbits, words, k);
        else hutch_kernel<FSLD_MODE_TRI, false><<<nblocks, kThreads, 0, s>>>(a, zbits, words, k);
    } else {
        if (det) hutch_kernel<FSLD_MODE_NN, true><<<nblocks, kThreads, 0, s>>>(a, zbits, words, k);
        else hutch_kernel<FSLD_MODE_NN, false><<<nblocks, kThreads, 0, s>>>(a, zbits, words, k);
    }
    return cudaGetLastError();
}

// z: (k, n) float64 +-1 -> zbits (n, words); one thread per (voxel, word).
__global__ void pack_probes_kernel(int64_t n, int k, int words, const double* __restrict__ z,
                                   uint32_t* __restrict__ zbits, int* bad) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= n * words) return;
    const int64_t j = tid / words;
    const int wd = (int)(tid - j * words);
    uint32_t bitsv = 0;
    int err = 0;
    for (int q = 0; q < 32; ++q) {
        const int p = wd * 32 + q;
        if (p >= k) break;
        const double zv = z[(size_t)p * n + j];
        if (zv == 1.0) bitsv |= 1u << q;
        else if (zv != -1.0) err = 1;
    }
    zbits[tid] = bitsv;
    if (err && bad) atomicOr(bad, 1);
}

cudaError_t launch_pack_probes(int64_t n, int k, const double* z, uint32_t* zbits, int* bad, cudaStream_t s) {
    const int words = (k + 31) / 32;
    const int64_t tot = n * words;
    pack_probes_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(n, k, words, z, zbits, bad);
    return cudaGetLastError();
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// Counter-based Rademacher probes (seed, voxel, word) -> 32 sign bits; unused
// bits of the last word are zero (required by the popcount identity).
__global__ void gen_probes_kernel(int64_t n, int k, int words, uint64_t seed, uint32_t* __restrict__ zbits) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= n * words) return;
    const int wd = words == 1 ? 0 : (int)((uint32_t)tid % (uint32_t)words);  // n * words < 2^32
    uint32_t bitsv = (uint32_t)splitmix64(seed ^ splitmix64((uint64_t)tid));
    const int valid = k - wd * 32;
    if (valid < 32) bitsv &= (1u << valid) - 1u;
    zbits[tid] = bitsv;
}

cudaError_t launch_gen_probes(int64_t n, int k, uint64_t seed, uint32_t* zbits, cudaStream_t s) {
    const int words = (k + 31) / 32;
    const int64_t tot = n * words;
    gen_probes_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(n, k, words, seed, zbits);
    return cudaGetLastError();
}

}  // namespace fsld
