// fsld_metrics.cu -- the per-epoch metric and the ingest step of the path as kernels.
//
//   fsc_kernel       : Fourier shell correlation (metrics.py:38-63): per shell r of rounded radius
//                      <= R, sums Re(u conj(v)), |u|^2, |v|^2 in fp64.  One pass over the volume;
//                      each CTA accumulates its voxels per shell in shared memory, writes its own
//                      partial row, and one small kernel adds the rows in CTA order.
//   mask_images_kernel: FSD1 ingest (io.py:91-125): full M^2 complex128 images -> the compact masked
//                      complex64 rows of the dataset (x = images[:, mask], forward.py:527).
#include "fsld_kernels.cuh"

namespace fsld {

constexpr int kFscThreads = 256;

// Shell of voxel j: rounded |k| (grid.py:241-257; the rounding of np.round, half to even).
__device__ __forceinline__ int voxel_shell(int64_t j, int M) {
    const int c = (M + 1) / 2;
    const int x = (int)(j % M), y = (int)((j / M) % M), zi = (int)(j / ((int64_t)M * M));
    const int kx = x - c, ky = y - c, kz = zi < M - c ? zi : zi - M;
    const double r = sqrt((double)(kx * kx + ky * ky + kz * kz));
    return (int)rint(r);
}

__global__ void __launch_bounds__(kFscThreads) fsc_kernel(int M, int R, const float2* __restrict__ u,
                                                          const float2* __restrict__ v, double* __restrict__ part) {
    extern __shared__ double acc[];  // 3 (R + 1)
    const int nsh = R + 1;
    for (int t = threadIdx.x; t < 3 * nsh; t += blockDim.x) acc[t] = 0.0;
    __syncthreads();
    const int64_t n = (int64_t)M * M * M;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const int s = voxel_shell(j, M);
        if (s > R) continue;
        const float2 a = u[j], b = v[j];
        atomicAdd(acc + s, (double)a.x * b.x + (double)a.y * b.y);
        atomicAdd(acc + nsh + s, (double)a.x * a.x + (double)a.y * a.y);
        atomicAdd(acc + 2 * nsh + s, (double)b.x * b.x + (double)b.y * b.y);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 3 * nsh; t += blockDim.x) part[(size_t)blockIdx.x * 3 * nsh + t] = acc[t];
}

__global__ void fsc_reduce_kernel(const double* __restrict__ part, int nrows, int ncols, double* __restrict__ out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ncols) return;
    double s = 0.0;
    for (int r = 0; r < nrows; ++r) s += part[(size_t)r * ncols + t];  // fixed order
    out[t] = s;
}

int fsc_grid() { return 148 * 2; }

cudaError_t launch_fsc(int M, int R, const float2* u, const float2* v, double* part, double* out, cudaStream_t s) {
    const int grid = fsc_grid(), ncols = 3 * (R + 1);
    fsc_kernel<<<grid, kFscThreads, sizeof(double) * ncols, s>>>(M, R, u, v, part);
    fsc_reduce_kernel<<<(ncols + 127) / 128, 128, 0, s>>>(part, grid, ncols, out);
    return cudaGetLastError();
}

// One CTA row-chunk per (image, 256 mask entries): coalesced reads of the mask table, gathered
// 16-byte reads of the complex128 pixels, coalesced 8-byte writes.
__global__ void mask_images_kernel(int M, int n_mask, const int32_t* __restrict__ mask, int N,
                                   const double2* __restrict__ in, float2* __restrict__ out) {
    const int i = blockIdx.y;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N || p >= n_mask) return;
    const double2 z = in[(size_t)i * M * M + mask[p]];
    out[(size_t)i * n_mask + p] = make_float2((float)z.x, (float)z.y);
}

cudaError_t launch_mask_images(int M, int n_mask, const int32_t* mask, int N, const void* in, void* out,
                               cudaStream_t s) {
    if (N < 1) return cudaSuccess;
    dim3 grid((n_mask + 255) / 256, N);
    mask_images_kernel<<<grid, 256, 0, s>>>(M, n_mask, mask, N, reinterpret_cast<const double2*>(in),
                                           reinterpret_cast<float2*>(out));
    return cudaGetLastError();
}

// Mean over the pixels of one ring (rounded radius R) of each image's squared CTF, fp64 throughout
// (threshold_alpha's sum_i |C_i(R)|^2 for a non-radial CTF; optim.py:250-266): one CTA per image.
__global__ void __launch_bounds__(128) ctf_ring_power_kernel(const fsld_image_rec* __restrict__ recs, int N,
                                                             const short2* __restrict__ ring, int n_ring,
                                                             double* __restrict__ out) {
    __shared__ double red[4];
    const int i = blockIdx.x;
    const fsld_image_rec& R = recs[i];
    double s = 0.0;
    for (int p = threadIdx.x; p < n_ring; p += blockDim.x) {
        double c2 = 1.0;
        if (R.flags & FSLD_REC_CTF) {
            const double kx = ring[p].x, ky = ring[p].y, k2 = kx * kx + ky * ky;
            const double g = R.gamma[0] * k2 + R.gamma[1] * (kx * kx - ky * ky) + R.gamma[2] * (2.0 * kx * ky) +
                             R.gamma[3] * k2 * k2;
            const double c = -((double)R.wsin * sin(g) + (double)R.wcos * cos(g)) * exp(-R.env * k2);
            c2 = c * c;
        }
        s += c2;
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) out[i] = (red[0] + red[1] + red[2] + red[3]) / (double)n_ring;
}

cudaError_t launch_ctf_ring_power(const fsld_image_rec* recs, int N, const short2* ring, int n_ring, double* out,
                                  cudaStream_t s) {
    if (N < 1) return cudaSuccess;
    ctf_ring_power_kernel<<<N, 128, 0, s>>>(recs, N, ring, n_ring, out);
    return cudaGetLastError();
}

// complex64 -> complex128 (the numpy call path's gradient: cast on the device, copied out as complex128
// straight into the caller's array, so the host never casts it)
__global__ void cast_c64_c128_kernel(int64_t n, const float2* __restrict__ src, double2* __restrict__ dst) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float2 z = src[i];
        dst[i] = make_double2((double)z.x, (double)z.y);
    }
}

cudaError_t launch_cast_c64_c128(int64_t n, const void* src, void* dst, cudaStream_t s) {
    if (n < 1) return cudaSuccess;
    const int64_t blocks = (n + 255) / 256;
    cast_c64_c128_kernel<<<(int)(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, s>>>(
        n, reinterpret_cast<const float2*>(src), reinterpret_cast<double2*>(dst));
    return cudaGetLastError();
}

}  // namespace fsld
