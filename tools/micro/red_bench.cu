// Microbenchmark: L2 reduction throughput of red.global.add.{f32, v2.f32, v4.f32} on B200.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void red1(float* a, float x) { asm volatile("red.global.add.f32 [%0], %1;" ::"l"(a), "f"(x) : "memory"); }
__device__ __forceinline__ void red2(float* a, float x, float y) { asm volatile("red.global.add.v2.f32 [%0], {%1,%2};" ::"l"(a), "f"(x), "f"(y) : "memory"); }
__device__ __forceinline__ void red4(float* a, float x, float y, float z, float w) { asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(a), "f"(x), "f"(y), "f"(z), "f"(w) : "memory"); }
__device__ __forceinline__ unsigned hash(unsigned x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
// mode: 0 = v2 random, 1 = v4 random (16B aligned), 2 = f32 random, 3 = v2 "row" locality (lane-consecutive), 4 = v4 row
__global__ void kern(float* buf, int nelem2, int iters, int mode) {
    unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        unsigned r = hash(t * 131 + i * 7919);
        if (mode == 0) { unsigned j = r % nelem2; red2(buf + 2 * j, 1.f, 1.f); }
        else if (mode == 1) { unsigned j = (r % (nelem2 / 2)) * 2; red4(buf + 2 * j, 1.f, 1.f, 1.f, 1.f); }
        else if (mode == 2) { unsigned j = r % (2 * nelem2); red1(buf + j, 1.f); }
        else if (mode == 3) { unsigned j = (hash(t / 32 * 131 + i * 7919) % (nelem2 - 64)) + (threadIdx.x & 31); red2(buf + 2 * j, 1.f, 1.f); }
        else { unsigned j = ((hash(t / 32 * 131 + i * 7919) % (nelem2 / 2 - 64)) + (threadIdx.x & 31)) * 2; red4(buf + 2 * j, 1.f, 1.f, 1.f, 1.f); }
    }
}
int main() {
    int M = 128, n2 = M * M * M;  // complex voxels
    float* buf; cudaMalloc(&buf, sizeof(float) * 2 * n2);
    cudaMemset(buf, 0, sizeof(float) * 2 * n2);
    int blocks = 148 * 8, threads = 256, iters = 64;
    const char* names[] = {"v2 random", "v4 random", "f32 random", "v2 lane-consecutive", "v4 lane-consecutive"};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int mode = 0; mode < 5; ++mode) {
        kern<<<blocks, threads>>>(buf, n2, iters, mode);
        cudaEventRecord(e0);
        kern<<<blocks, threads>>>(buf, n2, iters, mode);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double ops = (double)blocks * threads * iters;
        printf("%-22s %8.3f ms  %8.1f Gops/s\n", names[mode], ms, ops / ms / 1e6);
    }
    return 0;
}
