// Host<->device transfer probe: copy-engine cudaMemcpyAsync vs kernels reading / writing pinned
// host memory directly (zero-copy over PCIe), each direction alone and both at once.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a zc_probe.cu -o zc_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void copy16(const int4* __restrict__ src, int4* __restrict__ dst, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

int main() {
    const size_t bytes = 128ull * 128 * 128 * 8, n = bytes / 16;
    void *h1, *h2, *d1, *d2;
    cudaHostAlloc(&h1, bytes, cudaHostAllocDefault);
    cudaHostAlloc(&h2, bytes, cudaHostAllocDefault);
    cudaMalloc(&d1, bytes);
    cudaMalloc(&d2, bytes);
    memset(h1, 1, bytes);
    memset(h2, 2, bytes);
    cudaStream_t s1, s2;
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char* name, auto fn) {
        for (int i = 0; i < 3; ++i) fn();
        cudaDeviceSynchronize();
        cudaEventRecord(a, 0);
        for (int i = 0; i < 20; ++i) fn();
        cudaEventRecord(b, 0);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 20;
        printf("%-28s %.4f ms  %.1f GB/s per direction\n", name, ms, bytes / ms / 1e6);
    };
    auto join = [&]() {
        cudaEvent_t e1, e2;
        cudaEventCreateWithFlags(&e1, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&e2, cudaEventDisableTiming);
        cudaEventRecord(e1, s1);
        cudaEventRecord(e2, s2);
        cudaStreamWaitEvent(0, e1, 0);
        cudaStreamWaitEvent(0, e2, 0);
        cudaEventDestroy(e1);
        cudaEventDestroy(e2);
    };
    auto fork = [&]() {
        cudaEvent_t e;
        cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        cudaEventRecord(e, 0);
        cudaStreamWaitEvent(s1, e, 0);
        cudaStreamWaitEvent(s2, e, 0);
        cudaEventDestroy(e);
    };
    for (int blocks : {148, 296, 592, 1184}) {
        char nm[64];
        snprintf(nm, 64, "kernel h2d (%d CTAs)", blocks);
        run(nm, [&]() { copy16<<<blocks, 512>>>((const int4*)h1, (int4*)d1, n); });
        snprintf(nm, 64, "kernel d2h (%d CTAs)", blocks);
        run(nm, [&]() { copy16<<<blocks, 512>>>((const int4*)d2, (int4*)h2, n); });
    }
    run("memcpy h2d", [&]() { cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice, 0); });
    run("memcpy d2h", [&]() { cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, 0); });
    run("memcpy both", [&]() {
        fork();
        cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice, s1);
        cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, s2);
        join();
    });
    run("kernel both (2x296 CTAs)", [&]() {
        fork();
        copy16<<<296, 512, 0, s1>>>((const int4*)h1, (int4*)d1, n);
        copy16<<<296, 512, 0, s2>>>((const int4*)d2, (int4*)h2, n);
        join();
    });
    run("memcpy h2d + kernel d2h", [&]() {
        fork();
        cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice, s1);
        copy16<<<296, 512, 0, s2>>>((const int4*)d2, (int4*)h2, n);
        join();
    });
    run("kernel h2d + memcpy d2h", [&]() {
        fork();
        copy16<<<296, 512, 0, s1>>>((const int4*)h1, (int4*)d1, n);
        cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, s2);
        join();
    });
    printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
