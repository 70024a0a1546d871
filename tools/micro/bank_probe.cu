// Shared-memory bank model probe: one warp issues ATOMS.ADD / LDS.32 / LDS.64 at word index
// lane * stride (+ perm) for several strides; read the wavefronts per instruction with ncu
// (l1tex__data_pipe_lsu_wavefronts_mem_shared_op_{atom,ld}.sum / smsp__inst_executed_op_shared_*).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a bank_probe.cu -o bank_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int STRIDE>
__global__ void atoms_probe(int* out, int reps) {
    __shared__ int s[32 * 64 + 64];
    for (int i = threadIdx.x; i < 32 * 64 + 64; i += blockDim.x) s[i] = 0;
    __syncthreads();
    const int a = (threadIdx.x * STRIDE) % (32 * 64);
    for (int r = 0; r < reps; ++r) atomicAdd(&s[a], r);
    __syncthreads();
    out[threadIdx.x] = s[threadIdx.x];
}

template <int STRIDE>
__global__ void lds64_probe(float* out, int reps) {
    __shared__ float2 s[32 * 64 + 64];
    for (int i = threadIdx.x; i < 32 * 64 + 64; i += blockDim.x) s[i] = make_float2(i, i);
    __syncthreads();
    int a = (threadIdx.x * STRIDE) % (32 * 64);
    float acc = 0.f;
    for (int r = 0; r < reps; ++r) {
        const float2 v = s[a];
        acc += v.x + v.y;
        a ^= (int)(acc == 12345.f);  // keep the load in the loop
    }
    out[threadIdx.x] = acc;
}

int main() {
    int* o;
    cudaMalloc(&o, 4096);
    const int reps = 1000;
    atoms_probe<1><<<1, 32>>>(o, reps);
    atoms_probe<2><<<1, 32>>>(o, reps);
    atoms_probe<3><<<1, 32>>>(o, reps);
    atoms_probe<4><<<1, 32>>>(o, reps);
    atoms_probe<32><<<1, 32>>>(o, reps);
    lds64_probe<1><<<1, 32>>>((float*)o, reps);
    lds64_probe<2><<<1, 32>>>((float*)o, reps);
    lds64_probe<3><<<1, 32>>>((float*)o, reps);
    lds64_probe<16><<<1, 32>>>((float*)o, reps);
    cudaDeviceSynchronize();
    printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
