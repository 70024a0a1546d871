// Shared-memory pipe throughput per access pattern (cycles per warp-instruction per SM), B200.
// 148 x 4 CTAs of 256 threads; each lane holds 8 precomputed word addresses (pattern), loops
// REPS times over them.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a smem_tput.cu -o /tmp/smem_tput
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int REPS = 2048;

__device__ int pat_addr(int pat, int lane, int q, unsigned seed) {
    unsigned h = (seed * 2654435761u) ^ (lane * 40503u + q * 977u + 12345u);
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    switch (pat) {
        case 0: return lane + 32 * q;                          // conflict-free
        case 1: return (int)(h % 1024u);                        // random over 1024 words
        case 2: return (lane & 15) + 32 * (lane >> 4) + 64 * q; // 16 banks used twice: 2-way
        case 3: return 64 * q;                                  // all lanes one address
        case 4: return 2 * ((lane & 15) + 16 * q) + (lane >> 4);  // int2 re/im trick: halves take re / im
        case 5: return 2 * (lane + 32 * q);                     // int2 interleaved re only: 2-way
        case 6: return (int)(h % 16u) + 32 * q + 16 * (lane >> 4);  // random bank within 16, no same addr? (dups)
        default: return 0;
    }
}

__global__ void __launch_bounds__(256) atoms_k(int pat, int* out, unsigned seed) {
    __shared__ int s[4096];
    for (int i = threadIdx.x; i < 4096; i += 256) s[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = pat_addr(pat, lane, q, seed + w);
    for (int r = 0; r < REPS; ++r) {
#pragma unroll
        for (int q = 0; q < 8; ++q) atomicAdd(&s[a[q]], 1);
    }
    __syncthreads();
    out[blockIdx.x * 256 + threadIdx.x] = s[threadIdx.x];
}

// float2 gathers: word index l -> 8-byte element
__global__ void __launch_bounds__(256) lds64_k(int pat, float* out, unsigned seed) {
    __shared__ float2 s[2048];
    for (int i = threadIdx.x; i < 2048; i += 256) s[i] = make_float2(i, -i);
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        int l;
        unsigned h = ((seed + w) * 2654435761u) ^ (lane * 40503u + q * 977u + 12345u);
        h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        switch (pat) {
            case 0: l = lane + 32 * q; break;                            // contiguous
            case 1: l = (int)(h % 729u); break;                          // random in a 9^3 brick
            case 2: l = (lane & 15) + 16 * 7 * (lane >> 4) + 64 * q; break;  // halves distinct mod 16, halves equal
            case 3: l = 2 * lane + 64 * q; break;                        // 2-way within half
            case 4: l = (lane & 15) * 17 % 16 + 16 * ((lane >> 4) * 3 + 5 * q); break;  // perm within halves
            case 5: l = (int)(h % 16u) + 16 * (lane >> 4) + 64 * q; break;  // random within half (dups same addr)
            case 6: l = lane + 32 * ((lane * 7 + q) % 5); break;           // distinct mod 32, different rows
            default: l = 0;
        }
        a[q] = l;
    }
    float2 acc = make_float2(0.f, 0.f);
    for (int r = 0; r < REPS; ++r) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            float vx, vy;
            asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(vx), "=f"(vy) : "r"((unsigned)__cvta_generic_to_shared(s + a[q])));
            acc.x += vx; acc.y += vy;
        }
        if (acc.x == 1.2345e30f) a[0] ^= 1;
    }
    out[blockIdx.x * 256 + threadIdx.x] = acc.x + acc.y;
}

int main() {
    int nsm = 148, per = 4;
    int* o;
    cudaMalloc(&o, (size_t)nsm * per * 256 * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double instr_per_sm = (double)per * 8 * REPS * 8;  // warps * reps * 8
    const char* an[] = {"conflict-free", "random/1024", "2-way (16 banks x2)", "same address", "int2 re|im halves",
                        "int2 re only", "random bank/16 + half"};
    for (int p = 0; p < 7; ++p) {
        atoms_k<<<nsm * per, 256>>>(p, o, 1);
        cudaEventRecord(e0);
        atoms_k<<<nsm * per, 256>>>(p, o, 7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("ATOMS  %-24s %.3f ms  %.2f cycles/instr/SM (at 1.965 GHz)\n", an[p], ms, ms * 1e-3 * 1.965e9 / instr_per_sm);
    }
    const char* ln[] = {"contiguous", "random/729", "halves distinct mod16", "2-way within half", "perm within halves", "rand in half, dup addr", "distinct mod32 rows"};
    for (int p = 0; p < 7; ++p) {
        lds64_k<<<nsm * per, 256>>>(p, (float*)o, 1);
        cudaEventRecord(e0);
        lds64_k<<<nsm * per, 256>>>(p, (float*)o, 7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("LDS.64 %-24s %.3f ms  %.2f cycles/instr/SM\n", ln[p], ms, ms * 1e-3 * 1.965e9 / instr_per_sm);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
