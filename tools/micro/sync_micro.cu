// Microbenchmark: cost of __syncthreads() after global atomics / stores (one CTA, 512 threads).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(uint32_t* g, uint32_t mask, long long* cyc, int reps) {
    __shared__ uint32_t sm[1024];
    uint32_t x = threadIdx.x * 2654435761u;
    __syncthreads();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        x = x * 1664525u + 1013904223u;
        if (MODE == 1) atomicOr(g + (x & mask), 1u);                 // RED.OR global
        if (MODE == 2) g[(x & mask)] = x;                            // STG
        if (MODE == 3) atomicOr(sm + (x & 1023), 1u);                // ATOMS
        if (MODE == 4 && threadIdx.x < 13) atomicAdd((unsigned long long*)g + (threadIdx.x * 8), 1ull);
        if (MODE == 5) { if (threadIdx.x == 0) atomicOr(g, 1u); }
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
}

int main() {
    uint32_t* g; long long* cyc; long long h;
    cudaMalloc(&g, 64 << 20); cudaMalloc(&cyc, 1024); cudaMemset(g, 0, 64 << 20);
    const char* names[] = {"sync only", "RED.OR global + sync", "STG + sync", "ATOMS + sync", "13x RED.ADD.64 + sync", "1x RED + sync"};
#define RUN(M) k<M><<<1, 512>>>(g, (1u << 22) - 1, cyc, 200); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("%-24s %lld cycles/iter\n", names[M], h);
    RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5)
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
