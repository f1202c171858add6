// Microbenchmark: latency of perm_apply (keyed Feistel + Philox) per thread, one CTA of 512 threads.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2511_13724_b200/csrc/common.cuh"
using namespace seneca;
namespace seneca { void set_error(const char*, ...) {} seneca_status cuda_status(cudaError_t, const char*) { return SENECA_ECUDA; } }

__global__ void k_perm(uint32_t n, uint64_t key, uint32_t* out, long long* cyc, int reps) {
    const PermDomain d = perm_domain(n);
    uint32_t acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) acc += perm_apply(key + r, d, (threadIdx.x * 7919u + r) % n);
    __syncthreads();
    long long t1 = clock64();
    out[threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
}

__global__ void k_philox(uint64_t key, uint32_t* out, long long* cyc, int reps) {
    uint32_t x = threadIdx.x;
    __syncthreads();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) x = philox_w0(x, r, (uint32_t)key, (uint32_t)(key >> 32));
    __syncthreads();
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
}

__global__ void k_ldcg_chain(const uint32_t* __restrict__ buf, uint32_t mask, uint32_t* out, long long* cyc, int reps) {
    uint32_t x = threadIdx.x * 4099u;
    __syncthreads();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) x = __ldcg(buf + (x & mask)) + r;
    __syncthreads();
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
}

int main() {
    uint32_t* out; long long* cyc; uint32_t* buf;
    cudaMalloc(&out, 1 << 16); cudaMalloc(&cyc, 4096);
    const size_t nbuf = 64u << 20;  // 256 MB of u32
    cudaMalloc(&buf, nbuf * 4);
    cudaMemset(buf, 0, nbuf * 4);
    long long h;
    for (int threads : {32, 512}) {
        k_philox<<<1, threads>>>(0x1234567890abcdefull, out, cyc, 200);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("philox4x32-10 latency, %3d threads/CTA: %lld cycles\n", threads, h);
        for (uint32_t n : {1000u, 1190000u, 2100000u, 4380000u, 14197122u}) {
            k_perm<<<1, threads>>>(n, 0xfeedbeefcafef00dull, out, cyc, 50);
            cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
            printf("perm_apply n=%9u, %3d threads/CTA: %lld cycles per call (CTA max)\n", n, threads, h);
        }
        for (uint32_t mb : {1u, 16u, 256u}) {
            uint32_t mask = (mb << 18) - 1;   // mb MB region
            k_ldcg_chain<<<1, threads>>>(buf, mask, out, cyc, 100);
            cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
            printf("dependent ldcg chain over %3u MB, %3d threads: %lld cycles per load\n", mb, threads, h);
        }
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
