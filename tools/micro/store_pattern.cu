// Store-pattern microbenchmark for the MDP grid write (10,000 or 100,000 rows of
// 5,151 doubles): which write pattern reaches the write bandwidth?
//   A  the paired sweep's pattern: groups of 64 threads per row, pair table order
//      (i0 ascending within a triangle row, i1 descending), 8-B stores
//   B  each group writes its row front to back, 8-B stores, coalesced
//   C  each group writes its row front to back, 16-B stores (aligned body)
//   D  the grid as one flat array, 16-B stores, grid-stride
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int kThreads = 256, kGroups = 4, kPairs = 2601, kSplits = 5151;
__global__ void __launch_bounds__(256, 3) patA(double* g, int rows, const uint2* tab) {
    __shared__ uint2 s[kPairs];
    for (int t = threadIdx.x; t < kPairs; t += blockDim.x) s[t] = tab[t];
    __syncthreads();
    const int gid = threadIdx.x / 64, gt = threadIdx.x % 64;
    for (int pi = blockIdx.x * kGroups + gid; pi < rows; pi += gridDim.x * kGroups) {
        double* row = g + (size_t)pi * kSplits;
#pragma unroll 2
        for (int t = gt; t < kPairs; t += 64) {
            const uint2 w = s[t];
            __stcs(row + (w.y & 0xffff), 1.0 * t);
            __stcs(row + (w.y >> 16), 2.0 * t);
        }
    }
}
__global__ void __launch_bounds__(256, 3) patB(double* g, int rows) {
    const int gid = threadIdx.x / 64, gt = threadIdx.x % 64;
    for (int pi = blockIdx.x * kGroups + gid; pi < rows; pi += gridDim.x * kGroups) {
        double* row = g + (size_t)pi * kSplits;
        for (int i = gt; i < kSplits; i += 64) __stcs(row + i, 1.0 * i);
    }
}
__global__ void __launch_bounds__(256, 3) patC(double* g, int rows) {
    const int gid = threadIdx.x / 64, gt = threadIdx.x % 64;
    for (int pi = blockIdx.x * kGroups + gid; pi < rows; pi += gridDim.x * kGroups) {
        double* row = g + (size_t)pi * kSplits;
        const int head = ((uintptr_t)row & 15) ? 1 : 0;
        if (gt == 0 && head) row[0] = 0.5;
        const int nv = (kSplits - head) / 2;
        double2* v = reinterpret_cast<double2*>(row + head);
        for (int i = gt; i < nv; i += 64) __stcs(v + i, make_double2(1.0 * i, 2.0 * i));
        if (gt == 0 && (kSplits - head) % 2) row[kSplits - 1] = 0.25;
    }
}
// E: each CTA writes whole rows, one row at a time, 16-B stores by all 256 threads
__global__ void __launch_bounds__(256, 3) patE(double* g, int rows) {
    for (int pi = blockIdx.x; pi < rows; pi += gridDim.x) {
        double* row = g + (size_t)pi * kSplits;
        const int head = ((uintptr_t)row & 15) ? 1 : 0;
        if (threadIdx.x == 0 && head) row[0] = 0.5;
        const int nv = (kSplits - head) / 2;
        double2* v = reinterpret_cast<double2*>(row + head);
        for (int i = threadIdx.x; i < nv; i += blockDim.x) __stcs(v + i, make_double2(1.0 * i, 2.0 * i));
        if (threadIdx.x == 0 && (kSplits - head) % 2) row[kSplits - 1] = 0.25;
    }
}
// F: each CTA fills a 41 KB shared row buffer (double-buffered) and writes it with one
// TMA bulk store (cp.async.bulk.global.shared::cta), head/tail 8 B by thread 0
__global__ void __launch_bounds__(256, 2) patF(double* g, int rows) {
    extern __shared__ __align__(128) double sbuf[];                 // [2][kSplits + 3]
    int it = 0;
    for (int pi = blockIdx.x; pi < rows; pi += gridDim.x, ++it) {
        double* buf = sbuf + (it & 1) * (kSplits + 3);
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncthreads();
        double* row = g + (size_t)pi * kSplits;
        const int head = ((uintptr_t)row & 15) ? 1 : 0;
        for (int i = threadIdx.x; i < kSplits; i += blockDim.x) buf[i + (head ? 1 : 0)] = 1.0 * i;   // buf index 16-B aligned with row
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            if (head) row[0] = buf[1];
            const int nb = ((kSplits - head) / 2) * 16;
            const uint32_t sa = (uint32_t)__cvta_generic_to_shared(buf + 2 * head);
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(row + head), "r"(sa), "r"(nb) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            if ((kSplits - head) % 2) row[kSplits - 1] = 0.25;
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__global__ void patD(double* g, size_t n) {
    double2* v = reinterpret_cast<double2*>(g);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n / 2; i += (size_t)gridDim.x * blockDim.x)
        __stcs(v + i, make_double2(1.0, 2.0));
}
int main(int argc, char** argv) {
    const int rows = argc > 1 ? atoi(argv[1]) : 10000;
    uint2 tab[kPairs];
    int t = 0;
    for (int a = 0; a <= 100; ++a) for (int b = 0; b <= a / 2; ++b) {
        const int i0 = a * (a + 1) / 2;
        tab[t++] = make_uint2(0, (i0 + b) | (i0 + a - b) << 16);
    }
    uint2* dtab; cudaMalloc(&dtab, sizeof tab); cudaMemcpy(dtab, tab, sizeof tab, cudaMemcpyHostToDevice);
    double* g; const size_t n = (size_t)rows * kSplits; cudaMalloc(&g, n * 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int blocks = 148 * 3;
    cudaFuncSetAttribute(patF, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * (kSplits + 3) * 8);
    const int nb = argc > 2 ? atoi(argv[2]) : 3;     // CTAs per SM for patterns A, B, C, E
    const int blocks2 = 148 * nb;
    for (int p = 0; p < 6; ++p) {
        float best = 1e9;
        for (int it = 0; it < 12; ++it) {
            cudaEventRecord(e0);
            if (p == 0) patA<<<blocks2, 256>>>(g, rows, dtab);
            if (p == 1) patB<<<blocks2, 256>>>(g, rows);
            if (p == 2) patC<<<blocks2, 256>>>(g, rows);
            if (p == 3) patD<<<148 * 8, 256>>>(g, n);
            if (p == 4) patE<<<blocks2, 256>>>(g, rows);
            if (p == 5) patF<<<148 * (nb < 2 ? nb : 2), 256, 2 * (kSplits + 3) * 8>>>(g, rows);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (it >= 2 && ms < best) best = ms;
        }
        printf("ctas/sm %d rows %d pattern %c: %.1f us  %.0f GB/s\n", nb, rows, "ABCDEF"[p], best * 1e3, n * 8 / (best * 1e-3) / 1e9);
    }
    return cudaGetLastError() != cudaSuccess;
}
