// common.cuh -- shared device helpers of libseneca.so (sm_100a).
//
// Counter-based randomness for the ODS replay (reading R-O17; the
// paper only says "a pseudo-random number generator", §5.2, and a
// "predetermined pseudo-random sequence", §1):
//   philox4x32-10 (Salmon et al., SC'11), splitmix64 key derivation, and a
//   4-round Feistel network on Z_a x Z_b (a*b just above n) restricted to [0,n)
//   by cycle walking -- a keyed bijection, so "a permutation slice" needs no sort.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>     // header-only NVTX v3: no-op unless a profiler injects itself

#include "../../include/seneca.h"

namespace seneca {

// ---------------------------------------------------------------- error plumbing
void set_error(const char* fmt, ...);
seneca_status cuda_status(cudaError_t e, const char* what);

// Host-side NVTX range over a C-ABI call (tracing: nsys / ncu --nvtx timelines
// show init, each round launch, the ring generation and the MDP sweep).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

#define SENECA_CUDA_TRY(expr)                                              \
    do {                                                                   \
        cudaError_t _e = (expr);                                           \
        if (_e != cudaSuccess) return ::seneca::cuda_status(_e, #expr);    \
    } while (0)

// ---------------------------------------------------------------- PRNG (device)
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

enum : uint32_t { PUR_INIT = 1, PUR_REQ = 2, PUR_SUB = 3, PUR_REFILL = 4 };

// key(seed, purpose, a, b, c) = splitmix64(seed ^ splitmix64(purpose<<56 ^ a<<48 ^ c<<44 ^ b))
__device__ __forceinline__ uint64_t derive_key(uint64_t seed, uint64_t purpose, uint64_t a,
                                               uint64_t b, uint64_t c) {
    return splitmix64(seed ^ splitmix64((purpose << 56) ^ (a << 48) ^ (c << 44) ^ b));
}

// philox4x32-10 on counter (c0, c1, 0, 0); only word 0 of the output is used.
__device__ __forceinline__ uint32_t philox_w0(uint32_t c0, uint32_t c1, uint32_t k0, uint32_t k1) {
    uint32_t c2 = 0, c3 = 0;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    return c0;
}

// Domain of a keyed permutation of [0, n): Z_a x Z_b with a = ceil(sqrt(n)),
// b = ceil(n / a), so a*b - n < a and a cycle-walk step happens with
// probability < 1/b -- no warp divergence in practice (a binary domain walks
// up to 2x on average and ~6x for the slowest lane of a warp).
struct PermDomain {
    uint32_t n, a, b;
};

__device__ __forceinline__ PermDomain perm_domain(uint32_t n) {
    PermDomain d;
    d.n = n;
    if (n <= 1) { d.a = d.b = 1; return d; }
    uint32_t a = (uint32_t)ceil(sqrt((double)n));
    while ((uint64_t)(a - 1) * (a - 1) >= n) --a;
    while ((uint64_t)a * a < n) ++a;
    d.a = a;
    d.b = (n + a - 1) / a;
    return d;
}

// Feistel on Z_a x Z_b (x = L*b + R): even rounds L += F mod a, odd rounds
// R += F mod b, F = philox((other part, round, 0, 0), key)[0] scaled to the
// modulus by multiply-high; cycle-walked into [0, n).  4 rounds; 12 when
// n < 64 (halves of <= 8 values need more rounds to mix, R-O17) -- a
// CTA-uniform branch in every caller (one pool size per call site).
__device__ __forceinline__ uint32_t perm_apply(uint64_t key, const PermDomain& d, uint32_t x) {
    if (d.n <= 1u) return 0u;
    const uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
    if (d.n < 64u) {
        do {
            uint32_t L = x / d.b, R = x - L * d.b;
#pragma unroll 1
            for (uint32_t rd = 0; rd < 12u; rd += 2) {
                L += __umulhi(philox_w0(R, rd, k0, k1), d.a); L = L >= d.a ? L - d.a : L;
                R += __umulhi(philox_w0(L, rd + 1, k0, k1), d.b); R = R >= d.b ? R - d.b : R;
            }
            x = L * d.b + R;
        } while (x >= d.n);
        return x;
    }
    do {
        uint32_t L = x / d.b, R = x - L * d.b;
        L += __umulhi(philox_w0(R, 0u, k0, k1), d.a); L = L >= d.a ? L - d.a : L;
        R += __umulhi(philox_w0(L, 1u, k0, k1), d.b); R = R >= d.b ? R - d.b : R;
        L += __umulhi(philox_w0(R, 2u, k0, k1), d.a); L = L >= d.a ? L - d.a : L;
        R += __umulhi(philox_w0(L, 3u, k0, k1), d.b); R = R >= d.b ? R - d.b : R;
        x = L * d.b + R;
    } while (x >= d.n);
    return x;
}

// ---------------------------------------------------------------- block scan
// Exclusive scan of one uint32 per thread across the block (blockDim.x a
// multiple of 32, <= 1024).  scratch: 33 uint32 of shared memory.  Every
// thread must call it; it ends with a barrier so scratch can be reused
// (kTail = false: no trailing barrier -- the caller's next barrier must come
// before scratch is written again).
template <bool kTail = true>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* total, uint32_t* scratch) {
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t nwarps = blockDim.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += y;
    }
    if (lane == 31) scratch[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < nwarps ? scratch[lane] : 0u;
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= (uint32_t)o) wi += y;
        }
        if (lane < nwarps) scratch[lane] = wi - w;
        if (lane == 31) scratch[32] = wi;
    }
    __syncthreads();
    const uint32_t res = scratch[warp] + incl - v;
    if (total) *total = scratch[32];
    if (kTail) __syncthreads();
    return res;
}

// Exclusive scan of a per-thread count given as two flag bits (v = f0 + f1,
// each 0 or 1) across the block: in-warp prefixes from two ballots, then one
// warp scans the per-warp totals.  Same contract as block_exclusive_scan
// (every thread calls it, ends with a barrier), far fewer instructions.
__device__ __forceinline__ uint32_t block_flag_scan(bool f0, bool f1, uint32_t* total, uint32_t* scratch) {
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t nwarps = blockDim.x >> 5;
    const uint32_t b0 = __ballot_sync(0xffffffffu, f0), b1 = __ballot_sync(0xffffffffu, f1);
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t ex_w = __popc(b0 & lt) + __popc(b1 & lt);
    if (lane == 0) scratch[warp] = __popc(b0) + __popc(b1);
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < nwarps ? scratch[lane] : 0u;
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= (uint32_t)o) wi += y;
        }
        if (lane < nwarps) scratch[lane] = wi - w;
        if (lane == 31) scratch[32] = wi;
    }
    __syncthreads();
    const uint32_t res = scratch[warp] + ex_w;
    if (total) *total = scratch[32];
    __syncthreads();
    return res;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace seneca
