// mdp.cu -- Model-Driven Partitioning sweep.
//
// One warp per hardware profile:
//   prologue  Eqs. 1-4 tier throughputs with the ring-reduce
//             overhead C = 2(n-1)/n * betaN; integer capacity tables
//             capAD[p], capE[p] (Eqs. 5-7 floored exactly, R-M6) and the Eq. 9
//             terms that depend on one coordinate only, in the warp's slice of
//             shared memory;
//   main loop every split of the grid: clamped counts (Eqs. 5-8) and
//             DSI_overall (Eq. 9) in the literal order of R-M7; optional
//             coalesced write of the full grid row;
//   epilogue  warp argmax, exact ties -> smallest enumeration index (R-M8).
//
// Bit-exactness with the oracle: every binary64 operation is an explicit
// round-to-nearest intrinsic (__dadd_rn/__dmul_rn/__ddiv_rn, never contracted
// into an FMA), integer->double conversions are __ull2double_rn, and a term
// taken from a table is the same operation on the same operands as the one the
// oracle performs per split.
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace seneca {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxSteps = 101;  // grid step 1 % -> 101 values per coordinate

enum : uint8_t { L_CACHE = 0, L_NIC = 1, L_PCIE = 2, L_CPU_AUG = 3, L_CPU_DEC_AUG = 4, L_GPU = 5, L_STORAGE = 6 };

__device__ __forceinline__ double u2d(uint64_t x) { return __ull2double_rn(x); }

__device__ __forceinline__ void take_min(double term, uint8_t code, double& best, uint8_t& lim) {
    if (term < best) { best = term; lim = code; }
}

// C = 2(n-1)/n x betaN
__device__ __forceinline__ double comm_overhead(uint64_t p, double model_bytes) {
    if (p <= 1) return 0.0;
    const double frac = __ddiv_rn(u2d(2ull * (p - 1ull)), u2d(p));
    return __dmul_rn(frac, model_bytes);
}

__device__ __forceinline__ bool finite_pos(double x) { return isfinite(x) && x > 0.0; }

__device__ bool profile_valid(const seneca_mdp_profile& p) {
    if (!finite_pos(p.t_gpu) || !finite_pos(p.t_decode_augment) || !finite_pos(p.t_augment)) return false;
    if (!finite_pos(p.b_nic) || !finite_pos(p.b_pcie) || !finite_pos(p.b_cache) || !finite_pos(p.b_storage)) return false;
    if (!isfinite(p.model_bytes) || p.model_bytes < 0.0) return false;
    if (p.n_total == 0 || p.s_data == 0 || p.m_den == 0 || p.m_num < p.m_den) return false;
    if (p.nodes == 0 || p.gpus_per_node == 0) return false;
    if (p.cache_bytes > (~0ull / 100ull) / p.m_den) return false;   // 100*cache*m_den < 2^64
    if (p.s_data > (~0ull / 100ull) / p.m_num) return false;        // 100*m_num*s_data < 2^64
    return true;
}

// Eqs. 1-4; dsi/lim index 0 A, 1 D, 2 E, 3 S.
__device__ void tier_throughputs(const seneca_mdp_profile& p, double dsi[4], uint8_t lim[4]) {
    const double Sd = u2d(p.s_data);
    const double MS = __ddiv_rn(u2d((uint64_t)p.m_num * p.s_data), u2d(p.m_den));   // M x S_data
    const uint64_t p_nw = p.comm_mapping ? p.gpus_per_node : p.nodes;                 // R-M1
    const uint64_t p_pc = p.comm_mapping ? p.nodes : p.gpus_per_node;
    const double C_nw = p.nvlink_inter ? 0.0 : comm_overhead(p_nw, p.model_bytes);
    const double C_pc = (p.nvlink_intra || p.nvlink_inter) ? 0.0 : comm_overhead(p_pc, p.model_bytes);
    const double nd = u2d(p.nodes);
    const double nic = __dmul_rn(nd, p.b_nic);
    const double pcie = __dmul_rn(nd, p.b_pcie);
    const double gpu = __dmul_rn(nd, p.t_gpu);
    const double cache_ms = __ddiv_rn(p.b_cache, MS);
    const double nic_ms = __ddiv_rn(nic, __dadd_rn(MS, C_nw));
    const double pcie_ms = __ddiv_rn(pcie, __dadd_rn(MS, C_pc));

    // Eq. 1
    double a = __longlong_as_double(0x7ff0000000000000ll); uint8_t la = 0xff;
    take_min(cache_ms, L_CACHE, a, la);
    take_min(nic_ms, L_NIC, a, la);
    take_min(pcie_ms, L_PCIE, a, la);
    take_min(gpu, L_GPU, a, la);
    // Eq. 2 (R-M4: the PCIe and GPU terms are separate)
    double d = __longlong_as_double(0x7ff0000000000000ll); uint8_t ld = 0xff;
    take_min(cache_ms, L_CACHE, d, ld);
    take_min(nic_ms, L_NIC, d, ld);
    take_min(__dmul_rn(nd, p.t_augment), L_CPU_AUG, d, ld);
    take_min(pcie_ms, L_PCIE, d, ld);
    take_min(gpu, L_GPU, d, ld);
    // Eq. 3: cache and NIC terms over the encoded size S_data
    double e = __longlong_as_double(0x7ff0000000000000ll); uint8_t le = 0xff;
    take_min(__ddiv_rn(p.b_cache, Sd), L_CACHE, e, le);
    take_min(__ddiv_rn(nic, __dadd_rn(Sd, C_nw)), L_NIC, e, le);
    take_min(__dmul_rn(nd, p.t_decode_augment), L_CPU_DEC_AUG, e, le);
    take_min(pcie_ms, L_PCIE, e, le);
    take_min(gpu, L_GPU, e, le);
    // Eq. 4
    const double st = __ddiv_rn(p.b_storage, Sd);
    double s = e; uint8_t ls = le;
    if (st < e) { s = st; ls = L_STORAGE; }
    dsi[0] = a; dsi[1] = d; dsi[2] = e; dsi[3] = s;
    lim[0] = la; lim[1] = ld; lim[2] = le; lim[3] = ls;
}

// Per-warp shared tables for one profile: capacities clamped to N (exact
// integers), and the Eq. 9 terms that depend on a single coordinate.
struct WarpTables {
    uint64_t capc[kMaxSteps];    // min(N, capAD(p))  -- A and D tiers (M x S_data per sample)
    uint64_t cape[kMaxSteps];    // min(N, capE(p))   -- E tier (S_data per sample)
    double tA[kMaxSteps];        // (capc/N) DSI_A
    double tD[kMaxSteps];        // (capc/N) DSI_D        (D unclamped)
    double tDc[kMaxSteps];       // ((N - capc)/N) DSI_D  (D clamped by the A count, indexed by p_A)
    double tE[kMaxSteps];        // (cape/N) DSI_E        (E unclamped)
};

// x / N correctly rounded, for integers 0 <= x <= N < 2^53, with y = RN(1/N)
// precomputed: q = RN(x y); the residual x - N q is exact; q' = RN(q + r y) is
// RN(x/N) (Markstein).  x/N is never an exact tie between two doubles here (a
// dyadic x/N is exactly representable), so q' equals __ddiv_rn(x, N) bit for bit.
__device__ __forceinline__ double div_by_n(double x, double dN, double y) {
    const double q = __dmul_rn(x, y);
    const double r = __fma_rn(-dN, q, x);
    return __fma_rn(r, y, q);
}

// The sweep of one profile by one warp; U = uint32_t when N < 2^31 (every
// count fits, 32-bit integer ops), uint64_t otherwise.  Each split needs one
// division at most: a clamped tier forces every later count to 0 (a zero term
// is exactly +0.0 in the oracle's arithmetic too), so either the clamped E
// count or the storage count is the only per-split quotient.
template <typename U>
__device__ __forceinline__ void sweep_profile(const WarpTables& W, const uint32_t* __restrict__ s_split, uint64_t N64,
                                              const double dsi[4], uint32_t n_splits, double* grow, double& best,
                                              uint32_t& best_i) {
    const uint32_t lane = threadIdx.x & 31;
    const U N = (U)N64;
    const double dN = u2d(N64);
    const double y = __drcp_rn(dN);
    constexpr bool kExact = sizeof(U) == 4;                          // div_by_n needs N < 2^53
    if (grow) grow += lane;
    for (uint32_t idx = lane; idx < n_splits; idx += 32) {
        const uint32_t packed = s_split[idx];                        // p_A | p_D << 8 | p_E << 16 (table indices)
        const uint32_t ia = packed & 0xffu, id = (packed >> 8) & 0xffu, ie = packed >> 16;
        const U r1 = N - (U)W.capc[ia];                              // Eq. 5: N_A = capc[p_A]
        const U cD = (U)W.capc[id];
        double tD, tE, tS;
        if (cD <= r1) {                                              // Eq. 6 unclamped
            tD = W.tD[id];
            const U r2 = r1 - cD;
            const U cE = (U)W.cape[ie];
            if (cE <= r2) {                                          // Eq. 7 unclamped, Eq. 8 remainder
                tE = W.tE[ie];
                tS = __dmul_rn(kExact ? div_by_n(u2d(r2 - cE), dN, y) : __ddiv_rn(u2d(r2 - cE), dN), dsi[3]);
            } else {                                                 // E takes the rest, N_S = 0
                tE = __dmul_rn(kExact ? div_by_n(u2d(r2), dN, y) : __ddiv_rn(u2d(r2), dN), dsi[2]);
                tS = 0.0;
            }
        } else {                                                     // D takes the rest: N_E = N_S = 0
            tD = W.tDc[ia];
            tE = 0.0;
            tS = 0.0;
        }
        const double v = __dadd_rn(__dadd_rn(__dadd_rn(W.tA[ia], tD), tE), tS);   // Eq. 9, R-M7
        if (grow) { __stcs(grow, v); grow += 32; }
        if (v > best) { best = v; best_i = idx; }                   // idx increases per lane
    }
}

// One WARP per profile (8 profiles per CTA in flight): the prologue needs only
// warp-level synchronisation, so one warp's setup overlaps the other warps'
// sweeps; each warp iteration stores 32 consecutive grid values (256 B).
__global__ void __launch_bounds__(kThreads)
mdp_sweep_kernel(const seneca_mdp_profile* __restrict__ profiles, uint32_t n_profiles, uint32_t g,
                 uint32_t steps, uint32_t n_splits, seneca_mdp_result* __restrict__ results,
                 double* __restrict__ grid) {
    constexpr int kWarps = kThreads / 32;
    __shared__ WarpTables s_tab[kWarps];
    extern __shared__ uint32_t s_split[];                           // [n_splits] packed split coordinates
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    WarpTables& W = s_tab[w];
    // enumeration index -> table indices (R-M9 order): row a has p_E = 100 - a g and
    // positions b = 0..a with p_A = b g, p_D = (a - b) g
    for (uint32_t a = 0, base = 0; a <= steps; base += a + 1, ++a)
        for (uint32_t b = threadIdx.x; b <= a; b += blockDim.x)
            s_split[base + b] = b | ((a - b) << 8) | ((steps - a) << 16);
    __syncthreads();

    for (uint32_t pi = blockIdx.x * kWarps + w; pi < n_profiles; pi += gridDim.x * kWarps) {
        const seneca_mdp_profile p = profiles[pi];
        if (!profile_valid(p)) {
            if (lane == 0) {
                seneca_mdp_result r = {};
                r.status = 1;
                results[pi] = r;
            }
            continue;
        }
        double dsi[4];
        uint8_t lim[4];
        tier_throughputs(p, dsi, lim);            // every lane (no shared state, no barrier)
        const uint64_t N = p.n_total;
        const double dN = u2d(N);
        const uint64_t Xad = p.cache_bytes * p.m_den, Dad = 100ull * p.m_num * p.s_data;
        const uint64_t De = 100ull * p.s_data;
        const bool exact_div = N < (1ull << 53);
        const double yN = __drcp_rn(dN);
        for (uint32_t k = lane; k <= steps; k += 32) {
            const uint64_t pct = (uint64_t)k * g;
            uint64_t cad = (pct * Xad) / Dad, ce = (pct * p.cache_bytes) / De;   // Eqs. 5-7, exact floors
            cad = cad < N ? cad : N;
            ce = ce < N ? ce : N;
            W.capc[k] = cad;
            W.cape[k] = ce;
            const double fa = exact_div ? div_by_n(u2d(cad), dN, yN) : __ddiv_rn(u2d(cad), dN);
            const double fc = exact_div ? div_by_n(u2d(N - cad), dN, yN) : __ddiv_rn(u2d(N - cad), dN);
            const double fe = exact_div ? div_by_n(u2d(ce), dN, yN) : __ddiv_rn(u2d(ce), dN);
            W.tA[k] = __dmul_rn(fa, dsi[0]);
            W.tD[k] = __dmul_rn(fa, dsi[1]);
            W.tDc[k] = __dmul_rn(fc, dsi[1]);
            W.tE[k] = __dmul_rn(fe, dsi[2]);
        }
        __syncwarp();
        double best = __longlong_as_double(0xfff0000000000000ll);
        uint32_t best_i = 0xffffffffu;
        double* grow = grid ? grid + (uint64_t)pi * n_splits : nullptr;
        if (N < (1ull << 31)) sweep_profile<uint32_t>(W, s_split, N, dsi, n_splits, grow, best, best_i);
        else sweep_profile<uint64_t>(W, s_split, N, dsi, n_splits, grow, best, best_i);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, best, o);
            const uint32_t oi = __shfl_xor_sync(0xffffffffu, best_i, o);
            if (ov > best || (ov == best && oi < best_i)) { best = ov; best_i = oi; }
        }
        if (lane == 0) {
            uint32_t ra = 0, rb = best_i;
            while (rb > ra) { rb -= ra + 1; ++ra; }
            seneca_mdp_result r;
            r.p_e = (uint8_t)(100 - ra * g);
            r.p_d = (uint8_t)((ra - rb) * g);
            r.p_a = (uint8_t)(rb * g);
            r.lim_a = lim[0]; r.lim_d = lim[1]; r.lim_e = lim[2]; r.lim_s = lim[3];
            r.status = 0;
            r.v_best = best;
            r.dsi_a = dsi[0]; r.dsi_d = dsi[1]; r.dsi_e = dsi[2]; r.dsi_s = dsi[3];
            results[pi] = r;
        }
        __syncwarp();
    }
}

}  // namespace
}  // namespace seneca

extern "C" uint64_t seneca_mdp_num_splits(uint32_t g) {
    if (g == 0 || g > 100 || 100 % g) return 0;
    const uint64_t s = 100 / g;
    return (s + 1) * (s + 2) / 2;
}

extern "C" seneca_status seneca_mdp_sweep(const seneca_mdp_profile* d_profiles, uint32_t n_profiles,
                                          uint32_t grid_step_pct, seneca_mdp_result* d_results,
                                          double* d_grid, void* stream) {
    using namespace seneca;
    if (grid_step_pct == 0 || grid_step_pct > 100 || 100 % grid_step_pct) {
        set_error("seneca_mdp_sweep: grid_step_pct %u does not divide 100", grid_step_pct);
        return SENECA_EINVAL;
    }
    if (n_profiles == 0 || !d_profiles || !d_results) {
        set_error("seneca_mdp_sweep: empty input or NULL pointer");
        return SENECA_EINVAL;
    }
    const uint32_t steps = 100 / grid_step_pct;
    const uint32_t ns = (uint32_t)seneca_mdp_num_splits(grid_step_pct);
    const uint32_t per_cta = kThreads / 32;
    uint32_t blocks = (n_profiles + per_cta - 1) / per_cta;
    blocks = blocks < 65535u * 8u ? blocks : 65535u * 8u;
    static bool attr_set = false;
    if (!attr_set) {
        SENECA_CUDA_TRY(cudaFuncSetAttribute(mdp_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)(5151 * sizeof(uint32_t))));
        attr_set = true;
    }
    mdp_sweep_kernel<<<blocks, kThreads, ns * sizeof(uint32_t), (cudaStream_t)stream>>>(
        d_profiles, n_profiles, grid_step_pct, steps, ns, d_results, d_grid);
    SENECA_CUDA_TRY(cudaGetLastError());
    return SENECA_OK;
}
