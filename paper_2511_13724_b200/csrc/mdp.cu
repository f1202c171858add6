// mdp.cu -- Model-Driven Partitioning sweep.
//
// One CTA per hardware profile (persistent CTAs walk a grid-stride list):
//   prologue  (warp 0, one profile ahead, double-buffered) Eqs. 1-4 tier
//             throughputs with the ring-reduce overhead
//             C = 2(n-1)/n * betaN; integer capacity tables capAD[p],
//             capE[p] (Eqs. 5-7 floored exactly, R-M6) and the Eq. 9 terms that
//             depend on one coordinate only, as rows in shared memory;
//   main loop every split of the grid, 256 threads: clamped counts (Eqs. 5-8)
//             and DSI_overall (Eq. 9) in the literal order of R-M7, branch-free;
//             optional coalesced streaming write of the full grid row;
//   epilogue  argmax per thread / warp / CTA, exact ties -> smallest
//             enumeration index (R-M8).
//
// Bit-exactness with the oracle: every binary64 operation is an explicit
// round-to-nearest intrinsic (__dadd_rn/__dmul_rn/__ddiv_rn, never contracted
// into an FMA), integer->double conversions are exact (__ull2double_rn, or the
// 2^52 trick for 32-bit counts), and a term
// taken from a table is the same operation on the same operands as the one the
// oracle performs per split.
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace seneca {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxSteps = 101;  // grid step 1 % -> 101 values per coordinate
#ifndef SENECA_MDP_CHUNK
#define SENECA_MDP_CHUNK 512
#endif
#ifndef SENECA_MDP_UNROLL
#define SENECA_MDP_UNROLL 4
#endif
#ifndef SENECA_MDP_FASTDIV
#define SENECA_MDP_FASTDIV 1      // 0: capacity floors by the u64 division routine (A/B knob)
#endif
#ifndef SENECA_MDP_PARHDR
#define SENECA_MDP_PARHDR 1       // 1: the header's divisions spread over lanes (two levels); 0: serial
#endif
#ifndef SENECA_MDP_REDUX
#define SENECA_MDP_REDUX 1        // warp argmax by fmax butterfly + REDUX.MIN of the index (A/B knob)
#endif
#ifndef SENECA_MDP_DENSE
#define SENECA_MDP_DENSE 2        // rows as dense arrays; 2: capc|cape in one 8-B slot, pre-scaled pair offsets (A/B knob)
#endif
#ifndef SENECA_MDP_MINB
#define SENECA_MDP_MINB 3
#endif
#ifndef SENECA_MDP_PAIRS
#define SENECA_MDP_PAIRS 1        // 1: the paired sweep (mdp_sweep_pairs); 0: mdp_sweep_kernel (A/B knob)
#endif
constexpr uint32_t kChunk = SENECA_MDP_CHUNK;  // splits per sweep work item (16 per lane)
constexpr int kUnroll = SENECA_MDP_UNROLL;      // splits in flight per lane

enum : uint8_t { L_CACHE = 0, L_NIC = 1, L_PCIE = 2, L_CPU_AUG = 3, L_CPU_DEC_AUG = 4, L_GPU = 5, L_STORAGE = 6 };

__device__ __forceinline__ double u2d(uint64_t x) { return __ull2double_rn(x); }

// Exact u32 -> double on the FP64 pipe: (2^52 + x) - 2^52 is exact for x < 2^32
// and equals __ull2double_rn(x); the I2F.F64 conversion runs on the narrow XU
// pipe, which ncu showed to be the sweep's bottleneck.
__device__ __forceinline__ double u32_to_d(uint32_t x) {
    return __dsub_rn(__hiloint2double(0x43300000, (int)x), 4503599627370496.0);
}

#ifndef SENECA_MDP_STCS
#define SENECA_MDP_STCS 1         // grid stores: 1 st.global.cs (evict-first), 0 plain st.global (A/B knob)
#endif
__device__ __forceinline__ void st_grid(double* p, double v) {
#if SENECA_MDP_STCS
    __stcs(p, v);
#else
    *p = v;
#endif
}

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

// Eqs. 1-4 by one warp with the nine divisions spread over lanes in two
// dependency levels (the same IEEE operations on the same operands as
// tier_throughputs, so the same bits); every lane ends with the results.
__device__ void tier_throughputs_warp(const seneca_mdp_profile& p, double dsi[4], uint8_t lim[4]) {
    const uint32_t lane = threadIdx.x & 31;
    const double Sd = u2d(p.s_data);
    const uint64_t p_nw = p.comm_mapping ? p.gpus_per_node : p.nodes;                 // R-M1
    const uint64_t p_pc = p.comm_mapping ? p.nodes : p.gpus_per_node;
    const double nd = u2d(p.nodes);
    const double nic = __dmul_rn(nd, p.b_nic);
    const double pcie = __dmul_rn(nd, p.b_pcie);
    const double gpu = __dmul_rn(nd, p.t_gpu);
    // level 1: M x S_data, the two ring fractions 2(n-1)/n, B_cache/S_data, B_storage/S_data
    double num = 1.0, den = 1.0;
    if (lane == 0) { num = u2d((uint64_t)p.m_num * p.s_data); den = u2d(p.m_den); }
    else if (lane == 1 && p_nw > 1) { num = u2d(2ull * (p_nw - 1ull)); den = u2d(p_nw); }
    else if (lane == 2 && p_pc > 1) { num = u2d(2ull * (p_pc - 1ull)); den = u2d(p_pc); }
    else if (lane == 3) { num = p.b_cache; den = Sd; }
    else if (lane == 4) { num = p.b_storage; den = Sd; }
    const double q1 = __ddiv_rn(num, den);
    const double MS = __shfl_sync(0xffffffffu, q1, 0);
    const double f_nw = __shfl_sync(0xffffffffu, q1, 1), f_pc = __shfl_sync(0xffffffffu, q1, 2);
    const double e_cache = __shfl_sync(0xffffffffu, q1, 3), st = __shfl_sync(0xffffffffu, q1, 4);
    const double C_nw = (p.nvlink_inter || p_nw <= 1) ? 0.0 : __dmul_rn(f_nw, p.model_bytes);
    const double C_pc = (p.nvlink_intra || p.nvlink_inter || p_pc <= 1) ? 0.0 : __dmul_rn(f_pc, p.model_bytes);
    // level 2: the cache, NIC and PCIe terms over M S_data, the NIC term over S_data
    num = 1.0; den = 1.0;
    if (lane == 0) { num = p.b_cache; den = MS; }
    else if (lane == 1) { num = nic; den = __dadd_rn(MS, C_nw); }
    else if (lane == 2) { num = pcie; den = __dadd_rn(MS, C_pc); }
    else if (lane == 3) { num = nic; den = __dadd_rn(Sd, C_nw); }
    const double q2 = __ddiv_rn(num, den);
    const double cache_ms = __shfl_sync(0xffffffffu, q2, 0), nic_ms = __shfl_sync(0xffffffffu, q2, 1);
    const double pcie_ms = __shfl_sync(0xffffffffu, q2, 2), e_nic = __shfl_sync(0xffffffffu, q2, 3);

    double a = __longlong_as_double(0x7ff0000000000000ll); uint8_t la = 0xff;       // Eq. 1
    take_min(cache_ms, L_CACHE, a, la);
    take_min(nic_ms, L_NIC, a, la);
    take_min(pcie_ms, L_PCIE, a, la);
    take_min(gpu, L_GPU, a, la);
    double d = __longlong_as_double(0x7ff0000000000000ll); uint8_t ld = 0xff;       // Eq. 2 (R-M4)
    take_min(cache_ms, L_CACHE, d, ld);
    take_min(nic_ms, L_NIC, d, ld);
    take_min(__dmul_rn(nd, p.t_augment), L_CPU_AUG, d, ld);
    take_min(pcie_ms, L_PCIE, d, ld);
    take_min(gpu, L_GPU, d, ld);
    double e = __longlong_as_double(0x7ff0000000000000ll); uint8_t le = 0xff;       // Eq. 3
    take_min(e_cache, L_CACHE, e, le);
    take_min(e_nic, L_NIC, e, le);
    take_min(__dmul_rn(nd, p.t_decode_augment), L_CPU_DEC_AUG, e, le);
    take_min(pcie_ms, L_PCIE, e, le);
    take_min(gpu, L_GPU, e, le);
    double s2 = e; uint8_t ls = le;                                                   // Eq. 4
    if (st < e) { s2 = st; ls = L_STORAGE; }
    dsi[0] = a; dsi[1] = d; dsi[2] = e; dsi[3] = s2;
    lim[0] = la; lim[1] = ld; lim[2] = le; lim[3] = ls;
}

// One row per grid coordinate value k (p = k g %): the capacities clamped to N
// (exact integers, Eqs. 5-7, R-M6) and the Eq. 9 terms that depend on a single
// coordinate.  Array-of-rows so that one byte offset per coordinate addresses
// every field with an immediate displacement.
struct Row {
    uint32_t capc;   // min(N, capAD(p))  -- A and D tiers (M x S_data per sample); used when N < 2^31
    uint32_t cape;   // min(N, capE(p))   -- E tier (S_data per sample)
    double tA;       // (capc/N) DSI_A
    double tD;       // (capc/N) DSI_D        (D unclamped)
    double tDc;      // ((N - capc)/N) DSI_D  (D clamped by the A count, indexed by p_A)
    double tE;       // (cape/N) DSI_E        (E unclamped)
};
static_assert(sizeof(Row) == 40, "Row layout");

// Per-profile header: Eqs. 1-4 results and what the row build needs.
struct Header {
    double dsi[4];
    uint64_t N, Xad, Dad, De, cache_bytes;
    double rDad, rDe;          // RN(1/Dad), RN(1/De): estimates for the exact floors of Eqs. 5-7
    uint8_t lim[4];
    uint32_t valid;
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

// Eqs. 1-4 of profile `pi` into a header (one warp; every lane computes the
// same values, lane 0 stores).
__device__ void build_header(const seneca_mdp_profile* __restrict__ profiles, uint32_t pi, Header& H) {
    const uint32_t lane = threadIdx.x & 31;
    const seneca_mdp_profile p = profiles[pi];
    const bool ok = profile_valid(p);
    double dsi[4] = {0.0, 0.0, 0.0, 0.0};
    uint8_t lim[4] = {0, 0, 0, 0};
#if SENECA_MDP_PARHDR
    if (ok) tier_throughputs_warp(p, dsi, lim);                   // ok is warp-uniform
#else
    if (ok) tier_throughputs(p, dsi, lim);
#endif
    if (lane == 0) {
        H.valid = ok;
        for (int t = 0; t < 4; ++t) { H.dsi[t] = dsi[t]; H.lim[t] = lim[t]; }
        H.N = p.n_total;
        H.Xad = p.cache_bytes * p.m_den;
        H.Dad = 100ull * p.m_num * p.s_data;
        H.De = 100ull * p.s_data;
        H.cache_bytes = p.cache_bytes;
        H.rDad = __drcp_rn(u2d(H.Dad));
        H.rDe = __drcp_rn(u2d(H.De));
    }
}

// floor(num / den) exactly, for den < 2^62: q0 = trunc(RN(num) * RN(1/den)) is
// within 1 of the quotient while it is < 2^50 (relative error < 2^-51); the
// residual num - q0 den, exact in two's complement because |residual| < 2 den,
// corrects it.  Larger quotients (or den) take the u64 division routine.
__device__ __forceinline__ uint64_t floor_div(uint64_t num, uint64_t den, double rden) {
#if SENECA_MDP_FASTDIV
    const double qe = __dmul_rn(u2d(num), rden);
    if (den < (1ull << 62) && qe < 1125899906842624.0) {          // 2^50
        uint64_t q = (uint64_t)qe;
        const int64_t r = (int64_t)(num - q * den);
        if (r < 0) --q;
        else if ((uint64_t)r >= den) ++q;
        return q;
    }
#endif
    (void)rden;
    return num / den;
}

// Rows k0 .. k0+31 (one per lane, k <= steps) of a valid profile's tables.
__device__ void build_rows(const Header& H, uint32_t k0, uint32_t g, uint32_t steps, Row* rows) {
    const uint32_t k = k0 + (threadIdx.x & 31);
    if (k > steps) return;
    const uint64_t N = H.N;
    const double dN = u2d(N);
    const bool exact_div = N < (1ull << 53);
    const double yN = __drcp_rn(dN);
    const uint64_t pct = (uint64_t)k * g;
    uint64_t cad = floor_div(pct * H.Xad, H.Dad, H.rDad), ce = floor_div(pct * H.cache_bytes, H.De, H.rDe);   // Eqs. 5-7, exact floors
    cad = cad < N ? cad : N;
    ce = ce < N ? ce : N;
    Row& R = rows[k];
    R.capc = (uint32_t)cad;                                          // used only when N < 2^31
    R.cape = (uint32_t)ce;
    const double fa = exact_div ? div_by_n(u2d(cad), dN, yN) : __ddiv_rn(u2d(cad), dN);
    const double fc = exact_div ? div_by_n(u2d(N - cad), dN, yN) : __ddiv_rn(u2d(N - cad), dN);
    const double fe = exact_div ? div_by_n(u2d(ce), dN, yN) : __ddiv_rn(u2d(ce), dN);
    R.tA = __dmul_rn(fa, H.dsi[0]);
    R.tD = __dmul_rn(fa, H.dsi[1]);
    R.tDc = __dmul_rn(fc, H.dsi[1]);
    R.tE = __dmul_rn(fe, H.dsi[2]);
}

__device__ __forceinline__ const Row& row_at(const Row* rows, uint32_t byte_off) {
    return *reinterpret_cast<const Row*>(reinterpret_cast<const char*>(rows) + byte_off);
}

// One chunk of kChunk consecutive splits of one profile (N < 2^31: every count
// fits 32 bits), kChunk / 32 per lane.  Branch-free: each split needs exactly
// one quotient -- the clamped E count or the storage count (a clamped tier
// forces every later count to 0) -- so the numerator and its multiplier are
// selected.  Eq. 9 in the order of R-M7 is ((tA + tD) + tE) + tS; with E
// clamped it is ((tA + tD) + tE) + 0 and is computed as ((tA + tD) + 0) + tE,
// the same value (x + 0 = x for x >= +0).
struct Sweep32 {        // per-profile constants of the 32-bit sweep, hoisted out of the chunks
    uint32_t N;
    double dN, y, dsiE, dsiS;
};

template <bool kGrid, bool kFull>
__device__ __forceinline__ void sweep32_chunk(const Sweep32& P, const Row* rows, const uint2* __restrict__ s_split,
                                              uint32_t i0, uint32_t n_splits, double* __restrict__ grow,
                                              double& best, uint32_t& best_i) {
    const uint32_t N = P.N;
    const double dN = P.dN, y = P.y, dsiE = P.dsiE, dsiS = P.dsiS;
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll (kUnroll)
    for (uint32_t u = 0; u < kChunk / 32; ++u) {
        const uint32_t idx = i0 + u * 32 + lane;
        if (!kFull && idx >= n_splits) break;
        const uint2 w = s_split[idx];                              // byte offsets of rows p_A | p_D << 16, p_E
        const Row& ra = row_at(rows, w.x & 0xffffu);
        const Row& rd = row_at(rows, w.x >> 16);
        const Row& re = row_at(rows, w.y);
        const uint32_t r1 = N - ra.capc;                           // Eq. 5: N_A = capc[p_A]
        const uint32_t cD = rd.capc;
        const bool dfree = cD <= r1;                               // Eq. 6 unclamped
        const uint32_t r2 = dfree ? r1 - cD : 0u;
        const uint32_t cE = re.cape;
        const bool efree = dfree && cE <= r2;                      // Eq. 7 unclamped
        const uint32_t x = efree ? r2 - cE : r2;                   // N_S, or the clamped N_E (0 if D clamped)
        const double q = div_by_n(u32_to_d(x), dN, y);
        const double prod = __dmul_rn(q, efree ? dsiS : dsiE);
        const double tD = dfree ? rd.tD : ra.tDc;
        const double tX = efree ? re.tE : 0.0;
        const double v = __dadd_rn(__dadd_rn(__dadd_rn(ra.tA, tD), tX), prod);
        if (kGrid) st_grid(grow + idx, v);
        if (v > best) { best = v; best_i = idx; }                 // a lane's idx only increases
    }
}

// The general chunk (N >= 2^31): the same split arithmetic with 64-bit counts
// and __ddiv_rn; the capacities (Eqs. 5-7 exact floors) recomputed on the fly
// -- a rare path, kept simple rather than fast.
__device__ void sweep64_chunk(const Header& H, const Row* rows, uint32_t g, const uint2* __restrict__ s_split,
                              uint32_t i0, uint32_t n_splits, double* grow, double& best, uint32_t& best_i) {
    const uint64_t N = H.N;
    const double dN = u2d(N);
    auto capc = [&](uint32_t k) { const uint64_t c = ((uint64_t)k * g * H.Xad) / H.Dad; return c < N ? c : N; };
    auto cape = [&](uint32_t k) { const uint64_t c = ((uint64_t)k * g * H.cache_bytes) / H.De; return c < N ? c : N; };
    for (uint32_t idx = i0 + (threadIdx.x & 31); idx < i0 + kChunk && idx < n_splits; idx += 32) {
        const uint2 w = s_split[idx];
        const uint32_t ka = (w.x & 0xffffu) / sizeof(Row), kd = (w.x >> 16) / sizeof(Row), ke = w.y / sizeof(Row);
        const uint64_t r1 = N - capc(ka);
        const uint64_t cD = capc(kd);
        const bool dfree = cD <= r1;
        const uint64_t r2 = dfree ? r1 - cD : 0ull;
        const uint64_t cE = cape(ke);
        const bool efree = dfree && cE <= r2;
        const uint64_t x = efree ? r2 - cE : r2;
        const double prod = __dmul_rn(__ddiv_rn(u2d(x), dN), efree ? H.dsi[3] : H.dsi[2]);
        const double tD = dfree ? rows[kd].tD : rows[ka].tDc;
        const double tX = efree ? rows[ke].tE : 0.0;
        const double v = __dadd_rn(__dadd_rn(__dadd_rn(rows[ka].tA, tD), tX), prod);
        if (grow) __stcs(grow + idx, v);
        if (v > best) { best = v; best_i = idx; }
    }
}

// One CTA per profile, persistent over a grid-stride list of profiles
// (iteration i sweeps profile blockIdx + i gridDim).  The work of an iteration
// is a list of items that warps take from a shared counter, so the serial
// per-profile setup never idles the CTA:
//   item 0                 Eqs. 1-4 header of profile i+2   (4 header buffers)
//   items 1 .. nrow        32 table rows each of profile i+1 (2 row buffers)
//   the rest               kChunk-split chunks of profile i's sweep
// Rows live once per CTA (uniform addresses, immediate field displacements);
// each iteration stores one contiguous grid row with streaming stores.  A
// warp's items come in increasing order, so a lane's split indices increase
// and `v > best` keeps the first maximum; argmax per lane / warp / CTA, exact
// ties -> smallest enumeration index (R-M8).
__global__ void __launch_bounds__(kThreads, SENECA_MDP_MINB)
mdp_sweep_kernel(const seneca_mdp_profile* __restrict__ profiles, uint32_t n_profiles, uint32_t g,
                 uint32_t steps, uint32_t n_splits, seneca_mdp_result* __restrict__ results,
                 double* __restrict__ grid) {
    constexpr int kWarps = kThreads / 32;
    __shared__ Header s_hdr[4];
    __shared__ Row s_rows[2][kMaxSteps];
    __shared__ double s_red_v[2][kWarps];
    __shared__ uint32_t s_red_i[2][kWarps];
    __shared__ uint32_t s_ctr[2];
    extern __shared__ uint2 s_split[];                              // [n_splits] row byte offsets
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t G = gridDim.x;
    const uint32_t nrow = (steps + 32) / 32;                        // row items per profile
    const uint32_t nchunk = (n_splits + kChunk - 1) / kChunk;
    const uint32_t n_items = 1 + nrow + nchunk;
    // enumeration index -> rows (R-M9 order): row a has p_E = 100 - a g and
    // positions b = 0..a with p_A = b g, p_D = (a - b) g
    for (uint32_t idx = threadIdx.x; idx < n_splits; idx += blockDim.x) {
        uint32_t a = (uint32_t)((sqrtf((float)(8u * idx + 1u)) - 1.0f) * 0.5f);   // row of idx, then exact fix-up
        while ((a + 1) * (a + 2) / 2 <= idx) ++a;
        while (a * (a + 1) / 2 > idx) --a;
        const uint32_t b = idx - a * (a + 1) / 2;
        s_split[idx] = make_uint2((uint32_t)(b * sizeof(Row)) | (uint32_t)((a - b) * sizeof(Row)) << 16,
                                  (uint32_t)((steps - a) * sizeof(Row)));
    }
    if (threadIdx.x < 2) s_ctr[threadIdx.x] = 0;
    if (w < 2 && blockIdx.x + w * G < n_profiles) build_header(profiles, blockIdx.x + w * G, s_hdr[w]);
    __syncthreads();
    if (w < nrow && s_hdr[0].valid) build_rows(s_hdr[0], w * 32, g, steps, s_rows[0]);
    __syncthreads();

    uint32_t it = 0;
    for (uint32_t pi = blockIdx.x; pi < n_profiles; pi += G, ++it) {
        const uint32_t buf = it & 1;
        const Header& H = s_hdr[it & 3];
        const bool valid = H.valid;
        double* grow = (grid && valid) ? grid + (uint64_t)pi * n_splits : nullptr;
        double best = __longlong_as_double(0xfff0000000000000ll);
        uint32_t best_i = 0xffffffffu;
        const bool narrow = H.N < (1ull << 31);
        Sweep32 P;
        P.N = (uint32_t)H.N;
        P.dN = u2d(H.N);
        P.y = __drcp_rn(P.dN);
        P.dsiE = H.dsi[2];
        P.dsiS = H.dsi[3];
        if (threadIdx.x == 0) s_ctr[buf ^ 1] = 0;                  // next iteration's counter (idle since the last barrier)
        for (;;) {
            uint32_t t = 0;
            if (lane == 0) t = atomicAdd(&s_ctr[buf], 1u);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (t >= n_items) break;
            if (t == 0) {
                if (pi + 2 * G < n_profiles) build_header(profiles, pi + 2 * G, s_hdr[(it + 2) & 3]);
            } else if (t <= nrow) {
                const Header& Hn = s_hdr[(it + 1) & 3];
                if (pi + G < n_profiles && Hn.valid) build_rows(Hn, (t - 1) * 32, g, steps, s_rows[buf ^ 1]);
            } else if (valid) {
                const uint32_t i0 = (t - 1 - nrow) * kChunk;
                if (narrow) {
                    const bool full = i0 + kChunk <= n_splits;
                    if (grow) {
                        if (full) sweep32_chunk<true, true>(P, s_rows[buf], s_split, i0, n_splits, grow, best, best_i);
                        else sweep32_chunk<true, false>(P, s_rows[buf], s_split, i0, n_splits, grow, best, best_i);
                    } else {
                        if (full) sweep32_chunk<false, true>(P, s_rows[buf], s_split, i0, n_splits, nullptr, best, best_i);
                        else sweep32_chunk<false, false>(P, s_rows[buf], s_split, i0, n_splits, nullptr, best, best_i);
                    }
                } else {
                    sweep64_chunk(H, s_rows[buf], g, s_split, i0, n_splits, grow, best, best_i);
                }
            }
        }
#if SENECA_MDP_REDUX
        {   // warp argmax: the maximum by butterfly (values are finite or -inf, no NaN),
            // then the smallest index among the lanes that hold it (REDUX.MIN) -- the
            // same (max, first index) as the pairwise reduction
            double m = best;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
            best_i = __reduce_min_sync(0xffffffffu, best == m ? best_i : 0xffffffffu);
            best = m;
        }
#else
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, best, o);
            const uint32_t oi = __shfl_xor_sync(0xffffffffu, best_i, o);
            if (ov > best || (ov == best && oi < best_i)) { best = ov; best_i = oi; }
        }
#endif
        if (lane == 0) { s_red_v[buf][w] = best; s_red_i[buf][w] = best_i; }
        __syncthreads();                                            // publishes next rows / headers, this reduction
        if (threadIdx.x == 0) {
            seneca_mdp_result r = {};
            if (!valid) {
                r.status = 1;
            } else {
                best = s_red_v[buf][0]; best_i = s_red_i[buf][0];
                for (int k = 1; k < kWarps; ++k) {
                    const double ov = s_red_v[buf][k];
                    const uint32_t oi = s_red_i[buf][k];
                    if (ov > best || (ov == best && oi < best_i)) { best = ov; best_i = oi; }
                }
                uint32_t ra = 0, rb = best_i;
                while (rb > ra) { rb -= ra + 1; ++ra; }
                r.p_e = (uint8_t)(100 - ra * g);
                r.p_d = (uint8_t)((ra - rb) * g);
                r.p_a = (uint8_t)(rb * g);
                r.lim_a = H.lim[0]; r.lim_d = H.lim[1]; r.lim_e = H.lim[2]; r.lim_s = H.lim[3];
                r.status = 0;
                r.v_best = best;
                r.dsi_a = H.dsi[0]; r.dsi_d = H.dsi[1]; r.dsi_e = H.dsi[2]; r.dsi_s = H.dsi[3];
            }
            results[pi] = r;
        }
        // header buffer (it & 3) is rewritten at iteration it + 2, after the
        // next barrier, which thread 0 reaches only after this store
    }
}

// ------------------------------------------------------------------ the paired sweep
// Splits mirrored in (p_A, p_D) -- (b, m) and (m, b) with the same p_E -- share
// every count of Eqs. 5-8 but N_A / N_D: the A and D tiers hold the same
// number of samples per byte (M x S_data), so capAD(p_A) + capAD(p_D) decides
// whether D is clamped (capAD(p_D) <= N - capAD(p_A) <=> the sum <= N) and
// N_E, N_S -- and with them the one per-split quotient N_S/N (or N_E/N) -- are
// identical for the two.  One pair = one quotient, two Eq. 9 sums: the same
// IEEE operations on the same operands as the per-split definition (tests
// compare the whole grid bit for bit).
//
// A group of kPairW warps sweeps one profile (named barrier per group, no CTA
// barrier): every warp derives the header (Eqs. 1-4) itself, the group builds
// the profile's rows (Eqs. 5-7 exact floors + one-coordinate Eq. 9 terms) in its
// shared buffer, then its threads take the pairs.  The pair table (row offsets
// of p_A = b, p_D = m, p_E and the two enumeration indices) is built once per CTA.
#ifndef SENECA_MDP_PAIRW
#define SENECA_MDP_PAIRW 2
#endif
#ifndef SENECA_MDP_PUNROLL
#define SENECA_MDP_PUNROLL 2      // pairs in flight per thread
#endif
#ifndef SENECA_MDP_HDR1
#define SENECA_MDP_HDR1 1         // 1: the group's first warp derives the header, shared via shared memory (A/B)
#endif
constexpr uint32_t kPairW = SENECA_MDP_PAIRW;                 // warps per profile group
constexpr int kPUnroll = SENECA_MDP_PUNROLL;
constexpr uint32_t kGroups = kThreads / 32 / kPairW;          // groups per CTA
constexpr uint32_t kMaxPairs = 2601;                          // 1 % grid: sum over rows of ceil((a + 1) / 2)
static_assert(kPairW * 32 >= kMaxSteps / 2 + 1, "a thread must meet at most one pair per row (argmax order)");

__device__ __forceinline__ void group_sync(uint32_t gid) {
    asm volatile("bar.sync %0, %1;" :: "r"(gid + 1), "r"(kPairW * 32) : "memory");
}

// Eqs. 1-4 of a profile for this warp (all lanes), and its validity.
struct Hdr {
    double dsi[4];
    uint8_t lim[4];
    bool valid;
};

__device__ __forceinline__ Hdr warp_header(const seneca_mdp_profile& p) {
    Hdr h;
    h.valid = profile_valid(p);
    for (int t = 0; t < 4; ++t) { h.dsi[t] = 0.0; h.lim[t] = 0; }
    if (h.valid) tier_throughputs_warp(p, h.dsi, h.lim);            // valid is warp-uniform
    return h;
}

// enumeration index -> (row a, position b) of R-M9: a(a+1)/2 <= i < (a+1)(a+2)/2
__device__ __forceinline__ void index_to_split(uint32_t i, uint32_t& a, uint32_t& b) {
    a = (uint32_t)((sqrtf((float)(8u * i + 1u)) - 1.0f) * 0.5f);
    while ((a + 1) * (a + 2) / 2 <= i) ++a;
    while (a * (a + 1) / 2 > i) --a;
    b = i - a * (a + 1) / 2;
}

// The pair table of a grid step (every CTA of mdp_sweep_pairs copies it into
// shared memory): row a (p_E = 100 - a g) holds positions b = 0..a (p_A = b g,
// p_D = (a - b) g) at enumeration index a(a+1)/2 + b (R-M9); pair (b, a - b) for
// b <= a / 2.  x = row offset of p_A=b | of p_D=a-b << 12 | p_E row << 24,
// y = index of (b, a - b) | index of (a - b, b) << 16.  Rows before a = 2m hold
// m(m + 1) pairs, before a = 2m + 1: (m + 1)^2.
// one table per grid step (steps = 100 / g for the 9 divisors g of 100), never
// rewritten once built: concurrent sweeps on other streams may read them
constexpr uint32_t kStepSlots = 9;
__device__ __align__(16) uint2 g_pairs[kStepSlots][kMaxPairs + 1];
// the same pairs for the structure-of-arrays rows (SENECA_MDP_DENSE): x = row
// index of p_A = b | of p_D = a - b << 8 | of p_E << 16, y as above
__device__ __align__(16) uint2 g_pairs_dense[kStepSlots][kMaxPairs + 1];
__host__ __device__ constexpr uint32_t step_slot(uint32_t steps) {
    return steps == 100 ? 0 : steps == 50 ? 1 : steps == 25 ? 2 : steps == 20 ? 3 : steps == 10 ? 4
         : steps == 5 ? 5 : steps == 4 ? 6 : steps == 2 ? 7 : 8;
}

__global__ void mdp_pair_table(uint32_t steps, uint32_t n_pairs) {
    uint2* tab = g_pairs[step_slot(steps)];
    auto pairs_before = [](uint32_t a) { const uint32_t m = a >> 1; return (a & 1) ? (m + 1) * (m + 1) : m * (m + 1); };
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n_pairs; t += gridDim.x * blockDim.x) {
        uint32_t a = 2u * (uint32_t)sqrtf((float)t);                 // row of pair t, then exact fix-up
        while (a > 0 && pairs_before(a) > t) --a;
        while (pairs_before(a + 1) <= t) ++a;
        const uint32_t b = t - pairs_before(a), m = a - b, i0 = a * (a + 1) / 2;
        tab[t] = make_uint2((uint32_t)(b * sizeof(Row)) | (uint32_t)(m * sizeof(Row)) << 12 | (steps - a) << 24,
                                (i0 + b) | (i0 + m) << 16);
#if SENECA_MDP_DENSE == 2
        // byte offsets of 8-B row slots and of grid entries, ready to add
        g_pairs_dense[step_slot(steps)][t] = make_uint2(8 * b | 8 * m << 10 | 8 * (steps - a) << 20,
                                                        8 * (i0 + b) | 8 * (i0 + m) << 16);
#else
        g_pairs_dense[step_slot(steps)][t] = make_uint2(b | m << 8 | (steps - a) << 16, (i0 + b) | (i0 + m) << 16);
#endif
    }
}

// The pairs of one profile taken by thread gt of its group (N < 2^31), AoS rows.
template <bool kGrid>
__device__ __forceinline__ void aos_pairs(const Row* rows, const uint2* __restrict__ s_pair, uint32_t n_pairs, uint32_t gt,
                                          uint32_t N, double dN, double y, double dsiE, double dsiS,
                                          double* __restrict__ grow, double& best, uint32_t& best_i) {
    const char* rb0 = reinterpret_cast<const char*>(rows);
#pragma unroll (kPUnroll)
    for (uint32_t t = gt; t < n_pairs; t += kPairW * 32) {
        const uint2 w = s_pair[t];
        const Row& rb = *reinterpret_cast<const Row*>(rb0 + (w.x & 0xfffu));
        const Row& rm = *reinterpret_cast<const Row*>(rb0 + ((w.x >> 12) & 0xfffu));
        const Row& re = rows[w.x >> 24];
        const uint32_t cb = rb.capc, cm = rm.capc;
        const uint32_t sum = cb + cm;                       // <= 2N < 2^32
        const bool dfree = sum <= N;                        // Eq. 6 unclamped (both splits)
        const uint32_t r2 = dfree ? N - sum : 0u;
        const uint32_t cE = re.cape;
        const bool efree = dfree && cE <= r2;               // Eq. 7 unclamped
        const uint32_t x = efree ? r2 - cE : r2;            // N_S, or the clamped N_E (0 if D clamped)
        const double q = div_by_n(u32_to_d(x), dN, y);
        const double prod = __dmul_rn(q, efree ? dsiS : dsiE);
        const double tX = efree ? re.tE : 0.0;
        const double v0 = __dadd_rn(__dadd_rn(__dadd_rn(rb.tA, dfree ? rm.tD : rb.tDc), tX), prod);
        const double v1 = __dadd_rn(__dadd_rn(__dadd_rn(rm.tA, dfree ? rb.tD : rm.tDc), tX), prod);
        const uint32_t i0 = w.y & 0xffffu, i1 = w.y >> 16;
        if (kGrid) { st_grid(grow + i0, v0); st_grid(grow + i1, v1); }
        // a thread meets at most one pair per row (kPairW * 32 >= the 51 pairs
        // of the longest row) and i0 <= i1, so its indices only increase:
        // strict > keeps the first maximum = the smallest index (R-M8)
        if (v0 > best) { best = v0; best_i = i0; }
        if (v1 > best) { best = v1; best_i = i1; }
    }
}

// Structure-of-arrays rows of one group: capc u32[104] | cape u32[104] | tA | tD |
// tDc | tE f64[104] -- a lane reading consecutive rows reads consecutive words
// (one wavefront for a 4-B field, two for an 8-B one), where the 40-B Row
// stride costs two for either.
constexpr uint32_t kDR = 104;
#if SENECA_MDP_DENSE == 2
// (2: capc and cape interleaved in one 8-B slot per row, so every field of row k
// is at 8k + a constant: one address per row index, the fields by immediates)
constexpr uint32_t kDCapc = 0, kDCape = 4, kDTA = 8 * kDR, kDTD = 16 * kDR, kDTDC = 24 * kDR, kDTE = 32 * kDR,
                   kDBytes = 40 * kDR;
#else
constexpr uint32_t kDCapc = 0, kDCape = 4 * kDR, kDTA = 8 * kDR, kDTD = 16 * kDR, kDTDC = 24 * kDR, kDTE = 32 * kDR,
                   kDBytes = 40 * kDR;
#endif
constexpr uint32_t kDIdx = SENECA_MDP_DENSE == 2 ? 2 : 1;   // u32 index scale of capc / cape
struct DenseRows {
    char* p;
    __device__ uint32_t& capc(uint32_t k) const { return reinterpret_cast<uint32_t*>(p + kDCapc)[kDIdx * k]; }
    __device__ uint32_t& cape(uint32_t k) const { return reinterpret_cast<uint32_t*>(p + kDCape)[kDIdx * k]; }
    __device__ double& tA(uint32_t k) const { return reinterpret_cast<double*>(p + kDTA)[k]; }
    __device__ double& tD(uint32_t k) const { return reinterpret_cast<double*>(p + kDTD)[k]; }
    __device__ double& tDc(uint32_t k) const { return reinterpret_cast<double*>(p + kDTDC)[k]; }
    __device__ double& tE(uint32_t k) const { return reinterpret_cast<double*>(p + kDTE)[k]; }
};

// Rows k0 .. k0+31 (one per lane) of a valid profile, dense layout (the same
// values as build_rows).
__device__ void build_rows_dense(const Header& H, uint32_t k0, uint32_t g, uint32_t steps, DenseRows R) {
    const uint32_t k = k0 + (threadIdx.x & 31);
    if (k > steps) return;
    const uint64_t N = H.N;
    const double dN = u2d(N);
    const bool exact_div = N < (1ull << 53);
    const double yN = __drcp_rn(dN);
    const uint64_t pct = (uint64_t)k * g;
    uint64_t cad = floor_div(pct * H.Xad, H.Dad, H.rDad), ce = floor_div(pct * H.cache_bytes, H.De, H.rDe);   // Eqs. 5-7, exact floors
    cad = cad < N ? cad : N;
    ce = ce < N ? ce : N;
    const double fa = exact_div ? div_by_n(u2d(cad), dN, yN) : __ddiv_rn(u2d(cad), dN);
    const double fc = exact_div ? div_by_n(u2d(N - cad), dN, yN) : __ddiv_rn(u2d(N - cad), dN);
    const double fe = exact_div ? div_by_n(u2d(ce), dN, yN) : __ddiv_rn(u2d(ce), dN);
    R.capc(k) = (uint32_t)cad;                                       // used only when N < 2^31
    R.cape(k) = (uint32_t)ce;
    R.tA(k) = __dmul_rn(fa, H.dsi[0]);
    R.tD(k) = __dmul_rn(fa, H.dsi[1]);
    R.tDc(k) = __dmul_rn(fc, H.dsi[1]);
    R.tE(k) = __dmul_rn(fe, H.dsi[2]);
}

template <uint32_t kOff>
__device__ __forceinline__ uint32_t ldsd_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1+%2];" : "=r"(v) : "r"(a), "n"(kOff));
    return v;
}
template <uint32_t kOff>
__device__ __forceinline__ double ldsd_f64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(a), "n"(kOff));
    return v;
}

// The pairs of one profile taken by thread gt of its group (N < 2^31), dense
// rows at shared address sb: the arithmetic of aos_pairs.
template <bool kGrid>
__device__ __forceinline__ void dense_pairs(uint32_t sb, const uint2* __restrict__ s_pair, uint32_t n_pairs, uint32_t gt,
                                            uint32_t N, double dN, double y, double dsiE, double dsiS,
                                            double* __restrict__ grow, double& best, uint32_t& best_i) {
    constexpr uint32_t kDelta = kDTDC - kDTD;
#pragma unroll (kPUnroll)
    for (uint32_t t = gt; t < n_pairs; t += kPairW * 32) {
        const uint2 w = s_pair[t];
#if SENECA_MDP_DENSE == 2
        const uint32_t b8 = sb + (w.x & 0x3ffu), m8 = sb + ((w.x >> 10) & 0x3ffu), e8 = sb + (w.x >> 20);
        const uint32_t sum = ldsd_u32<kDCapc>(b8) + ldsd_u32<kDCapc>(m8);   // <= 2N < 2^32
        const uint32_t cE = ldsd_u32<kDCape>(e8);
#else
        const uint32_t b = w.x & 0xffu, m = __byte_perm(w.x, 0, 0x4441), e = w.x >> 16;
        const uint32_t b4 = sb + 4 * b, m4 = sb + 4 * m, b8 = sb + 8 * b, m8 = sb + 8 * m, e8 = sb + 8 * e;
        const uint32_t sum = ldsd_u32<kDCapc>(b4) + ldsd_u32<kDCapc>(m4);   // <= 2N < 2^32
        const uint32_t cE = ldsd_u32<kDCape>(sb + 4 * e);
#endif
        const bool dfree = sum <= N;                        // Eq. 6 unclamped (both splits)
        const uint32_t r2 = dfree ? N - sum : 0u;
        const bool efree = dfree && cE <= r2;               // Eq. 7 unclamped
        const uint32_t x = efree ? r2 - cE : r2;            // N_S, or the clamped N_E (0 if D clamped)
        const double q = div_by_n(u32_to_d(x), dN, y);
        const double prod = __dmul_rn(q, efree ? dsiS : dsiE);
        const double tX = efree ? ldsd_f64<kDTE>(e8) : 0.0;
        // Eq. 6: tD of the other coordinate when D is free, else tDc of this one
        const double d0 = ldsd_f64<kDTDC>(dfree ? m8 - kDelta : b8);
        const double d1 = ldsd_f64<kDTDC>(dfree ? b8 - kDelta : m8);
        const double v0 = __dadd_rn(__dadd_rn(__dadd_rn(ldsd_f64<kDTA>(b8), d0), tX), prod);
        const double v1 = __dadd_rn(__dadd_rn(__dadd_rn(ldsd_f64<kDTA>(m8), d1), tX), prod);
        const uint32_t i0 = w.y & 0xffffu, i1 = w.y >> 16;   // (DENSE 2: byte offsets, 8 x the index)
#if SENECA_MDP_DENSE == 2
        if (kGrid) {
            st_grid(reinterpret_cast<double*>(reinterpret_cast<char*>(grow) + i0), v0);
            st_grid(reinterpret_cast<double*>(reinterpret_cast<char*>(grow) + i1), v1);
        }
#else
        if (kGrid) { st_grid(grow + i0, v0); st_grid(grow + i1, v1); }
#endif
        if (v0 > best) { best = v0; best_i = i0; }
        if (v1 > best) { best = v1; best_i = i1; }
    }
}

__global__ void __launch_bounds__(kThreads, SENECA_MDP_MINB)
mdp_sweep_pairs(const seneca_mdp_profile* __restrict__ profiles, uint32_t n_profiles, uint32_t g,
                uint32_t steps, uint32_t n_splits, uint32_t n_pairs, seneca_mdp_result* __restrict__ results,
                double* __restrict__ grid) {
#if SENECA_MDP_DENSE
    __shared__ __align__(16) char s_drows[kGroups][kDBytes];
#else
    __shared__ Row s_rows[kGroups][kMaxSteps];
#endif
    __shared__ double s_red_v[kGroups][kPairW];
    __shared__ uint32_t s_red_i[kGroups][kPairW];
    extern __shared__ uint2 s_pair[];                               // [n_pairs]
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t gid = warp / kPairW, gw = warp % kPairW, gt = gw * 32 + lane;   // group, warp / thread in it
    // pair table: row a (p_E = 100 - a g) holds positions b = 0..a (p_A = b g,
    // p_D = (a - b) g) at enumeration index a(a+1)/2 + b (R-M9); pair (b, a - b)
    // for b <= a / 2.  x = row offset of p_A=b | of p_D=a-b << 12 | p_E row << 24,
    // y = index of (b, a - b) | index of (a - b, b) << 16.
    // rows before a = 2m hold m(m + 1) pairs, before a = 2m + 1: (m + 1)^2
    // (built once per device and grid step by mdp_pair_table into g_pairs; copied
    // here with 16-B loads)
    {
#if SENECA_MDP_DENSE
        const uint2* tab = g_pairs_dense[step_slot(steps)];
#else
        const uint2* tab = g_pairs[step_slot(steps)];
#endif
        const uint4* src = reinterpret_cast<const uint4*>(tab);
        uint4* dst = reinterpret_cast<uint4*>(s_pair);
        for (uint32_t t = threadIdx.x; t < n_pairs / 2; t += blockDim.x) dst[t] = src[t];
        if ((n_pairs & 1u) && threadIdx.x == 0) s_pair[n_pairs - 1] = tab[n_pairs - 1];
    }
    __syncthreads();
#if SENECA_MDP_DENSE
    const DenseRows DR{s_drows[gid]};
#else
    Row* rows = s_rows[gid];
#endif
    const uint32_t n_groups = gridDim.x * kGroups;
    for (uint32_t pi = blockIdx.x * kGroups + gid; pi < n_profiles; pi += n_groups) {
        const seneca_mdp_profile prof = profiles[pi];
#if SENECA_MDP_HDR1
        // Eqs. 1-4 by the group's first warp, shared through shared memory
        __shared__ Hdr s_h[kGroups];
        if (gw == 0) {
            const Hdr h0 = warp_header(prof);
            if (lane == 0) s_h[gid] = h0;
        }
        group_sync(gid);
        const Hdr H = s_h[gid];
#else
        const Hdr H = warp_header(prof);
#endif
        double best = __longlong_as_double(0xfff0000000000000ll);
        uint32_t best_i = 0xffffffffu;
        if (H.valid) {                                              // group-uniform
            // rows (Eqs. 5-7 exact floors, clamped to N; one-coordinate Eq. 9 terms)
            Header B;
            for (int t = 0; t < 4; ++t) B.dsi[t] = H.dsi[t];
            B.N = prof.n_total;
            B.Xad = prof.cache_bytes * prof.m_den;
            B.Dad = 100ull * prof.m_num * prof.s_data;
            B.De = 100ull * prof.s_data;
            B.cache_bytes = prof.cache_bytes;
            B.rDad = __drcp_rn(u2d(B.Dad));
            B.rDe = __drcp_rn(u2d(B.De));
#if SENECA_MDP_DENSE
            for (uint32_t k0 = gw * 32; k0 <= steps; k0 += kPairW * 32) build_rows_dense(B, k0, g, steps, DR);
#else
            for (uint32_t k0 = gw * 32; k0 <= steps; k0 += kPairW * 32) build_rows(B, k0, g, steps, rows);
#endif
            group_sync(gid);
            double* grow = grid ? grid + (uint64_t)pi * n_splits : nullptr;
            if (B.N < (1ull << 31)) {
                const double dN = u2d(B.N), y = __drcp_rn(dN);
#if SENECA_MDP_DENSE
                const uint32_t sb = (uint32_t)__cvta_generic_to_shared(DR.p);
                if (grow) dense_pairs<true>(sb, s_pair, n_pairs, gt, (uint32_t)B.N, dN, y, H.dsi[2], H.dsi[3], grow, best, best_i);
                else dense_pairs<false>(sb, s_pair, n_pairs, gt, (uint32_t)B.N, dN, y, H.dsi[2], H.dsi[3], nullptr, best, best_i);
#else
                if (grow) aos_pairs<true>(rows, s_pair, n_pairs, gt, (uint32_t)B.N, dN, y, H.dsi[2], H.dsi[3], grow, best, best_i);
                else aos_pairs<false>(rows, s_pair, n_pairs, gt, (uint32_t)B.N, dN, y, H.dsi[2], H.dsi[3], nullptr, best, best_i);
#endif
            } else {                                                // N >= 2^31: 64-bit counts (rare)
                const uint64_t N = B.N;
                const double dN = u2d(N);
                auto capc = [&](uint32_t k) { const uint64_t c = ((uint64_t)k * g * B.Xad) / B.Dad; return c < N ? c : N; };
                auto cape = [&](uint32_t k) { const uint64_t c = ((uint64_t)k * g * B.cache_bytes) / B.De; return c < N ? c : N; };
                for (uint32_t t = gt; t < n_pairs; t += kPairW * 32) {
                    const uint2 w = s_pair[t];
                    for (int h = 0; h < 2; ++h) {
#if SENECA_MDP_DENSE == 2
                        const uint32_t kb = (w.x & 0x3ffu) >> 3, km = ((w.x >> 10) & 0x3ffu) >> 3;
                        const uint32_t ka = h ? km : kb, kd = h ? kb : km, ke = w.x >> 23;
                        const auto row_tA = [&](uint32_t k) { return DR.tA(k); };
                        const auto row_tD = [&](uint32_t k) { return DR.tD(k); };
                        const auto row_tDc = [&](uint32_t k) { return DR.tDc(k); };
                        const auto row_tE = [&](uint32_t k) { return DR.tE(k); };
#elif SENECA_MDP_DENSE
                        const uint32_t kb = w.x & 0xffu, km = (w.x >> 8) & 0xffu;
                        const uint32_t ka = h ? km : kb, kd = h ? kb : km, ke = w.x >> 16;
                        const auto row_tA = [&](uint32_t k) { return DR.tA(k); };
                        const auto row_tD = [&](uint32_t k) { return DR.tD(k); };
                        const auto row_tDc = [&](uint32_t k) { return DR.tDc(k); };
                        const auto row_tE = [&](uint32_t k) { return DR.tE(k); };
#else
                        const uint32_t ka = (h ? (w.x >> 12) & 0xfffu : w.x & 0xfffu) / sizeof(Row);
                        const uint32_t kd = (h ? w.x & 0xfffu : (w.x >> 12) & 0xfffu) / sizeof(Row);
                        const uint32_t ke = w.x >> 24;
                        const auto row_tA = [&](uint32_t k) { return rows[k].tA; };
                        const auto row_tD = [&](uint32_t k) { return rows[k].tD; };
                        const auto row_tDc = [&](uint32_t k) { return rows[k].tDc; };
                        const auto row_tE = [&](uint32_t k) { return rows[k].tE; };
#endif
                        const uint32_t idx = (h ? w.y >> 16 : w.y & 0xffffu) / (SENECA_MDP_DENSE == 2 ? 8u : 1u);
                        const uint64_t r1 = N - capc(ka);
                        const uint64_t cD = capc(kd);
                        const bool dfree = cD <= r1;
                        const uint64_t r2 = dfree ? r1 - cD : 0ull;
                        const uint64_t cE = cape(ke);
                        const bool efree = dfree && cE <= r2;
                        const uint64_t x = efree ? r2 - cE : r2;
                        const double prod = __dmul_rn(__ddiv_rn(u2d(x), dN), efree ? H.dsi[3] : H.dsi[2]);
                        const double tD = dfree ? row_tD(kd) : row_tDc(ka);
                        const double tX = efree ? row_tE(ke) : 0.0;
                        const double v = __dadd_rn(__dadd_rn(__dadd_rn(row_tA(ka), tD), tX), prod);
                        if (grow) __stcs(grow + idx, v);
                        const uint32_t bidx = SENECA_MDP_DENSE == 2 ? 8u * idx : idx;   // (DENSE 2: byte offsets)
                        if (v > best || (v == best && bidx < best_i)) { best = v; best_i = bidx; }
                    }
                }
            }
        }
        // argmax: the maximum by butterfly, then the smallest index holding it (R-M8)
        double mx = best;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        best_i = __reduce_min_sync(0xffffffffu, best == mx ? best_i : 0xffffffffu);
        if (lane == 0) { s_red_v[gid][gw] = mx; s_red_i[gid][gw] = best_i; }
        group_sync(gid);                                            // rows free, per-warp maxima visible
        if (gt == 0) {
            seneca_mdp_result r = {};
            if (!H.valid) {
                r.status = 1;
            } else {
                double bv = s_red_v[gid][0];
                uint32_t bi = s_red_i[gid][0];
                for (uint32_t k = 1; k < kPairW; ++k) {
                    const double ov = s_red_v[gid][k];
                    const uint32_t oi = s_red_i[gid][k];
                    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
                }
                uint32_t ra, rb;
                if (SENECA_MDP_DENSE == 2) bi >>= 3;                // byte offset -> split index
                index_to_split(bi, ra, rb);
                r.p_e = (uint8_t)(100 - ra * g);
                r.p_d = (uint8_t)((ra - rb) * g);
                r.p_a = (uint8_t)(rb * g);
                r.lim_a = H.lim[0]; r.lim_d = H.lim[1]; r.lim_e = H.lim[2]; r.lim_s = H.lim[3];
                r.status = 0;
                r.v_best = bv;
                r.dsi_a = H.dsi[0]; r.dsi_d = H.dsi[1]; r.dsi_e = H.dsi[2]; r.dsi_s = H.dsi[3];
            }
            results[pi] = r;
        }
        // the next profile's rows are written after this barrier; the per-warp
        // maxima after the next profile's first barrier, which thread gt == 0
        // reaches only after reading these
    }
}

#ifndef SENECA_MDP_GRID_CTAS
#define SENECA_MDP_GRID_CTAS 0    // > 0: at most this many mdp_sweep_pairs CTAs per SM when it writes the grid
#endif
// (Two TMA-staged grid kernels -- whole profile rows written by one cp.async.bulk
// store each -- were built and measured slower than this sweep, DESIGN.md 7.3;
// they are in the history at commit 40d95f7.)

// ------------------------------------------------------------------ evaluation at given splits
constexpr uint32_t kMaxEvalSplits = 4096;
struct EvalSplits {
    uint32_t packed[kMaxEvalSplits];   // p_e | p_d << 8 | p_a << 16
};

// One warp per profile (grid-stride), lanes over the splits.  Eqs. 5-8 in exact
// integers (validity keeps pct * cache * m_den < 2^64), Eq. 9 with one IEEE
// operation per step in the order of R-M7: ((tA + tD) + tE) + tS, t = (n/N) DSI.
__global__ void __launch_bounds__(256)
mdp_eval_kernel(const seneca_mdp_profile* __restrict__ profiles, uint32_t n_profiles,
                const __grid_constant__ EvalSplits S, uint32_t n_splits, double* __restrict__ values,
                uint64_t* __restrict__ counts, seneca_mdp_result* __restrict__ tiers) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warps = gridDim.x * (blockDim.x / 32);
    for (uint32_t pi = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); pi < n_profiles; pi += warps) {
        const seneca_mdp_profile p = profiles[pi];
        double* vrow = values + (uint64_t)pi * n_splits;
        uint64_t* crow = counts ? counts + (uint64_t)pi * n_splits * 4 : nullptr;
        if (!profile_valid(p)) {
            for (uint32_t s = lane; s < n_splits; s += 32) {
                vrow[s] = __longlong_as_double(0x7ff8000000000000ll);
                if (crow) for (int t = 0; t < 4; ++t) crow[4 * s + t] = 0;
            }
            if (tiers && lane == 0) { seneca_mdp_result r = {}; r.status = 1; tiers[pi] = r; }
            continue;
        }
        double dsi[4];
        uint8_t lim[4];
        tier_throughputs(p, dsi, lim);
        if (tiers && lane == 0) {
            seneca_mdp_result r = {};
            r.lim_a = lim[0]; r.lim_d = lim[1]; r.lim_e = lim[2]; r.lim_s = lim[3];
            r.dsi_a = dsi[0]; r.dsi_d = dsi[1]; r.dsi_e = dsi[2]; r.dsi_s = dsi[3];
            tiers[pi] = r;
        }
        const uint64_t N = p.n_total;
        const double dN = u2d(N);
        const uint64_t Xad = p.cache_bytes * p.m_den, Dad = 100ull * p.m_num * p.s_data, De = 100ull * p.s_data;
        for (uint32_t s = lane; s < n_splits; s += 32) {
            const uint32_t w = S.packed[s];
            const uint64_t pe = w & 0xff, pd = (w >> 8) & 0xff, pa = (w >> 16) & 0xff;
            const uint64_t capA = (pa * Xad) / Dad, capD = (pd * Xad) / Dad, capE = (pe * p.cache_bytes) / De;
            const uint64_t nA = N < capA ? N : capA;                                   // Eq. 5
            const uint64_t nD = (N - nA) < capD ? (N - nA) : capD;                     // Eq. 6
            const uint64_t nE = (N - nA - nD) < capE ? (N - nA - nD) : capE;           // Eq. 7
            const uint64_t nS = N - nA - nD - nE;                                      // Eq. 8
            const double tA = __dmul_rn(__ddiv_rn(u2d(nA), dN), dsi[0]);
            const double tD = __dmul_rn(__ddiv_rn(u2d(nD), dN), dsi[1]);
            const double tE = __dmul_rn(__ddiv_rn(u2d(nE), dN), dsi[2]);
            const double tS = __dmul_rn(__ddiv_rn(u2d(nS), dN), dsi[3]);
            vrow[s] = __dadd_rn(__dadd_rn(__dadd_rn(tA, tD), tE), tS);              // Eq. 9, R-M7
            if (crow) { crow[4 * s] = nA; crow[4 * s + 1] = nD; crow[4 * s + 2] = nE; crow[4 * s + 3] = nS; }
        }
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
    seneca::NvtxRange nvtx("seneca_mdp_sweep");
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
#if SENECA_MDP_PAIRS
    {
        uint32_t np = 0;
        for (uint32_t a = 0; a <= steps; ++a) np += a / 2 + 1;
        static int pslots = 0, psms = 0;
        if (!pslots) {
            int dev = 0, sms = 0, per_sm = 0;
            SENECA_CUDA_TRY(cudaGetDevice(&dev));
            SENECA_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
            psms = sms;
            SENECA_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mdp_sweep_pairs, kThreads,
                                                                          kMaxPairs * sizeof(uint2)));
            pslots = sms * (per_sm > 0 ? per_sm : 1);
        }
        {   // the pair table of this grid step on this device (stream-ordered before the sweep)
            static uint16_t built[64] = {};                         // bit step_slot per device
            int dev = 0;
            SENECA_CUDA_TRY(cudaGetDevice(&dev));
            const uint16_t bit = (uint16_t)(1u << step_slot(steps));
            if (dev < 0 || dev >= 64 || !(built[dev] & bit)) {
                // first use of this grid step on this device: built once, synchronously,
                // so that a sweep on any other stream finds it complete
                mdp_pair_table<<<(np + 255) / 256, 256, 0, (cudaStream_t)stream>>>(steps, np);
                SENECA_CUDA_TRY(cudaGetLastError());
                SENECA_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
                if (dev >= 0 && dev < 64) built[dev] |= bit;
            }
        }
        const uint32_t want = (n_profiles + kGroups - 1) / kGroups;
        uint32_t blocks = want < (uint32_t)pslots ? want : (uint32_t)pslots;
        // with the grid requested, fewer profile rows in flight: the DRAM write rate of
        // the row-interleaved store pattern falls as concurrent row streams grow
        // (tools/micro/store_pattern.cu)
        const uint32_t gcap = (uint32_t)psms * SENECA_MDP_GRID_CTAS;
        if (d_grid && SENECA_MDP_GRID_CTAS > 0 && blocks > gcap) blocks = gcap;
        mdp_sweep_pairs<<<blocks, kThreads, np * sizeof(uint2), (cudaStream_t)stream>>>(
            d_profiles, n_profiles, grid_step_pct, steps, ns, np, d_results, d_grid);
        SENECA_CUDA_TRY(cudaGetLastError());
        return SENECA_OK;
    }
#endif
    // persistent grid: every resident CTA slot of the device, never more CTAs than profiles
    static int slots = 0;
    if (!slots) {
        SENECA_CUDA_TRY(cudaFuncSetAttribute(mdp_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)(5151 * sizeof(uint2))));
        int dev = 0, sms = 0, per_sm = 0;
        SENECA_CUDA_TRY(cudaGetDevice(&dev));
        SENECA_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        SENECA_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mdp_sweep_kernel, kThreads,
                                                                      5151 * sizeof(uint2)));
        slots = sms * (per_sm > 0 ? per_sm : 1);
    }
    const uint32_t blocks = n_profiles < (uint32_t)slots ? n_profiles : (uint32_t)slots;
    mdp_sweep_kernel<<<blocks, kThreads, ns * sizeof(uint2), (cudaStream_t)stream>>>(
        d_profiles, n_profiles, grid_step_pct, steps, ns, d_results, d_grid);
    SENECA_CUDA_TRY(cudaGetLastError());
    return SENECA_OK;
}

extern "C" seneca_status seneca_mdp_eval(const seneca_mdp_profile* d_profiles, uint32_t n_profiles,
                                         const seneca_split* h_splits, uint32_t n_splits, double* d_values,
                                         uint64_t* d_counts, seneca_mdp_result* d_tiers, void* stream) {
    using namespace seneca;
    if (n_profiles == 0 || !d_profiles || !h_splits || !d_values) {
        set_error("seneca_mdp_eval: empty input or NULL pointer");
        return SENECA_EINVAL;
    }
    if (n_splits == 0 || n_splits > kMaxEvalSplits) {
        set_error("seneca_mdp_eval: n_splits %u not in [1, %u]", n_splits, kMaxEvalSplits);
        return SENECA_EINVAL;
    }
    EvalSplits S;                    // by-value kernel parameter (copied at launch)
    for (uint32_t s = 0; s < n_splits; ++s) {
        const seneca_split& x = h_splits[s];
        if ((uint32_t)x.p_e + x.p_d + x.p_a != 100) {
            set_error("seneca_mdp_eval: split %u sums to %u, not 100", s, (uint32_t)x.p_e + x.p_d + x.p_a);
            return SENECA_EINVAL;
        }
        S.packed[s] = x.p_e | (uint32_t)x.p_d << 8 | (uint32_t)x.p_a << 16;
    }
    const uint32_t warps = 256 / 32;
    uint32_t blocks = (n_profiles + warps - 1) / warps;
    blocks = blocks < 148u * 16u ? blocks : 148u * 16u;
    mdp_eval_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(d_profiles, n_profiles, S, n_splits, d_values,
                                                              d_counts, d_tiers);
    SENECA_CUDA_TRY(cudaGetLastError());
    return SENECA_OK;
}
