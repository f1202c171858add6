// capi.cu -- error plumbing, host-side integer helpers and the epoch model
// (seneca_epoch_model, NEXT-1) of libseneca.so.
#include <cmath>
#include <cstdarg>
#include <cstdio>

#include <cuda_runtime.h>

#include "common.cuh"

namespace seneca {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

seneca_status cuda_status(cudaError_t e, const char* what) {
    set_error("CUDA error %s (%s) in %s", cudaGetErrorName(e), cudaGetErrorString(e), what);
    return SENECA_ECUDA;
}

}  // namespace seneca

extern "C" const char* seneca_last_error(void) { return seneca::g_err; }

// 1 bit per sample per job + 1 byte per sample (status + reference)
extern "C" uint64_t seneca_metadata_bytes(uint64_t n_total, uint32_t n_jobs) {
    return (uint64_t)n_jobs * ((n_total + 7) / 8) + n_total;
}

// Eqs. 5-8, floors exact in integers (R-M6); caps = {E, D, A, storage}
extern "C" seneca_status seneca_split_capacities(uint64_t n_total, uint64_t s_data, uint32_t m_num,
                                                 uint32_t m_den, uint64_t cache_bytes, uint32_t p_e,
                                                 uint32_t p_d, uint32_t p_a, uint64_t caps[4]) {
    using seneca::set_error;
    if (!caps || n_total == 0 || s_data == 0 || m_den == 0 || m_num < m_den || p_e + p_d + p_a != 100) {
        set_error("seneca_split_capacities: invalid argument");
        return SENECA_EINVAL;
    }
    if (cache_bytes > (~0ull / 100ull) / m_den || s_data > (~0ull / 100ull) / m_num) {
        set_error("seneca_split_capacities: 100*cache*m_den or 100*m_num*s_data overflows");
        return SENECA_EINVAL;
    }
    const uint64_t den_ad = 100ull * m_num * s_data, den_e = 100ull * s_data;
    const uint64_t cap_a = ((uint64_t)p_a * cache_bytes * m_den) / den_ad;
    const uint64_t cap_d = ((uint64_t)p_d * cache_bytes * m_den) / den_ad;
    const uint64_t cap_e = ((uint64_t)p_e * cache_bytes) / den_e;
    const uint64_t n_a = cap_a < n_total ? cap_a : n_total;
    const uint64_t n_d = cap_d < n_total - n_a ? cap_d : n_total - n_a;
    const uint64_t n_e = cap_e < n_total - n_a - n_d ? cap_e : n_total - n_a - n_d;
    caps[0] = n_e;
    caps[1] = n_d;
    caps[2] = n_a;
    caps[3] = n_total - n_a - n_d - n_e;
    return SENECA_OK;
}

// ------------------------------------------------------------------ epoch model (NEXT-1)
namespace seneca {
namespace {
__global__ void epoch_model_kernel(const seneca_job_epoch_stats* __restrict__ st, uint32_t n, uint64_t N,
                                   double dA, double dD, double dE, double dS, seneca_epoch_metrics* __restrict__ out) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const uint64_t sS = st[r].served[0], sE = st[r].served[1], sD = st[r].served[2], sA = st[r].served[3];
    const double dN = __ull2double_rn(N);
    const double cA = __ull2double_rn(sA), cD = __ull2double_rn(sD), cE = __ull2double_rn(sE),
                 cS = __ull2double_rn(sS);
    double t = __ddiv_rn(cA, dA);
    t = __dadd_rn(t, __ddiv_rn(cD, dD));
    t = __dadd_rn(t, __ddiv_rn(cE, dE));
    t = __dadd_rn(t, __ddiv_rn(cS, dS));
    double v = __dmul_rn(__ddiv_rn(cA, dN), dA);
    v = __dadd_rn(v, __dmul_rn(__ddiv_rn(cD, dN), dD));
    v = __dadd_rn(v, __dmul_rn(__ddiv_rn(cE, dN), dE));
    v = __dadd_rn(v, __dmul_rn(__ddiv_rn(cS, dN), dS));
    seneca_epoch_metrics m;
    m.epoch_seconds = t;
    m.dsi_mix = v;
    m.decode_aug_ops = sS + sE;
    m.aug_only_ops = sD;
    m.hit_rate = __ddiv_rn(__ull2double_rn(sE + sD + sA), dN);
    out[r] = m;
}
}  // namespace
}  // namespace seneca

extern "C" seneca_status seneca_epoch_model(const seneca_job_epoch_stats* d_stats, uint32_t n_rows, uint64_t n_total,
                                            const double h_dsi[4], seneca_epoch_metrics* d_out, void* stream) {
    using namespace seneca;
    if (!d_stats || !h_dsi || !d_out || n_rows == 0 || n_total == 0) {
        set_error("seneca_epoch_model: NULL pointer or empty input");
        return SENECA_EINVAL;
    }
    for (int t = 0; t < 4; ++t)
        if (!(h_dsi[t] > 0.0) || !std::isfinite(h_dsi[t])) {
            set_error("seneca_epoch_model: DSI[%d] must be finite and > 0", t);
            return SENECA_EINVAL;
        }
    epoch_model_kernel<<<(n_rows + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
        d_stats, n_rows, n_total, h_dsi[0], h_dsi[1], h_dsi[2], h_dsi[3], d_out);
    SENECA_CUDA_TRY(cudaGetLastError());
    return SENECA_OK;
}
