// capi.cu -- error plumbing and host-side integer helpers of libseneca.so.
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
