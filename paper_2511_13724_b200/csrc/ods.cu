// ods.cu -- Opportunistic Data Sampling replay on B200.
//
// §5.2 of the paper made concrete by readings R-O1..R-O20
// (DESIGN.md §3).  One round = one batch for each listed job, then maintain:
//
//   ods_request_classify  <<<jobs, 1024>>>  a1-a3: walk the job's current lap
//        list (its keyed permutation, then the lists of deferred misses) from
//        the cursor, test seen bits, compact the first `need` unseen ids
//        (ballot/scan), classify hits vs misses against the residency bitmaps and
//        the job's consumer set, mark hits seen and update the pool counts; the
//        number of substitutes per tier k_A, k_D, k_E follows from the pool sizes.
//   ods_select_apply      <<<jobs x 3, 512>>>  a4-a6: one CTA per (job, tier):
//        keyed ranks sigma(u) over the ascending pool, located through the
//        superblock/block count hierarchy (superblock prefix in shared memory,
//        then one 128-B row of block counts, then one 128-B row of bitmap words);
//        the last CTA of a job finishes it: storage misses, deferral lists,
//        counters, digest, transcript.
//   ods_maintain          <<<1, 1024>>>  a7: eviction of A entries consumed by
//        every active job, keyed refill from the storage pool, count updates.
//   epoch end (a8): memset of seen_j, ods_recount (pool counts of the job),
//        ods_perm_fill (the next epoch's permutation, whole-GPU, ALU-bound).
//
// Pool counts: for every pool (job x {A, D, E}, plus the storage pool) a count
// per 1024-id block, per 32-block superblock and a total, kept exact
// incrementally; a pool member is an id whose pool word bit is set:
//   A: tier_A & ~seen_j & ~cons_j    D: tier_D & ~seen_j    E: tier_E & ~seen_j
//   S: ~(tier_E | tier_D | tier_A)   (R-O2, R-O8)
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include <cuda_runtime.h>

#include "common.cuh"

namespace seneca {
namespace {

constexpr uint32_t T_S = 0, T_E = 1, T_D = 2, T_A = 3, SUBST = 4;
constexpr uint32_t kMaxJobs = 32;
constexpr uint32_t kMaxBatch = 4096;
constexpr uint32_t kReqThreads = 1024;
constexpr uint32_t kSelThreads = 512;
constexpr uint32_t kMaintThreads = 1024;
constexpr uint32_t kRecountThreads = 1024;   // one warp per block, 32 blocks = one superblock

struct JobDev {
    uint32_t cur_buf;    // list being walked: 0 the permutation, 1/2 deferral lists
    uint32_t nxt_buf;    // list receiving this lap's deferred misses
    uint32_t cursor;     // position in the current list
    uint32_t cur_len;
    uint32_t nxt_len;
    uint32_t wrap_slot;  // this round: first slot taken after a lap wrap (0 = no wrap)
    uint32_t m;          // this round: misses
    uint32_t k[3];       // this round: substitutes from A, D, E
    uint32_t done;       // select CTAs finished (last one finishes the job)
    uint32_t pad[5];
};
static_assert(sizeof(JobDev) == 64, "JobDev layout");

struct Cfg {
    uint32_t N, NW, NB, NS, NBp;  // samples, words/bitmap, blocks, superblocks, padded blocks
    uint32_t J, Bmax, maxT;
    uint32_t cap_a;
    uint32_t pad;
    uint64_t seed;
};

struct Lay {
    uint32_t *bm_e, *bm_d, *bm_a;   // [NW]
    uint32_t *seen, *cons;          // [J][NW]
    uint32_t *evmark;               // [NW]
    uint32_t *cnt_blk;              // [3J+1][NBp]
    uint32_t *cnt_sup;              // [3J+1][NS]
    uint32_t *cnt_tot;              // [3J+1]
    uint32_t *a_size;               // [1]
    uint32_t *lists;                // [J][3][N]
    JobDev *jobs;                   // [J]
    uint32_t *req;                  // [J][Bmax]
    uint32_t *miss;                 // [J][Bmax]
    uint32_t *out_ids;              // [J][Bmax] (replay scratch)
    uint8_t *out_src;               // [J][Bmax]
    uint32_t *evict_list;           // [max(cap_a,1)]
    uint32_t *fill_list;            // [max(cap_a,1)]
    seneca_job_epoch_stats *stats;  // [J][maxT]
    unsigned long long *evicted, *refilled;
    uint32_t *err;
    uint32_t *claim;                // [NW] scratch for request validation
};

struct RoundParams {
    uint64_t r;
    uint32_t nj;
    uint32_t active_after;   // active mask after this round's departures
    uint32_t full_scan;      // the active set changed: every A entry is a candidate (R-O6)
    uint32_t out_stride;     // row stride of out_ids / out_src / requested
    uint32_t job[kMaxJobs];
    uint32_t need[kMaxJobs];
    uint32_t nbase[kMaxJobs];
    uint32_t epoch[kMaxJobs];
    uint32_t* out_ids;
    uint8_t* out_src;
    const uint32_t* requested;   // mode 1: [nj][out_stride]
    unsigned long long* transcript;
};

__device__ __forceinline__ uint32_t pidx_of(uint32_t j, uint32_t t) {
    return j * 3u + (t == T_A ? 0u : (t == T_D ? 1u : 2u));
}

__device__ __forceinline__ uint32_t valid_mask(const Cfg& C, uint32_t w) {
    const uint64_t lo = (uint64_t)w * 32u;
    if (lo + 32u <= C.N) return 0xffffffffu;
    if (lo >= C.N) return 0u;
    return (1u << (C.N - lo)) - 1u;
}

// word w of pool (t, j)
__device__ __forceinline__ uint32_t pool_word(const Lay& L, const Cfg& C, uint32_t t, uint32_t j, uint32_t w) {
    if (t == T_S) return ~(L.bm_e[w] | L.bm_d[w] | L.bm_a[w]) & valid_mask(C, w);
    const uint32_t s = L.seen[(size_t)j * C.NW + w];
    if (t == T_A) return L.bm_a[w] & ~s & ~L.cons[(size_t)j * C.NW + w];
    if (t == T_D) return L.bm_d[w] & ~s;
    return L.bm_e[w] & ~s;
}

__device__ __forceinline__ void count_add(const Lay& L, const Cfg& C, uint32_t pidx, uint32_t id, int delta) {
    atomicAdd(L.cnt_blk + (size_t)pidx * C.NBp + (id >> 10), (uint32_t)delta);
    atomicAdd(L.cnt_sup + (size_t)pidx * C.NS + (id >> 15), (uint32_t)delta);
}

// Exclusive prefix of the superblock counts of pool pidx into shared memory.
__device__ void load_sup_prefix(const Lay& L, const Cfg& C, uint32_t pidx, uint32_t* s_pre, uint32_t* scratch) {
    const uint32_t per = (C.NS + blockDim.x - 1) / blockDim.x;
    const uint32_t lo = threadIdx.x * per;
    const uint32_t* src = L.cnt_sup + (size_t)pidx * C.NS;
    uint32_t sum = 0;
    for (uint32_t k = 0; k < per && lo + k < C.NS; ++k) sum += src[lo + k];
    uint32_t run = block_exclusive_scan(sum, nullptr, scratch);
    for (uint32_t k = 0; k < per && lo + k < C.NS; ++k) {
        const uint32_t v = src[lo + k];
        s_pre[lo + k] = run;
        run += v;
    }
    __syncthreads();
}

// The rank-th (0-based) member, in ascending id order, of pool (t, j).
__device__ uint32_t pool_select(const Lay& L, const Cfg& C, uint32_t pidx, uint32_t t, uint32_t j,
                                const uint32_t* s_pre, uint32_t rank) {
    uint32_t lo = 0, hi = C.NS - 1;
    while (lo < hi) {                                   // last superblock with prefix <= rank
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (s_pre[mid] <= rank) lo = mid; else hi = mid - 1;
    }
    uint32_t r = rank - s_pre[lo];
    const uint4* cb = reinterpret_cast<const uint4*>(L.cnt_blk + (size_t)pidx * C.NBp + (size_t)lo * 32u);
    uint32_t blk = lo * 32u;
    bool found = false;
#pragma unroll 1
    for (int q = 0; q < 8 && !found; ++q) {
        const uint4 v = cb[q];
        const uint32_t c[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (!found) {
                if (r < c[k]) { found = true; blk = lo * 32u + q * 4 + k; }
                else r -= c[k];
            }
        }
    }
    const uint32_t w0 = blk * 32u;
#pragma unroll 1
    for (uint32_t k = 0; k < 32; ++k) {
        uint32_t pw = pool_word(L, C, t, j, w0 + k);
        const uint32_t pc = __popc(pw);
        if (r < pc) {
            for (uint32_t s = 0; s < r; ++s) pw &= pw - 1u;
            return (w0 + k) * 32u + (uint32_t)(__ffs(pw) - 1);
        }
        r -= pc;
    }
    atomicOr(L.err, 1u);   // counts inconsistent with bitmaps
    return 0;
}

// ---------------------------------------------------------------------------
// a1-a3: request + classify.  One CTA per job of the round.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kReqThreads)
ods_request_classify(Lay L, Cfg C, RoundParams P, uint32_t mode) {
    extern __shared__ uint32_t smem[];
    uint32_t* s_req = smem;                         // [Bmax]
    __shared__ uint32_t s_scan[33];
    __shared__ uint32_t s_state[6];                 // cur_buf, nxt_buf, cursor, cur_len, nxt_len, wrap
    __shared__ uint32_t s_newcursor;
    __shared__ uint32_t s_hits[3];
    __shared__ uint32_t s_tot[3];

    const uint32_t x = blockIdx.x;
    const uint32_t j = P.job[x];
    const uint32_t need = P.need[x];
    const uint32_t tid = threadIdx.x, T = blockDim.x;
    uint32_t* seen_j = L.seen + (size_t)j * C.NW;
    uint32_t* cons_j = L.cons + (size_t)j * C.NW;

    if (tid == 0) {
        const JobDev& jd = L.jobs[j];
        s_state[0] = jd.cur_buf; s_state[1] = jd.nxt_buf; s_state[2] = jd.cursor;
        s_state[3] = jd.cur_len; s_state[4] = jd.nxt_len; s_state[5] = 0;
        s_hits[0] = s_hits[1] = s_hits[2] = 0;
        for (int k = 0; k < 3; ++k) s_tot[k] = L.cnt_tot[j * 3 + k];
    }
    __syncthreads();

    if (mode == 1) {
        for (uint32_t s = tid; s < need; s += T) s_req[s] = P.requested[(size_t)x * P.out_stride + s];
        __syncthreads();
    } else {
        // a1/a2: first `need` unseen ids of the lap list from the cursor (R-O1)
        uint32_t taken = 0;
        bool wrapped = false;
        while (taken < need) {
            if (s_state[2] >= s_state[3]) {         // lap ends: continue with the deferred list
                __syncthreads();
                if (wrapped || s_state[4] == 0) {
                    if (tid == 0) atomicOr(L.err, 2u);
                    break;
                }
                if (tid == 0) {
                    s_state[5] = taken;
                    s_state[0] = s_state[1];
                    s_state[3] = s_state[4];
                    s_state[2] = 0;
                    s_state[1] = s_state[0] == 1 ? 2 : 1;
                    s_state[4] = 0;
                }
                wrapped = true;
                __syncthreads();
            }
            const uint32_t cursor = s_state[2], len = s_state[3];
            const uint32_t* list = L.lists + ((size_t)j * 3 + s_state[0]) * C.N;
            uint32_t ids[4];
            uint32_t flags = 0, cnt = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t e = cursor + tid * 4 + k;
                ids[k] = 0;
                if (e < len) {
                    const uint32_t id = list[e];
                    ids[k] = id;
                    if (!((seen_j[id >> 5] >> (id & 31)) & 1u)) { flags |= 1u << k; ++cnt; }
                }
            }
            uint32_t tot;
            const uint32_t ex = block_exclusive_scan(cnt, &tot, s_scan);
            const uint32_t remaining = need - taken;
            uint32_t r = ex;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (flags & (1u << k)) {
                    if (r < remaining) s_req[taken + r] = ids[k];
                    if (r == remaining - 1) s_newcursor = cursor + tid * 4 + k + 1;
                    ++r;
                }
            }
            __syncthreads();
            if (tot >= remaining) {
                if (tid == 0) s_state[2] = s_newcursor;
                taken = need;
            } else {
                if (tid == 0) s_state[2] = min(cursor + 4 * T, len);
                taken += tot;
            }
            __syncthreads();
        }
    }

    // a3: classify.  Hits (E, D, or A not consumed by j, R-O13) join seen_j now.
    uint32_t* miss_j = L.miss + (size_t)j * C.Bmax;
    uint32_t mbase = 0;
    for (uint32_t base = 0; base < need; base += T) {
        const uint32_t s = base + tid;
        bool is_miss = false;
        if (s < need) {
            const uint32_t i = s_req[s];
            const uint32_t w = i >> 5, b = 1u << (i & 31);
            const uint32_t t = (L.bm_a[w] & b) ? T_A : (L.bm_d[w] & b) ? T_D : (L.bm_e[w] & b) ? T_E : T_S;
            const bool hit = (t == T_E || t == T_D || (t == T_A && !(cons_j[w] & b)));
            if (hit) {
                P.out_ids[(size_t)x * P.out_stride + s] = i;
                P.out_src[(size_t)x * P.out_stride + s] = (uint8_t)t;
                atomicOr(seen_j + w, b);
                if (t == T_A) atomicOr(cons_j + w, b);
                count_add(L, C, pidx_of(j, t), i, -1);
                atomicAdd(&s_hits[t == T_A ? 0 : (t == T_D ? 1 : 2)], 1u);
            } else {
                is_miss = true;
            }
        }
        uint32_t tot;
        const uint32_t ex = block_exclusive_scan(is_miss ? 1u : 0u, &tot, s_scan);
        if (is_miss) miss_j[mbase + ex] = s;
        mbase += tot;
    }
    if (mode == 1) {  // keep request ids for the storage / deferral phase
        for (uint32_t s = tid; s < need; s += T) L.req[(size_t)j * C.Bmax + s] = s_req[s];
    } else {
        for (uint32_t s = tid; s < need; s += T) L.req[(size_t)j * C.Bmax + s] = s_req[s];
    }
    __syncthreads();
    if (tid == 0) {
        // pool totals after the hits; substitutes per tier A -> D -> E (R-O2)
        uint32_t pa = s_tot[0] - s_hits[0], pd = s_tot[1] - s_hits[1], pe = s_tot[2] - s_hits[2];
        L.cnt_tot[j * 3 + 0] = pa; L.cnt_tot[j * 3 + 1] = pd; L.cnt_tot[j * 3 + 2] = pe;
        const uint32_t m = mbase;
        const uint32_t ka = min(m, pa), kd = min(m - ka, pd), ke = min(m - ka - kd, pe);
        JobDev& jd = L.jobs[j];
        jd.cur_buf = s_state[0]; jd.nxt_buf = s_state[1]; jd.cursor = s_state[2];
        jd.cur_len = s_state[3]; jd.nxt_len = s_state[4]; jd.wrap_slot = s_state[5];
        jd.m = m; jd.k[0] = ka; jd.k[1] = kd; jd.k[2] = ke;
    }
}

// ---------------------------------------------------------------------------
// a4-a6: substitution by keyed rank + apply; the last CTA of a job finishes it.
// ---------------------------------------------------------------------------
__device__ void finish_job(const Lay& L, const Cfg& C, const RoundParams& P, uint32_t x, uint32_t* s_scan,
                           unsigned long long* s_red) {
    const uint32_t j = P.job[x], need = P.need[x], tid = threadIdx.x, T = blockDim.x;
    const JobDev jd = L.jobs[j];
    const uint32_t q = jd.k[0] + jd.k[1] + jd.k[2];
    const uint32_t m = jd.m;
    const uint32_t* miss_j = L.miss + (size_t)j * C.Bmax;
    const uint32_t* req_j = L.req + (size_t)j * C.Bmax;
    uint32_t* seen_j = L.seen + (size_t)j * C.NW;
    const size_t row = (size_t)x * P.out_stride;

    // remaining misses are fetched from storage (R-O18)
    for (uint32_t u = q + tid; u < m; u += T) {
        const uint32_t s = miss_j[u], i = req_j[s];
        P.out_ids[row + s] = i;
        P.out_src[row + s] = (uint8_t)T_S;
        atomicOr(seen_j + (i >> 5), 1u << (i & 31));
    }
    // deferred (replaced) misses are requested again on the next lap (R-O1):
    // slots before the wrap belong to the lap that just ended -> end of the
    // (new) current list; the rest -> the next list.  Slot order = list order.
    uint32_t q1 = 0;
    if (jd.wrap_slot > 0) {
        uint32_t c = 0;
        for (uint32_t u = tid; u < q; u += T) c += miss_j[u] < jd.wrap_slot;
        block_exclusive_scan(c, &q1, s_scan);
    }
    uint32_t* cur_list = L.lists + ((size_t)j * 3 + jd.cur_buf) * C.N;
    uint32_t* nxt_list = L.lists + ((size_t)j * 3 + jd.nxt_buf) * C.N;
    for (uint32_t u = tid; u < q; u += T) {
        const uint32_t id = req_j[miss_j[u]];
        if (u < q1) cur_list[jd.cur_len + u] = id;
        else nxt_list[jd.nxt_len + (u - q1)] = id;
    }
    __syncthreads();

    // counters, digest, transcript (a6)
    unsigned long long acc[13];
#pragma unroll
    for (int k = 0; k < 13; ++k) acc[k] = 0;
    const uint32_t e = P.epoch[x], nbase = P.nbase[x];
    unsigned long long* trow = P.transcript ? P.transcript + ((size_t)j * C.maxT + e) * C.N : nullptr;
    for (uint32_t s = tid; s < need; s += T) {
        const uint32_t i = P.out_ids[row + s];
        const uint32_t src = P.out_src[row + s];
        const uint32_t t = src & 3u;
        acc[t] += 1;
        if (src & SUBST) acc[4 + t] += 1;
        else if (t != T_S) acc[8 + t] += 1;
        const uint64_t word = ((uint64_t)(nbase + s) << 35) | ((uint64_t)src << 32) | i;
        acc[12] += splitmix64(word);
        if (trow) trow[nbase + s] = ((unsigned long long)src << 32) | i;
    }
#pragma unroll
    for (int k = 0; k < 13; ++k) {
        unsigned long long v = warp_sum(acc[k]);
        if ((tid & 31) == 0) s_red[(tid >> 5) * 13 + k] = v;
    }
    __syncthreads();
    if (tid < 13) {
        unsigned long long v = 0;
        for (uint32_t w = 0; w < T / 32; ++w) v += s_red[w * 13 + tid];
        unsigned long long* st = reinterpret_cast<unsigned long long*>(L.stats + (size_t)j * C.maxT + e);
        st[tid] += v;
    }
    if (tid == 0) {
        JobDev& w = L.jobs[j];
        w.cur_len = jd.cur_len + q1;
        w.nxt_len = jd.nxt_len + (q - q1);
        w.done = 0;
    }
}

__global__ void __launch_bounds__(kSelThreads)
ods_select_apply(Lay L, Cfg C, RoundParams P) {
    extern __shared__ uint32_t smem[];
    uint32_t* s_pre = smem;                  // [NS]
    uint32_t* s_sub = smem + C.NS;           // [Bmax]
    __shared__ uint32_t s_scan[33];
    __shared__ unsigned long long s_red[(kSelThreads / 32) * 13];
    __shared__ int s_last;

    const uint32_t x = blockIdx.x / 3, tt = blockIdx.x % 3;
    const uint32_t t = tt == 0 ? T_A : (tt == 1 ? T_D : T_E);
    const uint32_t j = P.job[x];
    const uint32_t tid = threadIdx.x, T = blockDim.x;
    const JobDev jd = L.jobs[j];
    const uint32_t k = jd.k[tt];
    const uint32_t qoff = tt == 0 ? 0u : (tt == 1 ? jd.k[0] : jd.k[0] + jd.k[1]);

    if (k > 0) {
        const uint32_t pidx = j * 3 + tt;
        const uint32_t P_t = L.cnt_tot[pidx];
        load_sup_prefix(L, C, pidx, s_pre, s_scan);
        const uint64_t key = derive_key(C.seed, PUR_SUB, j, P.r, t);
        const PermDomain dom = perm_domain(P_t);
        const uint32_t* miss_j = L.miss + (size_t)j * C.Bmax;
        const size_t row = (size_t)x * P.out_stride;
        for (uint32_t u = tid; u < k; u += T) {
            const uint32_t rank = perm_apply(key, dom, u);
            const uint32_t id = pool_select(L, C, pidx, t, j, s_pre, rank);
            const uint32_t s = miss_j[qoff + u];
            P.out_ids[row + s] = id;
            P.out_src[row + s] = (uint8_t)(t | SUBST);
            s_sub[u] = id;
        }
        __syncthreads();
        uint32_t* seen_j = L.seen + (size_t)j * C.NW;
        uint32_t* cons_j = L.cons + (size_t)j * C.NW;
        for (uint32_t u = tid; u < k; u += T) {
            const uint32_t id = s_sub[u];
            const uint32_t w = id >> 5, b = 1u << (id & 31);
            atomicOr(seen_j + w, b);
            if (t == T_A) atomicOr(cons_j + w, b);
            count_add(L, C, pidx, id, -1);
        }
        if (tid == 0) L.cnt_tot[pidx] = P_t - k;
    }
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        const uint32_t old = atomicAdd(&L.jobs[j].done, 1u);
        s_last = (old == 2);
        if (s_last) __threadfence();
    }
    __syncthreads();
    if (s_last) finish_job(L, C, P, x, s_scan, s_red);
}

// ---------------------------------------------------------------------------
// a7: maintain -- eviction of A entries consumed by every active job (R-O5,
// R-O6) and keyed refill from the storage pool as of round start (R-O8).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kMaintThreads)
ods_maintain(Lay L, Cfg C, RoundParams P) {
    extern __shared__ uint32_t smem[];
    uint32_t* s_pre = smem;                        // [NS]
    __shared__ uint32_t s_scan[33];
    __shared__ uint32_t s_ne;
    __shared__ uint32_t s_add[kMaxJobs];
    const uint32_t tid = threadIdx.x, T = blockDim.x;
    const uint32_t active = P.active_after;
    if (active == 0) return;                       // replay over: no maintain work (R-O7)
    if (tid == 0) s_ne = 0;
    if (tid < kMaxJobs) s_add[tid] = 0;
    __syncthreads();

    auto consumed_by_all = [&](uint32_t w, uint32_t b) -> bool {
        for (uint32_t m = active; m; m &= m - 1) {
            const uint32_t a = __ffs(m) - 1;
            if (!(L.cons[(size_t)a * C.NW + w] & b)) return false;
        }
        return true;
    };

    if (P.full_scan) {
        // the active set changed: every A entry is a candidate
        for (uint32_t w = tid; w < C.NW; w += T) {
            uint32_t ev = L.bm_a[w];
            for (uint32_t m = active; m && ev; m &= m - 1) ev &= L.cons[(size_t)(__ffs(m) - 1) * C.NW + w];
            if (ev) {
                const uint32_t base = atomicAdd(&s_ne, (uint32_t)__popc(ev));
                uint32_t c = 0;
                for (uint32_t v = ev; v; v &= v - 1) L.evict_list[base + c++] = w * 32u + (__ffs(v) - 1);
            }
        }
    } else {
        // candidates: the A-served ids of this round (deduplicated by claiming)
        uint32_t total = 0;
        for (uint32_t x = 0; x < P.nj; ++x) total += P.need[x];
        for (uint32_t f = tid; f < total; f += T) {
            uint32_t x = 0, s = f;
            while (s >= P.need[x]) { s -= P.need[x]; ++x; }
            const size_t at = (size_t)x * P.out_stride + s;
            if ((P.out_src[at] & 3u) != T_A) continue;
            const uint32_t i = P.out_ids[at];
            const uint32_t w = i >> 5, b = 1u << (i & 31);
            if (!(L.bm_a[w] & b) || !consumed_by_all(w, b)) continue;
            if (atomicOr(L.evmark + w, b) & b) continue;      // already claimed
            L.evict_list[atomicAdd(&s_ne, 1u)] = i;
        }
    }
    __syncthreads();
    const uint32_t ne = s_ne;
    const uint32_t size_a = *L.a_size;
    const uint32_t deficit = C.cap_a - (size_a - ne);
    const uint32_t PS = L.cnt_tot[3 * C.J];
    const uint32_t k = min(deficit, PS);
    const uint32_t spidx = 3 * C.J;
    if (k > 0) {
        load_sup_prefix(L, C, spidx, s_pre, s_scan);
        const uint64_t key = derive_key(C.seed, PUR_REFILL, 0, P.r, 0);
        const PermDomain dom = perm_domain(PS);
        for (uint32_t u = tid; u < k; u += T)
            L.fill_list[u] = pool_select(L, C, spidx, T_S, 0, s_pre, perm_apply(key, dom, u));
    }
    __syncthreads();
    // apply evictions: A -> S, consumers cleared; the storage pool gains them
    for (uint32_t u = tid; u < ne; u += T) {
        const uint32_t i = L.evict_list[u];
        const uint32_t w = i >> 5, b = 1u << (i & 31);
        atomicAnd(L.bm_a + w, ~b);
        if (!P.full_scan) atomicAnd(L.evmark + w, ~b);
        for (uint32_t a = 0; a < C.J; ++a) atomicAnd(L.cons + (size_t)a * C.NW + w, ~b);
        count_add(L, C, spidx, i, +1);
    }
    // apply refills: S -> A with empty consumers; every active job that has not
    // seen the id gains it in its A pool
    for (uint32_t u = tid; u < k; u += T) {
        const uint32_t i = L.fill_list[u];
        const uint32_t w = i >> 5, b = 1u << (i & 31);
        atomicOr(L.bm_a + w, b);
        count_add(L, C, spidx, i, -1);
        for (uint32_t m = active; m; m &= m - 1) {
            const uint32_t a = __ffs(m) - 1;
            if (!(L.seen[(size_t)a * C.NW + w] & b)) {
                count_add(L, C, a * 3 + 0, i, +1);
                atomicAdd(&s_add[a], 1u);
            }
        }
    }
    __syncthreads();
    if (tid < C.J && s_add[tid]) L.cnt_tot[tid * 3 + 0] += s_add[tid];
    if (tid == 0) {
        L.cnt_tot[spidx] = PS + ne - k;
        *L.a_size = size_a - ne + k;
        *L.evicted += ne;
        *L.refilled += k;
    }
}

// ---------------------------------------------------------------------------
// pool recount: one CTA per superblock; one warp per 1024-id block.
// blockIdx.y selects a job of jobs_mask (in order); y == popc(mask) -> storage pool.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kRecountThreads)
ods_recount(Lay L, Cfg C, uint32_t jobs_mask, uint32_t with_storage) {
    __shared__ uint32_t s_c[32][3];
    const uint32_t sblk = blockIdx.x;
    const uint32_t nmask = __popc(jobs_mask);
    const uint32_t y = blockIdx.y;
    const bool storage = y >= nmask;
    if (storage && !with_storage) return;
    uint32_t j = 0;
    if (!storage) {
        uint32_t m = jobs_mask;
        for (uint32_t k = 0; k < y; ++k) m &= m - 1;
        j = __ffs(m) - 1;
    }
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t blk = sblk * 32 + warp;
    const uint32_t w = blk * 32 + lane;
    uint32_t ca = 0, cd = 0, ce = 0;
    if (blk < C.NB) {
        if (storage) {
            ca = __popc(~(L.bm_e[w] | L.bm_d[w] | L.bm_a[w]) & valid_mask(C, w));
        } else {
            const uint32_t s = L.seen[(size_t)j * C.NW + w];
            ca = __popc(L.bm_a[w] & ~s & ~L.cons[(size_t)j * C.NW + w]);
            cd = __popc(L.bm_d[w] & ~s);
            ce = __popc(L.bm_e[w] & ~s);
        }
    }
    ca = warp_sum(ca); cd = warp_sum(cd); ce = warp_sum(ce);
    if (lane == 0) {
        s_c[warp][0] = ca; s_c[warp][1] = cd; s_c[warp][2] = ce;
        if (storage) L.cnt_blk[(size_t)(3 * C.J) * C.NBp + blk] = ca;
        else {
            L.cnt_blk[(size_t)(j * 3 + 0) * C.NBp + blk] = ca;
            L.cnt_blk[(size_t)(j * 3 + 1) * C.NBp + blk] = cd;
            L.cnt_blk[(size_t)(j * 3 + 2) * C.NBp + blk] = ce;
        }
    }
    __syncthreads();
    if (warp == 0) {
        uint32_t a = s_c[lane][0], d = s_c[lane][1], e = s_c[lane][2];
        a = warp_sum(a); d = warp_sum(d); e = warp_sum(e);
        if (lane == 0) {
            if (storage) {
                L.cnt_sup[(size_t)(3 * C.J) * C.NS + sblk] = a;
                atomicAdd(L.cnt_tot + 3 * C.J, a);
            } else {
                L.cnt_sup[(size_t)(j * 3 + 0) * C.NS + sblk] = a;
                L.cnt_sup[(size_t)(j * 3 + 1) * C.NS + sblk] = d;
                L.cnt_sup[(size_t)(j * 3 + 2) * C.NS + sblk] = e;
                atomicAdd(L.cnt_tot + j * 3 + 0, a);
                atomicAdd(L.cnt_tot + j * 3 + 1, d);
                atomicAdd(L.cnt_tot + j * 3 + 2, e);
            }
        }
    }
}

// pi_j for epoch e: list[pos] = perm(key(seed, REQ, j, e), N, pos) (R-O3).
// Also resets the job's lap-list state (block 0, thread 0).
__global__ void ods_perm_fill(Lay L, Cfg C, uint32_t j, uint32_t epoch) {
    const uint64_t key = derive_key(C.seed, PUR_REQ, j, epoch, 0);
    const PermDomain dom = perm_domain(C.N);
    uint32_t* out = L.lists + (size_t)j * 3 * C.N;
    for (uint32_t pos = blockIdx.x * blockDim.x + threadIdx.x; pos < C.N; pos += gridDim.x * blockDim.x)
        out[pos] = perm_apply(key, dom, pos);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        JobDev& jd = L.jobs[j];
        jd.cur_buf = 0; jd.nxt_buf = 1; jd.cursor = 0; jd.cur_len = C.N; jd.nxt_len = 0;
        jd.wrap_slot = 0; jd.m = 0; jd.k[0] = jd.k[1] = jd.k[2] = 0; jd.done = 0;
    }
}

// warm start (R-O9): positions [0,cap_A) -> A, next cap_D -> D, next cap_E -> E
__global__ void ods_init_tiers(Lay L, Cfg C, uint32_t cap_e, uint32_t cap_d) {
    const uint64_t key = derive_key(C.seed, PUR_INIT, 0, 0, 0);
    const PermDomain dom = perm_domain(C.N);
    const uint32_t total = C.cap_a + cap_d + cap_e;
    for (uint32_t pos = blockIdx.x * blockDim.x + threadIdx.x; pos < total; pos += gridDim.x * blockDim.x) {
        const uint32_t i = perm_apply(key, dom, pos);
        uint32_t* bm = pos < C.cap_a ? L.bm_a : (pos < C.cap_a + cap_d ? L.bm_d : L.bm_e);
        atomicOr(bm + (i >> 5), 1u << (i & 31));
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *L.a_size = C.cap_a;
}

// caller-supplied requests (mode 1): range, duplicates within the row, seen
__global__ void ods_validate_requests(Lay L, Cfg C, RoundParams P) {
    extern __shared__ uint32_t s_row[];
    const uint32_t x = blockIdx.x, j = P.job[x], need = P.need[x];
    const uint32_t* R = P.requested + (size_t)x * P.out_stride;
    for (uint32_t s = threadIdx.x; s < need; s += blockDim.x) s_row[s] = R[s];
    __syncthreads();
    for (uint32_t s = threadIdx.x; s < need; s += blockDim.x) {
        const uint32_t i = s_row[s];
        if (i >= C.N) { atomicOr(L.err, 0x100u); continue; }
        if (L.seen[(size_t)j * C.NW + (i >> 5)] & (1u << (i & 31))) atomicOr(L.err, 0x100u);
        for (uint32_t s2 = 0; s2 < s; ++s2)
            if (s_row[s2] == i) { atomicOr(L.err, 0x100u); break; }
    }
}

inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace
}  // namespace seneca

// ===========================================================================
// host side
// ===========================================================================
using namespace seneca;

namespace {
enum KernelClass { K_REQUEST = 0, K_SELECT, K_MAINTAIN, K_RECOUNT, K_PERM, K_INIT, K_VALIDATE, K_NCLASS };
const char* const kKernelNames[K_NCLASS] = {"ods_request_classify", "ods_select_apply", "ods_maintain",
                                            "ods_recount", "ods_perm_fill", "ods_init_tiers",
                                            "ods_validate_requests"};

// Sampled kernel timing: CUDA events around the launches of every k-th round
// (and around every launch of the rare classes), on the launch stream, kept in
// a ring and resolved lazily so the host never waits on recent work.
struct KernelProfiler {
    struct Slot { cudaEvent_t a = nullptr, b = nullptr; int cls = -1; };
    uint32_t every = 0;
    std::vector<Slot> ring;
    size_t head = 0;
    uint64_t launches[K_NCLASS] = {};
    uint64_t sampled[K_NCLASS] = {};
    double ms[K_NCLASS] = {};

    void resolve(Slot& s) {
        if (s.cls < 0) return;
        float t = 0.f;
        cudaEventSynchronize(s.b);
        if (cudaEventElapsedTime(&t, s.a, s.b) == cudaSuccess) { sampled[s.cls]++; ms[s.cls] += t; }
        s.cls = -1;
    }
    Slot* acquire() {
        if (ring.empty()) {
            ring.resize(4096);
            for (auto& s : ring) { cudaEventCreate(&s.a); cudaEventCreate(&s.b); }
        }
        Slot& s = ring[head];
        head = (head + 1) % ring.size();
        resolve(s);
        return &s;
    }
    void flush() { for (auto& s : ring) resolve(s); }
    ~KernelProfiler() { for (auto& s : ring) { if (s.a) cudaEventDestroy(s.a); if (s.b) cudaEventDestroy(s.b); } }
};
}  // namespace

struct seneca_ctx {
    KernelProfiler prof;
    Cfg C;
    Lay L;
    uint32_t mode;
    uint32_t batch[kMaxJobs], target[kMaxJobs];
    uint64_t cap_e, cap_d;
    uint64_t e[kMaxJobs], n[kMaxJobs];
    uint32_t active;
    uint64_t r;
    uint64_t launches;
    size_t sel_smem, req_smem, maint_smem;
};

namespace {

seneca_status check_cfg(const seneca_cache_config* cfg) {
    if (!cfg) { set_error("NULL config"); return SENECA_EINVAL; }
    if (cfg->n_total == 0 || cfg->n_total >= (1ull << 31)) {
        set_error("n_total must be in [1, 2^31)"); return SENECA_EINVAL;
    }
    if (cfg->n_jobs == 0 || cfg->n_jobs > kMaxJobs) { set_error("n_jobs must be in [1, 32]"); return SENECA_EINVAL; }
    if (cfg->request_mode > 1) { set_error("request_mode must be 0 or 1"); return SENECA_EINVAL; }
    if (!cfg->batch_size || !cfg->target_epochs) { set_error("NULL batch_size/target_epochs"); return SENECA_EINVAL; }
    for (uint32_t j = 0; j < cfg->n_jobs; ++j) {
        if (cfg->batch_size[j] == 0 || cfg->batch_size[j] > kMaxBatch) {
            set_error("batch_size[%u] must be in [1, %u]", j, kMaxBatch); return SENECA_EINVAL;
        }
        if (cfg->target_epochs[j] == 0 || cfg->target_epochs[j] > 1000000) {
            set_error("target_epochs[%u] must be in [1, 1e6]", j); return SENECA_EINVAL;
        }
    }
    if (cfg->cap_e > cfg->n_total || cfg->cap_d > cfg->n_total || cfg->cap_a > cfg->n_total ||
        cfg->cap_e + cfg->cap_d + cfg->cap_a > cfg->n_total) {
        set_error("cap_e + cap_d + cap_a exceeds n_total"); return SENECA_EINVAL;
    }
    return SENECA_OK;
}

struct Sizes {
    Cfg C;
    size_t off[32];
    size_t total;
};

Sizes compute_sizes(const seneca_cache_config* cfg) {
    Sizes z{};
    Cfg& C = z.C;
    C.N = (uint32_t)cfg->n_total;
    C.NB = (C.N + 1023) / 1024;
    C.NS = (C.NB + 31) / 32;
    C.NBp = C.NS * 32;
    C.NW = C.NBp * 32;              // bitmaps padded to whole superblocks
    C.J = cfg->n_jobs;
    C.Bmax = 0;
    C.maxT = 0;
    for (uint32_t j = 0; j < C.J; ++j) {
        C.Bmax = std::max(C.Bmax, cfg->batch_size[j]);
        C.maxT = std::max(C.maxT, cfg->target_epochs[j]);
    }
    C.cap_a = (uint32_t)cfg->cap_a;
    C.seed = cfg->seed;
    const size_t W = (size_t)C.NW * 4, P = 3 * (size_t)C.J + 1;
    const size_t capl = std::max<size_t>(cfg->cap_a, 1) * 4;
    const size_t sz[] = {
        W, W, W,                                   // 0-2 bm_e, bm_d, bm_a
        W * C.J, W * C.J,                          // 3-4 seen, cons
        W,                                         // 5 evmark
        P * C.NBp * 4, P * C.NS * 4, P * 4,        // 6-8 counts
        4,                                         // 9 a_size
        (size_t)C.J * 3 * C.N * 4,                 // 10 lists
        (size_t)C.J * sizeof(JobDev),              // 11 jobs
        (size_t)C.J * C.Bmax * 4,                  // 12 req
        (size_t)C.J * C.Bmax * 4,                  // 13 miss
        (size_t)C.J * C.Bmax * 4,                  // 14 out_ids
        (size_t)C.J * C.Bmax,                      // 15 out_src
        capl, capl,                                // 16-17 evict, fill
        (size_t)C.J * C.maxT * sizeof(seneca_job_epoch_stats),  // 18 stats
        8, 8, 4,                                   // 19-21 evicted, refilled, err
        W,                                         // 22 claim
    };
    size_t at = 0;
    for (size_t k = 0; k < sizeof(sz) / sizeof(sz[0]); ++k) {
        z.off[k] = at;
        at += align256(sz[k]);
    }
    z.total = at;
    return z;
}

Lay carve(const Sizes& z, char* base) {
    Lay L;
    L.bm_e = (uint32_t*)(base + z.off[0]);
    L.bm_d = (uint32_t*)(base + z.off[1]);
    L.bm_a = (uint32_t*)(base + z.off[2]);
    L.seen = (uint32_t*)(base + z.off[3]);
    L.cons = (uint32_t*)(base + z.off[4]);
    L.evmark = (uint32_t*)(base + z.off[5]);
    L.cnt_blk = (uint32_t*)(base + z.off[6]);
    L.cnt_sup = (uint32_t*)(base + z.off[7]);
    L.cnt_tot = (uint32_t*)(base + z.off[8]);
    L.a_size = (uint32_t*)(base + z.off[9]);
    L.lists = (uint32_t*)(base + z.off[10]);
    L.jobs = (JobDev*)(base + z.off[11]);
    L.req = (uint32_t*)(base + z.off[12]);
    L.miss = (uint32_t*)(base + z.off[13]);
    L.out_ids = (uint32_t*)(base + z.off[14]);
    L.out_src = (uint8_t*)(base + z.off[15]);
    L.evict_list = (uint32_t*)(base + z.off[16]);
    L.fill_list = (uint32_t*)(base + z.off[17]);
    L.stats = (seneca_job_epoch_stats*)(base + z.off[18]);
    L.evicted = (unsigned long long*)(base + z.off[19]);
    L.refilled = (unsigned long long*)(base + z.off[20]);
    L.err = (uint32_t*)(base + z.off[21]);
    L.claim = (uint32_t*)(base + z.off[22]);
    return L;
}

int g_num_sms = 0;

int num_sms() {
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

template <class F>
void timed_launch(seneca_ctx* c, int cls, bool sample, cudaStream_t st, F&& launch) {
    c->launches++;
    c->prof.launches[cls]++;
    if (!sample || !c->prof.every) { launch(); return; }
    auto* s = c->prof.acquire();
    cudaEventRecord(s->a, st);
    launch();
    cudaEventRecord(s->b, st);
    s->cls = cls;
}

seneca_status launch_recount(seneca_ctx* c, uint32_t jobs_mask, bool storage, cudaStream_t st) {
    const uint32_t ny = __builtin_popcount(jobs_mask) + (storage ? 1 : 0);
    if (!ny) return SENECA_OK;
    // zero the totals being rebuilt
    for (uint32_t m = jobs_mask; m; m &= m - 1) {
        const uint32_t j = __builtin_ctz(m);
        SENECA_CUDA_TRY(cudaMemsetAsync(c->L.cnt_tot + j * 3, 0, 12, st));
    }
    if (storage) SENECA_CUDA_TRY(cudaMemsetAsync(c->L.cnt_tot + 3 * c->C.J, 0, 4, st));
    dim3 grid(c->C.NS, ny);
    timed_launch(c, K_RECOUNT, true, st, [&] {
        ods_recount<<<grid, kRecountThreads, 0, st>>>(c->L, c->C, jobs_mask, storage ? 1u : 0u);
    });
    SENECA_CUDA_TRY(cudaGetLastError());
    return SENECA_OK;
}

seneca_status launch_perm_fill(seneca_ctx* c, uint32_t j, uint32_t epoch, cudaStream_t st) {
    const uint32_t threads = 256;
    uint32_t blocks = (c->C.N + threads - 1) / threads;
    blocks = std::min<uint32_t>(blocks, (uint32_t)num_sms() * 8);
    timed_launch(c, K_PERM, true, st, [&] { ods_perm_fill<<<blocks, threads, 0, st>>>(c->L, c->C, j, epoch); });
    SENECA_CUDA_TRY(cudaGetLastError());
    return SENECA_OK;
}

// One round (R-O11) with the host's data-independent schedule.
seneca_status run_round(seneca_ctx* c, const uint32_t* jobs, uint32_t nj, const uint32_t* d_requested,
                        uint32_t* out_ids, uint8_t* out_src, uint32_t out_stride, unsigned long long* transcript,
                        uint32_t* h_lens, cudaStream_t st) {
    RoundParams P;
    std::memset(&P, 0, sizeof P);
    P.r = c->r;
    P.nj = nj;
    P.out_stride = out_stride;
    P.out_ids = out_ids;
    P.out_src = out_src;
    P.requested = d_requested;
    P.transcript = transcript;
    uint32_t departing = 0, ending = 0;
    for (uint32_t x = 0; x < nj; ++x) {
        const uint32_t j = jobs[x];
        const uint64_t need = std::min<uint64_t>(c->batch[j], (uint64_t)c->C.N - c->n[j]);
        P.job[x] = j;
        P.need[x] = (uint32_t)need;
        P.nbase[x] = (uint32_t)c->n[j];
        P.epoch[x] = (uint32_t)c->e[j];
        if (c->n[j] + need == c->C.N) {
            ending |= 1u << j;
            if (c->e[j] + 1 == c->target[j]) departing |= 1u << j;
        }
        if (h_lens) h_lens[x] = (uint32_t)need;
    }
    P.active_after = c->active & ~departing;
    P.full_scan = departing ? 1u : 0u;

    if (c->mode == 1) {
        timed_launch(c, K_VALIDATE, false, st, [&] {
            ods_validate_requests<<<nj, 256, (size_t)c->C.Bmax * 4, st>>>(c->L, c->C, P);
        });
        SENECA_CUDA_TRY(cudaGetLastError());
        uint32_t err = 0;
        SENECA_CUDA_TRY(cudaMemcpyAsync(&err, c->L.err, 4, cudaMemcpyDeviceToHost, st));
        SENECA_CUDA_TRY(cudaStreamSynchronize(st));
        if (err & 0x100u) {
            SENECA_CUDA_TRY(cudaMemsetAsync(c->L.err, 0, 4, st));
            set_error("supplied request ids out of range, duplicated or already seen");
            return SENECA_EPROTO;
        }
    }
    const bool sample = c->prof.every && (c->r % c->prof.every) == 0;
    timed_launch(c, K_REQUEST, sample, st, [&] {
        ods_request_classify<<<nj, kReqThreads, c->req_smem, st>>>(c->L, c->C, P, c->mode);
    });
    timed_launch(c, K_SELECT, sample, st, [&] {
        ods_select_apply<<<nj * 3, kSelThreads, c->sel_smem, st>>>(c->L, c->C, P);
    });
    timed_launch(c, K_MAINTAIN, sample, st, [&] {
        ods_maintain<<<1, kMaintThreads, c->maint_smem, st>>>(c->L, c->C, P);
    });
    SENECA_CUDA_TRY(cudaGetLastError());
    // epoch ends (a8, R-O16): reset seen, rebuild the job's pool counts, next permutation
    if (ending) {
        uint32_t recount = 0;
        for (uint32_t m = ending; m; m &= m - 1) {
            const uint32_t j = __builtin_ctz(m);
            SENECA_CUDA_TRY(cudaMemsetAsync(c->L.seen + (size_t)j * c->C.NW, 0, (size_t)c->C.NW * 4, st));
            if (!(departing & (1u << j))) {
                recount |= 1u << j;
                if (c->mode == 0) {
                    seneca_status s = launch_perm_fill(c, j, (uint32_t)(c->e[j] + 1), st);
                    if (s) return s;
                }
            }
        }
        seneca_status s = launch_recount(c, recount, false, st);
        if (s) return s;
    }
    // host mirror of the schedule
    for (uint32_t x = 0; x < nj; ++x) {
        const uint32_t j = jobs[x];
        c->n[j] += P.need[x];
        if (c->n[j] == c->C.N) {
            c->n[j] = 0;
            c->e[j] += 1;
        }
    }
    c->active &= ~departing;
    c->r += 1;
    return SENECA_OK;
}

}  // namespace

extern "C" seneca_status seneca_state_bytes(const seneca_cache_config* cfg, size_t* bytes) {
    seneca_status s = check_cfg(cfg);
    if (s) return s;
    if (!bytes) { set_error("NULL bytes"); return SENECA_EINVAL; }
    *bytes = compute_sizes(cfg).total;
    return SENECA_OK;
}

extern "C" seneca_status seneca_init_cache(const seneca_cache_config* cfg, void* d_workspace, size_t ws_bytes,
                                           void* stream, seneca_ctx** out) {
    seneca_status s = check_cfg(cfg);
    if (s) return s;
    if (!out || !d_workspace) { set_error("NULL workspace or out"); return SENECA_EINVAL; }
    if ((uintptr_t)d_workspace & 255) { set_error("workspace must be 256-byte aligned"); return SENECA_EINVAL; }
    Sizes z = compute_sizes(cfg);
    if (ws_bytes < z.total) {
        set_error("workspace %zu bytes < required %zu", ws_bytes, z.total);
        return SENECA_ENOSPC;
    }
    if ((size_t)z.C.NS * 4 + (size_t)z.C.Bmax * 4 > 200 * 1024) {
        set_error("dataset too large for the shared-memory superblock index");
        return SENECA_EINVAL;
    }
    seneca_ctx* c = new (std::nothrow) seneca_ctx();
    if (!c) { set_error("out of host memory"); return SENECA_EINVAL; }
    c->C = z.C;
    c->L = carve(z, (char*)d_workspace);
    c->mode = cfg->request_mode;
    for (uint32_t j = 0; j < cfg->n_jobs; ++j) {
        c->batch[j] = cfg->batch_size[j];
        c->target[j] = cfg->target_epochs[j];
    }
    c->cap_e = cfg->cap_e;
    c->cap_d = cfg->cap_d;
    c->active = cfg->n_jobs == 32 ? 0xffffffffu : ((1u << cfg->n_jobs) - 1);
    c->req_smem = (size_t)c->C.Bmax * 4;
    c->sel_smem = (size_t)c->C.NS * 4 + (size_t)c->C.Bmax * 4;
    c->maint_smem = (size_t)c->C.NS * 4;
    cudaStream_t st = (cudaStream_t)stream;
#define INIT_TRY(expr) do { cudaError_t _e = (expr); if (_e != cudaSuccess) { delete c; return cuda_status(_e, #expr); } } while (0)
    INIT_TRY(cudaFuncSetAttribute(ods_request_classify, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    INIT_TRY(cudaFuncSetAttribute(ods_select_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    INIT_TRY(cudaFuncSetAttribute(ods_maintain, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    INIT_TRY(cudaMemsetAsync(d_workspace, 0, z.total, st));
    {
        const uint32_t total = (uint32_t)(cfg->cap_a + cfg->cap_d + cfg->cap_e);
        uint32_t blocks = std::max<uint32_t>(1, std::min<uint32_t>((total + 255) / 256, num_sms() * 8));
        timed_launch(c, K_INIT, false, st, [&] {
            ods_init_tiers<<<blocks, 256, 0, st>>>(c->L, c->C, (uint32_t)cfg->cap_e, (uint32_t)cfg->cap_d);
        });
        INIT_TRY(cudaGetLastError());
    }
    s = launch_recount(c, c->active, true, st);
    if (s) { delete c; return s; }
    for (uint32_t j = 0; j < cfg->n_jobs; ++j) {
        if (c->mode == 0) {
            s = launch_perm_fill(c, j, 0, st);
            if (s) { delete c; return s; }
        }
    }
#undef INIT_TRY
    *out = c;
    return SENECA_OK;
}

extern "C" seneca_status seneca_ods_next_batch(seneca_ctx* c, const uint32_t* h_jobs, uint32_t n_jobs,
                                               const uint32_t* d_requested, uint32_t* d_out_ids,
                                               uint8_t* d_out_src, uint32_t* h_out_lens, void* stream) {
    if (!c || !h_jobs || n_jobs == 0 || n_jobs > c->C.J || !d_out_ids || !d_out_src) {
        set_error("seneca_ods_next_batch: bad arguments"); return SENECA_EINVAL;
    }
    if ((c->mode == 1) != (d_requested != nullptr)) {
        set_error("d_requested must be given exactly when request_mode = 1"); return SENECA_EINVAL;
    }
    uint32_t seenmask = 0;
    for (uint32_t x = 0; x < n_jobs; ++x) {
        const uint32_t j = h_jobs[x];
        if (j >= c->C.J || (seenmask & (1u << j))) { set_error("bad or duplicate job %u", j); return SENECA_EINVAL; }
        seenmask |= 1u << j;
        if (!(c->active & (1u << j))) { set_error("job %u has departed", j); return SENECA_ESTATE; }
    }
    return run_round(c, h_jobs, n_jobs, d_requested, d_out_ids, d_out_src, c->C.Bmax, nullptr, h_out_lens,
                     (cudaStream_t)stream);
}

static seneca_status replay(seneca_ctx* c, uint64_t max_rounds, uint32_t n_epochs, bool by_epochs,
                            uint64_t* d_transcript, uint64_t* h_rounds, cudaStream_t st) {
    if (c->mode != 0) { set_error("replay requires request_mode 0"); return SENECA_ESTATE; }
    if (!c->active) { set_error("no active job"); return SENECA_ESTATE; }
    uint64_t goal[kMaxJobs];
    const uint32_t tracked = c->active;
    for (uint32_t j = 0; j < c->C.J; ++j) goal[j] = c->e[j] + n_epochs;
    uint64_t done = 0;
    uint32_t jobs[kMaxJobs];
    for (;;) {
        if (!by_epochs && done >= max_rounds) break;
        if (by_epochs) {
            bool pending = false;
            for (uint32_t m = tracked & c->active; m; m &= m - 1) {
                const uint32_t j = __builtin_ctz(m);
                if (c->e[j] < goal[j]) pending = true;
            }
            if (!pending) break;
        }
        if (!c->active) break;
        uint32_t nj = 0;
        for (uint32_t m = c->active; m; m &= m - 1) jobs[nj++] = __builtin_ctz(m);
        seneca_status s = run_round(c, jobs, nj, nullptr, c->L.out_ids, c->L.out_src, c->C.Bmax,
                                    (unsigned long long*)d_transcript, nullptr, st);
        if (s) return s;
        ++done;
    }
    if (h_rounds) *h_rounds = done;
    return SENECA_OK;
}

extern "C" seneca_status seneca_replay_epochs(seneca_ctx* c, uint32_t n_epochs, uint64_t* d_transcript,
                                              uint64_t* h_rounds, void* stream) {
    if (!c || n_epochs == 0) { set_error("bad arguments"); return SENECA_EINVAL; }
    return replay(c, 0, n_epochs, true, d_transcript, h_rounds, (cudaStream_t)stream);
}

extern "C" seneca_status seneca_replay_rounds(seneca_ctx* c, uint64_t n_rounds, uint64_t* d_transcript,
                                              uint64_t* h_rounds, void* stream) {
    if (!c) { set_error("bad arguments"); return SENECA_EINVAL; }
    return replay(c, n_rounds, 0, false, d_transcript, h_rounds, (cudaStream_t)stream);
}

extern "C" seneca_status seneca_read_state(const seneca_ctx* c, seneca_state_view* v) {
    if (!c || !v) { set_error("bad arguments"); return SENECA_EINVAL; }
    std::memset(v, 0, sizeof *v);
    v->n_total = c->C.N;
    v->n_jobs = c->C.J;
    v->max_target = c->C.maxT;
    v->words = c->C.NW;
    v->d_tier_e = c->L.bm_e;
    v->d_tier_d = c->L.bm_d;
    v->d_tier_a = c->L.bm_a;
    v->d_seen = c->L.seen;
    v->d_cons = c->L.cons;
    v->d_stats = c->L.stats;
    v->d_evicted = (const uint64_t*)c->L.evicted;
    v->d_refilled = (const uint64_t*)c->L.refilled;
    v->round = c->r;
    for (uint32_t j = 0; j < c->C.J; ++j) { v->epoch[j] = c->e[j]; v->consumed[j] = c->n[j]; }
    v->active_mask = c->active;
    return SENECA_OK;
}

extern "C" seneca_status seneca_sync_status(seneca_ctx* c, void* stream) {
    if (!c) { set_error("bad arguments"); return SENECA_EINVAL; }
    uint32_t err = 0;
    SENECA_CUDA_TRY(cudaMemcpyAsync(&err, c->L.err, 4, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    SENECA_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    if (err) { set_error("device consistency check failed (flags 0x%x)", err); return SENECA_ESTATE; }
    return SENECA_OK;
}

extern "C" uint64_t seneca_launch_count(const seneca_ctx* c) { return c ? c->launches : 0; }

extern "C" seneca_status seneca_profile(seneca_ctx* c, uint32_t sample_every_rounds) {
    if (!c) { set_error("bad arguments"); return SENECA_EINVAL; }
    c->prof.every = sample_every_rounds;
    return SENECA_OK;
}

extern "C" seneca_status seneca_profile_read(seneca_ctx* c, seneca_kernel_stat* out, uint32_t cap, uint32_t* n_out) {
    if (!c || (!out && cap)) { set_error("bad arguments"); return SENECA_EINVAL; }
    c->prof.flush();
    const uint32_t n = std::min<uint32_t>(cap, K_NCLASS);
    for (uint32_t k = 0; k < n; ++k) {
        out[k].name = kKernelNames[k];
        out[k].launches = c->prof.launches[k];
        out[k].sampled = c->prof.sampled[k];
        out[k].sampled_ms = c->prof.ms[k];
    }
    if (n_out) *n_out = K_NCLASS;
    return SENECA_OK;
}

extern "C" void seneca_destroy(seneca_ctx* c) { delete c; }
