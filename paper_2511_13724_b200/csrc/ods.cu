// ods.cu -- Opportunistic Data Sampling replay on B200.
//
// §5.2 of the paper made concrete by readings R-O1..R-O20
// (DESIGN.md §3).  A round is one batch for each listed job, then maintain.
//
// Execution:
//   ods_perm_all      the (job, epoch) permutations pi_j,e(pos) =
//                     perm(key(seed, REQ, j, e), N, pos) (R-O3) into a ring of
//                     K = min(max epochs, 2) slots per job (epoch e in slot e % K),
//                     publishing a ready flag per (job, epoch); the host fills the
//                     ring ahead of each round launch and bounds the launch so no
//                     job enters an epoch that has no slot yet (launch_rounds).
//   ods_rounds        ONE cooperative launch runs R rounds.  CTA x < J owns job
//                     x; CTA J is the maintain CTA.  Per round:
//       job CTAs      classify (a3) -> select (a4, a5) -> finish (a6, a8)
//       maintain CTA  speculative refill selection from the round-start storage
//                     pool (it cannot change before maintain)            [overlapped]
//       -- signal "job phases of round r done" (job CTAs -> maintain CTA) --
//       maintain CTA  eviction of A entries consumed by every active job, apply
//                     evictions + refills (a7)
//       job CTAs      walk of the NEXT round (a1, a2): it reads only the job's
//                     own seen bitmap and lists                          [overlapped]
//       -- signal "maintain(r) applied" (maintain CTA -> job CTAs) --
//   The signals are release/acquire counters; nobody waits for anything it does
//   not depend on.  With no tracked tier (cap_A = 0, evict_tiers = A) jobs never interact and
//   the job CTAs run their rounds without any signal.
//
// Pool counts: for each pool (job x {A, D, E}, plus the storage pool S) a count
// per 256-id block, per 32-block superblock and a total, kept exact
// incrementally.  A pool member is an id whose pool word bit is set:
//   A: tier_A & ~seen_j & ~cons_j    D: tier_D & ~seen_j    E: tier_E & ~seen_j
//   S: ~(tier_E | tier_D | tier_A)   (R-O2, R-O8)
// Selecting the rank-th member is a binary search over the superblock prefix
// (shared memory), one 128-B row of block counts, one 32-B row per bitmap.
//
// Mutable state shared between CTAs of the persistent kernel is read with
// ld.global.cg (L2, never a stale L1 line); the barrier is release/acquire.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "common.cuh"

namespace seneca {
namespace {

constexpr uint32_t T_S = 0, T_E = 1, T_D = 2, T_A = 3, SUBST = 4;
constexpr uint32_t kNewCons = 0x80;          // internal s_osrc flag: consumer set joined this round
constexpr uint32_t kMaxJobs = 32;
constexpr uint32_t kMaxReplicas = 64;        // independent replay instances per context
constexpr uint32_t kMaxShards = 8;           // sample-ID-range shards of one replay
constexpr uint32_t kMaxBatch = 4096;
#ifndef SENECA_LATE_WALK
#define SENECA_LATE_WALK 1          // storage-list walk once all of a job's pools are empty (Cfg.late)
#endif
#ifndef SENECA_LATE_BULK
#define SENECA_LATE_BULK 1          // late rounds of an uncoupled job decided in one pass (late_bulk)
#endif
#ifndef SENECA_BULK_MIN
#define SENECA_BULK_MIN 1           // fewest rounds worth a bulk pass
#endif
constexpr uint32_t kBulkMin = SENECA_BULK_MIN;
#ifndef SENECA_HOIST_KEYS
#define SENECA_HOIST_KEYS 1         // substitution keys and rank domains derived once per round and tier
#endif
#ifndef SENECA_EMPTY_POOLS_FAST
#define SENECA_EMPTY_POOLS_FAST 1    // skip the classification gathers when every pool of the job is empty
#endif
#ifndef SENECA_ODS_THREADS
#define SENECA_ODS_THREADS 512
#endif
constexpr uint32_t kThreads = SENECA_ODS_THREADS;   // CTA size of the persistent kernel
constexpr uint32_t kBlockShift = 7;          // 128 ids (4 words, one 16-B vector) per count block
constexpr uint32_t kSuperShift = 12;         // 32 blocks = 4096 ids per superblock
constexpr uint32_t kWordsPerBlock = 4;
constexpr uint32_t kWalkPerThread = 8;       // list entries examined per thread per walk step
constexpr uint32_t kWinMax = 1024;           // prefetched walk window (list entries)
constexpr uint32_t kGenChunk = 16384;        // positions per permutation-generation chunk
// the prefetched walk step covers 2 window entries per thread: window = min(kWinMax, 2 T)

// ------------------------------------------------------------------ layouts
struct JobDev {           // per-job persistent walk state (workspace)
    uint32_t cur_buf;     // 0: this epoch's permutation; 1/2: deferral (lap) lists
    uint32_t nxt_buf;     // lap list receiving this lap's deferred misses (1/2)
    uint32_t cursor;      // position in the current list
    uint32_t cur_len;
    uint32_t nxt_len;
    uint32_t recount;     // pools must be rebuilt before the next classify (epoch start)
    uint32_t late;        // storage-list walk of this epoch (see Cfg.late)
    uint32_t lc, lk;      // late walk position in lap 1: storage-list segment lc, entry lk
    uint32_t fl, fc, fk, fpos;   // seen-marking frontier of the late rounds (see catch_up_seen)
    uint32_t pad[3];
};

struct Cfg {
    uint32_t N, NW, NB, NS, NBp;     // samples, words/bitmap, blocks, superblocks, padded blocks
    uint32_t J, Bmax, maxT, cap_a, cap_d, cap_e;
    uint32_t K;                      // permutation ring slots per job: min(maxT, 2), a power of two
    uint32_t evict_all;              // evict_tiers = ALL (R-O21): every cached tier is tracked
    uint32_t cap_t;                  // capacity of the tracked tiers (cap_a, or cap_a + cap_d + cap_e; 0 baseline)
    uint32_t baseline;               // the uniform no-evict sampler (R-O22): no substitution, static tiers
    uint32_t cold;                   // cold start (R-O24): empty tiers, round-end admission until full
    uint32_t Nrow;                   // row stride of the permutation / lap lists (N rounded up to 64)
    uint32_t FL;                     // capacity of one refill buffer
    uint32_t late;                   // storage lists: static tiers (no tracked tier, no cold start, ODS sampler,
                                     // generated requests, one unsharded replica) -- once all of a job's pools
                                     // are empty its walk takes the epoch's storage ids in permutation order
                                     // (every unseen id ahead of the cursor is then storage-resident, every
                                     // cached one seen), no seen test (§7.1 "late rounds")
    uint32_t nch;                    // generation chunks (16 K positions) per permutation
    uint32_t G;                      // sample-ID-range shards (1: unsharded), SURVEY §8(e)
    uint32_t xsys;                   // exchange scope: 1 system (peers on other devices), 0 this device
    uint32_t mb_c1, mb_c2, mb_rf, mb_fl;   // mailbox offsets (u32) of the shard exchange, see Lay.mbox
    uint64_t seed;
    uint32_t batch[kMaxJobs];
    uint32_t target[kMaxJobs];
};

struct Lay {
    uint32_t *bm_e, *bm_d, *bm_a;    // [NW]
    uint32_t *seen, *cons;           // [J][NW]
    uint32_t *cons_cnt;              // [N] active consumers of each A entry (R-O5)
    uint32_t *cnt8;                  // [3J+1][NBp] u8 block counts, 4 per word (one 32-B row per superblock)
    uint32_t *cnt_sup;               // [3J+1][NS] superblock counts (kept in shared memory while running)
    uint32_t *cnt_tot;               // [3J+1]
    uint32_t *tsize;                 // [4] tier sizes by tier code (E 1, D 2, A 3)
    uint32_t *perms;                 // [J][K][Nrow] ring: epoch e of job j in slot e % K
    uint32_t *laps;                  // [J][2][N]
    uint32_t *perm_ready;            // [J][maxT]
    uint32_t *perm_done;             // [J][maxT] positions finished
    uint32_t *epoch_at;              // [J] epoch job j plays (published at each epoch start, release):
                                     //     the concurrent ring generator refills slot e % K once it is >= e - K + 1
    uint32_t *gen_next;              // [1] work counter of the ring generator CTAs
    uint32_t *ring_pairs;            // [kRingPairs] (job << 24 | epoch) the generator CTAs fill, in order
    uint32_t *slist;                 // Cfg.late: [J][K][Nrow] per ring slot, per 16 K-position chunk of the
                                     //   permutation its storage-resident ids in position order (a segment)
    uint32_t *scnt;                  //   [J][K][nch] entries of each segment
    uint32_t *cbits;                 //   [J][K][Nrow/32] bit p: position p holds a storage-resident id
    JobDev *jobs;                    // [J]
    uint32_t *out_ids;               // [J][Bmax] replay scratch
    uint8_t *out_src;                // [J][Bmax]
    uint32_t *evict_push;            // ring [J*Bmax]: entries whose consumer count reached |active|
    uint32_t *fill_n;                // [2][4] per round parity: refills k, of which to A, to D (rest E)
    uint32_t *evict_list;            // [max(cap_t,1)] full-scan eviction candidates
    uint32_t *fill_list;             // [2][FL], FL = max(cap_t,1) + J*Bmax; buffer = round parity
    uint32_t *ev_ed;                 // [2][max(cap_e+cap_d,1)] evicted E/D ids (bit 31: E) per parity
    uint32_t *ev_ed_n;               // [2]
    uint32_t *fetch;                 // [J][Bmax] storage fetches of the round (cold start, R-O24)
    uint32_t *fetch_n;               // [J]
    uint32_t *warm;                  // [1] every tier has been full once (cold start ends)
    uint32_t *claim;                 // [NW] admission de-duplication scratch (all zero between rounds)
    seneca_job_epoch_stats *stats;   // [J][maxT]
    unsigned long long *evicted, *refilled;
    uint32_t *err;                   // latched consistency flags (control block, see kCtlBytes)
    uint32_t *verr;                  // caller-supplied request validation flag (control block)
    uint32_t *dbg;                   // [4] first consistency failure: site | pool, rank / round, ... (control block)
    uint32_t *bar;                   // [4] signals: u64 {job phases done | evictions pushed << 32},
                                     //     maintain rounds applied, eviction ring position (control block)
    unsigned long long *phase;       // [32] accumulated cycles per phase (see seneca.h)
    uint64_t seed;                   // this replica's seed (cfg seed + replica index)
    // sample-ID-range sharding: this slice is shard `shard` of G and
    // keeps the pool counts of ids [id_lo, id_hi) = superblocks [sb_lo, sb_hi) only;
    // everything else is replicated.  Unsharded: shard 0 of 1, the whole range.
    uint32_t shard, sb_lo, sb_hi, id_lo, id_hi;
    uint32_t *mbox;                  // this shard's mailbox (peers write into it):
                                     //   c1 [2][J+1][G][4]  per-shard pool totals (stamp, 3 values)
                                     //   c2 [2][J][Bmax]    resolved substitute ids
                                     //   rf [2][FL]         resolved refill ids
                                     //   fl [2][J+1][G]     "ids of round r written" stamps
    uint32_t *peer[kMaxShards];      // every shard's mailbox as seen from here (peer[shard] == mbox)
};

// Per-replica layouts: a kernel parameter (constant bank), indexed by the CTA's
// replica -- no per-CTA copy, and the compiler may hoist every field.
struct Lays {
    Lay r[kMaxReplicas];
};

struct Launch {
    uint64_t r0;
    uint32_t rounds;
    uint32_t subset;                 // jobs taking part in every round (& active)
    uint32_t mode;                   // 0 generated requests, 1 caller-supplied
    uint32_t active0;
    uint32_t pending0;               // jobs that have not arrived yet (R-O23)
    uint32_t arrival[kMaxJobs];      // arrival round of each job
    uint32_t n0[kMaxJobs];           // consumed samples of the current epoch at launch
    uint32_t e0[kMaxJobs];           // epoch at launch
    uint32_t row_of_job[kMaxJobs];   // output row of each job
    uint32_t out_stride;
    uint32_t timing;
    uint32_t* out_ids;
    uint8_t* out_src;
    const uint32_t* requested;       // mode 1: [row][out_stride]
    unsigned long long* transcript;  // [replica][J][maxT][N] or null
    uint64_t out_rep;                // elements of out_ids / out_src per replica
    uint64_t tr_rep;                 // elements of transcript per replica
    uint32_t gen_ctas;               // trailing CTAs of the launch that refill the permutation ring (§7.2)
    uint32_t gen_pairs;              // (job, epoch) pairs they fill, L.ring_pairs of slice 0
    uint32_t cluster;                // 1: the J + 1 round CTAs are one thread-block cluster (DSMEM signals)
};

__device__ __forceinline__ uint32_t ldcg(const uint32_t* p) { return __ldcg(p); }
__device__ __forceinline__ uint4 ldcg4(const uint32_t* p) { return __ldcg(reinterpret_cast<const uint4*>(p)); }

// asynchronous 16-B global -> shared copies (L2 only, never a stale L1 line)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ------------------------------------------------------------------ shard exchange
// Mailboxes live in device memory of the receiving shard: in one context (all
// shards on one device, emulation) the peers' slices of the same workspace; with
// one shard per device, peer memory mapped over NVLink.  Writers store payloads,
// fence, then store a per-(round parity, slot, sender) stamp = round + 1;
// readers poll the stamps, fence, then read the payload uncached (the fence +
// relaxed store / relaxed load + fence pairs are release / acquire).  Scope:
// the device (gpu) when every shard is on this device, the system when the
// peers are other devices (Cfg.xsys).  Lane g of warp 0 serves peer g, so an
// exchange costs two fences and one poll round trip, not 2G.  Round parity
// double-buffers: every shard waits for every other shard's round-r values
// before it can publish round r + 1's, so a buffer is never overwritten while a
// peer may still read it.
__device__ __forceinline__ void xfence(const Cfg& C) {
    if (C.xsys) __threadfence_system(); else __threadfence();
}
__device__ __forceinline__ void st_stamp(const Cfg& C, uint32_t* p, uint32_t v) {
    if (C.xsys) asm volatile("st.relaxed.sys.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
    else asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_stamp(const Cfg& C, const uint32_t* p) {
    uint32_t v;
    if (C.xsys) asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    else asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_mbox(const uint32_t* p) { return __ldcv(p); }

// Failure detection for the exchange: a peer that has not published within
// kPeerTimeoutNs (a dead or never-launched shard) latches err bit 4 and traps
// the launch instead of spinning forever.
constexpr unsigned long long kPeerTimeoutNs = 20ull * 1000 * 1000 * 1000;
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void wait_stamp(const Lay& L, const Cfg& C, const uint32_t* p, uint32_t stamp) {
    if (ld_stamp(C, p) == stamp) return;
    const unsigned long long t0 = globaltimer_ns();
    while (ld_stamp(C, p) != stamp) {
        if (globaltimer_ns() - t0 > kPeerTimeoutNs) { atomicOr(L.err, 4u); __threadfence_system(); __trap(); }
    }
}

// C1 (warp 0 of the calling CTA, every lane): publish (v0, v1, v2) of slot s for
// round r to every shard, wait for every shard's, lane g stores shard g's values
// into out[g][0..2].
__device__ void shard_c1(const Lay& L, const Cfg& C, uint32_t slot, uint64_t r, uint32_t v0, uint32_t v1, uint32_t v2,
                         uint32_t (*out)[3]) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t stamp = (uint32_t)r + 1u;
    const size_t row = C.mb_c1 + (((size_t)(r & 1) * (C.J + 1) + slot) * C.G) * 4;
    if (lane < C.G) {
        uint32_t* q = L.peer[lane] + row + (size_t)L.shard * 4;
        q[1] = v0; q[2] = v1; q[3] = v2;
    }
    xfence(C);
    if (lane < C.G) st_stamp(C, L.peer[lane] + row + (size_t)L.shard * 4, stamp);
    if (lane < C.G) wait_stamp(L, C, L.mbox + row + (size_t)lane * 4, stamp);
    xfence(C);
    if (lane < C.G) {
        const uint32_t* q = L.mbox + row + (size_t)lane * 4;
        out[lane][0] = ld_mbox(q + 1); out[lane][1] = ld_mbox(q + 2); out[lane][2] = ld_mbox(q + 3);
    }
    __syncwarp();
}

// C2 flags (every thread calls it after storing its resolved ids into every
// shard's mailbox): the barrier orders the CTA's stores before warp 0's fence
// and stamps (cumulativity), then warp 0 waits for every shard's stamp.
__device__ void shard_c2_sync(const Lay& L, const Cfg& C, uint32_t slot, uint64_t r) {
    __syncthreads();
    if (threadIdx.x < 32) {
        const uint32_t lane = threadIdx.x;
        const uint32_t stamp = (uint32_t)r + 1u;
        const size_t row = C.mb_fl + ((size_t)(r & 1) * (C.J + 1) + slot) * C.G;
        xfence(C);
        if (lane < C.G) st_stamp(C, L.peer[lane] + row + L.shard, stamp);
        if (lane < C.G) wait_stamp(L, C, L.mbox + row + lane, stamp);
        xfence(C);
    }
    __syncthreads();
}

// The shard owning global pool rank `rank` of pool column t (counts cnt[g][t],
// shards in ascending id order) and the rank within that shard.
__device__ __forceinline__ uint32_t shard_owner(const Cfg& C, const uint32_t (*cnt)[3], uint32_t t, uint32_t rank,
                                                uint32_t* local) {
    uint32_t acc = 0, g = 0;
    for (; g + 1 < C.G; ++g) {
        if (rank < acc + cnt[g][t]) break;
        acc += cnt[g][t];
    }
    *local = rank - acc;
    return g;
}

__device__ __forceinline__ uint32_t valid_mask(const Cfg& C, uint32_t w) {
    const uint64_t lo = (uint64_t)w * 32u;
    if (lo + 32u <= C.N) return 0xffffffffu;
    if (lo >= C.N) return 0u;
    return (1u << (C.N - lo)) - 1u;
}

__device__ __forceinline__ uint32_t pool_of(uint32_t j, uint32_t t) {   // t: T_A, T_D, T_E
    return j * 3u + (t == T_A ? 0u : (t == T_D ? 1u : 2u));
}

// Pool counts: a u8 count per 128-id block in global memory (L2-resident; the
// byte is updated with a 32-bit add of +-1 shifted into place -- a count never
// leaves [0, 128], so no carry/borrow crosses bytes), and a u32 count per
// 4096-id superblock in the shared memory of the CTA that owns the pool.
// kSh: a shard counts only the ids of its own range (returns whether it did).
template <bool kSh = false>
__device__ __forceinline__ bool count_add(const Lay& L, const Cfg& C, uint32_t pidx, uint32_t id, uint32_t delta,
                                          uint32_t* s_sup_pool) {
    if (kSh && (id < L.id_lo || id >= L.id_hi)) return false;
    const uint32_t blk = id >> kBlockShift;
    atomicAdd(L.cnt8 + (size_t)pidx * (C.NBp >> 2) + (blk >> 2), delta << (8u * (blk & 3u)));
    atomicAdd(s_sup_pool + (id >> kSuperShift), delta);
    return true;
}

// Exclusive prefix of the superblock counts (shared memory -> shared memory).
__device__ void prefix_from_smem(const Cfg& C, const uint32_t* s_sup_pool, uint32_t* s_pre_pool, uint32_t* scratch) {
    const uint32_t per = (C.NS + blockDim.x - 1) / blockDim.x;
    const uint32_t lo = threadIdx.x * per;
    const uint32_t hi = min(lo + per, C.NS);
    uint32_t sum = 0;
    if (per <= 8) {                          // (ImageNet-22K: 3,467 superblocks, 7 per thread) counts in registers
        uint32_t v[8];
#pragma unroll
        for (uint32_t k = 0; k < 8; ++k) { v[k] = lo + k < hi ? s_sup_pool[lo + k] : 0u; sum += v[k]; }
        uint32_t run = block_exclusive_scan<false>(sum, nullptr, scratch);   // the barrier below ends it
#pragma unroll
        for (uint32_t k = 0; k < 8; ++k) {
            if (lo + k < hi) s_pre_pool[lo + k] = run;
            run += v[k];
        }
    } else {
        for (uint32_t k = lo; k < hi; ++k) sum += s_sup_pool[k];
        uint32_t run = block_exclusive_scan<false>(sum, nullptr, scratch);
        for (uint32_t k = lo; k < hi; ++k) {
            s_pre_pool[k] = run;
            run += s_sup_pool[k];
        }
    }
    __syncthreads();
}

// Position of the r-th (0-based) set bit of x, r < popc(x): a branch-free
// halving search on popcounts (5 steps, no data-dependent loop).
__device__ __forceinline__ uint32_t select_bit(uint32_t x, uint32_t r) {
    uint32_t pos = 0, c;
    c = __popc(x & 0xffffu); if (r >= c) { r -= c; x >>= 16; pos += 16; }
    c = __popc(x & 0xffu);   if (r >= c) { r -= c; x >>= 8;  pos += 8; }
    c = __popc(x & 0xfu);    if (r >= c) { r -= c; x >>= 4;  pos += 4; }
    c = __popc(x & 0x3u);    if (r >= c) { r -= c; x >>= 2;  pos += 2; }
    c = x & 1u;              if (r >= c) { pos += 1; }
    return pos;
}

// The rank-th (0-based) member, in ascending id order, of pool (t, j):
// superblock by binary search in shared memory, then the superblock's 32-B
// row of block counts (two 16-B loads), then one 16-B vector of each bitmap.
// The row is scanned word-wise: each word's four byte counts (<= 128 each) are
// summed in two 16-bit lanes, a running sum over the 8 words picks the word,
// then at most 3 byte steps pick the block -- a 12-step chain instead of 32.
__device__ uint32_t pool_select(const Lay& L, const Cfg& C, uint32_t pidx, uint32_t t, uint32_t j,
                                const uint32_t* s_pre, uint32_t rank) {
    uint32_t lo = 0, hi = C.NS - 1;
    while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (s_pre[mid] <= rank) lo = mid; else hi = mid - 1;
    }
    uint32_t r = rank - s_pre[lo];
    const uint32_t* crow = L.cnt8 + (size_t)pidx * (C.NBp >> 2) + (size_t)lo * 8u;
    const uint4 c0 = ldcg4(crow), c1 = ldcg4(crow + 4);
    const uint32_t cw[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
    uint32_t run = 0, before = 0, qsel = 0, wsel = cw[0];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const uint32_t x = (cw[q] & 0x00ff00ffu) + ((cw[q] >> 8) & 0x00ff00ffu);
        run += (x & 0xffffu) + (x >> 16);
        if (q < 7 && run <= r) { before = run; qsel = q + 1; wsel = cw[q < 7 ? q + 1 : 7]; }
    }
    if (run <= r) {                                      // counts inconsistent with the bitmaps
        if (atomicCAS(L.dbg, 0u, 0x10000u | pidx) == 0u) L.dbg[1] = rank;
        atomicOr(L.err, 1u);
        return 0;
    }
    r -= before;
    uint32_t k = 0, b = wsel & 0xffu;
    if (r >= b) {
        r -= b; k = 1; b = (wsel >> 8) & 0xffu;
        if (r >= b) {
            r -= b; k = 2; b = (wsel >> 16) & 0xffu;
            if (r >= b) { r -= b; k = 3; }
        }
    }
    const uint32_t w0 = (lo * 32u + qsel * 4u + k) * kWordsPerBlock;
    uint32_t pw[4];
    if (t == T_S) {
        const uint4 a = ldcg4(L.bm_a + w0), e = ldcg4(L.bm_e + w0), d = ldcg4(L.bm_d + w0);
        pw[0] = ~(a.x | e.x | d.x) & valid_mask(C, w0 + 0);
        pw[1] = ~(a.y | e.y | d.y) & valid_mask(C, w0 + 1);
        pw[2] = ~(a.z | e.z | d.z) & valid_mask(C, w0 + 2);
        pw[3] = ~(a.w | e.w | d.w) & valid_mask(C, w0 + 3);
    } else {
        const uint4 sv = ldcg4(L.seen + (size_t)j * C.NW + w0);
        const uint4 bv = ldcg4((t == T_A ? L.bm_a : (t == T_D ? L.bm_d : L.bm_e)) + w0);
        pw[0] = bv.x & ~sv.x; pw[1] = bv.y & ~sv.y; pw[2] = bv.z & ~sv.z; pw[3] = bv.w & ~sv.w;
        if (t == T_A) {
            const uint4 cv = ldcg4(L.cons + (size_t)j * C.NW + w0);
            pw[0] &= ~cv.x; pw[1] &= ~cv.y; pw[2] &= ~cv.z; pw[3] &= ~cv.w;
        }
    }
    uint32_t ksel = 0, xsel = pw[0];
    {
        const uint32_t p0 = __popc(pw[0]), p1 = __popc(pw[1]), p2 = __popc(pw[2]);
        if (r >= p0) {
            r -= p0; ksel = 1; xsel = pw[1];
            if (r >= p1) {
                r -= p1; ksel = 2; xsel = pw[2];
                if (r >= p2) { r -= p2; ksel = 3; xsel = pw[3]; }
            }
        }
    }
    if (r >= (uint32_t)__popc(xsel)) {                  // counts inconsistent with the bitmaps
        if (atomicCAS(L.dbg, 0u, 0x20000u | pidx) == 0u) L.dbg[1] = rank;
        atomicOr(L.err, 1u);
        return 0;
    }
    return (w0 + ksel) * 32u + select_bit(xsel, r);
}

// ------------------------------------------------------------------ barrier among the round CTAs
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long ld_acquire64(const uint32_t* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Signals through distributed shared memory (the round CTAs of one replica are one
// cluster): the writer releases at cluster scope into the reader CTA's shared
// word, the reader polls its own shared memory with acquire loads.
__device__ __forceinline__ uint32_t dsmem_addr_raw(uint32_t local_shared, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_shared), "r"(rank));
    return r;
}
__device__ __forceinline__ uint32_t dsmem_addr(const void* local, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"((uint32_t)__cvta_generic_to_shared(local)), "r"(rank));
    return r;
}
__device__ __forceinline__ void dsmem_red_release_add64(uint32_t addr, unsigned long long v) {
    asm volatile("red.release.cluster.shared::cluster.add.u64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}
constexpr uint32_t kFillBuf = 512;   // refill ids pushed into each job CTA's shared memory (DSMEM signals)
__device__ __forceinline__ void dsmem_st32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void dsmem_st_release64(uint32_t addr, unsigned long long v) {
    asm volatile("st.release.cluster.shared::cluster.u64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}
__device__ __forceinline__ void dsmem_st_release32(uint32_t addr, uint32_t v) {
    asm volatile("st.release.cluster.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long smem_ld_acquire64(const void* p) {
    unsigned long long v;
    asm volatile("ld.acquire.cluster.shared::cta.u64 %0, [%1];" : "=l"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t smem_ld_acquire32(const void* p) {
    uint32_t v;
    asm volatile("ld.acquire.cluster.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)) : "memory");
    return v;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// ------------------------------------------------------------------ per-CTA phase timer (profiling)
// kOn = false (the timed replays) compiles every tick out; the kernel with
// kOn = true is launched only when seneca_profile bit 1 asks for phase counters.
template <bool kOn>
struct PhaseTimer {
    long long last;
    unsigned long long acc[16];
    uint32_t on;
    __device__ __forceinline__ void tick(uint32_t slot) {
        if (kOn && on && threadIdx.x == 0) {
            const long long t = clock64();
            acc[slot] += (unsigned long long)(t - last);
            last = t;
        }
    }
    __device__ __forceinline__ void count(uint32_t slot, unsigned long long v) {
        if (kOn && on && threadIdx.x == 0) acc[slot] += v;
    }
};

// ------------------------------------------------------------------ shared state of a job CTA
struct JobSmem {
    uint32_t cur_buf, nxt_buf, cursor, cur_len, nxt_len;
    uint32_t wrap_slot, need, newcursor, walk_err;
    uint32_t m, k[3], tot[3], hits[3];
    unsigned long long key[3];               // this round's substitution key per tier (A, D, E)
    PermDomain dom[3];                       // and rank domain of the pool after the hits
    uint32_t hits_loc[3], own[3], glob[3];   // sharded: hits / substitutes in this shard's range, global pool sizes
    uint32_t hg[kMaxShards][3], sg[kMaxShards][3];   // sharded, static tiers: this round's hits / substitutes
    uint32_t c1;                                     //   per shard range; 1: the next round exchanges C1
    uint32_t cnt[kMaxShards][3];             // sharded: every shard's pool sizes of this round (C1)
    uint32_t recount;
    uint32_t late, lc, lk; // storage-list walk (Cfg.late): on, lap-1 segment and entry
    uint32_t lcnt;         // entries of segment lc (cached while the walk stays in it)
    uint32_t fl, fc, fk, fpos; // late rounds' seen-marking frontier: fl 0 lap-1 (segment fc, entry fk), 1 lap list fpos
    uint32_t perm_seen;   // epoch+1 whose permutation was observed published (0: none)
    float dens;           // unseen fraction observed by the last walk step (window sizing)
    uint32_t npush;       // evictions pushed by this job this round
    uint32_t rep;         // replica of this CTA
    uint32_t warm;        // cold start over (read at the round start, R-O24)
    // prefetch of the next walk window (R-O1 walk, see job_walk_prefetched)
    uint32_t pf_state;    // 0 none, 1 list window requested, 2 seen chunks requested
    uint32_t pf_buf, pf_epoch, pf_base, pf_len, pf_vlen;
    uint32_t scan[33];
    // this job-epoch's counters, accumulated across rounds and added to memory at
    // the epoch end / launch end (flush_stats): the digest one running sum per
    // thread (a sum mod 2^64 is order-free), counter c in acc_cnt[c]
    unsigned long long acc_cnt[12];
    unsigned long long acc_dig[kThreads];
};

__device__ __forceinline__ const uint32_t* list_ptr(const Lay& L, const Cfg& C, uint32_t j, uint32_t e, uint32_t buf) {
    return buf == 0 ? L.perms + ((size_t)j * C.K + (e & (C.K - 1))) * C.Nrow
                    : L.laps + ((size_t)j * 2 + (buf - 1)) * C.Nrow;
}

// Stage 1 (right after a walk): the next walk window of the current list into
// shared memory.  The list content below cur_len never changes.
__device__ void prefetch_window(const Lay& L, const Cfg& C, JobSmem& S, uint32_t* s_win, uint32_t j, uint32_t e,
                                uint32_t want) {
    const uint32_t tid = threadIdx.x;
    const uint32_t base = S.cursor & ~3u;
    uint32_t len = min(min(kWinMax, 2 * blockDim.x), (want + (S.cursor - base) + 3) & ~3u);
    len = min(len, C.Nrow - base);
    const uint32_t* list = list_ptr(L, C, j, e, S.cur_buf);
    for (uint32_t t = tid; t * 4 < len; t += blockDim.x) cp_async16(s_win + 4 * t, list + base + 4 * t);
    cp_async_commit();
    if (tid == 0) {
        S.pf_state = 1; S.pf_buf = S.cur_buf; S.pf_epoch = e; S.pf_base = base; S.pf_len = len;
    }
}

// Stage 2 (once this round's hits and substitutes are marked seen): the 16-B
// seen chunk of every window id, asynchronously.  Exactness: seen_j is written
// only by this CTA, and the only bits set after this point in the round belong
// to storage-served requested ids, which lie before the window in the list.
__device__ void prefetch_seen(const Lay& L, const Cfg& C, JobSmem& S, const uint32_t* s_win, uint4* s_wseen, uint32_t j) {
    const uint32_t tid = threadIdx.x;
    cp_async_wait_all();
    __syncthreads();
    const uint32_t vlen = S.cur_len > S.pf_base ? min(S.pf_len, S.cur_len - S.pf_base) : 0u;
    const uint32_t* seen_j = L.seen + (size_t)j * C.NW;
    for (uint32_t t = tid; t < vlen; t += blockDim.x) {
        const uint32_t id = s_win[t];
        cp_async16(s_wseen + t, seen_j + ((id >> 5) & ~3u));
    }
    cp_async_commit();
    __syncthreads();
    if (tid == 0) { S.pf_state = 2; S.pf_vlen = vlen; }
}

// a1/a2 (R-O1): the first `need` ids of the job's current lap list, from the
// cursor, that are not in seen_j.  At a lap end the walk continues with the
// list of deferred misses of the lap (slot order = position order).
struct WalkPrefetch {
    const uint4* wseen;      // [kWinMax] prefetched 16-B seen chunks
};

template <class TMr>
__device__ void job_walk(const Lay& L, const Cfg& C, JobSmem& S, uint32_t* s_req, uint32_t j, uint32_t e, uint32_t need,
                         TMr& TM, const uint32_t* s_win, const WalkPrefetch* pf) {
    unsigned long long* iters = TM.on ? &TM.acc[7] : nullptr;
    const uint32_t tid = threadIdx.x, T = blockDim.x;
    const uint32_t* seen_j = L.seen + (size_t)j * C.NW;
    // (thread 0 alone reads and writes the walk bookkeeping here; everyone reads it
    // after the barrier -- compute-sanitizer racecheck)
    if (tid == 0) {
        S.wrap_slot = 0; S.need = need;
        if (S.cur_buf == 0 && S.perm_seen != e + 1) {   // the epoch's permutation must be published
            const uint32_t* f = L.perm_ready + (size_t)j * C.maxT + e;
            while (ld_acquire(f) == 0) { }
            S.perm_seen = e + 1;
        }
    }
    __syncthreads();
    uint32_t taken = 0;
    bool wrapped = false;
    if (pf && S.pf_state != 0) {
        // first step from the prefetched window and its prefetched seen chunks
        // (the bookkeeping is read before the barrier: thread 0 resets pf_state below)
        const bool usable = S.pf_state == 2 && S.pf_buf == S.cur_buf && S.pf_epoch == e &&
                            S.cursor >= S.pf_base && S.cursor < S.pf_base + S.pf_vlen;
        cp_async_wait_all();
        __syncthreads();
        if (usable) {
            const uint32_t cursor = S.cursor, wend = S.pf_base + S.pf_vlen;
            if (iters && tid == 0) *iters += 1;
            const uint32_t p0 = S.pf_base + tid * 2;
            uint32_t flags = 0, cnt = 0, ids[2];
#pragma unroll
            for (uint32_t k = 0; k < 2; ++k) {
                const uint32_t p = p0 + k;
                ids[k] = 0;
                if (p >= cursor && p < wend) {
                    const uint32_t t = p - S.pf_base, id = s_win[t];
                    const uint4 ch = pf->wseen[t];
                    const uint32_t q = (id >> 5) & 3u;
                    const uint32_t w = q == 0 ? ch.x : (q == 1 ? ch.y : (q == 2 ? ch.z : ch.w));
                    ids[k] = id;
                    if (!((w >> (id & 31)) & 1u)) { flags |= 1u << k; ++cnt; }
                }
            }
            uint32_t tot;
            const uint32_t ex = block_flag_scan(flags & 1u, (flags >> 1) & 1u, &tot, S.scan);
            uint32_t r = ex;
#pragma unroll
            for (uint32_t k = 0; k < 2; ++k) {
                if (flags & (1u << k)) {
                    if (r < need) s_req[r] = ids[k];
                    if (r == need - 1) S.newcursor = p0 + k + 1;
                    ++r;
                }
            }
            __syncthreads();
            if (tot >= need) {
                if (tid == 0) {
                    S.cursor = S.newcursor;
                    S.dens = (float)need / (float)max(1u, S.newcursor - cursor);
                }
                taken = need;
            } else {
                if (tid == 0) {
                    S.cursor = wend;
                    S.dens = (float)tot / (float)max(1u, wend - cursor);
                }
                taken = tot;
            }
        }
        if (tid == 0) S.pf_state = 0;
        __syncthreads();
        TM.tick(12);
    }
    while (taken < need) {
        if (S.cursor >= S.cur_len) {
            // read by every thread before the barrier: thread 0 rewrites the lap
            // bookkeeping after it (a read after it raced with that write -- found by
            // compute-sanitizer racecheck/synccheck: a thread could take the error
            // exit alone and leave the block's barriers unmatched)
            const bool dead = wrapped || S.nxt_len == 0;
            __syncthreads();
            if (dead) {
                if (tid == 0) atomicOr(L.err, 2u);
                break;
            }
            if (tid == 0) {
                S.wrap_slot = taken;
                S.cur_buf = S.nxt_buf;
                S.cur_len = S.nxt_len;
                S.cursor = 0;
                S.nxt_buf = S.cur_buf == 1 ? 2 : 1;
                S.nxt_len = 0;
            }
            wrapped = true;
            __syncthreads();
        }
        const uint32_t cursor = S.cursor, len = S.cur_len;
        const uint32_t* list = list_ptr(L, C, j, e, S.cur_buf);
        if (iters && tid == 0) *iters += 1;
        // window [base, base + 8*nt): base = cursor rounded down to 4 entries (16 B);
        // nt threads load two aligned 16-B vectors each; the window is sized from the
        // last observed unseen density (scattered seen gathers cost ~1 L1 wavefront each)
        const uint32_t base = cursor & ~3u;
        const float want = (float)(need - taken) / fmaxf(S.dens, 1.0f / 64.0f) * 1.15f + 64.0f;
        const uint32_t nt = min(T, max(32u, ((uint32_t)want + (cursor - base) + 8 * 32 - 1) / (8 * 32) * 32));
        const uint32_t p0 = base + tid * kWalkPerThread;
        uint32_t ids[kWalkPerThread];
        uint32_t flags = 0, cnt = 0;
        if (tid < nt) {
            if (p0 + kWalkPerThread <= len) {
                const uint4 v0 = ldcg4(list + p0), v1 = ldcg4(list + p0 + 4);
                ids[0] = v0.x; ids[1] = v0.y; ids[2] = v0.z; ids[3] = v0.w;
                ids[4] = v1.x; ids[5] = v1.y; ids[6] = v1.z; ids[7] = v1.w;
            } else {
#pragma unroll
                for (uint32_t k = 0; k < kWalkPerThread; ++k) ids[k] = p0 + k < len ? ldcg(list + p0 + k) : 0u;
            }
#pragma unroll
            for (uint32_t k = 0; k < kWalkPerThread; ++k) {
                const uint32_t p = p0 + k;
                if (p >= cursor && p < len) {
                    const uint32_t id = ids[k];
                    if (!((ldcg(seen_j + (id >> 5)) >> (id & 31)) & 1u)) { flags |= 1u << k; ++cnt; }
                }
            }
        }
        uint32_t tot;
        const uint32_t ex = block_exclusive_scan(cnt, &tot, S.scan);
        const uint32_t remaining = need - taken;
        uint32_t r = ex;
#pragma unroll
        for (uint32_t k = 0; k < kWalkPerThread; ++k) {
            if (flags & (1u << k)) {
                if (r < remaining) s_req[taken + r] = ids[k];
                if (r == remaining - 1) S.newcursor = p0 + k + 1;
                ++r;
            }
        }
        __syncthreads();
        const uint32_t wend = min(base + kWalkPerThread * nt, len);
        if (tot >= remaining) {
            if (tid == 0) {
                S.cursor = S.newcursor;
                S.dens = (float)remaining / (float)max(1u, S.newcursor - cursor);
            }
            taken = need;
        } else {
            if (tid == 0) {
                S.cursor = wend;
                S.dens = (float)tot / (float)max(1u, wend - cursor);
            }
            taken += tot;
        }
        __syncthreads();
    }
}

// Cfg.late: once every pool of job j is empty (static tiers), every unseen id
// ahead of the lap-1 cursor is storage-resident and every cached id is seen, and
// every entry of the lap lists (the deferred, replaced misses: storage ids) is
// unseen.  The walk then takes the next `need` ids of the epoch's storage-list
// segments in order, then of the lap lists -- the same ids the seen-testing
// walk would take, with no seen test.
__device__ void late_walk(const Lay& L, const Cfg& C, JobSmem& S, uint32_t* s_req, uint32_t j, uint32_t e,
                          uint32_t need, const uint32_t* s_win) {
    const uint32_t tid = threadIdx.x, T = blockDim.x;
    const size_t slot = (size_t)j * C.K + (e & (C.K - 1));
    if (tid == 0) { S.wrap_slot = 0; S.need = need; }
    uint32_t s = 0;
    if (S.pf_state == 3) {                           // the first entries, prefetched one round ahead
        const bool usable = S.pf_buf == S.cur_buf &&
                            (S.cur_buf == 0 ? (S.pf_epoch == S.lc && S.pf_base == S.lk) : S.pf_base == S.cursor);
        const uint32_t n = min(S.pf_len, need), off = S.pf_vlen;
        cp_async_wait_all();
        __syncthreads();
        if (usable) {
            for (uint32_t t = tid; t < n; t += T) s_req[t] = s_win[off + t];
            s = n;
            __syncthreads();
            if (tid == 0) {
                if (S.cur_buf == 0) {
                    S.lk += n;
                    if (S.lk == S.lcnt) {
                        S.lc += 1; S.lk = 0;
                        S.lcnt = S.lc < C.nch ? ldcg(L.scnt + slot * C.nch + S.lc) : 0u;
                    }
                } else {
                    S.cursor += n;
                }
            }
        }
        if (tid == 0) S.pf_state = 0;
    }
    while (s < need) {
        __syncthreads();                             // state of the previous step visible
        uint32_t take;
        if (S.cur_buf == 0) {
            if (S.lc >= C.nch) {                     // lap 1 done: the deferred misses are next
                __syncthreads();
                if (tid == 0) {
                    S.wrap_slot = s;
                    S.cur_buf = S.nxt_buf; S.cur_len = S.nxt_len; S.cursor = 0;
                    S.nxt_buf = S.cur_buf == 1 ? 2 : 1; S.nxt_len = 0;
                }
                continue;
            }
            const uint32_t cnt = S.lcnt;
            take = min(cnt - S.lk, need - s);
            const uint32_t* src = L.slist + slot * C.Nrow + (size_t)S.lc * kGenChunk + S.lk;
            for (uint32_t t = tid; t < take; t += T) s_req[s + t] = ldcg(src + t);
            __syncthreads();
            if (tid == 0) {
                S.lk += take;
                if (S.lk == cnt) {
                    S.lc += 1; S.lk = 0;
                    S.lcnt = S.lc < C.nch ? ldcg(L.scnt + slot * C.nch + S.lc) : 0u;
                }
            }
        } else {
            take = min(S.cur_len - S.cursor, need - s);
            if (take == 0) {                         // cannot happen while n_j < N
                if (tid == 0) atomicOr(L.err, 2u);
                break;
            }
            const uint32_t* src = L.laps + ((size_t)j * 2 + (S.cur_buf - 1)) * C.Nrow + S.cursor;
            for (uint32_t t = tid; t < take; t += T) s_req[s + t] = ldcg(src + t);
            __syncthreads();
            if (tid == 0) S.cursor += take;
        }
        s += take;
    }
    __syncthreads();
}

// The next late walk's first `want` entries -- as far as the current segment or
// lap list reaches -- copied into s_win with 16-B cp.async (the 16-B-aligned
// superset; the walk reads from offset pos mod 4): the storage lists stream
// from DRAM, so the copy is issued a round ahead (every thread calls it).
__device__ void late_prefetch(const Lay& L, const Cfg& C, JobSmem& S, uint32_t* s_win, uint32_t j, uint32_t e,
                              uint32_t want) {
    const uint32_t tid = threadIdx.x;
    const uint32_t* src;
    uint32_t pos, avail;
    if (S.cur_buf == 0) {
        if (S.lc >= C.nch) return;
        src = L.slist + ((size_t)j * C.K + (e & (C.K - 1))) * C.Nrow + (size_t)S.lc * kGenChunk;
        pos = S.lk;
        avail = S.lcnt - S.lk;
    } else {
        src = L.laps + ((size_t)j * 2 + (S.cur_buf - 1)) * C.Nrow;
        pos = S.cursor;
        avail = S.cur_len - S.cursor;
    }
    const uint32_t n = min(avail, min(want, kWinMax - 4));
    if (n == 0) return;
    const uint32_t al = pos & ~3u, end = (pos + n + 3) & ~3u;
    for (uint32_t t = tid; al + 4 * t < end; t += blockDim.x) cp_async16(s_win + 4 * t, src + al + 4 * t);
    cp_async_commit();
    __syncthreads();
    if (tid == 0) {
        S.pf_state = 3; S.pf_buf = S.cur_buf; S.pf_epoch = S.lc; S.pf_base = pos; S.pf_len = n; S.pf_vlen = pos - al;
    }
}

// Switch job j to the storage-list walk (all its pools are empty; every thread
// calls it): the lap-1 cursor becomes (segment, entry) by counting the
// storage-resident positions of its chunk before it.
__device__ __noinline__ void enter_late(const Lay& L, const Cfg& C, JobSmem& S, uint32_t j, uint32_t e) {
    const uint32_t tid = threadIdx.x;
    cp_async_wait_all();                              // the seen-testing walk's prefetch is dropped
    __syncthreads();
    if (S.cur_buf == 0) {
        const size_t slot = (size_t)j * C.K + (e & (C.K - 1));
        const uint32_t* cb = L.cbits + slot * (C.Nrow / 32);
        const uint32_t cur = S.cursor, lc = cur / kGenChunk;
        const uint32_t w0 = lc * (kGenChunk / 32), w1 = cur >> 5;
        uint32_t c = 0;
        for (uint32_t w = w0 + tid; w <= w1; w += blockDim.x) {
            if (w < w1) c += __popc(ldcg(cb + w));
            else if (cur & 31) c += __popc(ldcg(cb + w) & ((1u << (cur & 31)) - 1u));
        }
        uint32_t tot;
        block_exclusive_scan(c, &tot, S.scan);
        if (tid == 0) {
            S.lc = lc; S.lk = tot; S.fl = 0; S.fc = lc; S.fk = tot;
            S.lcnt = lc < C.nch ? ldcg(L.scnt + slot * C.nch + lc) : 0u;
        }
    } else if (tid == 0) {
        S.fl = 1; S.fpos = S.cursor;
    }
    if (tid == 0) { S.late = 1; S.pf_state = 0; }
    __syncthreads();
}

// Late rounds do not mark their deliveries in seen_j: nothing reads job j's seen
// bits while its pools are empty (no seen test in the walk, no pool selection,
// static tiers: no refills) and the epoch end clears them.  A launch that ends
// mid-epoch in late mode marks the ids delivered since the frontier -- the
// storage-list entries walked in lap 1, then the lap-list entries -- so the
// state is exact between launches (every thread calls it).
__device__ __noinline__ void catch_up_seen(const Lay& L, const Cfg& C, JobSmem& S, uint32_t j, uint32_t e) {
    const uint32_t tid = threadIdx.x, T = blockDim.x;
    uint32_t* seen_j = L.seen + (size_t)j * C.NW;
    __syncthreads();
    if (S.fl == 0) {
        const size_t slot = (size_t)j * C.K + (e & (C.K - 1));
        const bool in1 = S.cur_buf == 0;
        const uint32_t ec = in1 ? S.lc : C.nch, ek = in1 ? S.lk : 0u;
        for (uint32_t c = S.fc; c <= ec && c < C.nch; ++c) {
            const uint32_t k0 = c == S.fc ? S.fk : 0u;
            const uint32_t k1 = c == ec ? ek : ldcg(L.scnt + slot * C.nch + c);
            const uint32_t* seg = L.slist + slot * C.Nrow + (size_t)c * kGenChunk;
            for (uint32_t k = k0 + tid; k < k1; k += T) {
                const uint32_t i = ldcg(seg + k);
                atomicOr(seen_j + (i >> 5), 1u << (i & 31));
            }
        }
        __syncthreads();
        if (tid == 0) {
            if (in1) { S.fc = S.lc; S.fk = S.lk; }
            else { S.fl = 1; S.fpos = 0; }
        }
        __syncthreads();
    }
    if (S.fl == 1 && S.cur_buf != 0) {
        const uint32_t* list = L.laps + ((size_t)j * 2 + (S.cur_buf - 1)) * C.Nrow;
        for (uint32_t k = S.fpos + tid; k < S.cursor; k += T) {
            const uint32_t i = ldcg(list + k);
            atomicOr(seen_j + (i >> 5), 1u << (i & 31));
        }
        __syncthreads();
        if (tid == 0) S.fpos = S.cursor;
    }
    __syncthreads();
}

// Late bulk (Cfg.late, uncoupled jobs): once every pool of job j is empty its
// remaining rounds of the epoch are decided in advance -- each takes the next
// `need` entries of the storage-list stream (late_walk) and every one is a miss
// served from storage (no pool to substitute from, R-O2; no tracked tier, so no
// consumer, eviction or refill) -- and the rounds of an uncoupled job read no
// state another round writes.  So `cnt` = K full batches of the stream are
// decided in one pass, positions n .. n + cnt - 1 of the epoch: digest and
// transcript exactly as job_round writes them for source S, served[S] += cnt.
// The stream cursor (lc, lk / cur_buf, cursor) ends where K late walks would
// leave it, and the seen-marking frontier is untouched (catch_up_seen covers
// these ids like any other late round's).  Every thread calls it.
__device__ __forceinline__ unsigned long long late_digest(uint32_t id, uint32_t pos, unsigned long long* trow) {
    if (trow) trow[pos] = id;                                       // (T_S << 32) | id, T_S = 0
    return splitmix64(((uint64_t)pos << 35) | id);                  // source T_S = 0 (job_round's digest term)
}

__device__ __noinline__ void late_bulk(const Lay& L, const Cfg& C, const Launch& P, JobSmem& S, uint32_t j, uint32_t e,
                                       uint32_t n, uint32_t cnt) {
    const uint32_t tid = threadIdx.x, T = blockDim.x;
    const size_t slot = (size_t)j * C.K + (e & (C.K - 1));
    unsigned long long* trow = P.transcript ? P.transcript + S.rep * P.tr_rep + ((size_t)j * C.maxT + e) * C.N : nullptr;
    cp_async_wait_all();                                 // a prefetched window of the next walk is dropped
    __syncthreads();
    if (tid == 0) S.pf_state = 0;
    unsigned long long dig = 0;
    uint32_t done = 0;
    while (done < cnt) {
        __syncthreads();                                 // the cursor of the previous step visible
        const uint32_t* src;
        uint32_t take;
        if (S.cur_buf == 0) {
            if (S.lc >= C.nch) {                         // lap 1 done: the deferred misses are next
                __syncthreads();
                if (tid == 0) {
                    S.cur_buf = S.nxt_buf; S.cur_len = S.nxt_len; S.cursor = 0;
                    S.nxt_buf = S.cur_buf == 1 ? 2 : 1; S.nxt_len = 0;
                }
                continue;
            }
            take = min(S.lcnt - S.lk, cnt - done);
            src = L.slist + slot * C.Nrow + (size_t)S.lc * kGenChunk + S.lk;
            if (S.lc + 1 < C.nch && take < cnt - done) {  // the next segment's lines into L2 meanwhile
                const uint32_t* nx = L.slist + slot * C.Nrow + (size_t)(S.lc + 1) * kGenChunk;
                for (uint32_t l = tid; l < kGenChunk / 32; l += T) asm volatile("prefetch.global.L2 [%0];" :: "l"(nx + 32 * l));
            }
        } else {
            take = min(S.cur_len - S.cursor, cnt - done);
            if (take == 0) {                             // cannot happen while n_j < N
                if (tid == 0) atomicOr(L.err, 2u);
                break;
            }
            src = L.laps + ((size_t)j * 2 + (S.cur_buf - 1)) * C.Nrow + S.cursor;
        }
        const uint32_t pos0 = n + done;
        // 16-B vectors between a scalar head and tail (4 vectors in flight per thread)
        const uint32_t head = min(take, (uint32_t)((16u - ((uint32_t)(uintptr_t)src & 15u)) & 15u) / 4u);
        if (tid < head) dig += late_digest(ldcg(src + tid), pos0 + tid, trow);
        const uint4* v = reinterpret_cast<const uint4*>(src + head);
        const uint32_t nv = (take - head) / 4;
#pragma unroll 4
        for (uint32_t q = tid; q < nv; q += T) {
            const uint4 x = __ldcg(v + q);
            const uint32_t p = pos0 + head + 4 * q;
            dig += late_digest(x.x, p, trow) + late_digest(x.y, p + 1, trow) +
                   late_digest(x.z, p + 2, trow) + late_digest(x.w, p + 3, trow);
        }
        const uint32_t t = head + 4 * nv + tid;
        if (t < take) dig += late_digest(ldcg(src + t), pos0 + t, trow);
        __syncthreads();                                 // every thread has read the cursor
        if (tid == 0) {
            if (S.cur_buf == 0) {
                S.lk += take;
                if (S.lk == S.lcnt) {
                    S.lc += 1; S.lk = 0;
                    S.lcnt = S.lc < C.nch ? ldcg(L.scnt + slot * C.nch + S.lc) : 0u;
                }
            } else {
                S.cursor += take;
            }
        }
        done += take;
    }
    __syncthreads();
    S.acc_dig[tid] += dig;
    if (tid == 0) S.acc_cnt[0] += cnt;                   // served[S]
}

// Rebuild the three pool counts of job j (epoch start): block bytes in global
// memory, superblock counts in this CTA's shared memory, totals in tot3.
__device__ __noinline__ void job_recount(const Lay& L, const Cfg& C, uint32_t j, uint32_t* s_sup /* [3][NS] */, uint32_t* tot3) {
    const uint32_t tid = threadIdx.x, T = blockDim.x;
    for (uint32_t k = tid; k < 3 * C.NS; k += T) s_sup[k] = 0;
    __syncthreads();
    const uint32_t* cj = L.cons + (size_t)j * C.NW;
    const uint32_t* sj = L.seen + (size_t)j * C.NW;
    uint32_t ta = 0, td = 0, te = 0;
    for (uint32_t g = L.sb_lo * 8 + tid; g < L.sb_hi * 8; g += T) {   // 4 blocks = 16 words per step (own shard)
        uint32_t pa = 0, pd = 0, pe = 0;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const uint32_t w0 = (g * 4 + h) * kWordsPerBlock;
            const uint4 a = ldcg4(L.bm_a + w0), d = ldcg4(L.bm_d + w0), e = ldcg4(L.bm_e + w0);
            const uint4 c = ldcg4(cj + w0), s = ldcg4(sj + w0);
            const uint32_t ca = __popc(a.x & ~c.x & ~s.x) + __popc(a.y & ~c.y & ~s.y) + __popc(a.z & ~c.z & ~s.z) + __popc(a.w & ~c.w & ~s.w);
            const uint32_t cd = __popc(d.x & ~s.x) + __popc(d.y & ~s.y) + __popc(d.z & ~s.z) + __popc(d.w & ~s.w);
            const uint32_t ce = __popc(e.x & ~s.x) + __popc(e.y & ~s.y) + __popc(e.z & ~s.z) + __popc(e.w & ~s.w);
            pa |= ca << (8 * h); pd |= cd << (8 * h); pe |= ce << (8 * h);
            ta += ca; td += cd; te += ce;
            const uint32_t sb = (g * 4 + h) >> 5;
            if (ca) atomicAdd(s_sup + sb, ca);
            if (cd) atomicAdd(s_sup + C.NS + sb, cd);
            if (ce) atomicAdd(s_sup + 2 * C.NS + sb, ce);
        }
        L.cnt8[(size_t)(j * 3 + 0) * (C.NBp >> 2) + g] = pa;
        L.cnt8[(size_t)(j * 3 + 1) * (C.NBp >> 2) + g] = pd;
        L.cnt8[(size_t)(j * 3 + 2) * (C.NBp >> 2) + g] = pe;
    }
    ta = warp_sum(ta); td = warp_sum(td); te = warp_sum(te);
    __shared__ uint32_t s_t[3];
    if (tid == 0) s_t[0] = s_t[1] = s_t[2] = 0;
    __syncthreads();
    if ((tid & 31) == 0) { atomicAdd(&s_t[0], ta); atomicAdd(&s_t[1], td); atomicAdd(&s_t[2], te); }
    __syncthreads();
    if (tid == 0) { tot3[0] = s_t[0]; tot3[1] = s_t[1]; tot3[2] = s_t[2]; }
    __syncthreads();
}

// a3-a6 for job j in round r: classify, substitute, respond.  kSh: this CTA is
// one shard of a sample-ID-range-sharded replay: classification,
// ranks and responses are replicated; the pool counts and the rank -> id
// selection cover this shard's range, with two exchanges per round (C1: every
// shard's pool sizes; C2: the ids each shard resolved).
template <bool kSh, class TMr>
__device__ void job_round(const Lay& L, const Cfg& C, const Launch& P, JobSmem& S, uint32_t* s_req, uint32_t* s_miss,
                          uint32_t* s_sub, uint32_t* s_oid, uint8_t* s_osrc, uint32_t* s_pre, uint32_t j, uint64_t r,
                          uint32_t e, uint32_t nbase, uint32_t n_act, TMr& TM, const uint32_t* s_win,
                          uint4* s_wseen, uint32_t* s_sup) {
    const uint32_t tid = threadIdx.x, T = blockDim.x;
    const uint32_t need = S.need;
    uint32_t* seen_j = L.seen + (size_t)j * C.NW;
    uint32_t* cons_j = L.cons + (size_t)j * C.NW;
    const size_t row = S.rep * P.out_rep + (size_t)P.row_of_job[j] * P.out_stride;
    // (S.hits and S.npush are zero here: reset after their last use of the previous
    // round; the pool totals S.tot persist across rounds in shared memory)

    // a3: hits (E, D, or A not consumed by j, R-O13) join seen_j now
    uint32_t mbase = 0;
#if SENECA_EMPTY_POOLS_FAST
    // every request is unseen by j, and an unseen E or D id -- or an unseen A id
    // j has not consumed -- is by definition a member of j's pool of that tier
    // (R-O2): with all three pools empty no request can hit, so no residency
    // word needs gathering (the same decisions; not under the baseline sampler,
    // whose A hits ignore consumption, nor sharded, whose totals are local)
    // (sharded: S.tot is this shard's part; in late mode every pool is empty globally)
    const bool none_cached = (!kSh && !C.baseline && (S.tot[0] | S.tot[1] | S.tot[2]) == 0u) || (kSh && S.late);
#else
    const bool none_cached = false;
#endif
    for (uint32_t base = 0; base < need; base += T) {
        const uint32_t s = base + tid;
        bool is_miss = false;
        if (s < need) {
            const uint32_t i = s_req[s];
            const uint32_t w = i >> 5, b = 1u << (i & 31);
            // only the tiers that exist are gathered; the consumer word only for A ids
            const uint32_t wa = C.cap_a && !none_cached ? ldcg(L.bm_a + w) : 0u;
            const uint32_t wd = C.cap_d && !none_cached ? ldcg(L.bm_d + w) : 0u;
            const uint32_t we = C.cap_e && !none_cached ? ldcg(L.bm_e + w) : 0u;
            const uint32_t t = (wa & b) ? T_A : (wd & b) ? T_D : (we & b) ? T_E : T_S;
            const bool hit = (t == T_E || t == T_D || (t == T_A && (C.baseline || !(ldcg(cons_j + w) & b))));
            if (hit) {
                if (P.out_ids) { P.out_ids[row + s] = i; P.out_src[row + s] = (uint8_t)t; }
                s_oid[s] = i;
                // kNewCons: j joined the consumer set now (A hits always do; E/D hits
                // under evict_tiers = ALL unless j consumed them before, R-O21)
                uint32_t flag = 0;
                if (C.baseline) { /* no consumer sets (R-O22) */ }
                else if (t == T_A) { atomicOr(cons_j + w, b); flag = kNewCons; }
                else if (C.evict_all && !(atomicOr(cons_j + w, b) & b)) flag = kNewCons;
                s_osrc[s] = (uint8_t)(t | flag);
                atomicOr(seen_j + w, b);
                const bool mine = count_add<kSh>(L, C, pool_of(j, t), i, 0xffffffffu,
                                                 s_sup + (pool_of(j, t) - j * 3) * C.NS);
                atomicAdd(&S.hits[t == T_A ? 0 : (t == T_D ? 1 : 2)], 1u);
                if (kSh && mine) atomicAdd(&S.hits_loc[t == T_A ? 0 : (t == T_D ? 1 : 2)], 1u);
                if (kSh && C.late)           // every shard classifies every request: it counts every range's hits
                    atomicAdd(&S.hg[(i >> kSuperShift) / ((C.NS + C.G - 1) / C.G)][t == T_A ? 0 : (t == T_D ? 1 : 2)], 1u);
            } else {
                is_miss = true;
            }
        }
        uint32_t tot;
        const uint32_t ex = block_flag_scan(is_miss, false, &tot, S.scan);
        if (is_miss) s_miss[mbase + ex] = s;
        mbase += tot;
    }
    // C1: this shard's pool sizes after its hits, everyone's back (not in late mode: every
    // shard entered it in the same round, after which all pools stay empty globally
    // until the epoch ends -- no exchange until then)
    // With static tiers a shard's pools change only by the round's hits and substitutes,
    // which every shard sees (classification is replicated; the owner of every rank
    // follows from the sizes), so every shard keeps every shard's sizes itself and C1
    // is exchanged only in the first round of a launch and after an epoch-start recount.
    if (kSh && !S.late && tid < 32) {
        if (!C.late || S.c1) {
            shard_c1(L, C, j, r, S.tot[0] - S.hits_loc[0], S.tot[1] - S.hits_loc[1], S.tot[2] - S.hits_loc[2], S.cnt);
        } else {
            if (tid < C.G) { S.cnt[tid][0] -= S.hg[tid][0]; S.cnt[tid][1] -= S.hg[tid][1]; S.cnt[tid][2] -= S.hg[tid][2]; }
            __syncwarp();
        }
    }
    if (tid == 0) {
        uint32_t pa, pd, pe;                 // the pools' sizes after this round's hits
        if constexpr (kSh) {
            S.tot[0] -= S.hits_loc[0]; S.tot[1] -= S.hits_loc[1]; S.tot[2] -= S.hits_loc[2];
            pa = pd = pe = 0;
            if (!S.late)
                for (uint32_t g = 0; g < C.G; ++g) { pa += S.cnt[g][0]; pd += S.cnt[g][1]; pe += S.cnt[g][2]; }
            S.glob[0] = pa; S.glob[1] = pd; S.glob[2] = pe;
            if ((pa > C.N || pd > C.N || pe > C.N) && atomicCAS(L.dbg, 0u, 0x80000u | j) == 0u) {
                L.dbg[1] = (uint32_t)r; L.dbg[2] = S.cnt[0][0]; L.dbg[3] = C.G > 1 ? S.cnt[1][0] : 0u;
                atomicOr(L.err, 8u);                      // a global pool size above N (diagnostic)
            }
        } else {
            pa = S.tot[0] - S.hits[0]; pd = S.tot[1] - S.hits[1]; pe = S.tot[2] - S.hits[2];
            if ((pa > C.N || pd > C.N || pe > C.N) && atomicCAS(L.dbg, 0u, 0x40000u | j) == 0u) {
                L.dbg[1] = (uint32_t)r; L.dbg[2] = S.tot[0]; L.dbg[3] = S.hits[0];
                atomicOr(L.err, 8u);                      // a pool total below its hits (diagnostic)
            }
#if !SENECA_HOIST_KEYS
            S.tot[0] = pa; S.tot[1] = pd; S.tot[2] = pe;
#endif                                                    // (else: the hits leave S.tot at the round end)
        }
        const uint32_t m = mbase;
        S.m = m;
        S.k[0] = C.baseline ? 0u : min(m, pa);                  // R-O22: no substitution
        S.k[1] = C.baseline ? 0u : min(m - S.k[0], pd);
        S.k[2] = C.baseline ? 0u : min(m - S.k[0] - S.k[1], pe);
    }
#if SENECA_HOIST_KEYS
    // meanwhile, lane 0 of warps 1-3: the key and the rank domain of tier tt for
    // this round (every substituting thread derived them itself before; the same
    // values -- derive_key(seed, SUB, j, r, t) and the pool size after the hits)
    if (!kSh && (tid & 31) == 0 && tid >= 32 && tid <= 96) {
        const uint32_t tt = (tid >> 5) - 1;
        S.key[tt] = derive_key(L.seed, PUR_SUB, j, r, tt == 0 ? T_A : (tt == 1 ? T_D : T_E));
        S.dom[tt] = perm_domain(S.tot[tt] - S.hits[tt]);
    }
#endif
    __syncthreads();
    TM.tick(1);

    // a4/a5: misses in slot order take substitutes A -> D -> E at keyed ranks (R-O2)
    const uint32_t k0 = S.k[0], k1 = S.k[1], k2 = S.k[2];
    const uint32_t q = k0 + k1 + k2;
    if (q > 0) {
        for (uint32_t tt = 0; tt < 3; ++tt)
            if (S.k[tt]) prefix_from_smem(C, s_sup + tt * C.NS, s_pre + tt * C.NS, S.scan);
        TM.tick(8);
        for (uint32_t u = tid; u < q; u += T) {
            const uint32_t tt = u < k0 ? 0u : (u < k0 + k1 ? 1u : 2u);
            const uint32_t ul = u - (tt == 0 ? 0u : (tt == 1 ? k0 : k0 + k1));
            const uint32_t t = tt == 0 ? T_A : (tt == 1 ? T_D : T_E);
#if SENECA_HOIST_KEYS
            const uint32_t rank = kSh ? perm_apply(derive_key(L.seed, PUR_SUB, j, r, t), perm_domain(S.glob[tt]), ul)
                                      : perm_apply(S.key[tt], S.dom[tt], ul);
#else
            const uint64_t key = derive_key(L.seed, PUR_SUB, j, r, t);
            const uint32_t rank = perm_apply(key, perm_domain(kSh ? S.glob[tt] : S.tot[tt]), ul);
#endif
            if constexpr (kSh) {
                // the shard whose range holds global rank `rank` resolves it and
                // stores the id into every shard's mailbox (C2)
                uint32_t local;
                const uint32_t owner = shard_owner(C, S.cnt, tt, rank, &local);
                if (C.late) atomicAdd(&S.sg[owner][tt], 1u);
                if (owner == L.shard) {
                    const uint32_t id = pool_select(L, C, j * 3 + tt, t, j, s_pre + tt * C.NS, local);
                    const size_t at = C.mb_c2 + ((size_t)(r & 1) * C.J + j) * C.Bmax + u;
                    for (uint32_t g = 0; g < C.G; ++g) L.peer[g][at] = id;
                    atomicAdd(&S.own[tt], 1u);
                }
            } else {
                const uint32_t id = pool_select(L, C, j * 3 + tt, t, j, s_pre + tt * C.NS, rank);
                const uint32_t s = s_miss[u];
                if (P.out_ids) { P.out_ids[row + s] = id; P.out_src[row + s] = (uint8_t)(t | SUBST); }
                s_oid[s] = id;
                s_osrc[s] = (uint8_t)(t | SUBST);
                s_sub[u] = id;
            }
        }
        if constexpr (kSh) {
            shard_c2_sync(L, C, j, r);                                             // C2
            const uint32_t* in = L.mbox + C.mb_c2 + ((size_t)(r & 1) * C.J + j) * C.Bmax;
            for (uint32_t u = tid; u < q; u += T) {
                const uint32_t t = u < k0 ? T_A : (u < k0 + k1 ? T_D : T_E);
                const uint32_t id = ld_mbox(in + u), s = s_miss[u];
                if (P.out_ids) { P.out_ids[row + s] = id; P.out_src[row + s] = (uint8_t)(t | SUBST); }
                s_oid[s] = id;
                s_osrc[s] = (uint8_t)(t | SUBST);
                s_sub[u] = id;
            }
        }
        __syncthreads();
        TM.tick(9);
        for (uint32_t u = tid; u < q; u += T) {
            const uint32_t tt = u < k0 ? 0u : (u < k0 + k1 ? 1u : 2u);
            const uint32_t id = s_sub[u];
            const uint32_t w = id >> 5, b = 1u << (id & 31);
            atomicOr(seen_j + w, b);
            if (tt == 0) { atomicOr(cons_j + w, b); s_osrc[s_miss[u]] |= kNewCons; }
            else if (C.evict_all && !(atomicOr(cons_j + w, b) & b)) s_osrc[s_miss[u]] |= kNewCons;
            count_add<kSh>(L, C, j * 3 + tt, id, 0xffffffffu, s_sup + tt * C.NS);
        }
    }
    __syncthreads();
    if (P.mode == 0 && S.pf_state == 1) prefetch_seen(L, C, S, s_win, s_wseen, j);   // next walk, stage 2
    TM.tick(2);
    // remaining misses are fetched from storage (R-O18); during a cold start they
    // are also listed, in slot order, for the round-end admission (R-O24)
    const bool record = C.cold && !S.warm;
    const bool late = S.late != 0;
    for (uint32_t u = q + tid; u < S.m; u += T) {
        const uint32_t s = s_miss[u], i = s_req[s];
        if (P.out_ids) { P.out_ids[row + s] = i; P.out_src[row + s] = (uint8_t)T_S; }
        s_oid[s] = i;
        s_osrc[s] = (uint8_t)T_S;
        if (!late) atomicOr(seen_j + (i >> 5), 1u << (i & 31));     // late rounds: catch_up_seen
        if (record) L.fetch[(size_t)j * C.Bmax + (u - q)] = i;
    }
    if (record && tid == 0) L.fetch_n[j] = S.m - q;
    // deferred (replaced) misses are requested again on the next lap (R-O1):
    // before a wrap -> the end of the (new) current list, after -> the next list
    uint32_t q1 = 0;
    if (S.wrap_slot > 0) {
        uint32_t c = 0;
        for (uint32_t u = tid; u < q; u += T) c += s_miss[u] < S.wrap_slot;
        block_exclusive_scan(c, &q1, S.scan);
    }
    if (P.mode == 0 && q > 0) {
        uint32_t* cur_list = L.laps + ((size_t)j * 2 + (S.cur_buf - 1)) * C.Nrow;   // only used if q1 > 0
        uint32_t* nxt_list = L.laps + ((size_t)j * 2 + (S.nxt_buf - 1)) * C.Nrow;
        for (uint32_t u = tid; u < q; u += T) {
            const uint32_t id = s_req[s_miss[u]];
            if (u < q1) cur_list[S.cur_len + u] = id;
            else nxt_list[S.nxt_len + (u - q1)] = id;
        }
    }
    __syncthreads();
    TM.tick(10);
    if (tid == 0) {
        if (P.mode == 0) { S.cur_len += q1; S.nxt_len += q - q1; }
        if constexpr (kSh) {                 // this shard's own substitutes leave its pools
            S.tot[0] -= S.own[0]; S.tot[1] -= S.own[1]; S.tot[2] -= S.own[2];
            S.own[0] = S.own[1] = S.own[2] = 0;
            if (C.late && !S.late) {         // every shard's sizes after this round (C1 skipped next round)
                for (uint32_t g = 0; g < C.G; ++g)
                    for (uint32_t t3 = 0; t3 < 3; ++t3) { S.cnt[g][t3] -= S.sg[g][t3]; S.sg[g][t3] = 0; }
                S.c1 = 0;
            }
        } else {
#if SENECA_HOIST_KEYS
            S.tot[0] -= S.hits[0] + k0;
            S.tot[1] -= S.hits[1] + k1;
            S.tot[2] -= S.hits[2] + k2;
#else
            S.tot[0] -= k0;
            S.tot[1] -= k1;
            S.tot[2] -= k2;
#endif
        }
    }

    // a6: digest, transcript; a tracked entry whose consumer count reaches
    // |active| is pushed for eviction at the round end (R-O5, R-O21).  The per-tier counters follow
    // from the phase counts: hits per tier, k_t substitutes, m - q storage.
    unsigned long long dig = 0;
    unsigned long long* trow = P.transcript ? P.transcript + S.rep * P.tr_rep + ((size_t)j * C.maxT + e) * C.N : nullptr;
    const uint32_t lane = tid & 31;
    for (uint32_t s = tid; s < need; s += T) {
        const uint32_t i = s_oid[s];
        const uint32_t src = s_osrc[s] & 7u;
        dig += splitmix64(((uint64_t)(nbase + s) << 35) | ((uint64_t)src << 32) | i);
        if (trow) trow[nbase + s] = ((unsigned long long)src << 32) | i;
        if (s_osrc[s] & kNewCons) {
            if (atomicAdd(L.cons_cnt + i, 1u) + 1u == n_act) {
                L.evict_push[atomicAdd(L.bar + 3, 1u) % (C.J * C.Bmax)] = i;
                atomicAdd(&S.npush, 1u);
            }
        }
    }
    // this job-epoch's counters accumulate in registers (the digest is a sum mod
    // 2^64, order-free: one running sum per thread; counter c in lane c of warp 0)
    // and are added to the counters in memory at the epoch end / launch end
    // (flush_stats); S.npush (the coupled signal) is complete at the barrier below
    S.acc_dig[tid] += dig;
    TM.tick(11);
    if (tid < 12) {
        // hits/k indexed A=0, D=1, E=2; counter tiers S=0, E=1, D=2, A=3
        const uint32_t hA = S.hits[0], hD = S.hits[1], hE = S.hits[2];
        unsigned long long v = 0;
        switch (tid) {
            case 0: v = S.m - (k0 + k1 + k2); break;           // served[S]
            case 1: v = hE + k2; break;                        // served[E]
            case 2: v = hD + k1; break;                        // served[D]
            case 3: v = hA + k0; break;                        // served[A]
            case 5: v = k2; break;                             // subst[E]
            case 6: v = k1; break;                             // subst[D]
            case 7: v = k0; break;                             // subst[A]
            case 9: v = hE; break;                             // req_hits[E]
            case 10: v = hD; break;                            // req_hits[D]
            case 11: v = hA; break;                            // req_hits[A]
            default: break;
        }
        S.acc_cnt[tid] += v;
    }
    __syncthreads();
    if (tid < 3) { S.hits[tid] = 0; S.hits_loc[tid] = 0; }   // for the next round (barriers before next use)
    if (kSh && tid < kMaxShards * 3) (&S.hg[0][0])[tid] = 0;
    TM.tick(3);
}

// Add a job's register-held counters of epoch e to its counter row (every thread
// of the job CTA calls it: the digest is reduced per warp).
__device__ __forceinline__ void flush_stats(const Lay& L, const Cfg& C, JobSmem& S, uint32_t j, uint32_t e) {
    const uint32_t tid = threadIdx.x;
    unsigned long long* f = reinterpret_cast<unsigned long long*>(L.stats + (size_t)j * C.maxT + e);
    const unsigned long long d = warp_sum(S.acc_dig[tid]);
    if ((tid & 31) == 0 && d) atomicAdd(f + 12, d);
    if (tid < 12 && S.acc_cnt[tid]) atomicAdd(f + tid, S.acc_cnt[tid]);
    S.acc_dig[tid] = 0;
    if (tid < 12) S.acc_cnt[tid] = 0;
}

// ------------------------------------------------------------------ maintain (a7)
struct MaintSmem {
    uint32_t ne, kmax, kspec, deficit0, PS, prev_k;
    uint32_t size[4];        // tier sizes by tier code (E 1, D 2, A 3), live while running
    uint32_t def[4];         // round-start deficits cap_t - |t| of the tracked tiers
    uint32_t ne_t[4];        // evictions of this round by tier
    uint32_t ned;            // E/D evictions listed for the job CTAs
    uint32_t warm;           // cold start over (R-O24)
    uint32_t nadm;           // admission candidates of this round
    uint32_t ne_push, push_base;
    uint32_t add[kMaxJobs];
    uint32_t scan[33];
    uint32_t PSg;                        // sharded: the global storage pool at round start (C1)
    uint32_t pscnt[kMaxShards][3];       // sharded: every shard's storage pool ([g][0])
    uint32_t ne_loc, k_loc;              // sharded: evictions / refills inside this shard's range
    uint32_t relpk;                      // DSMEM signals: this round's refill split for the release word
};

// keyed refill ranks rho(u) over the storage pool as of round start (R-O8),
// located through the S-pool counts; the prefix s_pre must be loaded.
// kSh: the global rank's owning shard resolves it into every shard's mailbox,
// then every shard copies the complete list (C2 of the maintain CTA, slot J).
template <bool kSh>
__device__ void maint_refill_select(const Lay& L, const Cfg& C, MaintSmem& M, const uint32_t* s_pre, uint64_t r,
                                    uint32_t u0, uint32_t u1) {
    if (u1 <= u0) return;
    const uint64_t key = derive_key(L.seed, PUR_REFILL, 0, r, 0);
    const PermDomain dom = perm_domain(kSh ? M.PSg : M.PS);
    uint32_t* fill = L.fill_list + (size_t)(r & 1) * C.FL;
    for (uint32_t u = u0 + threadIdx.x; u < u1; u += blockDim.x) {
        const uint32_t rank = perm_apply(key, dom, u);
        if constexpr (kSh) {
            uint32_t local;
            if (shard_owner(C, M.pscnt, 0, rank, &local) == L.shard) {
                const uint32_t id = pool_select(L, C, 3 * C.J, T_S, 0, s_pre, local);
                const size_t at = C.mb_rf + (size_t)(r & 1) * C.FL + u;
                for (uint32_t g = 0; g < C.G; ++g) L.peer[g][at] = id;
            }
        } else {
            fill[u] = pool_select(L, C, 3 * C.J, T_S, 0, s_pre, rank);
        }
    }
    if constexpr (kSh) {
        shard_c2_sync(L, C, C.J, r);
        const uint32_t* in = L.mbox + C.mb_rf + (size_t)(r & 1) * C.FL;
        for (uint32_t u = u0 + threadIdx.x; u < u1; u += blockDim.x) fill[u] = ld_mbox(in + u);
    }
    __syncthreads();
}

// eviction of tracked entries (A, or every cached tier under evict_tiers = ALL)
// consumed by every active job (R-O5, R-O6, R-O21), refill from the storage pool
// as of round start, tier by tier A -> D -> E from one keyed rank stream (R-O8,
// R-O21), counts kept exact.
template <bool kSh, class TMr>
__device__ void maint_apply(const Lay& L, const Cfg& C, const Launch& P, MaintSmem& M, uint32_t* s_pre,
                            uint32_t* s_supS, uint64_t r, uint32_t active, uint32_t part_of_round, bool full_scan,
                            bool speculated, uint32_t ne_push, uint32_t push_base, TMr& TM,
                            uint32_t dfill = 0) {
    // dfill: shared address of the job CTAs' refill buffer (DSMEM signals), 0: none
    const uint32_t tid = threadIdx.x, T = blockDim.x;
    if (tid == 0) {
        M.ne = full_scan ? 0u : ne_push;
        M.ne_t[0] = M.ne_t[1] = M.ne_t[2] = M.ne_t[3] = 0;
        M.ned = 0;
        M.nadm = 0;
        M.ne_loc = 0;
        M.k_loc = 0;
    }
    __syncthreads();
    const bool admit = C.cold && !M.warm;
    uint32_t* fill_w = L.fill_list + (size_t)(r & 1) * C.FL;
    if (admit && active) {
        // cold start (R-O24): the storage fetches of the jobs of this round, in
        // ascending job order and slot order, first occurrence only, that were
        // storage-resident at round start (tiers read before any eviction applies)
        for (uint32_t m = part_of_round; m; m &= m - 1) {
            const uint32_t jj = __ffs(m) - 1;
            const uint32_t n = ldcg(L.fetch_n + jj);
            for (uint32_t base = 0; base < n; base += T) {
                const uint32_t u = base + tid;
                uint32_t i = 0;
                bool ok = false;
                if (u < n) {
                    i = ldcg(L.fetch + (size_t)jj * C.Bmax + u);
                    const uint32_t w = i >> 5, b = 1u << (i & 31);
                    const bool cached = ((ldcg(L.bm_a + w) | ldcg(L.bm_d + w) | ldcg(L.bm_e + w)) & b) != 0;
                    ok = !cached && !(atomicOr(L.claim + w, b) & b);     // ids within one job are distinct
                }
                uint32_t tot;
                const uint32_t ex = block_exclusive_scan(ok ? 1u : 0u, &tot, M.scan);
                if (ok) fill_w[M.nadm + ex] = i;
                __syncthreads();
                if (tid == 0) M.nadm += tot;
                __syncthreads();
            }
        }
        for (uint32_t u = tid; u < M.nadm; u += T) {                 // the scratch is zero between rounds
            const uint32_t i = fill_w[u];
            atomicAnd(L.claim + (i >> 5), ~(1u << (i & 31)));
        }
        __syncthreads();
    }
    if (full_scan) {
        // the active set changed (R-O6): every tracked entry is a candidate; the
        // consumer counts of the survivors are rebuilt for the new active set
        for (uint32_t w = tid; w < C.NW; w += T) {
            const uint32_t a_w = C.evict_all ? (ldcg(L.bm_a + w) | ldcg(L.bm_d + w) | ldcg(L.bm_e + w))
                                             : ldcg(L.bm_a + w);
            if (!a_w) continue;
            uint32_t ev = active ? a_w : 0u;                        // nothing is evicted with no active job
            for (uint32_t m = active; m; m &= m - 1) ev &= ldcg(L.cons + (size_t)(__ffs(m) - 1) * C.NW + w);
            if (ev) {
                const uint32_t base = atomicAdd(&M.ne, (uint32_t)__popc(ev));
                uint32_t c = 0;
                for (uint32_t v = ev; v; v &= v - 1) L.evict_list[base + c++] = w * 32u + (__ffs(v) - 1);
            }
            for (uint32_t v = a_w & ~ev; v; v &= v - 1) {
                const uint32_t bit = __ffs(v) - 1;
                uint32_t cnt = 0;
                for (uint32_t m = active; m; m &= m - 1)
                    cnt += (ldcg(L.cons + (size_t)(__ffs(m) - 1) * C.NW + w) >> bit) & 1u;
                L.cons_cnt[w * 32u + bit] = cnt;
            }
        }
        __syncthreads();
    }
    TM.tick(3);
    const uint32_t ne = M.ne;
    uint32_t k = active ? min(M.deficit0 + ne, kSh ? M.PSg : M.PS) : 0u;   // no refill with no active job
    if (admit) {
        k = active ? min(M.deficit0 + ne, M.nadm) : 0u;           // admissions instead of refills (R-O24)
    } else if (!speculated) {
        if (k) prefix_from_smem(C, s_supS, s_pre, M.scan);
        maint_refill_select<kSh>(L, C, M, s_pre, r, 0, k);
    } else if (k > M.kspec) {
        maint_refill_select<kSh>(L, C, M, s_pre, r, M.kspec, k);  // beyond the speculated ranks
    }
    const uint32_t spidx = 3 * C.J;
    const uint32_t ring = C.J * C.Bmax;
    uint32_t* ev_ed = L.ev_ed + (size_t)(r & 1) * max(C.cap_e + C.cap_d, 1u);
    for (uint32_t u = tid; u < ne; u += T) {
        const uint32_t i = full_scan ? L.evict_list[u] : ldcg(L.evict_push + (push_base + u) % ring);
        const uint32_t w = i >> 5, b = 1u << (i & 31);
        uint32_t t = T_A;
        if (C.evict_all) {
            t = (ldcg(L.bm_a + w) & b) ? T_A : ((ldcg(L.bm_d + w) & b) ? T_D : T_E);
            if (t != T_A) ev_ed[atomicAdd(&M.ned, 1u)] = i | (t == T_E ? 0x80000000u : 0u);
        }
        atomicAnd((t == T_A ? L.bm_a : (t == T_D ? L.bm_d : L.bm_e)) + w, ~b);
        if (C.evict_all) atomicAdd(&M.ne_t[t], 1u);      // A only: ne_t[A] = ne (set below)
        for (uint32_t a = 0; a < C.J; ++a) atomicAnd(L.cons + (size_t)a * C.NW + w, ~b);
        L.cons_cnt[i] = 0;
        if (count_add<kSh>(L, C, spidx, i, 1u, s_supS) && kSh) atomicAdd(&M.ne_loc, 1u);
    }
    if (!C.evict_all && tid == 0) M.ne_t[T_A] = ne;
    __syncthreads();
    // tier split of the k refill positions: A, then D, then E, each up to its deficit
    const uint32_t kA = min(M.def[T_A] + M.ne_t[T_A], k);
    const uint32_t kD = min(M.def[T_D] + M.ne_t[T_D], k - kA);
    // refills enter their tier with no consumers; each job CTA adds them to its
    // own pools before its next classification (R-O8)
    const uint32_t* fill = L.fill_list + (size_t)(r & 1) * C.FL;
    const bool push = dfill && k <= kFillBuf;       // the ids into every job CTA's shared memory
    for (uint32_t u = tid; u < k; u += T) {
        const uint32_t i = ldcg(fill + u);
        if (push)
            for (uint32_t jj = 0; jj < C.J; ++jj) dsmem_st32(dsmem_addr_raw(dfill + 4u * u, jj), i);
        uint32_t* bm = u < kA ? L.bm_a : (u < kA + kD ? L.bm_d : L.bm_e);
        atomicOr(bm + (i >> 5), 1u << (i & 31));
        if (count_add<kSh>(L, C, spidx, i, 0xffffffffu, s_supS) && kSh) atomicAdd(&M.k_loc, 1u);
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t* fn = L.fill_n + (r & 1) * 4;
        fn[0] = k; fn[1] = kA; fn[2] = kD;
        M.relpk = push ? (0x80000000u | k | (kA << 10) | (kD << 20)) : 0u;
        L.ev_ed_n[r & 1] = M.ned;
        M.PS = kSh ? M.PS + M.ne_loc - M.k_loc : M.PS + ne - k;   // storage pool and tier sizes live in
                                                                   // shared memory while running
        M.size[T_A] += kA - M.ne_t[T_A];
        M.size[T_D] += kD - M.ne_t[T_D];
        M.size[T_E] += (k - kA - kD) - M.ne_t[T_E];
        if (admit && M.size[T_A] == C.cap_a && M.size[T_D] == C.cap_d && M.size[T_E] == C.cap_e) {
            M.warm = 1;                                           // every tier full: the cold start ends
            *L.warm = 1;
        }
        *L.evicted += ne;
        *L.refilled += k;
        M.prev_k = k;
    }
    __syncthreads();
    TM.tick(4);
}

// Job j's pools follow round r's maintain (its CTA alone owns its pool counts;
// a recount at an epoch start covers everything instead): refills it has not
// seen join the pool of their tier (empty consumer sets), and under
// evict_tiers = ALL evicted E/D entries it has not seen leave its E/D pool (an
// evicted A entry was consumed by j, so it was in no A pool of j).
// relpk (DSMEM signals): bit 31 set -> the split k | kA << 10 | kD << 20 came with the
// release and the ids are in this CTA's shared buffer s_fill (pushed by maintain).
template <bool kSh>
__device__ void job_take_refills(const Lay& L, const Cfg& C, JobSmem& S, uint32_t j, uint64_t r, uint32_t* s_sup,
                                 uint32_t relpk = 0, const uint32_t* s_fill = nullptr) {
    const uint32_t* fn = L.fill_n + (r & 1) * 4;
    const uint32_t* fill = L.fill_list + (size_t)(r & 1) * C.FL;
    const bool local = (relpk >> 31) != 0;
    uint32_t i0, kf, kA, kD;
    if (local) {
        kf = relpk & 1023u; kA = (relpk >> 10) & 1023u; kD = (relpk >> 20) & 1023u;
        i0 = threadIdx.x < kf ? s_fill[threadIdx.x] : 0u;
    } else {
        // the first refill entry of this thread is loaded together with the counts (an
        // entry beyond kf is read but not used; the buffer holds FL entries)
        i0 = threadIdx.x < C.FL ? ldcg(fill + threadIdx.x) : 0u;
        kf = ldcg(fn); kA = ldcg(fn + 1); kD = ldcg(fn + 2);
    }
    const uint32_t* seen_j = L.seen + (size_t)j * C.NW;
    uint32_t addA = 0, addD = 0, addE = 0;   // registers (no indexed local array)
    for (uint32_t u = threadIdx.x; u < kf; u += blockDim.x) {
        const uint32_t i = u == threadIdx.x ? i0 : (local ? s_fill[u] : ldcg(fill + u));
        if (!((ldcg(seen_j + (i >> 5)) >> (i & 31)) & 1u)) {
            const uint32_t tt = u < kA ? 0u : (u < kA + kD ? 1u : 2u);
            if (count_add<kSh>(L, C, j * 3 + tt, i, 1u, s_sup + tt * C.NS)) {
                addA += tt == 0; addD += tt == 1; addE += tt == 2;
            }
        }
    }
    if (C.evict_all) {
        const uint32_t ne = ldcg(L.ev_ed_n + (r & 1));
        const uint32_t* ev = L.ev_ed + (size_t)(r & 1) * max(C.cap_e + C.cap_d, 1u);
        for (uint32_t u = threadIdx.x; u < ne; u += blockDim.x) {
            const uint32_t x = ldcg(ev + u), i = x & 0x7fffffffu;
            if (!((ldcg(seen_j + (i >> 5)) >> (i & 31)) & 1u)) {
                const uint32_t tt = (x >> 31) ? 2u : 1u;
                if (count_add<kSh>(L, C, j * 3 + tt, i, 0xffffffffu, s_sup + tt * C.NS)) {
                    addD -= tt == 1; addE -= tt == 2;   // wraps; the sums below are mod 2^32
                }
            }
        }
    }
    addA = __reduce_add_sync(0xffffffffu, addA);
    addD = __reduce_add_sync(0xffffffffu, addD);
    addE = __reduce_add_sync(0xffffffffu, addE);
    if ((threadIdx.x & 31) == 0) {
        if (addA) atomicAdd(&S.tot[0], addA);
        if (addD) atomicAdd(&S.tot[1], addD);
        if (addE) atomicAdd(&S.tot[2], addE);
    }
}

// ------------------------------------------------------------------ the persistent round kernel
// Grid: (J + 1) CTAs per replica; replicas are independent replays (their own
// workspace slice and seed) that share nothing but the launch.
__device__ __noinline__ void ring_generate(const Lay& L, const Cfg& C, uint32_t n_pairs);

// The schedule of rounds rs .. rs+K-1 advanced by warp 0 (lane = job) in
// closed form, as K calls of `advance` would: every active job of the subset
// consumes a batch per round (the last round of an epoch takes the rest),
// departs at the end of the round that completes its last epoch, and a pending
// job joins at the start of its arrival round (spans are cut at arrivals).
__device__ __noinline__ void skip_rounds_warp0(const Cfg& C, const Launch& P, uint64_t rs, uint32_t K, uint32_t* s_n,
                                               uint32_t* s_e, uint32_t& s_active, uint32_t& s_pending) {
    const uint32_t lane = threadIdx.x & 31u;
    while (K > 0) {
        uint64_t span = K;
        for (uint32_t m = s_pending; m; m &= m - 1) {
            const uint32_t jj = __ffs(m) - 1;
            if (P.arrival[jj] > rs) span = min(span, (uint64_t)P.arrival[jj] - rs);
        }
        const uint32_t part = s_active & P.subset;
        bool gone = false;
        if (lane < C.J && ((part >> lane) & 1u)) {
            const uint32_t B = C.batch[lane];
            uint32_t n = s_n[lane], e = s_e[lane];
            uint64_t R = span;
            while (R > 0) {
                const uint32_t r_ep = (C.N - n + B - 1) / B;    // rounds left in epoch e (the last may be short)
                if (R < r_ep) { n += (uint32_t)R * B; R = 0; }
                else {
                    R -= r_ep; n = 0; e += 1;
                    if (e == C.target[lane]) { gone = true; break; }   // departs after its last round
                }
            }
            s_n[lane] = n; s_e[lane] = e;
        }
        const uint32_t departed = __ballot_sync(0xffffffffu, gone);
        rs += span;
        K -= (uint32_t)span;
        if (lane == 0) {
            s_active &= ~departed;
            for (uint32_t m = s_pending; m; m &= m - 1) {       // arrivals at the start of round rs
                const uint32_t jj = __ffs(m) - 1;
                if (P.arrival[jj] <= rs) { s_active |= 1u << jj; s_pending &= ~(1u << jj); }
            }
        }
        __syncwarp();
    }
}

template <bool kTime, bool kCoupled, bool kShard>
__device__ __forceinline__ void ods_rounds_body(const Lays& LS, const Cfg& C, const Launch& P) {
    if (P.gen_ctas && blockIdx.x >= gridDim.x - P.gen_ctas) {     // the permutation-ring generator CTAs
        ring_generate(LS.r[0], C, P.gen_pairs);
        return;
    }
    extern __shared__ __align__(16) uint32_t smem[];
    __shared__ JobSmem S;
    __shared__ MaintSmem M;
    __shared__ uint32_t s_n[kMaxJobs], s_e[kMaxJobs], s_active, s_pending;
    __shared__ uint32_t s_part, s_departing;     // schedule of the current round (warp 0 computes it)
    const uint32_t tid = threadIdx.x;
    const uint32_t rep = blockIdx.x / (C.J + 1);
    const uint32_t cta = blockIdx.x - rep * (C.J + 1);
    const Lay& L = LS.r[rep];
    const bool is_maint = cta == C.J;
    const uint32_t j = cta;
    __shared__ PhaseTimer<kTime> TM;
    if (tid == 0) {
        TM.on = P.timing;
        TM.last = clock64();
        for (int k = 0; k < 16; ++k) TM.acc[k] = 0;
    }

    // shared memory carve: job CTA s_req | s_miss | s_sub | s_oid [Bmax] + s_pre [3][NS] + s_osrc [Bmax];
    // maintain CTA s_pre [NS]
    uint32_t* s_req = smem;
    uint32_t* s_miss = smem + C.Bmax;
    uint32_t* s_sub = smem + 2 * C.Bmax;
    uint32_t* s_oid = smem + 3 * C.Bmax;
    uint32_t* s_sup = smem + 4 * C.Bmax;                            // [3][NS] superblock counts (maint: S pool)
    uint32_t* s_pre = s_sup + 3 * C.NS;                             // [3][NS] prefixes
    const uint32_t o_win = (4 * C.Bmax + 6 * C.NS + 3) & ~3u;       // 16-B aligned (cp.async)
    uint32_t* s_win = smem + o_win;
    const uint32_t win = min(kWinMax, 2 * blockDim.x);              // prefetched walk window
    const uint32_t o_wseen = o_win + win;
    uint4* s_wseen = reinterpret_cast<uint4*>(smem + o_wseen);
    uint8_t* s_osrc = reinterpret_cast<uint8_t*>(smem + o_wseen + 4 * win);
    WalkPrefetch pfs;
    pfs.wseen = s_wseen;
    const WalkPrefetch* pf = P.mode == 0 ? &pfs : nullptr;
    // with no tracked tier (cap_A = 0 and evict_tiers = A) there is no cross-job
    // interaction at all (E and D are static, maintain has nothing to do): the job
    // CTAs run their rounds independently
    // (kCoupled == (C.cap_t > 0 || C.cold), chosen by the host: the uncoupled
    // instantiation contains no maintain, refill or signal code at all)
    constexpr bool coupled = kCoupled;
    if (is_maint && !coupled) return;
    // DSMEM signals (coupled, one cluster of J + 1 CTAs): s_sig in the maintain CTA counts
    // job phases | evictions pushed << 32; s_rel in each job CTA counts maintains applied
    __shared__ unsigned long long s_sig;
    __shared__ unsigned long long s_rel;           // rounds applied | refill split << 32
    __shared__ uint32_t s_fill[kFillBuf];          // the refill ids of the last maintain (job CTAs)
    __shared__ uint32_t s_relpk;
    const bool csig = coupled && !kShard && P.cluster != 0;
    if (csig) {
        if (tid == 0) { s_sig = 0; s_rel = 0; }
        __syncthreads();
        cluster_sync_all();              // every CTA's words are zero before any remote write
    }

    if (tid < kMaxJobs) { s_n[tid] = P.n0[tid]; s_e[tid] = P.e0[tid]; }
    if (tid == 0) {
        s_active = P.active0;
        s_pending = P.pending0;
        for (uint32_t m = s_pending; m; m &= m - 1) {         // arrivals of the first round (R-O23)
            const uint32_t jj = __ffs(m) - 1;
            if (P.arrival[jj] <= P.r0) { s_active |= 1u << jj; s_pending &= ~(1u << jj); }
        }
    }
    if (!is_maint && tid == 0) {
        const JobDev jd = L.jobs[j];
        S.cur_buf = jd.cur_buf; S.nxt_buf = jd.nxt_buf; S.cursor = jd.cursor;
        S.cur_len = jd.cur_len; S.nxt_len = jd.nxt_len; S.recount = jd.recount;
        S.late = jd.late; S.lc = jd.lc; S.lk = jd.lk;
        if (S.late && S.cur_buf == 0 && S.lc < C.nch)
            S.lcnt = ldcg(L.scnt + ((size_t)j * C.K + (P.e0[j] & (C.K - 1))) * C.nch + S.lc);
        S.fl = jd.fl; S.fc = jd.fc; S.fk = jd.fk; S.fpos = jd.fpos;
        // a job that has not arrived took no maintain results: its pools are rebuilt
        // from the bitmaps when it arrives (R-O23)
        if ((P.pending0 >> j) & 1u) S.recount = 1;
        S.perm_seen = 0;
        S.rep = rep;
        S.dens = 1.0f;
        S.pf_state = 0;
        S.npush = 0;
    }
    if (!is_maint) {
        S.acc_dig[tid] = 0;
        if (tid < 12) S.acc_cnt[tid] = 0;
        if (tid < kMaxShards * 3) { (&S.hg[0][0])[tid] = 0; (&S.sg[0][0])[tid] = 0; }
        if (tid == 0) S.c1 = 1;
        if (tid < 3) { S.hits[tid] = 0; S.hits_loc[tid] = 0; S.own[tid] = 0; }   // (shared memory is not zeroed
        if (tid < 3) S.tot[tid] = ldcg(L.cnt_tot + j * 3 + tid);                   //  at launch: initcheck-blind)
        for (uint32_t k = tid; k < 3 * C.NS; k += blockDim.x) s_sup[k] = ldcg(L.cnt_sup + (size_t)j * 3 * C.NS + k);
    } else {
        if (tid == 0) {
            M.prev_k = blockDim.x;
            M.PS = ldcg(L.cnt_tot + 3 * C.J);
            for (int t = 0; t < 4; ++t) M.size[t] = ldcg(L.tsize + t);
            M.warm = C.cold ? ldcg(L.warm) : 1u;
        }
        for (uint32_t k = tid; k < C.NS; k += blockDim.x) s_sup[k] = ldcg(L.cnt_sup + (size_t)3 * C.J * C.NS + k);
    }
    __syncthreads();

    auto need_of = [&](uint32_t jj) -> uint32_t { return min(C.batch[jj], C.N - s_n[jj]); };
    // data-independent schedule of the current round (R-O12): warp 0 computes it
    // (lane jj = job jj) after the launch setup and at every round end, every
    // thread reads it
    auto schedule_warp0 = [&]() {
        const uint32_t part = s_active & P.subset;
        const bool dep = tid < C.J && ((part >> tid) & 1u) && s_n[tid] + need_of(tid) == C.N &&
                         s_e[tid] + 1 == C.target[tid];
        const uint32_t departing = __ballot_sync(0xffffffffu, dep);
        if (tid == 0) { s_part = part; s_departing = departing; }
    };
    auto schedule = [&](uint32_t& part, uint32_t& departing) {
        part = s_part;
        departing = s_departing;
    };
    // end of round r: progress, departures, then the arrivals of round r + 1
    auto advance = [&](uint32_t part, uint32_t departing, uint64_t r) {
        __syncthreads();
        if (tid < 32) {
            if ((part >> tid) & 1u) {
                uint32_t n = s_n[tid] + need_of(tid);
                if (n == C.N) { n = 0; s_e[tid] += 1; }
                s_n[tid] = n;
            }
            if (tid == 0) {
                s_active &= ~departing;
                for (uint32_t m = s_pending; m; m &= m - 1) {
                    const uint32_t jj = __ffs(m) - 1;
                    if (P.arrival[jj] <= r + 1) { s_active |= 1u << jj; s_pending &= ~(1u << jj); }
                }
            }
            __syncwarp();
            schedule_warp0();
        }
        __syncthreads();
    };
    if (tid < 32) schedule_warp0();
    __syncthreads();

    // Coupled rounds synchronise through two one-directional signals (zeroed by
    // the host before every launch): L.bar[0] counts job phases completed, L.bar[1]
    // counts rounds whose maintain has been applied.  A job CTA only waits for
    // maintain(r-1) before classifying round r; the maintain CTA only waits for
    // the job phases of round r -- the next round's walk and speculative refill
    // overlap everything else.
    if (is_maint) {
        uint32_t expect = 0, push_total = 0;
        bool spec = false;
        // speculative refill ranks for the round about to be played: the storage
        // pool as of round start cannot change before this round's maintain
        // round-start deficits of the tracked tiers (A; D and E under evict_tiers = ALL)
        auto set_deficits = [&]() {
            M.def[T_S] = 0;
            M.def[T_A] = C.cap_a - M.size[T_A];
            const bool all = C.evict_all || (C.cold && !M.warm);        // cold start fills every tier
            M.def[T_D] = all ? C.cap_d - M.size[T_D] : 0u;
            M.def[T_E] = all ? C.cap_e - M.size[T_E] : 0u;
            M.deficit0 = M.def[T_A] + M.def[T_D] + M.def[T_E];
        };
        auto speculate = [&](uint64_t r, uint32_t part, uint32_t departing) -> bool {
            if (kShard) return false;            // sharded: refill ranks resolved after C1 of the storage pool
            const uint32_t active_after = s_active & ~departing;
            if (!(active_after && C.cap_t > 0) || departing || (C.cold && !M.warm)) return false;
            if (tid == 0) set_deficits();
            if (tid == 0) {
                uint32_t cand = 0;
                for (uint32_t m = part; m; m &= m - 1) cand += need_of(__ffs(m) - 1);
                M.kmax = min(M.deficit0 + cand, M.PS);
                M.kspec = min(M.kmax, min(blockDim.x, M.deficit0 + M.prev_k + 64u));
            }
            __syncthreads();
            if (M.kspec) prefix_from_smem(C, s_sup, s_pre, M.scan);
            TM.tick(0);
            maint_refill_select<false>(L, C, M, s_pre, r, 0, M.kspec);
            TM.tick(1);
            return true;
        };
        {
            uint32_t part, departing;
            schedule(part, departing);
            spec = speculate(P.r0, part, departing);
        }
        for (uint32_t rr = 0; rr < P.rounds; ++rr) {
            const uint64_t r = P.r0 + rr;
            uint32_t part, departing;
            schedule(part, departing);
            const uint32_t active_after = s_active & ~departing;
            expect += __popc(part);
            if (kShard && tid < 32) {        // C1 of the storage pool as of round start
                shard_c1(L, C, C.J, r, M.PS, 0u, 0u, M.pscnt);
                if (tid == 0) {
                    uint32_t t = 0;
                    for (uint32_t g = 0; g < C.G; ++g) t += M.pscnt[g][0];
                    M.PSg = t;
                }
            }
            if (tid == 0) {                  // job phases of round r done; evictions they pushed
                unsigned long long v;
                if (csig) { while ((uint32_t)(v = smem_ld_acquire64(&s_sig)) < expect) { } }
                else { while ((uint32_t)(v = ld_acquire64(L.bar)) < expect) { } }
                const uint32_t pushed = (uint32_t)(v >> 32);
                M.ne_push = pushed - push_total;
                M.push_base = push_total;
                push_total = pushed;
            }
            __syncthreads();
            TM.tick(2);
            // a departure rebuilds the consumer counts for the remaining jobs even when
            // none remains but arrivals are pending (no eviction, no refill then): a
            // job arriving later must not inherit counts of departed consumers (R-O23)
            if ((active_after || (departing && s_pending)) && (C.cap_t > 0 || (C.cold && !M.warm))) {
                if (!spec && tid == 0) set_deficits();
                __syncthreads();
                maint_apply<kShard>(L, C, P, M, s_pre, s_sup, r, active_after, part, departing != 0, spec,
                                    M.ne_push, M.push_base, TM,
                                    csig ? (uint32_t)__cvta_generic_to_shared(s_fill) : 0u);
            } else if (tid == 0) {          // nothing maintained: the job CTAs take an empty round
                uint32_t* fn = L.fill_n + (r & 1) * 4;
                fn[0] = fn[1] = fn[2] = 0;
                L.ev_ed_n[r & 1] = 0;
                M.relpk = 0x80000000u;       // (DSMEM signals: an empty split with the release)
            }
            __syncthreads();
            if (csig) {                     // release round r's tiers into every job CTA (lane = job)
                if (tid < C.J) dsmem_st_release64(dsmem_addr(&s_rel, tid), ((unsigned long long)M.relpk << 32) | (rr + 1));
            } else if (tid == 0) {
                __threadfence(); atomicExch(L.bar + 2, rr + 1);
            }
            TM.tick(5);
            advance(part, departing, r);
            spec = false;
            if (rr + 1 < P.rounds) {
                uint32_t part2, departing2;
                schedule(part2, departing2);
                spec = speculate(r + 1, part2, departing2);
            }
        }
    } else {
        // prologue: the walk of the first round
        if ((s_active & P.subset) >> j & 1u) {
            const uint32_t need = need_of(j);
            if (P.mode == 1) {
                for (uint32_t s = tid; s < need; s += blockDim.x)
                    s_req[s] = P.requested[(size_t)P.row_of_job[j] * P.out_stride + s];
                if (tid == 0) { S.need = need; S.wrap_slot = 0; }
                __syncthreads();
            } else if (S.late) {
                late_walk(L, C, S, s_req, j, s_e[j], need, s_win);
            } else {
                job_walk(L, C, S, s_req, j, s_e[j], need, TM, s_win, nullptr);
                if (P.rounds > 1)
                    prefetch_window(L, C, S, s_win, j, s_e[j], (uint32_t)(C.batch[j] / fmaxf(S.dens, 1.0f / 64.0f) * 1.15f) + 64);
            }
        }
        for (uint32_t rr = 0; rr < P.rounds; ++rr) {
            const uint64_t r = P.r0 + rr;
            uint32_t part, departing;
            schedule(part, departing);
            const uint32_t active_after = s_active & ~departing;
            if (coupled && rr > 0) {                   // maintain(r-1) applied?
                if (tid == 0) {
                    s_relpk = 0;
                    if (csig) {
                        unsigned long long v;
                        while ((uint32_t)(v = smem_ld_acquire64(&s_rel)) < rr) { }
                        if ((uint32_t)v == rr) s_relpk = (uint32_t)(v >> 32);
                    } else {
                        while (ld_acquire(L.bar + 2) < rr) { }
                    }
                }
                __syncthreads();
            }
            TM.tick(4);
            if (C.cold && tid == 0) S.warm = ldcg(L.warm);        // stable until this round's maintain
            if ((part >> j) & 1u) {
                if (S.recount) {
                    job_recount(L, C, j, s_sup, S.tot);
                    if (tid == 0) { S.recount = 0; S.c1 = 1; }     // (sharded: the recounted sizes are exchanged)
                    __syncthreads();
                }
                else if (coupled && rr > 0) { job_take_refills<kShard>(L, C, S, j, r - 1, s_sup, s_relpk, s_fill); __syncthreads(); }
                TM.tick(0);
                job_round<kShard>(L, C, P, S, s_req, s_miss, s_sub, s_oid, s_osrc, s_pre, j, r, s_e[j], s_n[j],
                          __popc(active_after), TM, s_win, s_wseen, s_sup);
                // a8 (R-O16): the epoch ends with this batch -> reset seen_j and the walk
                if (s_n[j] + S.need == C.N) {
                    flush_stats(L, C, S, j, s_e[j]);
                    uint4* sj = reinterpret_cast<uint4*>(L.seen + (size_t)j * C.NW);
                    for (uint32_t k = tid; k < C.NW / 4; k += blockDim.x) sj[k] = make_uint4(0, 0, 0, 0);
                    if (tid == 0) {
                        S.cur_buf = 0; S.nxt_buf = 1; S.cursor = 0; S.cur_len = C.N; S.nxt_len = 0;
                        S.recount = 1;
                        S.late = 0;
                    }
                    // epoch e is over: no read of its ring slot is in flight any more (the
                    // prefetched window copies of this CTA are drained), so the slot may be
                    // refilled with epoch e + K by the concurrent generator
                    cp_async_wait_all();
                    __syncthreads();
                    if (tid == 0) { __threadfence(); atomicExch(L.epoch_at + j, s_e[j] + 1); }
                    if (tid == 0) S.pf_state = 0;
                }
                if (coupled && tid == 0) {                 // job phase done (+ evictions pushed)
                    if (csig) {
                        dsmem_red_release_add64(dsmem_addr(&s_sig, C.J), 1ull + ((unsigned long long)S.npush << 32));
                    } else {
                        __threadfence();
                        atomicAdd(reinterpret_cast<unsigned long long*>(L.bar), 1ull + ((unsigned long long)S.npush << 32));
                    }
                    S.npush = 0;
                }
                TM.tick(0);
            }
            advance(part, departing, r);
            if (rr + 1 < P.rounds && ((s_active & P.subset) >> j & 1u)) {
                // (C.late: all pools of the job empty, not at an epoch start -> storage-list walk)
                // (sharded: the global pool sizes after this round's hits less its substitutes)
                const bool empty = kShard ? ((S.glob[0] - S.k[0]) | (S.glob[1] - S.k[1]) | (S.glob[2] - S.k[2])) == 0u
                                          : (S.tot[0] | S.tot[1] | S.tot[2]) == 0u;
                if (C.late && !S.late && !S.recount && empty)
                    enter_late(L, C, S, j, s_e[j]);
#if SENECA_LATE_BULK
                // late bulk: rounds rr+1 .. rr+K of an uncoupled job in late mode, all
                // but the last round of its epoch and of the launch, decided in one
                // pass; the schedule (progress of every job, departures, arrivals)
                // advances round by round in warp 0 as `advance` would
                if (!coupled && S.late && P.mode == 0 && !P.out_ids) {
                    const uint32_t B = C.batch[j], left = (C.N - s_n[j] + B - 1) / B;   // rounds of epoch s_e[j] left
                    const uint32_t lrest = P.rounds - (rr + 1);                        // rounds of the launch left
                    const uint32_t K = min(left, lrest) - 1;
                    if (left >= 2 && lrest >= 2 && K >= kBulkMin) {
                        late_bulk(L, C, P, S, j, s_e[j], s_n[j], K * B);
                        if (tid < 32) skip_rounds_warp0(C, P, P.r0 + rr + 1, K, s_n, s_e, s_active, s_pending);
                        __syncwarp();
                        if (tid < 32) schedule_warp0();
                        __syncthreads();
                        rr += K;
                        TM.tick(6);
                        TM.count(15, K);                 // rounds decided in bulk
                    }
                }
#endif
                if (S.late) {
                    late_walk(L, C, S, s_req, j, s_e[j], need_of(j), s_win);
                    TM.tick(13);
                    if (rr + 2 < P.rounds) {              // the round after: prefetch its requests
                        const uint32_t n2 = s_n[j] + need_of(j);
                        if (n2 < C.N) late_prefetch(L, C, S, s_win, j, s_e[j], min(C.batch[j], C.N - n2));
                    }
                    TM.tick(14);
                } else {
                    job_walk(L, C, S, s_req, j, s_e[j], need_of(j), TM, s_win, pf);   // next request
                    TM.tick(13);
                    if (rr + 2 < P.rounds)
                        prefetch_window(L, C, S, s_win, j, s_e[j], (uint32_t)(C.batch[j] / fmaxf(S.dens, 1.0f / 64.0f) * 1.15f) + 64);
                    TM.tick(14);
                }
            }
            TM.tick(5);
        }
    }
    // epilogue: the current epoch's counters, the last round's refills into this
    // job's A pool; persist the totals
    if (!is_maint) {
        flush_stats(L, C, S, j, s_e[j]);
        if (S.late) catch_up_seen(L, C, S, j, s_e[j]);
        if (coupled && P.rounds > 0 && (s_active >> j & 1u)) {
            if (tid == 0) {
                s_relpk = 0;
                if (csig) {
                    unsigned long long v;
                    while ((uint32_t)(v = smem_ld_acquire64(&s_rel)) < P.rounds) { }
                    if ((uint32_t)v == P.rounds) s_relpk = (uint32_t)(v >> 32);
                } else {
                    while (ld_acquire(L.bar + 2) < P.rounds) { }
                }
            }
            __syncthreads();
            if (!S.recount) job_take_refills<kShard>(L, C, S, j, P.r0 + P.rounds - 1, s_sup, s_relpk, s_fill);
            __syncthreads();
        }
        if (tid < 3) L.cnt_tot[j * 3 + tid] = S.tot[tid];
        for (uint32_t k = tid; k < 3 * C.NS; k += blockDim.x) L.cnt_sup[(size_t)j * 3 * C.NS + k] = s_sup[k];
    } else {
        if (tid == 0) { L.cnt_tot[3 * C.J] = M.PS; for (int t = 0; t < 4; ++t) L.tsize[t] = M.size[t]; }
        for (uint32_t k = tid; k < C.NS; k += blockDim.x) L.cnt_sup[(size_t)3 * C.J * C.NS + k] = s_sup[k];
    }
    cp_async_wait_all();
    // persist the walk state
    if (!is_maint && tid == 0) {
        JobDev& jd = L.jobs[j];
        jd.cur_buf = S.cur_buf; jd.nxt_buf = S.nxt_buf; jd.cursor = S.cursor;
        jd.cur_len = S.cur_len; jd.nxt_len = S.nxt_len; jd.recount = S.recount;
        jd.late = S.late; jd.lc = S.lc; jd.lk = S.lk;
        jd.fl = S.fl; jd.fc = S.fc; jd.fk = S.fk; jd.fpos = S.fpos;
    }
    if (kTime && P.timing && tid == 0 && (is_maint || cta == 0)) {
        const uint32_t base = is_maint ? 16 : 0;
        for (int k = 0; k < 16; ++k) atomicAdd(L.phase + base + k, TM.acc[k]);
    }
    if (csig) cluster_sync_all();        // no CTA leaves while a peer may still write its signal word
}

// Two instantiations: 512 threads, one CTA per SM (a single replay: the most
// memory parallelism per job), and 256 threads, two CTAs per SM (replicas that
// would not fit one per SM: twice the independent replays per SM).
// (kTime: the phase-counter build, launched only under seneca_profile bit 1;
// kCoupled: a tracked tier or a cold start, i.e. jobs interact through maintain.)
template <bool kTime, bool kCoupled>
__global__ void __launch_bounds__(kThreads, 1)
ods_rounds(const __grid_constant__ Lays LS, const __grid_constant__ Cfg C, const __grid_constant__ Launch P) {
    ods_rounds_body<kTime, kCoupled, false>(LS, C, P);
}

template <bool kTime, bool kCoupled>
__global__ void __launch_bounds__(kThreads / 2, 2)
ods_rounds_x2(const __grid_constant__ Lays LS, const __grid_constant__ Cfg C, const __grid_constant__ Launch P) {
    ods_rounds_body<kTime, kCoupled, false>(LS, C, P);
}

// One shard of a sample-ID-range-sharded replay per (J + 1)-CTA group (SURVEY
// §8(e)): the slices of one launch are the shards of ONE replay (emulation on
// one device), or the launch is this device's shard and its peers' mailboxes
// are mapped peer memory.
template <bool kTime, bool kCoupled>
__global__ void __launch_bounds__(kThreads, 1)
ods_rounds_sh(const __grid_constant__ Lays LS, const __grid_constant__ Cfg C, const __grid_constant__ Launch P) {
    ods_rounds_body<kTime, kCoupled, true>(LS, C, P);
}

// 256 threads, one CTA per SM: independent jobs whose longest chain of rounds
// has batches of <= 256 (each round is shorter with fewer, fuller warps)
template <bool kTime, bool kCoupled>
__global__ void __launch_bounds__(kThreads / 2, 1)
ods_rounds_half(const __grid_constant__ Lays LS, const __grid_constant__ Cfg C, const __grid_constant__ Launch P) {
    ods_rounds_body<kTime, kCoupled, false>(LS, C, P);
}

// the round kernel for (variant: 0 512 threads, 1 256 threads two CTAs per SM,
// 2 256 threads one CTA per SM; phase counters; coupled)
const void* round_kernel(int variant, bool timed, bool coupled) {
    if (variant == 3) {
        if (coupled) return timed ? (const void*)ods_rounds_sh<true, true> : (const void*)ods_rounds_sh<false, true>;
        return timed ? (const void*)ods_rounds_sh<true, false> : (const void*)ods_rounds_sh<false, false>;
    }
    if (variant == 2) {
        if (coupled) return timed ? (const void*)ods_rounds_half<true, true> : (const void*)ods_rounds_half<false, true>;
        return timed ? (const void*)ods_rounds_half<true, false> : (const void*)ods_rounds_half<false, false>;
    }
    if (variant == 1) {
        if (coupled) return timed ? (const void*)ods_rounds_x2<true, true> : (const void*)ods_rounds_x2<false, true>;
        return timed ? (const void*)ods_rounds_x2<true, false> : (const void*)ods_rounds_x2<false, false>;
    }
    if (coupled) return timed ? (const void*)ods_rounds<true, true> : (const void*)ods_rounds<false, true>;
    return timed ? (const void*)ods_rounds<true, false> : (const void*)ods_rounds<false, false>;
}

// ------------------------------------------------------------------ one-off kernels
// The (job, epoch) pairs one generator launch fills, in the order given
// (epoch-major, so the earliest needed permutations complete first).
struct PermWork {
    uint32_t n;
    uint32_t j[2 * kMaxJobs], e[2 * kMaxJobs];
};

// The epochs a single-replica launch's jobs enter during the launch, in the
// order their ring slots free (refilled by the launch's generator CTAs).
constexpr uint32_t kRingPairs = 1024;
struct PermRing {
    uint32_t n;
    uint32_t j[kRingPairs], e[kRingPairs];
};

// One 16 K-position chunk [lo, hi) of pi_j,e into ring slot e % K; with
// Cfg.late also the chunk's storage-list segment (its storage-resident ids in
// position order, by a block scan per 512 positions), their count, and a bit per
// position (storage-resident) for locating a cursor in the segments.  Every
// thread of the CTA calls it (blockDim a multiple of 32, lo a multiple of 16 K).
__device__ void gen_chunk(const Lay& L, const Cfg& C, uint32_t j, uint32_t e, uint32_t part, uint64_t key,
                          const PermDomain& dom, uint32_t* s_scan /* 33 u32 */) {
    const uint32_t lo = part * kGenChunk, hi = min(lo + kGenChunk, C.N);
    const size_t slot = (size_t)j * C.K + (e & (C.K - 1));
    uint32_t* out = L.perms + slot * C.Nrow;
    if (!C.late) {
        for (uint32_t pos = lo + threadIdx.x; pos < hi; pos += blockDim.x) out[pos] = perm_apply(key, dom, pos);
        return;
    }
    uint32_t* seg = L.slist + slot * C.Nrow + lo;
    uint32_t* cb = L.cbits + slot * (C.Nrow / 32);
    uint32_t run = 0;
    for (uint32_t base = lo; base < hi; base += blockDim.x) {
        const uint32_t pos = base + threadIdx.x;
        bool st = false;
        uint32_t id = 0;
        if (pos < hi) {
            id = perm_apply(key, dom, pos);
            out[pos] = id;
            const uint32_t w = id >> 5;
            const uint32_t cached = (C.cap_e ? ldcg(L.bm_e + w) : 0u) | (C.cap_d ? ldcg(L.bm_d + w) : 0u);
            st = !((cached >> (id & 31)) & 1u);
        }
        const uint32_t ball = __ballot_sync(0xffffffffu, st);
        const uint32_t wbase = base + (threadIdx.x & ~31u);
        if ((threadIdx.x & 31) == 0 && wbase < hi) cb[wbase >> 5] = ball;
        uint32_t tot;
        const uint32_t ex = block_flag_scan(st, false, &tot, s_scan);
        if (st) seg[run + ex] = id;
        run += tot;
    }
    if (threadIdx.x == 0) L.scnt[slot * C.nch + part] = run;
}

// pi_j,e for the listed (job, epoch) pairs, in chunks, into ring slot e % K; the
// CTA finishing the last chunk of (j, e) publishes perm_ready[j][e] (release).
__global__ void ods_perm_all(const __grid_constant__ Lays LS, const __grid_constant__ Cfg C,
                             const __grid_constant__ PermWork W, uint32_t chunk) {
    const Lay& L = LS.r[blockIdx.y];
    (void)chunk;
    const uint32_t per = C.nch;
    const uint64_t total = (uint64_t)W.n * per;
    const PermDomain dom = perm_domain(C.N);
    __shared__ uint32_t s_last, s_scan[33];
    for (uint64_t c = blockIdx.x; c < total; c += gridDim.x) {
        const uint32_t pair = (uint32_t)(c / per);
        const uint32_t e = W.e[pair], j = W.j[pair];
        const uint32_t part = (uint32_t)(c % per);
        const uint64_t key = derive_key(L.seed, PUR_REQ, j, e, 0);
        const uint32_t lo = part * kGenChunk, hi = min(lo + kGenChunk, C.N);
        gen_chunk(L, C, j, e, part, key, dom, s_scan);
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            const uint32_t old = atomicAdd(L.perm_done + (size_t)j * C.maxT + e, hi - lo);
            s_last = old + (hi - lo) == C.N;
            if (s_last) {
                __threadfence();
                atomicExch(L.perm_ready + (size_t)j * C.maxT + e, 1u);
            }
        }
        __syncthreads();
    }
}

// The ring generator CTAs of a single-replica round launch (the trailing
// P.gen_ctas CTAs of the cooperative grid, so they are co-resident with the job
// CTAs by construction -- no reliance on two concurrent kernels, which a
// serialising profiler would deadlock): slot e % K is refilled with epoch e of
// job j as soon as job j has started epoch e - K + 1 (epoch_at, released by the
// job CTA at its epoch reset), so no launch has to stop at an epoch boundary.
// Work items (pair, 16 K-position chunk) are taken in list order (pairs sorted
// by the round their slot frees); a waiting CTA sleeps.
__device__ __noinline__ void ring_generate(const Lay& L, const Cfg& C, uint32_t n_pairs) {
    const uint32_t per = C.nch;
    const uint32_t total = n_pairs * per;
    const PermDomain dom = perm_domain(C.N);
    __shared__ uint32_t s_item, s_last, s_scan[33];
    for (;;) {
        if (threadIdx.x == 0) s_item = atomicAdd(L.gen_next, 1u);
        __syncthreads();
        const uint32_t item = s_item;
        if (item >= total) break;
        const uint32_t pair = item / per, part = item % per;
        const uint32_t pj = ldcg(L.ring_pairs + pair);
        const uint32_t e = pj & 0xffffffu, j = pj >> 24;
        if (threadIdx.x == 0)
            while (ld_acquire(L.epoch_at + j) + C.K - 1 < e) __nanosleep(1000);
        __syncthreads();
        const uint64_t key = derive_key(L.seed, PUR_REQ, j, e, 0);
        const uint32_t lo = part * kGenChunk, hi = min(lo + kGenChunk, C.N);
        gen_chunk(L, C, j, e, part, key, dom, s_scan);
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            const uint32_t old = atomicAdd(L.perm_done + (size_t)j * C.maxT + e, hi - lo);
            s_last = old + (hi - lo) == C.N;
            if (s_last) {
                __threadfence();
                atomicExch(L.perm_ready + (size_t)j * C.maxT + e, 1u);
            }
        }
        __syncthreads();
    }
}

// warm start (R-O9): positions [0,cap_A) -> A, next cap_D -> D, next cap_E -> E
__global__ void ods_init_tiers(const __grid_constant__ Lays LS, const __grid_constant__ Cfg C, uint32_t cap_e,
                               uint32_t cap_d) {
    const Lay& L = LS.r[blockIdx.y];
    const uint64_t key = derive_key(L.seed, PUR_INIT, 0, 0, 0);
    const PermDomain dom = perm_domain(C.N);
    const uint32_t total = C.cold ? 0u : C.cap_a + cap_d + cap_e;    // cold start: empty tiers (R-O24)
    for (uint32_t pos = blockIdx.x * blockDim.x + threadIdx.x; pos < total; pos += gridDim.x * blockDim.x) {
        const uint32_t i = perm_apply(key, dom, pos);
        uint32_t* bm = pos < C.cap_a ? L.bm_a : (pos < C.cap_a + cap_d ? L.bm_d : L.bm_e);
        atomicOr(bm + (i >> 5), 1u << (i & 31));
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        L.tsize[T_S] = 0;
        L.tsize[T_E] = C.cold ? 0u : cap_e; L.tsize[T_D] = C.cold ? 0u : cap_d; L.tsize[T_A] = C.cold ? 0u : C.cap_a;
    }
}

// Pool counts of every job and of the storage pool (init): the bitmap pass.
// One warp per 4096-id superblock, one 128-id block (a 16-B vector of each
// bitmap) per lane: the residency vectors are read once, then each job's seen
// and consumer vectors (every bitmap byte read exactly once, 512 contiguous
// bytes per warp and bitmap), and the 3J + 1 pool counts are formed in
// registers: block count = 4 popcounts, 4 lanes' counts packed into one word
// of the superblock's 32-B count row, the superblock total by a warp sum.
// blockIdx.z is the job: few registers, many warps in flight (memory-level
// parallelism); the residency vectors are re-read per job (from L2).
constexpr uint32_t kRecountWarps = 8;        // superblocks per CTA of the init bitmap pass
__global__ void __launch_bounds__(kRecountWarps * 32)
ods_recount_all(const __grid_constant__ Lays LS, const __grid_constant__ Cfg C) {
    const Lay& L = LS.r[blockIdx.y];
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t sblk = blockIdx.x * kRecountWarps + (threadIdx.x >> 5);   // grid (NS/8, replicas, J)
    __shared__ uint32_t s_tot[4];                                  // this CTA's pool totals: S, A, D, E
    if (threadIdx.x < 4) s_tot[threadIdx.x] = 0;
    __syncthreads();
    const bool live = sblk >= L.sb_lo && sblk < L.sb_hi;      // this shard's superblocks (all: unsharded)
    const uint32_t blk = sblk * 32 + lane, w0 = blk * kWordsPerBlock;
    const uint4 z4 = make_uint4(0, 0, 0, 0);
    const uint4 a = live ? __ldcs(reinterpret_cast<const uint4*>(L.bm_a + w0)) : z4;
    const uint4 d = live ? __ldcs(reinterpret_cast<const uint4*>(L.bm_d + w0)) : z4;
    const uint4 e = live ? __ldcs(reinterpret_cast<const uint4*>(L.bm_e + w0)) : z4;
    auto emit = [&](uint32_t pool, uint32_t slot, uint4 x) {
        const uint32_t c = __popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w);   // <= 128: one byte
        const uint32_t c1 = __shfl_down_sync(0xffffffffu, c, 1);
        const uint32_t c2 = __shfl_down_sync(0xffffffffu, c, 2);
        const uint32_t c3 = __shfl_down_sync(0xffffffffu, c, 3);
        if (live && (lane & 3) == 0)
            L.cnt8[(size_t)pool * (C.NBp >> 2) + (blk >> 2)] = c | (c1 << 8) | (c2 << 16) | (c3 << 24);
        const uint32_t t = warp_sum(c);
        if (live && lane == 0) {
            L.cnt_sup[(size_t)pool * C.NS + sblk] = t;
            if (t) atomicAdd(&s_tot[slot], t);
        }
    };
    const uint32_t j = blockIdx.z;
    const uint4 S_ = live ? __ldcs(reinterpret_cast<const uint4*>(L.seen + (size_t)j * C.NW + w0)) : z4;
    const uint4 Cv = live ? __ldcs(reinterpret_cast<const uint4*>(L.cons + (size_t)j * C.NW + w0)) : z4;
    if (j == 0)
        emit(3 * C.J, 0, make_uint4(~(a.x | d.x | e.x) & valid_mask(C, w0 + 0), ~(a.y | d.y | e.y) & valid_mask(C, w0 + 1),
                                    ~(a.z | d.z | e.z) & valid_mask(C, w0 + 2), ~(a.w | d.w | e.w) & valid_mask(C, w0 + 3)));
    emit(j * 3 + 0, 1, make_uint4(a.x & ~S_.x & ~Cv.x, a.y & ~S_.y & ~Cv.y, a.z & ~S_.z & ~Cv.z, a.w & ~S_.w & ~Cv.w));
    emit(j * 3 + 1, 2, make_uint4(d.x & ~S_.x, d.y & ~S_.y, d.z & ~S_.z, d.w & ~S_.w));
    emit(j * 3 + 2, 3, make_uint4(e.x & ~S_.x, e.y & ~S_.y, e.z & ~S_.z, e.w & ~S_.w));
    __syncthreads();                                                // one global add per pool per CTA
    if (threadIdx.x < 4 && s_tot[threadIdx.x])
        atomicAdd(L.cnt_tot + (threadIdx.x == 0 ? 3 * C.J : j * 3 + threadIdx.x - 1), s_tot[threadIdx.x]);
}

__global__ void ods_init_jobs(const __grid_constant__ Lays LS, const __grid_constant__ Cfg C) {
    const Lay& L = LS.r[blockIdx.x];
    const uint32_t j = threadIdx.x;
    if (j < C.J) {
        JobDev& jd = L.jobs[j];
        jd.cur_buf = 0; jd.nxt_buf = 1; jd.cursor = 0; jd.cur_len = C.N; jd.nxt_len = 0; jd.recount = 0;
        jd.late = 0; jd.lc = 0; jd.lk = 0;
        jd.fl = 0; jd.fc = 0; jd.fk = 0; jd.fpos = 0;
    }
}

// caller-supplied requests (mode 1): range, duplicates within the row, seen
__global__ void ods_validate_requests(const __grid_constant__ Lays LS, const __grid_constant__ Cfg C,
                                      const __grid_constant__ Launch P) {
    const Lay& L = LS.r[0];                     // caller-supplied requests: one replica
    extern __shared__ uint32_t s_row[];
    uint32_t x = 0;
    uint32_t j = 0xffffffffu;
    for (uint32_t m = P.subset; m; m &= m - 1) {
        if (x == blockIdx.x) { j = __ffs(m) - 1; break; }
        ++x;
    }
    if (j == 0xffffffffu) return;
    const uint32_t need = min(C.batch[j], C.N - P.n0[j]);
    const uint32_t* R = P.requested + (size_t)P.row_of_job[j] * P.out_stride;
    for (uint32_t s = threadIdx.x; s < need; s += blockDim.x) s_row[s] = R[s];
    __syncthreads();
    for (uint32_t s = threadIdx.x; s < need; s += blockDim.x) {
        const uint32_t i = s_row[s];
        if (i >= C.N) { atomicOr(L.verr, 1u); continue; }
        if (L.seen[(size_t)j * C.NW + (i >> 5)] & (1u << (i & 31))) atomicOr(L.verr, 1u);
        for (uint32_t s2 = 0; s2 < s; ++s2)
            if (s_row[s2] == i) { atomicOr(L.verr, 1u); break; }
    }
}

inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// Control block at the start of the workspace, one 64-B slot per replica:
// bar[4] at +0, err at +16, verr at +20.  Kept contiguous (not inside the
// replica slices) so the per-launch signal reset and the status read are one
// small strided copy whatever the replica slice size.
constexpr size_t kCtlBytes = 64;
inline size_t ctl_bytes(uint32_t R) { return align256((size_t)R * kCtlBytes); }

enum KernelClass { K_ROUNDS = 0, K_PERM, K_RECOUNT, K_INIT, K_VALIDATE, K_NCLASS };
const char* const kKernelNames[K_NCLASS] = {"ods_rounds", "ods_perm_all", "ods_recount_all", "ods_init_tiers",
                                            "ods_validate_requests"};

}  // namespace
}  // namespace seneca

// ===========================================================================
// host side
// ===========================================================================
using namespace seneca;

struct seneca_ctx {
    Cfg C;
    Lay L;                 // replica 0
    Lays LS;               // every replica
    uint32_t R;            // replicas
    size_t rep_stride;     // workspace bytes per replica
    char* ctl;             // control block (kCtlBytes per replica) at the workspace start
    uint32_t mode;
    uint64_t cap_e, cap_d;
    uint64_t e[kMaxJobs], n[kMaxJobs];
    uint32_t active;
    uint32_t pending;              // jobs that have not arrived (R-O23)
    uint64_t arrival[kMaxJobs];
    uint64_t r;
    uint64_t gen_hi[kMaxJobs];     // permutations of epochs < gen_hi[j] have been generated (ring, C.K slots)
    uint32_t shard_mode;           // sharded (C.G > 1): 0 all shards in this context, 1 one shard
    uint32_t gen_ctas;             // ring generator CTAs appended to single-replica launches (0: none)
    uint32_t ring_host[1024];      // staging of the generator work list (cudaMemcpyAsync from pageable memory)
    bool attached;                 // shard_mode 1: the peers' mailboxes are known
    uint64_t launches;
    uint64_t klaunch[K_NCLASS];
    double kms[K_NCLASS];
    uint64_t ksampled[K_NCLASS];
    uint32_t profiling;
    size_t round_smem;
    const void* round_fn;      // ods_rounds (512 threads, 1 CTA / SM) or ods_rounds_x2 (256, 2 / SM)
    const void* round_fn_timed; // the same with the phase counters compiled in (seneca_profile bit 1)
    uint32_t round_threads;
    int device;
    cudaStream_t side;
    cudaEvent_t ev_init;
    cudaEvent_t ev_a, ev_b;
};

namespace {

seneca_status check_cfg(const seneca_cache_config* cfg) {
    if (!cfg) { set_error("NULL config"); return SENECA_EINVAL; }
    if (cfg->n_total == 0 || cfg->n_total >= (1ull << 31)) { set_error("n_total must be in [1, 2^31)"); return SENECA_EINVAL; }
    if (cfg->n_jobs == 0 || cfg->n_jobs > kMaxJobs) { set_error("n_jobs must be in [1, 32]"); return SENECA_EINVAL; }
    if (cfg->request_mode > 1) { set_error("request_mode must be 0 or 1"); return SENECA_EINVAL; }
    if (!cfg->batch_size || !cfg->target_epochs) { set_error("NULL batch_size/target_epochs"); return SENECA_EINVAL; }
    for (uint32_t j = 0; j < cfg->n_jobs; ++j) {
        if (cfg->batch_size[j] == 0 || cfg->batch_size[j] > kMaxBatch) {
            set_error("batch_size[%u] must be in [1, %u]", j, kMaxBatch); return SENECA_EINVAL;
        }
        if (cfg->target_epochs[j] == 0 || cfg->target_epochs[j] > 100000) {
            set_error("target_epochs[%u] must be in [1, 1e5]", j); return SENECA_EINVAL;
        }
    }
    if (cfg->replicas > kMaxReplicas) { set_error("replicas must be <= %u", kMaxReplicas); return SENECA_EINVAL; }
    if (cfg->evict_tiers > 1) { set_error("evict_tiers must be 0 (A only) or 1 (all)"); return SENECA_EINVAL; }
    if (cfg->sampler > 1) { set_error("sampler must be 0 (ODS) or 1 (uniform no-evict baseline)"); return SENECA_EINVAL; }
    if (cfg->cold_start > 1) { set_error("cold_start must be 0 or 1"); return SENECA_EINVAL; }
    if (cfg->replicas > 1 && cfg->request_mode != 0) {
        set_error("caller-supplied requests (request_mode 1) need replicas <= 1"); return SENECA_EINVAL;
    }
    if (cfg->shards > kMaxShards) { set_error("shards must be <= %u", kMaxShards); return SENECA_EINVAL; }
    if (cfg->shards > 1) {
        if (cfg->shard_mode > 1) { set_error("shard_mode must be 0 (all shards here) or 1 (one)"); return SENECA_EINVAL; }
        if (cfg->shard_mode == 1 && cfg->shard_rank >= cfg->shards) {
            set_error("shard_rank must be < shards"); return SENECA_EINVAL;
        }
        if (cfg->replicas > 1 || cfg->request_mode != 0) {
            set_error("a sharded replay needs replicas <= 1 and request_mode 0"); return SENECA_EINVAL;
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
    size_t off[48];
    size_t total;          // one replica
    uint32_t R;
};

Sizes compute_sizes(const seneca_cache_config* cfg) {
    Sizes z{};
    Cfg& C = z.C;
    C.N = (uint32_t)cfg->n_total;
    C.NB = (C.N + 127) / 128;
    C.NS = (C.NB + 31) / 32;
    C.NBp = C.NS * 32;
    C.NW = C.NBp * kWordsPerBlock;          // bitmaps padded to whole superblocks
    C.J = cfg->n_jobs;
    C.Bmax = 0;
    C.maxT = 0;
    for (uint32_t j = 0; j < C.J; ++j) {
        C.Bmax = std::max(C.Bmax, cfg->batch_size[j]);
        C.maxT = std::max(C.maxT, cfg->target_epochs[j]);
        C.batch[j] = cfg->batch_size[j];
        C.target[j] = cfg->target_epochs[j];
    }
    C.K = std::min<uint32_t>(C.maxT, 2);
    C.cap_a = (uint32_t)cfg->cap_a;
    C.cap_d = (uint32_t)cfg->cap_d;
    C.cap_e = (uint32_t)cfg->cap_e;
    C.evict_all = cfg->evict_tiers;
    C.baseline = cfg->sampler;
    C.cold = cfg->cold_start ? 1u : 0u;
    C.cap_t = C.baseline ? 0u : (C.evict_all ? C.cap_a + C.cap_d + C.cap_e : C.cap_a);
    C.seed = cfg->seed;
    C.Nrow = (C.N + 63) & ~63u;
    C.FL = (uint32_t)(std::max<size_t>(C.cap_t, 1) + (size_t)C.J * C.Bmax);
    C.nch = (C.N + kGenChunk - 1) / kGenChunk;
    C.late = (SENECA_LATE_WALK && cfg->cap_a == 0 && !cfg->evict_tiers && !cfg->cold_start && !cfg->sampler &&
              cfg->request_mode == 0 && cfg->replicas <= 1) ? 1u : 0u;
    C.G = cfg->shards > 1 ? cfg->shards : 1u;
    C.xsys = C.G > 1 && cfg->shard_mode == 1 ? 1u : 0u;
    C.mb_c1 = 0;
    C.mb_c2 = C.mb_c1 + 2 * (C.J + 1) * C.G * 4;
    C.mb_rf = C.mb_c2 + 2 * C.J * C.Bmax;
    C.mb_fl = C.mb_rf + (C.G > 1 ? 2 * C.FL : 0u);
    const size_t mbox_u32 = C.G > 1 ? (size_t)C.mb_fl + 2 * (C.J + 1) * C.G : 1;
    const size_t W = (size_t)C.NW * 4, P = 3 * (size_t)C.J + 1;
    const size_t capl = std::max<size_t>(C.cap_t, 1) * 4;
    const size_t edl = std::max<size_t>(C.cap_e + C.cap_d, 1) * 4;
    const size_t sz[] = {
        W, W, W,                                            // 0-2 bm_e, bm_d, bm_a
        W * C.J, W * C.J,                                   // 3-4 seen, cons
        (size_t)C.Nrow * 4,                                 // 5 cons_cnt
        P * C.NBp, P * C.NS * 4, P * 4,                     // 6-8 counts
        16,                                                 // 9 tsize
        (size_t)C.J * C.K * C.Nrow * 4,                     // 10 perms (ring of K epochs per job)
        (size_t)C.J * 2 * C.Nrow * 4,                       // 11 laps
        (size_t)C.J * C.maxT * 4, (size_t)C.J * C.maxT * 4, // 12-13 perm_ready, perm_done
        (size_t)C.J * sizeof(JobDev),                       // 14 jobs
        (size_t)C.J * C.Bmax * 4, (size_t)C.J * C.Bmax,     // 15-16 out_ids, out_src
        (size_t)C.J * C.Bmax * 4, 32,                       // 17-18 evict_push, fill_n
        capl, 2 * (capl + (size_t)C.J * C.Bmax * 4),        // 19-20 evict, fill [2]
        (size_t)C.J * C.maxT * sizeof(seneca_job_epoch_stats),  // 21 stats
        8, 8, 0, 0, 256,                                    // 22-26 evicted, refilled, (control block x2), phase
        C.evict_all ? 2 * edl : 4, 8,                       // 27-28 ev_ed, ev_ed_n
        C.cold ? (size_t)C.J * C.Bmax * 4 : 4, (size_t)C.J * 4,   // 29-30 fetch, fetch_n
        4, C.cold ? W : 4,                                  // 31-32 warm, claim
        (size_t)C.J * 4, 4,                                 // 33-34 epoch_at, gen_next
        mbox_u32 * 4,                                       // 35 shard mailbox
        (size_t)kRingPairs * 4,                             // 36 ring generator work list
        C.late ? (size_t)C.J * C.K * C.Nrow * 4 : 4,        // 37 storage-list segments
        C.late ? (size_t)C.J * C.K * C.nch * 4 : 4,         // 38 segment counts
        C.late ? (size_t)C.J * C.K * (C.Nrow / 32) * 4 : 4, // 39 storage bit per position
    };
    size_t at = 0;
    for (size_t k = 0; k < sizeof(sz) / sizeof(sz[0]); ++k) {
        z.off[k] = at;
        at += align256(sz[k]);
    }
    z.total = at;
    z.R = cfg->replicas ? cfg->replicas : 1;
    if (C.G > 1 && cfg->shard_mode == 0) z.R = C.G;          // emulation: one slice per shard
    return z;
}

Lay carve(const Sizes& z, char* base, char* ctl, uint64_t seed) {
    Lay L;
    L.seed = seed;
    L.bm_e = (uint32_t*)(base + z.off[0]);
    L.bm_d = (uint32_t*)(base + z.off[1]);
    L.bm_a = (uint32_t*)(base + z.off[2]);
    L.seen = (uint32_t*)(base + z.off[3]);
    L.cons = (uint32_t*)(base + z.off[4]);
    L.cons_cnt = (uint32_t*)(base + z.off[5]);
    L.cnt8 = (uint32_t*)(base + z.off[6]);
    L.cnt_sup = (uint32_t*)(base + z.off[7]);
    L.cnt_tot = (uint32_t*)(base + z.off[8]);
    L.tsize = (uint32_t*)(base + z.off[9]);
    L.perms = (uint32_t*)(base + z.off[10]);
    L.laps = (uint32_t*)(base + z.off[11]);
    L.perm_ready = (uint32_t*)(base + z.off[12]);
    L.perm_done = (uint32_t*)(base + z.off[13]);
    L.jobs = (JobDev*)(base + z.off[14]);
    L.out_ids = (uint32_t*)(base + z.off[15]);
    L.out_src = (uint8_t*)(base + z.off[16]);
    L.evict_push = (uint32_t*)(base + z.off[17]);
    L.fill_n = (uint32_t*)(base + z.off[18]);
    L.evict_list = (uint32_t*)(base + z.off[19]);
    L.fill_list = (uint32_t*)(base + z.off[20]);
    L.stats = (seneca_job_epoch_stats*)(base + z.off[21]);
    L.evicted = (unsigned long long*)(base + z.off[22]);
    L.refilled = (unsigned long long*)(base + z.off[23]);
    L.bar = (uint32_t*)ctl;
    L.err = (uint32_t*)(ctl + 16);
    L.verr = (uint32_t*)(ctl + 20);
    L.dbg = (uint32_t*)(ctl + 24);
    L.phase = (unsigned long long*)(base + z.off[26]);
    L.ev_ed = (uint32_t*)(base + z.off[27]);
    L.ev_ed_n = (uint32_t*)(base + z.off[28]);
    L.fetch = (uint32_t*)(base + z.off[29]);
    L.fetch_n = (uint32_t*)(base + z.off[30]);
    L.warm = (uint32_t*)(base + z.off[31]);
    L.claim = (uint32_t*)(base + z.off[32]);
    L.epoch_at = (uint32_t*)(base + z.off[33]);
    L.gen_next = (uint32_t*)(base + z.off[34]);
    L.mbox = (uint32_t*)(base + z.off[35]);
    L.ring_pairs = (uint32_t*)(base + z.off[36]);
    L.slist = (uint32_t*)(base + z.off[37]);
    L.scnt = (uint32_t*)(base + z.off[38]);
    L.cbits = (uint32_t*)(base + z.off[39]);
    for (uint32_t g = 0; g < kMaxShards; ++g) L.peer[g] = nullptr;
    L.shard = 0; L.sb_lo = 0; L.sb_hi = z.C.NS; L.id_lo = 0; L.id_hi = z.C.NS * 4096u;
    return L;
}

int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

template <class F>
void timed(seneca_ctx* c, int cls, cudaStream_t st, F&& launch) {
    c->launches++;
    c->klaunch[cls]++;
    if (!(c->profiling & 1u)) { launch(); return; }
    cudaEventRecord(c->ev_a, st);
    launch();
    cudaEventRecord(c->ev_b, st);
    cudaEventSynchronize(c->ev_b);
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, c->ev_a, c->ev_b) == cudaSuccess) { c->kms[cls] += ms; c->ksampled[cls]++; }
}

// Host mirror of the data-independent schedule (R-O12, R-O23): per job the
// consumed count and epoch, the active and not-yet-arrived sets, the round.
struct Sched {
    uint64_t n[kMaxJobs], e[kMaxJobs], arrival[kMaxJobs];
    uint32_t active, pending;
    uint64_t r;
};

Sched sched_of(const seneca_ctx* c) {
    Sched s;
    for (uint32_t j = 0; j < kMaxJobs; ++j) { s.n[j] = c->n[j]; s.e[j] = c->e[j]; s.arrival[j] = c->arrival[j]; }
    s.active = c->active;
    s.pending = c->pending;
    s.r = c->r;
    return s;
}

void sched_arrive(Sched& s) {               // start of round s.r
    for (uint32_t m = s.pending; m; m &= m - 1) {
        const uint32_t j = __builtin_ctz(m);
        if (s.arrival[j] <= s.r) { s.active |= 1u << j; s.pending &= ~(1u << j); }
    }
}

// one round of the jobs in mask (after sched_arrive); an idle round if none is active
void sched_round(const Cfg& C, Sched& s, uint32_t mask) {
    const uint32_t part = s.active & mask;
    uint32_t departing = 0;
    for (uint32_t m = part; m; m &= m - 1) {
        const uint32_t j = __builtin_ctz(m);
        s.n[j] += std::min<uint64_t>(C.batch[j], (uint64_t)C.N - s.n[j]);
        if (s.n[j] == C.N) { s.n[j] = 0; s.e[j] += 1; if (s.e[j] == C.target[j]) departing |= 1u << j; }
    }
    s.active &= ~departing;
    s.r += 1;
}

// Rounds (<= R) a launch may play when the ring is filled only between launches:
// it stops before the first round in which a participating job would play an
// epoch whose permutation has not been generated.
uint64_t rounds_allowed(const seneca_ctx* c, uint64_t R, uint32_t jobs_mask) {
    if (c->mode != 0) return R;
    Sched s = sched_of(c);
    uint64_t k = 0;
    for (; k < R; ++k) {
        sched_arrive(s);
        bool ok = true;
        for (uint32_t m = s.active & jobs_mask; m; m &= m - 1) {
            const uint32_t j = __builtin_ctz(m);
            if (s.e[j] >= c->gen_hi[j]) { ok = false; break; }
        }
        if (!ok) break;
        sched_round(c->C, s, jobs_mask);
    }
    return k;
}

// The permutation ring ahead of a launch of (up to) R rounds; returns in *R_out
// the rounds the launch may play.
//  * Epochs a job may need at once (its current one up to K - 1 beyond) that are
//    not generated yet: ods_perm_all over the whole GPU, before the launch.  Their
//    slots hold epochs the job has finished (every earlier launch is ordered
//    before this generator), so no live permutation is overwritten.  One
//    replica: on the side stream, overlapping the round launch, which waits on
//    the ready flags; several replicas may fill every SM with round CTAs, so
//    their generator runs first on the caller's stream.
//  * One replica with more epochs than slots: the epochs the jobs will enter
//    during the launch are generated DURING it by ods_perm_ring on the side stream
//    (a few CTAs beside the J + 1 round CTAs; each slot is refilled once its job
//    has started the epoch after the slot's old one), so jobs whose epochs end at
//    different rounds never have to meet at a launch boundary.
//  * Several replicas: the launch stops before a job would enter an epoch that
//    is not in the ring (rounds_allowed); the next launch refills it.
seneca_status prepare_perms(seneca_ctx* c, cudaStream_t st, uint64_t R, uint32_t jobs_mask, uint64_t* R_out,
                            uint32_t* gen_pairs) {
    *gen_pairs = 0;
    NvtxRange nvtx("seneca permutation ring");
    *R_out = R;
    if (c->mode != 0) return SENECA_OK;
    const uint32_t K = c->C.K;
    uint64_t gen[kMaxJobs];
    for (uint32_t j = 0; j < kMaxJobs; ++j) gen[j] = c->gen_hi[j];
    PermWork W;
    W.n = 0;
    for (uint32_t k = 0; k < K; ++k)                           // epoch-major
        for (uint32_t j = 0; j < c->C.J; ++j) {
            if (!(((c->active | c->pending) >> j) & 1u)) continue;
            const uint64_t e = c->e[j] + k;
            if (e < gen[j] || e >= c->C.target[j]) continue;
            W.j[W.n] = j; W.e[W.n] = (uint32_t)e; ++W.n;
            gen[j] = e + 1;
        }
    const uint32_t chunk = 16384;
    if (W.n) {
        cudaStream_t ps = st;
        if (c->R == 1) {
            SENECA_CUDA_TRY(cudaEventRecord(c->ev_init, st));
            SENECA_CUDA_TRY(cudaStreamWaitEvent(c->side, c->ev_init, 0));
            ps = c->side;
        }
        const uint32_t gx = std::max<uint32_t>(1, (uint32_t)num_sms() * 4 / c->R);
        timed(c, K_PERM, ps, [&] { ods_perm_all<<<dim3(gx, c->R), 512, 0, ps>>>(c->LS, c->C, W, chunk); });
        SENECA_CUDA_TRY(cudaGetLastError());
        for (uint32_t j = 0; j < kMaxJobs; ++j) c->gen_hi[j] = gen[j];
    }
    if (c->R > 1 || c->C.maxT <= K || c->gen_ctas == 0) {
        *R_out = rounds_allowed(c, R, jobs_mask);
        return SENECA_OK;
    }
    // one replica: the epochs entered during the launch, refilled concurrently
    PermRing Q;
    Q.n = 0;
    Sched s = sched_of(c);
    uint64_t k = 0;
    for (; k < R; ++k) {
        sched_arrive(s);
        Sched t = s;
        sched_round(c->C, t, jobs_mask);
        uint32_t add = 0;
        for (uint32_t m = s.active & jobs_mask; m; m &= m - 1) {    // jobs entering epoch e' this round
            const uint32_t j = __builtin_ctz(m);
            const uint64_t e = t.e[j] + K - 1;                     // its slot frees now
            if (t.e[j] != s.e[j] && e < c->C.target[j] && e >= gen[j]) ++add;
        }
        if (Q.n + add > kRingPairs) break;                         // the next launch takes over
        for (uint32_t m = s.active & jobs_mask; m; m &= m - 1) {
            const uint32_t j = __builtin_ctz(m);
            const uint64_t e = t.e[j] + K - 1;
            if (t.e[j] != s.e[j] && e < c->C.target[j] && e >= gen[j]) {
                Q.j[Q.n] = j; Q.e[Q.n] = (uint32_t)e; ++Q.n;
                gen[j] = e + 1;
            }
        }
        s = t;
    }
    *R_out = k;
    if (Q.n) {
        // the launch's trailing generator CTAs fill them (ring_generate)
        for (uint32_t x = 0; x < Q.n; ++x) c->ring_host[x] = Q.j[x] << 24 | Q.e[x];
        SENECA_CUDA_TRY(cudaMemcpyAsync(c->L.ring_pairs, c->ring_host, (size_t)Q.n * 4, cudaMemcpyHostToDevice, st));
        SENECA_CUDA_TRY(cudaMemsetAsync(c->L.gen_next, 0, 4, st));
        *gen_pairs = Q.n;
        for (uint32_t j = 0; j < kMaxJobs; ++j) c->gen_hi[j] = gen[j];
    }
    return SENECA_OK;
}

// Launch up to *Rio rounds (fewer when the permutation ring bounds the launch,
// prepare_perms); *Rio returns the rounds launched.  jobs_mask: the jobs of every
// round (replay: all active).
seneca_status launch_rounds(seneca_ctx* c, uint64_t* Rio, uint32_t jobs_mask, const uint32_t* d_requested,
                            uint32_t* out_ids, uint8_t* out_src, uint32_t out_stride, const uint32_t* row_of_job,
                            unsigned long long* transcript, cudaStream_t st) {
    NvtxRange nvtx("seneca round launch");
    uint64_t R = *Rio;
    if (!c->attached) { set_error("sharded context: attach the peers' mailboxes first"); return SENECA_ESTATE; }
    Launch P;
    std::memset(&P, 0, sizeof P);
    P.r0 = c->r;
    P.rounds = (uint32_t)R;
    P.subset = jobs_mask;
    P.mode = c->mode;
    P.active0 = c->active;
    P.pending0 = c->pending;
    for (uint32_t j = 0; j < c->C.J; ++j) {
        P.n0[j] = (uint32_t)c->n[j];
        P.e0[j] = (uint32_t)c->e[j];
        P.row_of_job[j] = row_of_job ? row_of_job[j] : j;
        P.arrival[j] = (uint32_t)std::min<uint64_t>(c->arrival[j], 0xffffffffu);
    }
    P.out_stride = out_stride;
    P.out_ids = out_ids;
    P.out_src = out_src;
    P.requested = d_requested;
    P.transcript = transcript;
    P.out_rep = (uint64_t)out_stride * (row_of_job ? __builtin_popcount(jobs_mask) : c->C.J);
    P.tr_rep = (uint64_t)c->C.J * c->C.maxT * c->C.N;
    P.timing = (c->profiling >> 1) & 1u;
    {
        uint64_t Rp = R;
        uint32_t gp = 0;
        seneca_status ps = prepare_perms(c, st, R, jobs_mask, &Rp, &gp);
        if (ps) return ps;
        P.gen_pairs = gp;
        P.gen_ctas = gp ? c->gen_ctas : 0u;
        if (Rp == 0) { set_error("internal: no round playable within the permutation ring"); return SENECA_ESTATE; }
        R = Rp;
        P.rounds = (uint32_t)R;
        *Rio = R;
    }
    if (c->mode == 1) {
        timed(c, K_VALIDATE, st, [&] {
            ods_validate_requests<<<__builtin_popcount(jobs_mask), 256, (size_t)c->C.Bmax * 4, st>>>(c->LS, c->C, P);
        });
        SENECA_CUDA_TRY(cudaGetLastError());
        uint32_t err = 0;
        SENECA_CUDA_TRY(cudaMemcpyAsync(&err, c->L.verr, 4, cudaMemcpyDeviceToHost, st));
        SENECA_CUDA_TRY(cudaStreamSynchronize(st));
        if (err) {                      // only the validation flag is cleared; latched flags stay
            SENECA_CUDA_TRY(cudaMemsetAsync(c->L.verr, 0, 4, st));
            set_error("supplied request ids out of range, duplicated or already seen");
            return SENECA_EPROTO;
        }
    }
    SENECA_CUDA_TRY(cudaMemset2DAsync(c->ctl, kCtlBytes, 0, 16, c->R, st));   // every replica's bar[4]
    // One replica's J + 1 round CTAs are launched as one thread-block cluster (same GPC,
    // hence same die; ImageNet-1K 9.01 -> 8.93 us per round, tools/s4q.sh); the generator
    // CTAs are padded so the grid is a multiple of the cluster size.  SENECA_ROUND_CLUSTER=0
    // turns it off; a cluster launch the device refuses falls back to the plain one.
    // (Nsight Compute cannot replay a cooperative cluster launch -- "LaunchFailed" --
    // so under an injected tool (ncu's NV_COMPUTE_PROFILER_PERFWORKS_DIR / NV_TPS_* /
    // NV_NSIGHT_INJECTION_*, any CUDA_INJECTION64_PATH) the plain cooperative launch
    // with global-memory signals is used)
    static const int want_cluster = [] {
        const char* e = getenv("SENECA_ROUND_CLUSTER");
        if (e) return atoi(e);
        for (const char* v : {"CUDA_INJECTION64_PATH", "NV_COMPUTE_PROFILER_PERFWORKS_DIR", "NV_TPS_LAUNCH_TOKEN",
                              "NV_NSIGHT_INJECTION_TRANSPORT_TYPE"}) {
            const char* x = getenv(v);
            if (x && *x) return 0;
        }
        return 1;
    }();
    const uint32_t cs = c->C.J + 1;
    const bool clustered = want_cluster && c->R == 1 && cs >= 2 && cs <= 8;
    if (clustered && P.gen_ctas) P.gen_ctas += (cs - (cs + P.gen_ctas) % cs) % cs;
    static const int want_dsig = [] { const char* e = getenv("SENECA_DSMEM_SIGNALS"); return e ? atoi(e) : 1; }();
    P.cluster = clustered && want_dsig ? 1u : 0u;
    void* args[] = {&c->LS, &c->C, &P};
    cudaError_t le = cudaSuccess;
    timed(c, K_ROUNDS, st, [&] {
        if (clustered) {
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3((c->C.J + 1) * c->R + P.gen_ctas);
            lc.blockDim = dim3(c->round_threads);
            lc.dynamicSmemBytes = c->round_smem;
            lc.stream = st;
            cudaLaunchAttribute at[2];
            at[0].id = cudaLaunchAttributeCooperative;
            at[0].val.cooperative = 1;
            at[1].id = cudaLaunchAttributeClusterDimension;
            at[1].val.clusterDim.x = cs; at[1].val.clusterDim.y = 1; at[1].val.clusterDim.z = 1;
            lc.attrs = at;
            lc.numAttrs = 2;
            le = cudaLaunchKernelExC(&lc, P.timing ? c->round_fn_timed : c->round_fn, args);
            if (le != cudaSuccess) {     // (a configuration error: nothing was launched)
                (void)cudaGetLastError();
                P.cluster = 0;
                le = cudaLaunchCooperativeKernel(P.timing ? c->round_fn_timed : c->round_fn,
                                                 lc.gridDim, lc.blockDim, args, c->round_smem, st);
            }
        } else {
            le = cudaLaunchCooperativeKernel(P.timing ? c->round_fn_timed : c->round_fn,
                                             dim3((c->C.J + 1) * c->R + P.gen_ctas), dim3(c->round_threads), args,
                                             c->round_smem, st);
        }
    });
    if (le != cudaSuccess) return cuda_status(le, "cudaLaunchCooperativeKernel(ods_rounds)");
    // host mirror of the data-independent schedule
    Sched sc = sched_of(c);
    for (uint64_t k = 0; k < R; ++k) {
        sched_arrive(sc);
        sched_round(c->C, sc, jobs_mask);
    }
    // (arrivals are applied at round starts only: a job stays pending until a
    // launch runs its arrival round, whose kernel rebuilds the job's pools)
    for (uint32_t j = 0; j < kMaxJobs; ++j) { c->n[j] = sc.n[j]; c->e[j] = sc.e[j]; }
    c->active = sc.active;
    c->pending = sc.pending;
    c->r = sc.r;
    return SENECA_OK;
}

}  // namespace

extern "C" seneca_status seneca_state_bytes(const seneca_cache_config* cfg, size_t* bytes) {
    seneca_status s = check_cfg(cfg);
    if (s) return s;
    if (!bytes) { set_error("NULL bytes"); return SENECA_EINVAL; }
    const Sizes z = compute_sizes(cfg);
    *bytes = ctl_bytes(z.R) + z.total * z.R;
    return SENECA_OK;
}

extern "C" seneca_status seneca_init_cache(const seneca_cache_config* cfg, void* d_workspace, size_t ws_bytes,
                                           void* stream, seneca_ctx** out) {
    NvtxRange nvtx("seneca_init_cache");
    seneca_status s = check_cfg(cfg);
    if (s) return s;
    if (!out || !d_workspace) { set_error("NULL workspace or out"); return SENECA_EINVAL; }
    if ((uintptr_t)d_workspace & 255) { set_error("workspace must be 256-byte aligned"); return SENECA_EINVAL; }
    Sizes z = compute_sizes(cfg);
    const size_t need_bytes = ctl_bytes(z.R) + z.total * z.R;
    if (ws_bytes < need_bytes) {
        set_error("workspace %zu bytes < required %zu", ws_bytes, need_bytes); return SENECA_ENOSPC;
    }
    // dynamic shared memory of a round CTA with T threads (window min(kWinMax, 2 T))
    auto smem_for = [&](uint32_t T) -> size_t {
        const size_t win = std::min<size_t>(kWinMax, 2 * (size_t)T);
        const size_t o_win = ((size_t)4 * z.C.Bmax + 6 * z.C.NS + 3) & ~(size_t)3;
        return (o_win + win + 4 * win) * 4 + z.C.Bmax;
    };
    const size_t round_smem = smem_for(kThreads);
    if (round_smem > 200 * 1024) { set_error("batch/dataset too large for the shared-memory indices"); return SENECA_EINVAL; }
    seneca_ctx* c = new (std::nothrow) seneca_ctx();
    if (!c) { set_error("out of host memory"); return SENECA_EINVAL; }
    c->C = z.C;
    c->R = z.R;
    c->rep_stride = z.total;
    c->ctl = (char*)d_workspace;
    const bool sharded = z.C.G > 1;
    c->shard_mode = sharded ? cfg->shard_mode : 0u;
    c->attached = !sharded || cfg->shard_mode == 0;
    for (uint32_t k = 0; k < z.R; ++k) {
        // emulated shards replay ONE instance: every slice has the configured seed
        c->LS.r[k] = carve(z, (char*)d_workspace + ctl_bytes(z.R) + k * z.total, c->ctl + k * kCtlBytes,
                           sharded ? cfg->seed : cfg->seed + k);
        if (sharded) {
            Lay& L = c->LS.r[k];
            const uint32_t g = cfg->shard_mode == 0 ? k : cfg->shard_rank;
            const uint32_t per = (z.C.NS + z.C.G - 1) / z.C.G;
            L.shard = g;
            L.sb_lo = std::min(z.C.NS, g * per);
            L.sb_hi = std::min(z.C.NS, (g + 1) * per);
            L.id_lo = L.sb_lo * 4096u;
            L.id_hi = L.sb_hi * 4096u;
        }
    }
    if (sharded) {
        for (uint32_t k = 0; k < z.R; ++k)
            for (uint32_t g = 0; g < z.C.G; ++g)
                c->LS.r[k].peer[g] = cfg->shard_mode == 0 ? c->LS.r[g].mbox
                                                          : (g == c->LS.r[k].shard ? c->LS.r[k].mbox : nullptr);
    }
    c->L = c->LS.r[0];
    c->mode = cfg->request_mode;
    c->cap_e = cfg->cap_e;
    c->cap_d = cfg->cap_d;
    c->active = cfg->n_jobs == 32 ? 0xffffffffu : ((1u << cfg->n_jobs) - 1);
    c->pending = 0;
    for (uint32_t j = 0; j < cfg->n_jobs; ++j) {
        c->arrival[j] = cfg->arrival_round ? cfg->arrival_round[j] : 0;
        if (c->arrival[j] > 0) { c->active &= ~(1u << j); c->pending |= 1u << j; }
    }
    c->round_smem = round_smem;
    cudaStream_t st = (cudaStream_t)stream;
    cudaGetDevice(&c->device);
#define INIT_TRY(expr) do { cudaError_t _e = (expr); if (_e != cudaSuccess) { delete c; return cuda_status(_e, #expr); } } while (0)
    const bool coupled = z.C.cap_t > 0 || z.C.cold;
    for (int v = 0; v < 4; ++v)
        for (int tm = 0; tm < 2; ++tm)
            INIT_TRY(cudaFuncSetAttribute(round_kernel(v, tm, coupled), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          200 * 1024));
    INIT_TRY(cudaFuncSetAttribute(ods_validate_requests, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    {   // the cooperative round launch needs every replica's CTAs co-resident: one
        // 512-thread CTA per SM when they fit, else two 256-thread CTAs per SM
        const uint64_t need = (uint64_t)(z.C.J + 1) * z.R;
        int per_sm = 0;
        // (occupancy of the timed variants is checked too: a profiled replay
        // must fit the same co-resident grid)
        int per_sm_t = 0;
        INIT_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, round_kernel(0, false, coupled), kThreads,
                                                               round_smem));
        INIT_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_t, round_kernel(0, true, coupled), kThreads,
                                                               round_smem));
        per_sm = std::min(per_sm, per_sm_t);
        uint64_t slots = (uint64_t)per_sm * num_sms();
        c->round_fn = round_kernel(0, false, coupled);
        c->round_fn_timed = round_kernel(0, true, coupled);
        c->round_threads = kThreads;
        if (sharded) {                       // 512 threads, one CTA per SM, every shard's CTAs co-resident
            int per_shd = 0, per_shd_t = 0;
            INIT_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_shd, round_kernel(3, false, coupled), kThreads,
                                                                   round_smem));
            INIT_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_shd_t, round_kernel(3, true, coupled), kThreads,
                                                                   round_smem));
            if (need > (uint64_t)std::min(per_shd, per_shd_t) * num_sms()) {
                set_error("%u shards x %u CTAs exceed the co-resident CTA slots", z.R, z.C.J + 1);
                delete c;
                return SENECA_EINVAL;
            }
            c->round_fn = round_kernel(3, false, coupled);
            c->round_fn_timed = round_kernel(3, true, coupled);
            slots = need;                    // no other variant below
        }
        // independent jobs (no maintain coupling): the replay lasts as long as the job
        // with the most rounds; when that job's batch fits 256 threads, 256-thread
        // CTAs run its rounds faster (measured: OpenImages)
        uint32_t jdom = 0;
        uint64_t rdom = 0;
        for (uint32_t jj = 0; jj < z.C.J; ++jj) {
            const uint64_t rj = (uint64_t)z.C.target[jj] * ((z.C.N + z.C.batch[jj] - 1) / z.C.batch[jj]);
            if (rj > rdom || (rj == rdom && z.C.batch[jj] > z.C.batch[jdom])) { rdom = rj; jdom = jj; }
        }
        if (!sharded && !coupled && z.C.batch[jdom] <= kThreads / 2 && need <= slots) {
            const size_t smemh = smem_for(kThreads / 2);
            int per_smh = 0, per_smh_t = 0;
            INIT_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_smh, round_kernel(2, false, coupled),
                                                                   kThreads / 2, smemh));
            INIT_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_smh_t, round_kernel(2, true, coupled),
                                                                   kThreads / 2, smemh));
            if (need <= (uint64_t)std::min(per_smh, per_smh_t) * num_sms()) {
                c->round_fn = round_kernel(2, false, coupled);
                c->round_fn_timed = round_kernel(2, true, coupled);
                c->round_threads = kThreads / 2;
                c->round_smem = smemh;
            }
        }
        if (need > slots) {
            const size_t smem2 = smem_for(kThreads / 2);
            int per_sm2 = 0;
            int per_sm2_t = 0;
            INIT_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, round_kernel(1, false, coupled),
                                                                   kThreads / 2, smem2));
            INIT_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2_t, round_kernel(1, true, coupled),
                                                                   kThreads / 2, smem2));
            per_sm2 = std::min(per_sm2, per_sm2_t);
            const uint64_t slots2 = (uint64_t)per_sm2 * num_sms();
            if (need > slots2) {
                set_error("%u replicas x %u CTAs exceed the %llu co-resident CTA slots", z.R, z.C.J + 1,
                          (unsigned long long)std::max(slots, slots2));
                delete c;
                return SENECA_EINVAL;
            }
            c->round_fn = round_kernel(1, false, coupled);
            c->round_fn_timed = round_kernel(1, true, coupled);
            c->round_threads = kThreads / 2;
            c->round_smem = smem2;
        }
    }
    if (z.R == 1 && z.C.maxT > z.C.K && cfg->request_mode == 0) {
        // ring generator CTAs appended to every launch that needs them: as many as
        // fit beside the J + 1 round CTAs, at most 16 (timed variant checked too)
        int per = 0, per_t = 0;
        INIT_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, c->round_fn, c->round_threads, c->round_smem));
        INIT_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_t, c->round_fn_timed, c->round_threads,
                                                               c->round_smem));
        const int64_t room = (int64_t)std::min(per, per_t) * num_sms() - (int64_t)(z.C.J + 1);
        c->gen_ctas = (uint32_t)std::max<int64_t>(0, std::min<int64_t>(16, room));
    }
    INIT_TRY(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
    INIT_TRY(cudaEventCreateWithFlags(&c->ev_init, cudaEventDisableTiming));
    INIT_TRY(cudaEventCreate(&c->ev_a));
    INIT_TRY(cudaEventCreate(&c->ev_b));
    INIT_TRY(cudaMemsetAsync(d_workspace, 0, need_bytes, st));
    {
        const uint32_t total = (uint32_t)(cfg->cap_a + cfg->cap_d + cfg->cap_e);
        const uint32_t blocks = std::max<uint32_t>(1, std::min<uint32_t>((total + 255) / 256, num_sms() * 8));
        timed(c, K_INIT, st, [&] {
            ods_init_tiers<<<dim3(blocks, c->R), 256, 0, st>>>(c->LS, c->C, (uint32_t)cfg->cap_e, (uint32_t)cfg->cap_d);
        });
        INIT_TRY(cudaGetLastError());
        timed(c, K_RECOUNT, st, [&] {
            ods_recount_all<<<dim3((c->C.NS + kRecountWarps - 1) / kRecountWarps, c->R, c->C.J), kRecountWarps * 32, 0,
                              st>>>(c->LS, c->C);
        });
        INIT_TRY(cudaGetLastError());
        ods_init_jobs<<<c->R, 32, 0, st>>>(c->LS, c->C);
        c->launches++;
        INIT_TRY(cudaGetLastError());
    }
    // the first ring of permutations (epochs 0 .. K-1 of every job), overlapping
    // the caller's next work when there is one replica (ensure_perms)
    {
        uint64_t unused = 0;
        uint32_t unused_pairs = 0;
        const seneca_status ps = prepare_perms(c, st, 0, 0xffffffffu, &unused, &unused_pairs);
        if (ps) { delete c; return ps; }
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
    uint32_t mask = 0, rows[kMaxJobs] = {0};
    for (uint32_t x = 0; x < n_jobs; ++x) {
        const uint32_t j = h_jobs[x];
        if (j >= c->C.J || (mask & (1u << j))) { set_error("bad or duplicate job %u", j); return SENECA_EINVAL; }
        mask |= 1u << j;
        rows[j] = x;
        const bool arrived = ((c->pending >> j) & 1u) && c->arrival[j] <= c->r;
        if (!(c->active & (1u << j)) && !arrived) {
            set_error((c->pending >> j) & 1u ? "job %u has not arrived yet" : "job %u has departed", j);
            return SENECA_ESTATE;
        }
    }
    for (uint32_t x = 0; x < n_jobs; ++x) {
        const uint32_t j = h_jobs[x];
        if (h_out_lens) h_out_lens[x] = (uint32_t)std::min<uint64_t>(c->C.batch[j], (uint64_t)c->C.N - c->n[j]);
    }
    uint64_t one = 1;
    return launch_rounds(c, &one, mask, d_requested, d_out_ids, d_out_src, c->C.Bmax, rows, nullptr,
                         (cudaStream_t)stream);
}

// Rounds needed until every tracked job (active or not yet arrived at the call)
// completed n more epochs or departed; idle rounds before an arrival included.
static uint64_t rounds_for_epochs(const seneca_ctx* c, uint32_t n_epochs) {
    Sched s = sched_of(c);
    const uint32_t tracked = s.active | s.pending;
    uint64_t goal[kMaxJobs];
    for (uint32_t j = 0; j < kMaxJobs; ++j) goal[j] = s.e[j] + n_epochs;
    uint64_t R = 0;
    for (;;) {
        sched_arrive(s);
        bool open = false;
        for (uint32_t m = tracked & (s.active | s.pending); m; m &= m - 1)
            if (s.e[__builtin_ctz(m)] < goal[__builtin_ctz(m)]) open = true;
        if (!open || !(s.active | s.pending)) break;
        sched_round(c->C, s, 0xffffffffu);
        ++R;
    }
    return R;
}

static seneca_status replay(seneca_ctx* c, uint64_t R, uint64_t* d_transcript, uint64_t* h_rounds, cudaStream_t st) {
    NvtxRange nvtx("seneca_replay");
    if (c->mode != 0) { set_error("replay requires request_mode 0"); return SENECA_ESTATE; }
    if (!(c->active | c->pending)) { set_error("no active job"); return SENECA_ESTATE; }
    uint64_t done = 0;
    // rounds per launch: the 32-bit signal counters (job phases, evictions pushed,
    // eviction ring position) count at most J (phases) / J * Bmax (pushes) per round
    // and are zeroed at every launch, so a launch never lets them wrap
    const uint64_t kChunk = std::min<uint64_t>(1u << 30, 0xffffffffull / ((uint64_t)c->C.J * (c->C.Bmax + 1)));
    while (done < R && (c->active | c->pending)) {
        uint64_t n = std::min<uint64_t>(R - done, kChunk);
        seneca_status s = launch_rounds(c, &n, 0xffffffffu, nullptr, nullptr, nullptr, c->C.Bmax, nullptr,
                                        (unsigned long long*)d_transcript, st);
        if (s) return s;
        done += n;
    }
    if (h_rounds) *h_rounds = done;
    return SENECA_OK;
}

extern "C" seneca_status seneca_replay_epochs(seneca_ctx* c, uint32_t n_epochs, uint64_t* d_transcript,
                                              uint64_t* h_rounds, void* stream) {
    if (!c || n_epochs == 0) { set_error("bad arguments"); return SENECA_EINVAL; }
    if (c->mode != 0) { set_error("replay requires request_mode 0"); return SENECA_ESTATE; }
    if (!(c->active | c->pending)) { set_error("no active job"); return SENECA_ESTATE; }
    return replay(c, rounds_for_epochs(c, n_epochs), d_transcript, h_rounds, (cudaStream_t)stream);
}

extern "C" seneca_status seneca_replay_epoch(seneca_ctx* c, uint32_t n_epochs, uint64_t* d_transcript,
                                             uint64_t* h_rounds, void* stream) {
    return seneca_replay_epochs(c, n_epochs, d_transcript, h_rounds, stream);
}

extern "C" seneca_status seneca_replay_rounds(seneca_ctx* c, uint64_t n_rounds, uint64_t* d_transcript,
                                              uint64_t* h_rounds, void* stream) {
    if (!c) { set_error("bad arguments"); return SENECA_EINVAL; }
    if (c->mode != 0) { set_error("replay requires request_mode 0"); return SENECA_ESTATE; }
    if (!(c->active | c->pending)) { set_error("no active job"); return SENECA_ESTATE; }
    // stop early when every job has departed (idle rounds before an arrival count)
    uint64_t R = 0;
    {
        Sched s = sched_of(c);
        for (;;) {
            sched_arrive(s);
            if (R >= n_rounds || !(s.active | s.pending)) break;
            sched_round(c->C, s, 0xffffffffu);
            ++R;
        }
    }
    return replay(c, R, d_transcript, h_rounds, (cudaStream_t)stream);
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
    v->d_phase_cycles = (const uint64_t*)c->L.phase;
    v->round = c->r;
    for (uint32_t j = 0; j < c->C.J; ++j) { v->epoch[j] = c->e[j]; v->consumed[j] = c->n[j]; }
    v->active_mask = c->active;
    for (uint32_t m = c->pending; m; m &= m - 1)             // arrived at the current round
        if (c->arrival[__builtin_ctz(m)] <= c->r) v->active_mask |= 1u << __builtin_ctz(m);
    v->replicas = c->R;
    v->replica_stride = c->rep_stride;
    return SENECA_OK;
}

extern "C" seneca_status seneca_shard_mailbox(const seneca_ctx* c, void** d_mailbox, size_t* bytes) {
    if (!c || !d_mailbox || !bytes) { set_error("bad arguments"); return SENECA_EINVAL; }
    if (c->C.G <= 1 || c->shard_mode != 1) { set_error("not a one-shard-per-context sharded replay"); return SENECA_EINVAL; }
    *d_mailbox = c->L.mbox;
    *bytes = ((size_t)c->C.mb_fl + 2 * (c->C.J + 1) * c->C.G) * 4;
    return SENECA_OK;
}

extern "C" seneca_status seneca_shard_attach(seneca_ctx* c, void* const* peers) {
    if (!c || !peers) { set_error("bad arguments"); return SENECA_EINVAL; }
    if (c->C.G <= 1 || c->shard_mode != 1) { set_error("not a one-shard-per-context sharded replay"); return SENECA_EINVAL; }
    Lay& L = c->LS.r[0];
    for (uint32_t g = 0; g < c->C.G; ++g) {
        void* p = peers[g] ? peers[g] : (g == L.shard ? (void*)L.mbox : nullptr);
        if (!p) { set_error("NULL mailbox of shard %u", g); return SENECA_EINVAL; }
        L.peer[g] = (uint32_t*)p;
    }
    c->L = L;
    c->attached = true;
    return SENECA_OK;
}

extern "C" seneca_status seneca_sync_status(seneca_ctx* c, void* stream) {
    if (!c) { set_error("bad arguments"); return SENECA_EINVAL; }
    uint32_t err[kMaxReplicas][8] = {{0}};
    SENECA_CUDA_TRY(cudaMemcpy2DAsync(err, 32, c->L.err, kCtlBytes, 32, c->R, cudaMemcpyDeviceToHost,
                                      (cudaStream_t)stream));
    SENECA_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    for (uint32_t k = 0; k < c->R; ++k)
        if (err[k][0]) {
            set_error("device consistency check failed (replica %u, flags 0x%x; first: site 0x%x pool/job %u, "
                      "%u %u %u)", k, err[k][0], err[k][2] >> 16, err[k][2] & 0xffffu, err[k][3], err[k][4], err[k][5]);
            return SENECA_ESTATE;
        }
    return SENECA_OK;
}

extern "C" uint64_t seneca_launch_count(const seneca_ctx* c) { return c ? c->launches : 0; }

extern "C" seneca_status seneca_profile(seneca_ctx* c, uint32_t enable) {
    if (!c) { set_error("bad arguments"); return SENECA_EINVAL; }
    c->profiling = enable & 3u;
    return SENECA_OK;
}

extern "C" seneca_status seneca_profile_read(seneca_ctx* c, seneca_kernel_stat* out, uint32_t cap, uint32_t* n_out) {
    if (!c || (!out && cap)) { set_error("bad arguments"); return SENECA_EINVAL; }
    const uint32_t n = std::min<uint32_t>(cap, K_NCLASS);
    for (uint32_t k = 0; k < n; ++k) {
        out[k].name = kKernelNames[k];
        out[k].launches = c->klaunch[k];
        out[k].sampled = c->ksampled[k];
        out[k].sampled_ms = c->kms[k];
    }
    if (n_out) *n_out = K_NCLASS;
    return SENECA_OK;
}

extern "C" void seneca_destroy(seneca_ctx* c) {
    if (!c) return;
    if (c->side) { cudaStreamSynchronize(c->side); cudaStreamDestroy(c->side); }
    if (c->ev_init) cudaEventDestroy(c->ev_init);
    if (c->ev_a) cudaEventDestroy(c->ev_a);
    if (c->ev_b) cudaEventDestroy(c->ev_b);
    delete c;
}
