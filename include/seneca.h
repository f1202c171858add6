/*
 * seneca.h -- C-ABI of libseneca.so, the B200 (sm_100a) hot path of Seneca
 * (arXiv 2511.13724, "Preparation Meets Opportunity: Enhancing Data
 * Preprocessing for ML Training With Seneca").
 *
 * Two parts:
 *   - MDP, Model-Driven Partitioning (§5.1; §5.3): the
 *     DSI throughput model (Eqs. 1-9) evaluated for every (x_E, x_D, x_A) split
 *     of a grid and every hardware profile, followed by an argmax.
 *   - ODS, Opportunistic Data Sampling (§5.2): trace-driven replay
 *     of N concurrent jobs over a cache partitioned into encoded (E), decoded
 *     (D) and augmented (A) forms.
 *
 * "P:Lnnn" cites /root/reference/PAPER.md line nnn; "R-xx" a reading recorded in
 * DESIGN.md §3 where the paper is silent or ambiguous.
 *
 * Conventions for every call:
 *   - Device memory is CALLER-OWNED.  Pointers prefixed d_ are device pointers
 *     (e.g. a torch tensor's data_ptr()); h_ are host pointers.  The library
 *     never allocates device memory: seneca_state_bytes() sizes one workspace.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Device work is enqueued and the call returns; device outputs are valid
 *     after the stream synchronises.  Host outputs that do not depend on device
 *     data (batch lengths, round counts) are returned synchronously.
 *   - Every call returns a seneca_status.  seneca_last_error() returns a
 *     thread-local message for the last failing call.  Invalid arguments never
 *     touch device memory.
 *   - A context is single-stream and not thread-safe; distinct contexts are
 *     independent (one process per GPU; see DESIGN.md §8 for multi-GPU).
 */
#ifndef SENECA_H
#define SENECA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SENECA_OK = 0,
    SENECA_EINVAL = 1,  /* invalid argument (SPEC "invalid-argument")                      */
    SENECA_ESTATE = 2,  /* call not valid in the current state (e.g. a departed job)       */
    SENECA_EPROTO = 3,  /* protocol violation by caller-supplied request ids       */
    SENECA_ECUDA = 4,   /* CUDA runtime error (message in seneca_last_error)                */
    SENECA_ENOSPC = 6   /* workspace smaller than seneca_state_bytes()                     */
} seneca_status;

/* ------------------------------------------------------------------------- */
/* MDP                                                                        */
/* ------------------------------------------------------------------------- */

/* One row of tab:model_vars: hardware x dataset x job.  Units are
 * canonical (bytes, bytes/s, samples/s; decimal SI, R-M11).  Layout: 112 bytes,
 * 8-byte aligned, no implicit padding.                                         */
typedef struct {
    double   t_gpu;            /* T_GPU    samples/s per node; finite, > 0           */
    double   t_decode_augment; /* T_{D+A}  samples/s per node; finite, > 0           */
    double   t_augment;        /* T_A      samples/s per node; finite, > 0           */
    double   b_nic;            /* B_NIC    bytes/s per node; finite, > 0             */
    double   b_pcie;           /* B_PCIe   bytes/s per node; finite, > 0             */
    double   b_cache;          /* B_cache  bytes/s; finite, > 0                      */
    double   b_storage;        /* B_storage bytes/s; finite, > 0                     */
    double   model_bytes;      /* beta*N in bytes (R-M2); finite, >= 0               */
    uint64_t cache_bytes;      /* S_cache = S_mem (R-M5); 100*cache_bytes*m_den < 2^64 */
    uint64_t n_total;          /* N_total >= 1                                       */
    uint64_t s_data;           /* S_data >= 1 bytes; 100*m_num*s_data < 2^64          */
    uint32_t m_num, m_den;     /* M = m_num/m_den >= 1 (5.12 = 128/25)        */
    uint32_t nodes;            /* n >= 1                                             */
    uint32_t gpus_per_node;    /* >= 1                                               */
    uint8_t  nvlink_intra;     /* intra-node NVLink -> C_PCIe = 0             */
    uint8_t  nvlink_inter;     /* inter-node NVLink -> C_PCIe = C_nw = 0      */
    uint8_t  comm_mapping;     /* R-M1: 0 network<->nodes, PCIe<->gpus_per_node;
                                  1 the literal (swapped) text of P:L529             */
    uint8_t  _pad[5];
} seneca_mdp_profile;

/* Argmax of Eq. 9 over the grid for one profile.  48 bytes.                  */
typedef struct {
    uint8_t p_e, p_d, p_a;     /* argmax split in integer percent, sums to 100        */
    uint8_t lim_a, lim_d, lim_e, lim_s; /* limiting term of Eqs. 1-4: 0 cache-bw, 1 nic,
                                  2 pcie, 3 cpu-augment, 4 cpu-decode-augment, 5 gpu,
                                  6 storage-bw (first minimal term wins, R-M8)       */
    uint8_t status;            /* 0 ok; 1 the profile violates the constraints above
                                  (all other fields then undefined)                  */
    double  v_best;            /* DSI_overall at the argmax (Eq. 9), samples/s        */
    double  dsi_a, dsi_d, dsi_e, dsi_s; /* Eqs. 1-4, samples/s                        */
} seneca_mdp_result;

/* Number of splits on a grid of step g percent (g divides 100):
 * (100/g + 1)(100/g + 2)/2, i.e. 5151 at 1 % and 66 at 10 %.          */
uint64_t seneca_mdp_num_splits(uint32_t grid_step_pct);

/* MDP sweep (a9-a12).  For every profile i < n_profiles: the tier throughputs
 * DSI_A/D/E/S (Eqs. 1-4, with the ring overhead 2(n-1)/n*betaN of
 * P:L529), the capacity-clamped counts N_A, N_D, N_E, N_S (Eqs. 5-8, floored
 * exactly in integers, R-M6) and DSI_overall (Eq. 9) for every split
 * of the grid, enumerated p_E = 100, 100-g, ..., 0 and, for each, p_D = 100-p_E,
 * ..., 0 (R-M9); then the argmax, exact ties to the smallest enumeration index
 * (R-M8).  Arithmetic is IEEE binary64 with one rounding per operation in the
 * literal order of R-M7 (bit-identical to the oracle).
 *   d_profiles  [n_profiles] device, read-only.
 *   d_results   [n_profiles] device, written.
 *   d_grid      NULL, or device [n_profiles][num_splits] doubles, row-major in
 *               enumeration order, written.
 * Errors: EINVAL if grid_step_pct does not divide 100, n_profiles == 0 or a
 * required pointer is NULL.  Per-profile constraint violations are reported in
 * seneca_mdp_result.status, not as a call error.                              */
seneca_status seneca_mdp_sweep(const seneca_mdp_profile* d_profiles, uint32_t n_profiles,
                               uint32_t grid_step_pct, seneca_mdp_result* d_results,
                               double* d_grid, void* stream);

/* Model evaluation at given splits (SPEC `evaluate`; SURVEY §8(f)
 * NEXT-4: fixed splits x dataset sizes, the Fig. 7 curves P:L837-909, are
 * profiles that differ in n_total).  For every profile i and every split s of
 * h_splits: V = DSI_overall (Eq. 9) with the same arithmetic as
 * seneca_mdp_sweep, and optionally the counts {N_A, N_D, N_E, N_S} (Eqs. 5-8).
 *   h_splits     host [n_splits], each p_e + p_d + p_a == 100 (integer %),
 *                1 <= n_splits <= 4096 (passed to the kernel by value).
 *   d_values     device [n_profiles][n_splits] doubles, written (NaN for an
 *                invalid profile).
 *   d_counts     NULL, or device [n_profiles][n_splits][4] uint64, written.
 *   d_tiers      NULL, or device [n_profiles] results: status, lim_* and dsi_*
 *                written, p_* = 0 and v_best = 0.
 * Errors: EINVAL on n_profiles == 0, NULL required pointers, n_splits out of
 * range or a split not summing to 100.                                        */
typedef struct {
    uint8_t p_e, p_d, p_a, _pad;
} seneca_split;

seneca_status seneca_mdp_eval(const seneca_mdp_profile* d_profiles, uint32_t n_profiles,
                              const seneca_split* h_splits, uint32_t n_splits, double* d_values,
                              uint64_t* d_counts, seneca_mdp_result* d_tiers, void* stream);

/* Eqs. 5-8 for one split on the host, in exact integer arithmetic (R-M6):
 * caps[0..3] = {N_E, N_D, N_A, N_storage} for a dataset of n_total samples of
 * s_data bytes, a cache of cache_bytes and M = m_num/m_den.  Used to size the
 * ODS tiers of seneca_cache_config.  EINVAL on p_e+p_d+p_a != 100, zero sizes,
 * m_num < m_den, or 100*cache_bytes*m_den / 100*m_num*s_data overflowing u64.  */
seneca_status seneca_split_capacities(uint64_t n_total, uint64_t s_data, uint32_t m_num,
                                      uint32_t m_den, uint64_t cache_bytes, uint32_t p_e,
                                      uint32_t p_d, uint32_t p_a, uint64_t caps[4]);

/* ODS metadata footprint as the paper counts it: 1 bit per sample
 * per job for `seen` plus 1 byte per sample for status+reference:
 * n_jobs*ceil(n_total/8) + n_total.  (This library's own layout is reported by
 * seneca_state_bytes; R-O14.)                                                   */
uint64_t seneca_metadata_bytes(uint64_t n_total, uint32_t n_jobs);

/* ------------------------------------------------------------------------- */
/* ODS                                                                        */
/* ------------------------------------------------------------------------- */

typedef struct seneca_ctx seneca_ctx;

typedef struct {
    uint64_t        n_total;       /* N, 1 <= N < 2^31 (and N/32768 + batch <= 51200)    */
    uint32_t        n_jobs;        /* J, 1..32                                           */
    uint32_t        request_mode;  /* 0: requests generated from each job's keyed
                                      permutation (R-O1, R-O3); 1: caller-supplied ids
                                      in seneca_ods_next_batch (R-O20)                   */
    const uint32_t* batch_size;    /* host [n_jobs], 1..4096 ("up to 1024")     */
    const uint32_t* target_epochs; /* host [n_jobs], >= 1; job departs after these     */
    uint64_t        cap_e, cap_d, cap_a; /* tier capacities in samples (Eqs. 5-7), sum <= N */
    uint64_t        seed;          /* all randomness derives from (seed, purpose, ...) R-O17 */
    uint32_t        replicas;      /* R independent replay instances in this context (0 or 1:
                                      one), replica k with seed + k, each with its own slice
                                      of the workspace; 1..64, R x (n_jobs + 1) CTAs must be
                                      co-resident (EINVAL otherwise); request_mode 1 needs
                                      R = 1.  SURVEY §8(e): replicas fill the GPU with
                                      independent replays (weak scaling inside one device). */
    uint32_t        evict_tiers;   /* 0: only augmented (A) entries carry consumer sets and are
                                      evicted / refilled (the default); 1: every
                                      cached tier (E, D, A) -- SURVEY 8c.3 "evict_tiers = ALL",
                                      DESIGN.md R-O21; E/D hits stay reusable              */
    uint32_t        sampler;       /* 0: ODS (the method); 1: the uniform no-evict baseline
                                      (MINIO-like, DESIGN.md R-O22): every
                                      cached id is a hit, misses go to storage, nothing is
                                      substituted, evicted or refilled                      */
    uint32_t        _pad0;
    const uint32_t* arrival_round; /* host [n_jobs] or NULL (all 0): job j takes part from round
                                      arrival_round[j] on (job-arrival / makespan traces, SURVEY
                                      8(f) NEXT-1, DESIGN.md R-O23); before it the job is not in
                                      the active set; a round with no active job while arrivals
                                      are pending is idle.  next_batch on a job that has not
                                      arrived is ESTATE                                        */
    uint32_t        cold_start;    /* 0: warm start (R-O9); 1: every tier starts empty and, until
                                      all three have been full once, each round's storage fetches
                                      (ascending job, slot order, first occurrence, storage-
                                      resident at round start) are admitted at the round end
                                      A -> D -> E up to each tier's capacity instead of random
                                      refills (DESIGN.md R-O24); refills and
                                      admissions are both counted in d_refilled               */
    uint32_t        _pad1;
    /* Sample-ID-range sharding of ONE replay (north_star "partitioned by
     * sample-ID range ... all-gathering per-shard candidate counts and selections each
     * batch").  Shard g of G keeps the pool counts of the ids of superblocks
     * [g*ceil(NS/G), (g+1)*ceil(NS/G)) (NS = ceil(N/4096)) and resolves the substitute /
     * refill ranks that fall into them; requests, classification, responses, seen and
     * consumer sets and eviction decisions are replicated on every shard.  Per round and
     * job two exchanges through device mailboxes: C1 = every shard's pool sizes, C2 = the
     * ids each shard resolved (the maintain CTA: the storage pool and the refill ids).
     * Results are identical for every G.                               */
    uint32_t        shards;        /* G, 0 or 1: unsharded; 2..8                                  */
    uint32_t        shard_rank;    /* shard_mode 1: this context's shard g < G                     */
    uint32_t        shard_mode;    /* 0: all G shards in this context on this device (one launch of
                                      G x (n_jobs + 1) CTAs; exchange through its own workspace);
                                      1: this context is shard shard_rank only (one per device);
                                      the peers' mailboxes are attached with seneca_shard_attach
                                      before the first round.  Both need replicas <= 1 and
                                      request_mode 0.                                         */
    uint32_t        _pad2;
} seneca_cache_config;

/* Per job-epoch counters (R-O10; digest in DESIGN.md §3).  104 bytes.       */
typedef struct {
    uint64_t served[4];    /* delivered samples by source tier: [0] storage, [1] E, [2] D, [3] A */
    uint64_t subst[4];     /* of which substituted for a miss, by tier                          */
    uint64_t req_hits[4];  /* requested samples that hit, by tier                               */
    uint64_t digest;       /* sum over delivery position q of splitmix64(q<<35 | src<<32 | id)  */
} seneca_job_epoch_stats;

/* Epoch model on top of a replay (SPEC `run` and
 * `preprocessing_ops`).  For every per job-epoch counter row:
 *   epoch_seconds  = served_A/DSI_A + served_D/DSI_D + served_E/DSI_E + served_S/DSI_S
 *                    (epoch time accounted over tiers), summed in that order;
 *   dsi_mix        = Eq. 9 with N_t := the epoch's served_t:
 *                    ((sA/N) DSI_A + (sD/N) DSI_D) + (sE/N) DSI_E) + (sS/N) DSI_S;
 *   decode_aug_ops = served_S + served_E, aug_only_ops = served_D;
 *   hit_rate       = (served_E + served_D + served_A) / N.
 * IEEE binary64, one rounding per operation, bit-identical to the oracle.    */
typedef struct {
    double   epoch_seconds;
    double   dsi_mix;
    uint64_t decode_aug_ops;
    uint64_t aug_only_ops;
    double   hit_rate;
} seneca_epoch_metrics;

/* d_stats: device [n_rows] counter rows (e.g. seneca_state_view.d_stats),
 * h_dsi: host {DSI_A, DSI_D, DSI_E, DSI_S} (finite, > 0; e.g. from
 * seneca_mdp_eval's d_tiers), d_out: device [n_rows].  EINVAL on NULL
 * pointers, n_rows == 0, n_total == 0 or a non-positive / non-finite DSI.   */
seneca_status seneca_epoch_model(const seneca_job_epoch_stats* d_stats, uint32_t n_rows, uint64_t n_total,
                                 const double h_dsi[4], seneca_epoch_metrics* d_out, void* stream);

/* Device views into the workspace, valid until seneca_destroy.              */
typedef struct {
    uint64_t n_total;
    uint32_t n_jobs, max_target;
    uint64_t words;                     /* 32-bit words per bitmap (bit i of word i/32)    */
    const uint32_t* d_tier_e;           /* residency bitmaps ("status")           */
    const uint32_t* d_tier_d;
    const uint32_t* d_tier_a;
    const uint32_t* d_seen;             /* [n_jobs][words] per-job seen           */
    const uint32_t* d_cons;             /* [n_jobs][words] consumer sets of A entries (R-O5) */
    const seneca_job_epoch_stats* d_stats; /* [n_jobs][max_target]                        */
    const uint64_t* d_evicted;          /* total evictions                                 */
    const uint64_t* d_refilled;         /* total refills                                   */
    const uint64_t* d_phase_cycles;     /* [32] SM cycles per phase when profiling.  Job CTA 0:
                                           [0] recount/epoch end [1] classify [2] substitute
                                           (apply) [3] respond [4] barrier-1 wait [5] next walk
                                           [6] barrier-2 wait [7] walk steps (a count)
                                           [8] substitute: pool prefixes [9] substitute: ranks
                                           and locate.  Maintain CTA (+16): [16] speculative
                                           prefix [17] speculative refill ranks [18] barrier-1
                                           wait [19] eviction decision [20] remaining refill
                                           ranks + apply [21] barrier-2 wait                    */
    uint64_t round;                     /* rounds executed                                 */
    uint64_t epoch[32];                 /* host mirror: current epoch of each job          */
    uint64_t consumed[32];              /* host mirror: samples consumed in current epoch  */
    uint32_t active_mask;               /* bit j set while job j has not departed          */
    uint32_t replicas;                  /* R slices (replicas, or the G shards of an emulated
                                           sharded replay); every d_ pointer above is slice
                                           0's --                                          */
    uint64_t replica_stride;            /* slice k's is at + k * replica_stride bytes       */
} seneca_state_view;

/* Workspace size for cfg (bytes, 256-aligned pieces; replicas x one replica's).
 * EINVAL on a bad cfg.                                                         */
seneca_status seneca_state_bytes(const seneca_cache_config* cfg, size_t* bytes);

/* init_cache (a warm start, R-O9): carve d_workspace (caller-owned, >= the
 * seneca_state_bytes size, 256-byte aligned), fill tiers with iota =
 * perm(key(seed, INIT), N, .) -- positions [0,cap_A) -> A, the next cap_D -> D,
 * the next cap_E -> E --, clear seen/consumer sets, build the pool counts and
 * every job's first permutation.  *out receives a host handle (free with
 * seneca_destroy).  EINVAL / ENOSPC on bad arguments.                          */
seneca_status seneca_init_cache(const seneca_cache_config* cfg, void* d_workspace,
                                size_t workspace_bytes, void* stream, seneca_ctx** out);

/* One round (R-O11): a batch for each job of h_jobs (distinct, active), then
 * maintain (eviction + refill, R-O7).  Per job j: need = min(B_j, N - n_j)
 * ids are requested (generated, or read from d_requested[x][0..need) when
 * request_mode = 1), misses are replaced by unseen cached samples tier by tier
 * A -> D -> E (§5.2 steps 1-4) and the response is written to
 * d_out_ids[k][x][s] / d_out_src[k][x][s] (k = replica, x = position in
 * h_jobs, row stride = max batch size; src bits 0-1 tier 0 S 1 E 2 D 3 A,
 * bit 2 substituted).  Every replica plays the same jobs.
 * h_out_lens[x] = need (host, synchronous).  A job whose epoch ends is reset
 * (step 6) and departs after its target epoch.
 * Errors: EINVAL (bad/duplicate job, NULL outputs, d_requested given in mode 0
 * or missing in mode 1), ESTATE (departed job), EPROTO (mode 1: a supplied id
 * out of range, duplicated or already seen -- checked synchronously, the round
 * is then not applied).                                                        */
seneca_status seneca_ods_next_batch(seneca_ctx* ctx, const uint32_t* h_jobs, uint32_t n_jobs,
                                    const uint32_t* d_requested, uint32_t* d_out_ids,
                                    uint8_t* d_out_src, uint32_t* h_out_lens, void* stream);

/* Replay whole rounds over all active jobs (request_mode 0 only) until every
 * job active at the call has completed n_epochs more epochs or departed.
 * d_transcript: NULL, or device [replicas][n_jobs][max_target][n_total] uint64 receiving
 * src<<32 | id at each delivery position.  *h_rounds = rounds executed.
 * ESTATE if no job is active or request_mode = 1.                            */
seneca_status seneca_replay_epochs(seneca_ctx* ctx, uint32_t n_epochs, uint64_t* d_transcript,
                                   uint64_t* h_rounds, void* stream);

/* The same call under the name north_star gives it (seneca_replay_epoch).      */
seneca_status seneca_replay_epoch(seneca_ctx* ctx, uint32_t n_epochs, uint64_t* d_transcript,
                                  uint64_t* h_rounds, void* stream);

/* As seneca_replay_epochs but for exactly n_rounds rounds (fewer if every job
 * departs).                                                                    */
seneca_status seneca_replay_rounds(seneca_ctx* ctx, uint64_t n_rounds, uint64_t* d_transcript,
                                   uint64_t* h_rounds, void* stream);

seneca_status seneca_read_state(const seneca_ctx* ctx, seneca_state_view* out);

/* Sharding with one shard per context (shard_mode 1).  seneca_shard_mailbox
 * returns this shard's mailbox (inside the workspace; peers write into it) so
 * the caller can map it into the other processes (e.g. CUDA IPC);
 * seneca_shard_attach takes d_peer_mailboxes[shards] -- every shard's mailbox
 * as addressable from this context's device (entry shard_rank may be NULL =
 * its own).  Rounds are ESTATE until attached; EINVAL for an unsharded or
 * shard_mode 0 context or a NULL peer.                                       */
seneca_status seneca_shard_mailbox(const seneca_ctx* ctx, void** d_mailbox, size_t* bytes);
seneca_status seneca_shard_attach(seneca_ctx* ctx, void* const* d_peer_mailboxes);

/* Synchronise `stream` and report a latched device-side error (an internal
 * consistency check failing) as ESTATE.                                        */
seneca_status seneca_sync_status(seneca_ctx* ctx, void* stream);

/* Number of kernel launches this context has issued (for gpu_launches).      */
uint64_t seneca_launch_count(const seneca_ctx* ctx);

/* Kernel timing.  seneca_profile(ctx, flags):
 *   bit 0  every kernel launch of this context is bracketed by CUDA events on
 *          its launch stream and the host waits for the end event (launches
 *          become synchronous; a replay is one launch); seneca_profile_read
 *          reports, per kernel, launches issued, launches timed and their
 *          summed event-measured duration;
 *   bit 1  the round kernel accumulates per-phase SM cycles into
 *          d_phase_cycles of the state view (clock reads inside the kernel:
 *          use for the phase split, not for timing).
 * Launch counts are always kept.                                              */
typedef struct {
    const char* name;      /* kernel name (static string)                       */
    uint64_t launches;     /* launches issued                                   */
    uint64_t sampled;      /* launches timed                                    */
    double   sampled_ms;   /* summed event-measured duration of timed launches  */
} seneca_kernel_stat;

seneca_status seneca_profile(seneca_ctx* ctx, uint32_t flags);
seneca_status seneca_profile_read(seneca_ctx* ctx, seneca_kernel_stat* out, uint32_t cap, uint32_t* n_classes);

void        seneca_destroy(seneca_ctx* ctx);
const char* seneca_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* SENECA_H */
