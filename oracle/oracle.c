/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU implementation of what the Seneca hot path
 * computes (arXiv 2511.13724, "Preparation Meets Opportunity"), written from the
 * paper and the readings listed in DESIGN.md §3.  It is the checker
 * the CUDA path is compared against.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  It shares no
 * source, header, table or helper with paper_2511_13724_b200/ and includes
 * nothing from it.
 *
 * Build (done by __graft_entry__.build() and oracle/__init__.py):
 *   gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -shared -fPIC
 * (no -march=native: the host has FMA and GCC would otherwise be free to
 *  contract a*b+c; -ffp-contract=off forbids it anyway).
 *
 * Citations: "P:Lnnn" = /root/reference/PAPER.md line nnn (the paper), with the
 * section / equation it falls in.  "R-xx" = a reading recorded in DESIGN.md §3.
 *
 * Parity status per function:
 *   philox4x32_10 ........ pinned (Random123 known-answer vectors)
 *   perm ................. pinned (exhaustive bijection; uniformity; independent Python transcription)
 *   MDP (Eqs. 1-9, grid) . pinned (Table 4 values, closed forms, exact-rational brute force)
 *   ODS replay ........... pinned by the SPEC worked example, closed forms (static tiers,
 *                          J=1 refill accounting), invariants I1-I10; exact decisions with
 *                          A-churn are "parity unpinned" beyond agreement with the second,
 *                          literal Python transcription (oracle/literal.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* ------------------------------------------------------------------------- */
/* Status codes (mirrors the meaning of the C-ABI codes; defined here anew).  */
enum { O_OK = 0, O_EINVAL = 1, O_ESTATE = 2, O_EPROTO = 3 };

/* Tier codes (R-O2): S = storage, E = encoded, D = decoded, A = augmented.   */
enum { T_S = 0, T_E = 1, T_D = 2, T_A = 3, SUBST = 4 };

/* ========================================================================= */
/* 1. PRNG.  The paper only says "a pseudo-random number generator" (P:L704,  */
/*    §5.2) and "predetermined pseudo-random sequence" (§1).  Reading  */
/*    R-O17: Philox4x32-10 (Salmon et al., Random123), splitmix64 key          */
/*    derivation, 6-round Feistel network with cycle walking.                 */
/* ========================================================================= */

void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }   /* key schedule */
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

uint64_t oracle_splitmix64(uint64_t x)
{
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* key(seed, purpose, a, b, c); purposes: INIT=1, REQ=2, SUB=3, REFILL=4 (R-O17) */
uint64_t oracle_key(uint64_t seed, uint64_t purpose, uint64_t a, uint64_t b, uint64_t c)
{
    uint64_t word = (purpose << 56) ^ (a << 48) ^ (c << 44) ^ b;
    return oracle_splitmix64(seed ^ oracle_splitmix64(word));
}

/* perm(K, n, x): keyed bijection of [0, n), 0 <= x < n (R-O17).  A Feistel
 * network on Z_a x Z_b with a = ceil(sqrt(n)), b = ceil(n / a)
 * (a*b >= n, a*b - n < a): x = L*b + R; even rounds L = (L + F) mod a with
 * F = floor(philox((R, rd, 0, 0), K)[0] * a / 2^32), odd rounds
 * R = (R + floor(philox((L, rd, 0, 0), K)[0] * b / 2^32)) mod b; restricted to
 * [0, n) by cycle walking (probability of a step < 1/b).  4 rounds for n >= 64;
 * 12 rounds for n < 64, where the halves are too small for 4 rounds to mix
 * (pairs chi-square, tests/test_oracle_prng.py; DESIGN.md R-O17).            */
static uint64_t isqrt_ceil(uint64_t n)   /* smallest a with a*a >= n */
{
    uint64_t a = (uint64_t)sqrt((double)n);
    while (a * a < n) ++a;
    while (a > 0 && (a - 1) * (a - 1) >= n) --a;
    return a;
}

uint64_t oracle_perm(uint64_t K, uint64_t n, uint64_t x)
{
    if (n <= 1) return 0;
    uint64_t a = isqrt_ceil(n);
    uint64_t b = (n + a - 1) / a;
    uint32_t key[2] = { (uint32_t)K, (uint32_t)(K >> 32) };
    do {
        uint64_t L = x / b, R = x % b;
        const uint32_t rounds = n < 64 ? 12u : 4u;
        for (uint32_t rd = 0; rd < rounds; ++rd) {
            uint32_t o[4];
            if ((rd & 1) == 0) {
                uint32_t ctr[4] = { (uint32_t)R, rd, 0, 0 };
                oracle_philox4x32_10(ctr, key, o);
                L = (L + (((uint64_t)o[0] * a) >> 32)) % a;
            } else {
                uint32_t ctr[4] = { (uint32_t)L, rd, 0, 0 };
                oracle_philox4x32_10(ctr, key, o);
                R = (R + (((uint64_t)o[0] * b) >> 32)) % b;
            }
        }
        x = L * b + R;
    } while (x >= n);
    return x;
}

/* perm(K, n, x) for x = x0 .. x0 + count - 1 into out[] (a loop over
 * oracle_perm, for the exhaustive / distribution pins in tests/).           */
void oracle_perm_block(uint64_t K, uint64_t n, uint64_t x0, uint64_t count, uint32_t* out)
{
    for (uint64_t t = 0; t < count; ++t) out[t] = (uint32_t)oracle_perm(K, n, x0 + t);
}

/* ========================================================================= */
/* 2. MDP: the DSI throughput model, §5.1, and the brute-force   */
/*    split search "for all combinations at 1% granularity" (§5.3).   */
/*    All arithmetic: IEEE binary64, one rounding per written operation, no   */
/*    contraction (R-M7).                                                     */
/* ========================================================================= */

typedef struct {                 /* one row of tab:model_vars     */
    double   t_gpu;              /* T_GPU      samples/s per node               */
    double   t_decode_augment;   /* T_{D+A}    samples/s per node               */
    double   t_augment;          /* T_A        samples/s per node               */
    double   b_nic;              /* B_NIC      bytes/s per node                 */
    double   b_pcie;             /* B_PCIe     bytes/s per node                 */
    double   b_cache;            /* B_cache    bytes/s                          */
    double   b_storage;          /* B_storage  bytes/s                          */
    double   model_bytes;        /* beta*N     bytes (R-M2)                     */
    uint64_t cache_bytes;        /* S_cache = S_mem (R-M5)                      */
    uint64_t n_total;            /* N_total                                     */
    uint64_t s_data;             /* S_data     bytes                            */
    uint32_t m_num, m_den;       /* M = m_num / m_den                           */
    uint32_t nodes;              /* n                                           */
    uint32_t gpus_per_node;
    uint8_t  nvlink_intra, nvlink_inter, comm_mapping, pad[5];
} oracle_profile;

typedef struct {
    uint8_t  p_e, p_d, p_a;
    uint8_t  lim_a, lim_d, lim_e, lim_s, pad;
    double   v, dsi_a, dsi_d, dsi_e, dsi_s;
} oracle_result;

/* limiting-factor codes (R-M8 / SPEC enumeration order) */
enum { L_CACHE = 0, L_NIC = 1, L_PCIE = 2, L_CPU_AUG = 3, L_CPU_DEC_AUG = 4, L_GPU = 5, L_STORAGE = 6 };

/* C = 2(n-1)/n x betaN, P:L529 (§5.1, ring all-reduce overhead) */
double oracle_comm_overhead(uint64_t participants, double model_bytes)
{
    if (participants <= 1) return 0.0;
    double frac = (double)(2 * (participants - 1)) / (double)participants;
    return frac * model_bytes;
}

/* first minimal term wins (ties -> earlier term, R-M8) */
static void take_min(double term, int code, double *best, int *lim)
{
    if (term < *best) { *best = term; *lim = code; }
}

/* Eqs. 1-4. */
void oracle_tiers(const oracle_profile *p, double dsi[4] /* A,D,E,S */, uint8_t lim[4])
{
    double Sd = (double)p->s_data;
    double MS = (double)((uint64_t)p->m_num * p->s_data) / (double)p->m_den;   /* M x S_data */
    uint64_t p_nw = p->comm_mapping ? p->gpus_per_node : p->nodes;             /* R-M1 */
    uint64_t p_pc = p->comm_mapping ? p->nodes : p->gpus_per_node;
    /* intra-node NVLink -> C_PCIe = 0; inter-node NVLink -> both 0 */
    double C_nw = p->nvlink_inter ? 0.0 : oracle_comm_overhead(p_nw, p->model_bytes);
    double C_pc = (p->nvlink_intra || p->nvlink_inter) ? 0.0 : oracle_comm_overhead(p_pc, p->model_bytes);
    double nd = (double)p->nodes;

    double nic_ms  = nd * p->b_nic;
    double pcie_ms = nd * p->b_pcie;
    double gpu     = nd * p->t_gpu;

    /* Eq. 1: DSI_A = min(B_cache/(M S), n B_NIC/(M S + C_nw), n B_PCIe/(M S + C_PCIe), n T_GPU) */
    double a = 1.0 / 0.0; int la = -1;
    take_min(p->b_cache / MS, L_CACHE, &a, &la);
    take_min(nic_ms / (MS + C_nw), L_NIC, &a, &la);
    take_min(pcie_ms / (MS + C_pc), L_PCIE, &a, &la);
    take_min(gpu, L_GPU, &a, &la);

    /* Eq. 2: DSI_D adds n T_A; missing comma read as two terms (R-M4) */
    double d = 1.0 / 0.0; int ld = -1;
    take_min(p->b_cache / MS, L_CACHE, &d, &ld);
    take_min(nic_ms / (MS + C_nw), L_NIC, &d, &ld);
    take_min(nd * p->t_augment, L_CPU_AUG, &d, &ld);
    take_min(pcie_ms / (MS + C_pc), L_PCIE, &d, &ld);
    take_min(gpu, L_GPU, &d, &ld);

    /* Eq. 3: DSI_E: cache and NIC over S_data (encoded), n T_{D+A}, PCIe over M S */
    double e = 1.0 / 0.0; int le = -1;
    take_min(p->b_cache / Sd, L_CACHE, &e, &le);
    take_min(nic_ms / (Sd + C_nw), L_NIC, &e, &le);
    take_min(nd * p->t_decode_augment, L_CPU_DEC_AUG, &e, &le);
    take_min(pcie_ms / (MS + C_pc), L_PCIE, &e, &le);
    take_min(gpu, L_GPU, &e, &le);

    /* Eq. 4: DSI_S = min(DSI_E, B_storage / S_data) */
    double st = p->b_storage / Sd;
    double s = e; int ls = le;
    if (st < e) { s = st; ls = L_STORAGE; }

    dsi[0] = a; dsi[1] = d; dsi[2] = e; dsi[3] = s;
    lim[0] = (uint8_t)la; lim[1] = (uint8_t)ld; lim[2] = (uint8_t)le; lim[3] = (uint8_t)ls;
}

/* Eqs. 5-8 with the
 * fractional counts floored (R-M6), exactly, in integers:
 *   x_A S_mem / (M S_data) = (p/100) S_mem m_den / (m_num S_data)
 * counts[] = {N_A, N_D, N_E, N_storage}.                                     */
void oracle_split_counts(const oracle_profile *p, uint32_t pe, uint32_t pd, uint32_t pa, uint64_t counts[4])
{
    typedef unsigned __int128 u128;
    u128 den_ad = (u128)100 * p->m_num * p->s_data;
    u128 den_e  = (u128)100 * p->s_data;
    uint64_t capA = (uint64_t)(((u128)pa * p->cache_bytes * p->m_den) / den_ad);
    uint64_t capD = (uint64_t)(((u128)pd * p->cache_bytes * p->m_den) / den_ad);
    uint64_t capE = (uint64_t)(((u128)pe * p->cache_bytes) / den_e);
    uint64_t N = p->n_total;
    uint64_t nA = N < capA ? N : capA;                                /* Eq. 5 */
    uint64_t nD = (N - nA) < capD ? (N - nA) : capD;                   /* Eq. 6 */
    uint64_t nE = (N - nA - nD) < capE ? (N - nA - nD) : capE;         /* Eq. 7 */
    uint64_t nS = N - nA - nD - nE;                                    /* Eq. 8 */
    counts[0] = nA; counts[1] = nD; counts[2] = nE; counts[3] = nS;
}

/* Eq. 9, literal term order (R-M7). */
double oracle_model_eval(const oracle_profile *p, uint32_t pe, uint32_t pd, uint32_t pa,
                         oracle_result *out, uint64_t counts_out[4])
{
    double dsi[4]; uint8_t lim[4]; uint64_t c[4];
    oracle_tiers(p, dsi, lim);
    oracle_split_counts(p, pe, pd, pa, c);
    double dN = (double)p->n_total;
    double fA = (double)c[0] / dN;
    double fD = (double)c[1] / dN;
    double fE = (double)c[2] / dN;
    double fS = (double)c[3] / dN;
    double tA = fA * dsi[0];
    double tD = fD * dsi[1];
    double tE = fE * dsi[2];
    double tS = fS * dsi[3];
    double v = tA + tD;
    v = v + tE;
    v = v + tS;
    if (out) {
        out->p_e = (uint8_t)pe; out->p_d = (uint8_t)pd; out->p_a = (uint8_t)pa;
        out->lim_a = lim[0]; out->lim_d = lim[1]; out->lim_e = lim[2]; out->lim_s = lim[3];
        out->pad = 0;
        out->v = v; out->dsi_a = dsi[0]; out->dsi_d = dsi[1]; out->dsi_e = dsi[2]; out->dsi_s = dsi[3];
    }
    if (counts_out) memcpy(counts_out, c, sizeof c);
    return v;
}

/* number of splits on a grid of step g (g | 100): (100/g+1)(100/g+2)/2 */
uint64_t oracle_num_splits(uint32_t g)
{
    uint64_t s = 100 / g;
    return (s + 1) * (s + 2) / 2;
}

/* Brute force over all splits summing to 100 % (R-M9), enumerated
 * p_E = 100, 100-g, ..., 0; for each, p_D = 100-p_E, ..., 0.  Argmax with
 * exact ties -> smallest enumeration index (higher x_E, then higher x_D; R-M8). */
int oracle_mdp_sweep(const oracle_profile *profiles, uint64_t n_profiles, uint32_t g,
                     oracle_result *results, double *grid /* may be NULL */)
{
    if (g == 0 || g > 100 || 100 % g) return O_EINVAL;
    uint64_t ns = oracle_num_splits(g);
    for (uint64_t i = 0; i < n_profiles; ++i) {
        const oracle_profile *p = &profiles[i];
        oracle_result best; int have = 0;
        uint64_t idx = 0;
        for (int pe = 100; pe >= 0; pe -= (int)g) {
            for (int pd = 100 - pe; pd >= 0; pd -= (int)g) {
                int pa = 100 - pe - pd;
                oracle_result r;
                double v = oracle_model_eval(p, (uint32_t)pe, (uint32_t)pd, (uint32_t)pa, &r, NULL);
                if (grid) grid[i * ns + idx] = v;
                if (!have || v > best.v) { best = r; have = 1; }
                ++idx;
            }
        }
        results[i] = best;
    }
    return O_OK;
}

/* ODS metadata formula, P:L707-710 (§5.2): 1 bit/sample/job + 1 B/sample. */
uint64_t oracle_metadata_bytes(uint64_t n_total, uint32_t n_jobs)
{
    return (uint64_t)n_jobs * ((n_total + 7) / 8) + n_total;
}

/* ========================================================================= */
/* 3. ODS replay: §5.2, steps 1-6 of fig:cache_aware_sampling,  */
/*    made concrete by readings R-O1..R-O20.                  */
/* ========================================================================= */

enum { PUR_INIT = 1, PUR_REQ = 2, PUR_SUB = 3, PUR_REFILL = 4 };

typedef struct {
    uint64_t served[4];     /* by tier code S,E,D,A                         */
    uint64_t subst[4];      /* substitutes by tier (S unused)               */
    uint64_t req_hits[4];   /* requested samples that hit, by tier          */
    uint64_t digest;        /* sum of splitmix64(q<<35 | src<<32 | id)      */
} oracle_stats;

typedef struct {
    uint64_t N, W;                 /* samples, 64-bit words per bitmap       */
    uint32_t J;
    uint32_t batch[32], target[32];
    uint64_t cap_e, cap_d, cap_a;
    uint64_t seed;
    uint64_t *bm_e, *bm_d, *bm_a;  /* residency ("status")           */
    uint64_t *seen;                /* [J][W]  per-job seen bit vector */
    uint64_t *cons;                /* [J][W]  per-job consumer set (R-O5)     */
    uint64_t c[32], e[32], n[32];  /* cursor, epoch, consumed in epoch        */
    int      active[32];
    uint64_t r;                    /* round counter                          */
    uint32_t max_target;
    oracle_stats *stats;           /* [J][max_target]                         */
    uint64_t evicted_total, refilled_total;
    uint64_t *transcript;          /* optional [J][max_target][N]: src<<32|id */
    int      evict_all;            /* evict_tiers = ALL (R-O21): consumer sets and
                                      eviction for every cached tier            */
    int      baseline;             /* the uniform no-evict sampler (R-O22)     */
    uint64_t arrival[32];          /* job arrival rounds (R-O23)              */
    int      pending[32];          /* not yet arrived                         */
    int      cold, warm;           /* cold start (R-O24): admission until full */
} ods_t;

/* tiers that carry consumer sets and can be evicted: A (R-O5), or all (R-O21);
 * none for the no-evict baseline sampler (R-O22) */
static int tracked(const ods_t *o, int t)
{
    if (o->baseline) return 0;
    return t == T_A || (o->evict_all && t != T_S);
}

static int  bit_get(const uint64_t *bm, uint64_t i) { return (int)((bm[i >> 6] >> (i & 63)) & 1u); }
static void bit_set(uint64_t *bm, uint64_t i)       { bm[i >> 6] |= (uint64_t)1 << (i & 63); }
static void bit_clr(uint64_t *bm, uint64_t i)       { bm[i >> 6] &= ~((uint64_t)1 << (i & 63)); }

static int tier_of(const ods_t *o, uint64_t i)
{
    if (bit_get(o->bm_a, i)) return T_A;
    if (bit_get(o->bm_d, i)) return T_D;
    if (bit_get(o->bm_e, i)) return T_E;
    return T_S;
}

static uint64_t valid_mask(const ods_t *o, uint64_t w)
{
    uint64_t lo = w * 64, hi = lo + 64;
    if (hi <= o->N) return ~(uint64_t)0;
    if (lo >= o->N) return 0;
    return ((uint64_t)1 << (o->N - lo)) - 1;
}

/* word w of pool_t for job j (R-O2):
 *   pool_t = {i : tier(i) = t, i not in seen_j, (t != A or i not in cons_j)}
 * t = T_S: storage-resident samples {i : tier(i) = S} (refill pool, R-O8).  */
static uint64_t pool_word(const ods_t *o, int t, uint32_t j, uint64_t w)
{
    if (t == T_S) return ~(o->bm_e[w] | o->bm_d[w] | o->bm_a[w]) & valid_mask(o, w);
    const uint64_t *sj = o->seen + (uint64_t)j * o->W;
    const uint64_t *cj = o->cons + (uint64_t)j * o->W;
    if (t == T_A) return o->bm_a[w] & ~sj[w] & ~cj[w];
    if (t == T_D) return o->bm_d[w] & ~sj[w];
    return o->bm_e[w] & ~sj[w];
}

static uint64_t pool_size(const ods_t *o, int t, uint32_t j)
{
    uint64_t P = 0;
    for (uint64_t w = 0; w < o->W; ++w) P += (uint64_t)__builtin_popcountll(pool_word(o, t, j, w));
    return P;
}

typedef struct { uint64_t rank; uint64_t u; } rank_pair;
static int cmp_rank(const void *a, const void *b)
{
    const rank_pair *x = a, *y = b;
    return x->rank < y->rank ? -1 : x->rank > y->rank;
}

/* ids[u] = pool_t[ranks[u]] where pool_t is read as the ASCENDING list of its
 * members (R-O2).  The ranks are sorted first (library qsort) so one pass over
 * the ascending bitmap words yields every requested element.               */
static void pool_select(const ods_t *o, int t, uint32_t j, const uint64_t *ranks, uint64_t k, uint64_t *ids)
{
    if (k == 0) return;
    rank_pair *rp = malloc(k * sizeof *rp);
    for (uint64_t u = 0; u < k; ++u) { rp[u].rank = ranks[u]; rp[u].u = u; }
    qsort(rp, k, sizeof *rp, cmp_rank);
    uint64_t next = 0, before = 0;              /* members in words < w */
    for (uint64_t w = 0; w < o->W && next < k; ++w) {
        uint64_t bits = pool_word(o, t, j, w);
        uint64_t pc = (uint64_t)__builtin_popcountll(bits);
        while (next < k && rp[next].rank < before + pc) {
            uint64_t want = rp[next].rank - before, b = bits;
            for (uint64_t s = 0; s < want; ++s) b &= b - 1;   /* drop lower members */
            ids[rp[next].u] = w * 64 + (uint64_t)__builtin_ctzll(b);
            ++next;
        }
        before += pc;
    }
    free(rp);
}

void oracle_ods_destroy(void *h)
{
    ods_t *o = h;
    if (!o) return;
    free(o->bm_e); free(o->bm_d); free(o->bm_a); free(o->seen); free(o->cons);
    free(o->stats); free(o->transcript); free(o);
}

/* init_cache, warm start (R-O9): iota = perm(key(seed, INIT), N, .);
 * positions [0,cap_A) -> A, next cap_D -> D, next cap_E -> E, rest -> S. */
void *oracle_ods_create(uint64_t N, uint32_t J, const uint32_t *batch, const uint32_t *target,
                        uint64_t cap_e, uint64_t cap_d, uint64_t cap_a, uint64_t seed,
                        int keep_transcript, int evict_all, int baseline)
{
    if (N == 0 || N >= ((uint64_t)1 << 32) || J == 0 || J > 32) return NULL;
    if (cap_e + cap_d + cap_a > N) return NULL;
    ods_t *o = calloc(1, sizeof *o);
    o->N = N; o->J = J; o->W = (N + 63) / 64;
    o->cap_e = cap_e; o->cap_d = cap_d; o->cap_a = cap_a; o->seed = seed;
    o->evict_all = evict_all != 0;
    o->baseline = baseline != 0;
    o->max_target = 0;
    for (uint32_t j = 0; j < J; ++j) {
        if (batch[j] == 0 || target[j] == 0) { free(o); return NULL; }
        o->batch[j] = batch[j]; o->target[j] = target[j];
        if (target[j] > o->max_target) o->max_target = target[j];
        o->active[j] = 1;
    }
    o->bm_e = calloc(o->W, 8); o->bm_d = calloc(o->W, 8); o->bm_a = calloc(o->W, 8);
    o->seen = calloc((size_t)J * o->W, 8); o->cons = calloc((size_t)J * o->W, 8);
    o->stats = calloc((size_t)J * o->max_target, sizeof(oracle_stats));
    if (keep_transcript) o->transcript = calloc((size_t)J * o->max_target * N, 8);
    uint64_t K = oracle_key(seed, PUR_INIT, 0, 0, 0);
    for (uint64_t pos = 0; pos < cap_a + cap_d + cap_e; ++pos) {
        uint64_t i = oracle_perm(K, N, pos);
        if (pos < cap_a) bit_set(o->bm_a, i);
        else if (pos < cap_a + cap_d) bit_set(o->bm_d, i);
        else bit_set(o->bm_e, i);
    }
    return o;
}

/* Job arrivals (R-O23, SURVEY 8(f) NEXT-1 job-arrival traces): job j takes
 * part from round arrival[j] on (0: from the start).  A round in which no job
 * is active while arrivals are pending is idle (it only advances the round
 * counter).  Call before the first round.                                    */
void oracle_ods_set_arrivals(void *h, const uint32_t *arrival)
{
    ods_t *o = h;
    for (uint32_t j = 0; j < o->J; ++j) {
        o->arrival[j] = arrival ? arrival[j] : 0;
        o->pending[j] = o->arrival[j] > o->r;
        if (o->pending[j]) o->active[j] = 0;
    }
}

/* jobs whose arrival round has come join the active set (start of a round) */
/* Cold start (R-O24): every tier starts empty; until all
 * three are full once, the storage-fetched samples of each round are admitted
 * at the round end instead of random refills.  Call before the first round. */
void oracle_ods_set_cold(void *h)
{
    ods_t *o = h;
    memset(o->bm_e, 0, o->W * 8); memset(o->bm_d, 0, o->W * 8); memset(o->bm_a, 0, o->W * 8);
    o->cold = 1;
    o->warm = 0;
}

static void arrive(ods_t *o)
{
    for (uint32_t j = 0; j < o->J; ++j)
        if (o->pending[j] && o->arrival[j] <= o->r) { o->pending[j] = 0; o->active[j] = 1; }
}

static int any_pending(const ods_t *o)
{
    for (uint32_t j = 0; j < o->J; ++j) if (o->pending[j]) return 1;
    return 0;
}

/* need_j = min(B_j, N - n_j) */
uint64_t oracle_ods_need(void *h, uint32_t j)
{
    ods_t *o = h;
    uint64_t rem = o->N - o->n[j];
    return o->batch[j] < rem ? o->batch[j] : rem;
}

/* One round = one ods_next_batch: a batch for every listed job, then maintain
 * (R-O7, R-O11).  jobs[] must be distinct active jobs.  requested: NULL for
 * the generated request stream (R-O1/R-O3), else [n_jobs][bmax] caller IDs
 * (R-O20).  Outputs in jobs[] order: out_ids/out_src [n_jobs][bmax],
 * out_lens [n_jobs].                                                       */
int oracle_ods_round(void *h, const uint32_t *jobs, uint32_t n_jobs, const uint32_t *requested,
                     uint32_t bmax, uint32_t *out_ids, uint8_t *out_src, uint32_t *out_lens)
{
    ods_t *o = h;
    arrive(o);
    if (n_jobs == 0 || n_jobs > o->J) return O_EINVAL;
    for (uint32_t x = 0; x < n_jobs; ++x) {
        if (jobs[x] >= o->J) return O_EINVAL;
        for (uint32_t y = 0; y < x; ++y) if (jobs[y] == jobs[x]) return O_EINVAL;
        if (!o->active[jobs[x]]) return O_ESTATE;
        if (oracle_ods_need(o, jobs[x]) > bmax) return O_EINVAL;
    }
    /* caller-supplied requests: distinct, unseen, in range (S:L303 pre) */
    if (requested) {
        for (uint32_t x = 0; x < n_jobs; ++x) {
            uint32_t j = jobs[x];
            uint64_t need = oracle_ods_need(o, j);
            const uint32_t *R = requested + (uint64_t)x * bmax;
            for (uint64_t s = 0; s < need; ++s) {
                if (R[s] >= o->N) return O_EPROTO;
                if (bit_get(o->seen + (uint64_t)j * o->W, R[s])) return O_EPROTO;
                for (uint64_t s2 = 0; s2 < s; ++s2) if (R[s2] == R[s]) return O_EPROTO;
            }
        }
    }

    uint64_t a_served_cap = 0;
    for (uint32_t x = 0; x < n_jobs; ++x) a_served_cap += oracle_ods_need(o, jobs[x]);
    uint64_t *a_served = malloc((a_served_cap + 1) * 8), n_a_served = 0;
    /* storage fetches of the round per job, slot order (cold-start admission, R-O24) */
    uint64_t *fetched[32] = {0}, n_fetched[32] = {0};
    int departing[32] = {0};

    for (uint32_t x = 0; x < n_jobs; ++x) {
        uint32_t j = jobs[x];
        uint64_t *seen_j = o->seen + (uint64_t)j * o->W;
        uint64_t *cons_j = o->cons + (uint64_t)j * o->W;
        uint64_t need = oracle_ods_need(o, j);
        uint64_t *R = malloc((need + 1) * 8);
        uint32_t *out = out_ids + (uint64_t)x * bmax;
        uint8_t *src = out_src + (uint64_t)x * bmax;

        /* step 1: the request.  Generated stream (R-O1): the first
         * `need` ids pi_j(pos), pos = c_j, c_j+1, ... (mod N), not in seen_j. */
        if (requested) {
            for (uint64_t s = 0; s < need; ++s) R[s] = requested[(uint64_t)x * bmax + s];
        } else {
            uint64_t K = oracle_key(o->seed, PUR_REQ, j, o->e[j], 0);
            uint64_t pos = o->c[j], taken = 0, last = pos;
            while (taken < need) {
                uint64_t i = oracle_perm(K, o->N, pos);
                if (!bit_get(seen_j, i)) { R[taken++] = i; last = pos; }
                pos = (pos + 1) % o->N;
            }
            o->c[j] = (last + 1) % o->N;
        }

        /* step 2: hits vs misses via status (R-O13/R-O19); hits join seen_j now */
        uint64_t *miss = malloc((need + 1) * 8), m = 0;
        for (uint64_t s = 0; s < need; ++s) {
            uint64_t i = R[s];
            int t = tier_of(o, i);
            if (t == T_E || t == T_D || (t == T_A && (o->baseline || !bit_get(cons_j, i)))) {
                out[s] = (uint32_t)i; src[s] = (uint8_t)t;
                bit_set(seen_j, i);
            } else {
                miss[m++] = s;
            }
        }

        /* step 2: replace misses with unseen cached samples,
         * tiers A -> D -> E, uniform by keyed ranks over the ascending pool (R-O2) */
        uint64_t q = 0;
        const int order[3] = { T_A, T_D, T_E };
        for (int ti = 0; ti < 3 && q < m && !o->baseline; ++ti) {   /* R-O22: no substitution */
            int t = order[ti];
            uint64_t P = pool_size(o, t, j);
            uint64_t k = (m - q) < P ? (m - q) : P;
            if (k == 0) continue;
            uint64_t K = oracle_key(o->seed, PUR_SUB, j, o->r, (uint64_t)t);
            uint64_t *ranks = malloc(k * 8), *ids = malloc(k * 8);
            for (uint64_t u = 0; u < k; ++u) ranks[u] = oracle_perm(K, P, u);
            pool_select(o, t, j, ranks, k, ids);
            for (uint64_t u = 0; u < k; ++u) {
                out[miss[q + u]] = (uint32_t)ids[u];
                src[miss[q + u]] = (uint8_t)(t | SUBST);
            }
            free(ranks); free(ids);
            q += k;
        }
        /* remaining misses are fetched from storage (R-O18) */
        for (uint64_t u = q; u < m; ++u) { out[miss[u]] = (uint32_t)R[miss[u]]; src[miss[u]] = T_S; }

        /* steps 3-4: respond, update seen; consumer set for A (R-O5)
         * -- for every cached source under evict_tiers = ALL (R-O21) */
        oracle_stats *st = &o->stats[(uint64_t)j * o->max_target + o->e[j]];
        for (uint64_t s = 0; s < need; ++s) {
            uint64_t i = out[s];
            int t = src[s] & 3, sub = (src[s] & SUBST) != 0;
            bit_set(seen_j, i);
            if (tracked(o, t)) { bit_set(cons_j, i); a_served[n_a_served++] = i; }
            if (src[s] == T_S && o->cold && !o->warm) {
                if (!fetched[j]) fetched[j] = malloc((need + 1) * 8);
                fetched[j][n_fetched[j]++] = i;
            }
            st->served[t]++;
            if (sub) st->subst[t]++;
            else if (t != T_S) st->req_hits[t]++;
            uint64_t qpos = o->n[j] + s;
            st->digest += oracle_splitmix64((qpos << 35) | ((uint64_t)src[s] << 32) | i);
            if (o->transcript)
                o->transcript[((uint64_t)j * o->max_target + o->e[j]) * o->N + qpos] = ((uint64_t)src[s] << 32) | i;
        }
        out_lens[x] = (uint32_t)need;

        /* step 6: epoch end resets seen_j (R-O16) */
        o->n[j] += need;
        if (o->n[j] == o->N) {
            memset(seen_j, 0, o->W * 8);
            o->e[j] += 1; o->c[j] = 0; o->n[j] = 0;
            if (o->e[j] == o->target[j]) departing[j] = 1;
        }
        free(R); free(miss);
    }

    /* step 5: maintain, once per round (R-O6, R-O7, R-O8). */
    int changed = 0, any_active = 0;
    for (uint32_t j = 0; j < o->J; ++j) {
        if (departing[j]) { o->active[j] = 0; changed = 1; }
        if (o->active[j]) any_active = 1;
    }
    if (any_active) {
        /* candidates, ascending and distinct: the cached-served ids of the round,
         * or every tracked entry when the active set changed (R-O6) */
        uint64_t *cand, nc = 0;
        if (changed) {
            cand = malloc((o->N + 1) * 8);
            for (uint64_t i = 0; i < o->N; ++i) if (tracked(o, tier_of(o, i))) cand[nc++] = i;
        } else {
            cand = malloc((n_a_served + 1) * 8);
            memcpy(cand, a_served, n_a_served * 8);
            rank_pair *tmp = malloc((n_a_served + 1) * sizeof *tmp);
            for (uint64_t u = 0; u < n_a_served; ++u) { tmp[u].rank = cand[u]; tmp[u].u = u; }
            qsort(tmp, n_a_served, sizeof *tmp, cmp_rank);
            for (uint64_t u = 0; u < n_a_served; ++u)
                if (nc == 0 || cand[nc - 1] != tmp[u].rank) cand[nc++] = tmp[u].rank;
            free(tmp);
        }
        /* evict candidates consumed by every active job */
        uint64_t *evict = malloc((nc + 1) * 8), ne = 0, ne_t[4] = {0, 0, 0, 0};
        for (uint64_t u = 0; u < nc; ++u) {
            uint64_t i = cand[u];
            int t = tier_of(o, i);
            if (!tracked(o, t)) continue;
            int all = 1;
            for (uint32_t a = 0; a < o->J; ++a)
                if (o->active[a] && !bit_get(o->cons + (uint64_t)a * o->W, i)) { all = 0; break; }
            if (all) { evict[ne++] = i; ne_t[t]++; }
        }
        /* refill (R-O8, R-O21): deficit_t = cap_t - |t| after eviction for the
         * tracked tiers; k = min(sum of deficits, |pool_S| at round start) ranks
         * rho(0..k-1) of one keyed stream, assigned tier by tier A -> D -> E.
         * Cold start (R-O24): until every tier has been full once, every tier's
         * deficit is filled instead from this round's storage fetches -- in
         * ascending job order, slot order, first occurrence, only ids that were
         * storage-resident at round start. */
        const int admit = o->cold && !o->warm;
        uint64_t deficit[4] = {0, 0, 0, 0};
        const uint64_t caps[4] = {0, o->cap_e, o->cap_d, o->cap_a};
        const uint64_t *bms[4] = {NULL, o->bm_e, o->bm_d, o->bm_a};
        for (int t = T_E; t <= T_A; ++t) {
            if (!tracked(o, t) && !admit) continue;
            uint64_t size = 0;
            for (uint64_t w = 0; w < o->W; ++w) size += (uint64_t)__builtin_popcountll(bms[t][w]);
            deficit[t] = caps[t] - (size - ne_t[t]);
        }
        uint64_t PS = pool_size(o, T_S, 0);
        uint64_t want = deficit[T_A] + deficit[T_D] + deficit[T_E];
        uint64_t k = want < PS ? want : PS;
        uint64_t *fill = NULL;
        if (admit) {
            uint64_t total = 0;
            for (uint32_t j = 0; j < o->J; ++j) total += n_fetched[j];
            fill = malloc((total + 1) * 8);
            uint64_t nf = 0;
            for (uint32_t j = 0; j < o->J; ++j)
                for (uint64_t u = 0; u < n_fetched[j]; ++u) {
                    uint64_t i = fetched[j][u];
                    if (tier_of(o, i) != T_S) continue;            /* cached at round start */
                    int dup = 0;
                    for (uint64_t v = 0; v < nf && !dup; ++v) dup = fill[v] == i;
                    if (!dup && nf < want) fill[nf++] = i;
                }
            k = nf;
        } else if (k) {
            uint64_t K = oracle_key(o->seed, PUR_REFILL, 0, o->r, 0);
            uint64_t *ranks = malloc(k * 8);
            fill = malloc(k * 8);
            for (uint64_t u = 0; u < k; ++u) ranks[u] = oracle_perm(K, PS, u);
            pool_select(o, T_S, 0, ranks, k, fill);
            free(ranks);
        }
        for (uint64_t u = 0; u < ne; ++u) {
            bit_clr(o->bm_a, evict[u]); bit_clr(o->bm_d, evict[u]); bit_clr(o->bm_e, evict[u]);
            for (uint32_t a = 0; a < o->J; ++a) bit_clr(o->cons + (uint64_t)a * o->W, evict[u]);
        }
        {
            const int order[3] = { T_A, T_D, T_E };
            uint64_t u = 0;
            for (int ti = 0; ti < 3; ++ti) {
                int t = order[ti];
                uint64_t end = u + deficit[t];
                if (end > k) end = k;
                uint64_t *bm = t == T_A ? o->bm_a : (t == T_D ? o->bm_d : o->bm_e);
                for (; u < end; ++u) bit_set(bm, fill[u]);
            }
        }
        if (admit) {                                            /* warm once every tier is full */
            uint64_t size[4] = {0, 0, 0, 0};
            for (uint64_t w = 0; w < o->W; ++w) {
                size[T_E] += (uint64_t)__builtin_popcountll(o->bm_e[w]);
                size[T_D] += (uint64_t)__builtin_popcountll(o->bm_d[w]);
                size[T_A] += (uint64_t)__builtin_popcountll(o->bm_a[w]);
            }
            if (size[T_E] == o->cap_e && size[T_D] == o->cap_d && size[T_A] == o->cap_a) o->warm = 1;
        }
        o->evicted_total += ne;
        o->refilled_total += k;
        free(cand); free(evict); free(fill);
    }
    o->r += 1;
    free(a_served);
    for (uint32_t j = 0; j < 32; ++j) free(fetched[j]);
    return O_OK;
}

/* Run n_rounds rounds over all active jobs (ascending).  Returns the number of
 * rounds executed (stops early when no job is active).                       */
uint64_t oracle_ods_replay_rounds(void *h, uint64_t n_rounds)
{
    ods_t *o = h;
    uint32_t jobs[32], *ids = NULL; uint8_t *src = NULL; uint32_t lens[32];
    uint32_t bmax = 0;
    for (uint32_t j = 0; j < o->J; ++j) if (o->batch[j] > bmax) bmax = o->batch[j];
    ids = malloc((size_t)o->J * bmax * 4); src = malloc((size_t)o->J * bmax);
    uint64_t done = 0;
    for (; done < n_rounds; ++done) {
        arrive(o);
        uint32_t nj = 0;
        for (uint32_t j = 0; j < o->J; ++j) if (o->active[j]) jobs[nj++] = j;
        if (nj == 0) {
            if (!any_pending(o)) break;
            o->r += 1;                                  /* idle round (R-O23) */
            continue;
        }
        oracle_ods_round(o, jobs, nj, NULL, bmax, ids, src, lens);
    }
    free(ids); free(src);
    return done;
}

/* Replay until every job active at the call has completed n_epochs more
 * epochs (or departed).  Returns the number of rounds executed.            */
uint64_t oracle_ods_replay_epochs(void *h, uint32_t n_epochs)
{
    ods_t *o = h;
    uint64_t goal[32]; int tracked[32];
    for (uint32_t j = 0; j < o->J; ++j) {
        tracked[j] = o->active[j] || o->pending[j];
        goal[j] = o->e[j] + n_epochs;
    }
    uint64_t rounds = 0;
    for (;;) {
        int pending = 0;
        for (uint32_t j = 0; j < o->J; ++j)
            if (tracked[j] && (o->active[j] || o->pending[j]) && o->e[j] < goal[j]) pending = 1;
        if (!pending) break;
        rounds += oracle_ods_replay_rounds(o, 1);
    }
    return rounds;
}

/* ---- state injection / readback for tests -------------------------------- */
/* Overwrite residency, seen and consumer sets (worked examples such as SPEC
 * S:L307 need a hand-built state).  tier: codes per sample; seen/cons: 0/1
 * bytes [J][N] (NULL = leave unchanged).                                    */
void oracle_ods_set_state(void *h, const uint8_t *tier, const uint8_t *seen, const uint8_t *cons)
{
    ods_t *o = h;
    memset(o->bm_e, 0, o->W * 8); memset(o->bm_d, 0, o->W * 8); memset(o->bm_a, 0, o->W * 8);
    for (uint64_t i = 0; i < o->N; ++i) {
        if (tier[i] == T_E) bit_set(o->bm_e, i);
        else if (tier[i] == T_D) bit_set(o->bm_d, i);
        else if (tier[i] == T_A) bit_set(o->bm_a, i);
    }
    for (uint32_t j = 0; j < o->J; ++j)
        for (uint64_t i = 0; i < o->N; ++i) {
            if (seen) { if (seen[(uint64_t)j * o->N + i]) bit_set(o->seen + (uint64_t)j * o->W, i);
                        else bit_clr(o->seen + (uint64_t)j * o->W, i); }
            if (cons) { if (cons[(uint64_t)j * o->N + i]) bit_set(o->cons + (uint64_t)j * o->W, i);
                        else bit_clr(o->cons + (uint64_t)j * o->W, i); }
        }
    /* n_j follows |seen_j| (I10) */
    if (seen)
        for (uint32_t j = 0; j < o->J; ++j) {
            uint64_t cnt = 0;
            for (uint64_t w = 0; w < o->W; ++w) cnt += (uint64_t)__builtin_popcountll(o->seen[(uint64_t)j * o->W + w]);
            o->n[j] = cnt;
        }
}

/* ---- state readback for tests ------------------------------------------- */
uint64_t oracle_ods_round_index(void *h) { return ((ods_t *)h)->r; }
uint32_t oracle_ods_max_target(void *h) { return ((ods_t *)h)->max_target; }

void oracle_ods_job_state(void *h, uint64_t *c, uint64_t *e, uint64_t *n, int32_t *active)
{
    ods_t *o = h;
    for (uint32_t j = 0; j < o->J; ++j) { c[j] = o->c[j]; e[j] = o->e[j]; n[j] = o->n[j]; active[j] = o->active[j]; }
}

/* tier codes per sample, seen/cons as 0/1 bytes [J][N] */
void oracle_ods_read_state(void *h, uint8_t *tier, uint8_t *seen, uint8_t *cons)
{
    ods_t *o = h;
    for (uint64_t i = 0; i < o->N; ++i) tier[i] = (uint8_t)tier_of(o, i);
    for (uint32_t j = 0; j < o->J; ++j)
        for (uint64_t i = 0; i < o->N; ++i) {
            if (seen) seen[(uint64_t)j * o->N + i] = (uint8_t)bit_get(o->seen + (uint64_t)j * o->W, i);
            if (cons) cons[(uint64_t)j * o->N + i] = (uint8_t)bit_get(o->cons + (uint64_t)j * o->W, i);
        }
}

/* stats [J][max_target] */
void oracle_ods_read_stats(void *h, oracle_stats *out, uint64_t *evicted, uint64_t *refilled)
{
    ods_t *o = h;
    memcpy(out, o->stats, (size_t)o->J * o->max_target * sizeof(oracle_stats));
    if (evicted) *evicted = o->evicted_total;
    if (refilled) *refilled = o->refilled_total;
}

/* transcript [J][max_target][N] of src<<32|id; returns 0 if not kept */
int oracle_ods_read_transcript(void *h, uint64_t *out)
{
    ods_t *o = h;
    if (!o->transcript) return 0;
    memcpy(out, o->transcript, (size_t)o->J * o->max_target * o->N * 8);
    return 1;
}

/* ========================================================================= */
/* 4. Epoch model on top of a replay (SPEC run and       */
/*    preprocessing_ops; hit rate P:L1293).                      */
/* ========================================================================= */

typedef struct {
    double   epoch_seconds;   /* sum over tiers of served_t / DSI_t         */
    double   dsi_mix;         /* Eq. 9 with N_t := served_t of the epoch */
    uint64_t decode_aug_ops;  /* storage fetches + encoded-tier hits         */
    uint64_t aug_only_ops;    /* decoded-tier hits                                    */
    double   hit_rate;        /* (served_E + served_D + served_A) / N       */
} oracle_epoch_row;

/* dsi[] = {DSI_A, DSI_D, DSI_E, DSI_S} (oracle_tiers order).  Served counts
 * are indexed by tier code S 0, E 1, D 2, A 3.  Sums in the tier order of
 * Eq. 9 (A, D, E, S), one IEEE operation per step.                           */
void oracle_epoch_metrics(const oracle_stats *st, uint64_t n_rows, uint64_t N, const double dsi[4],
                          oracle_epoch_row *out)
{
    double dN = (double)N;
    for (uint64_t r = 0; r < n_rows; ++r) {
        const uint64_t *sv = st[r].served;
        double cA = (double)sv[T_A], cD = (double)sv[T_D], cE = (double)sv[T_E], cS = (double)sv[T_S];
        double t = cA / dsi[0];
        t = t + cD / dsi[1];
        t = t + cE / dsi[2];
        t = t + cS / dsi[3];
        double v = (cA / dN) * dsi[0];
        v = v + (cD / dN) * dsi[1];
        v = v + (cE / dN) * dsi[2];
        v = v + (cS / dN) * dsi[3];
        out[r].epoch_seconds = t;
        out[r].dsi_mix = v;
        out[r].decode_aug_ops = sv[T_S] + sv[T_E];
        out[r].aug_only_ops = sv[T_D];
        out[r].hit_rate = (double)(sv[T_E] + sv[T_D] + sv[T_A]) / dN;
    }
}
