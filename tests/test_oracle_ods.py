"""Pins for the oracle's ODS replay (§5.2; readings R-O1..R-O20).

What fixes the oracle here:
  * SPEC's hand-worked example of the six fig:cache_aware_sampling steps;
  * closed forms: static tiers (cap_A = 0) give exactly cap_E + cap_D hits per
    job-epoch whatever the sampler; J = 1 pays every A hit with one refill;
    cache-less jobs decode every sample (P:L428's 7.16 M = 4 x 1.79 M);
  * invariants I1-I10 (each job-epoch delivers [0,N) exactly once, capacities,
    conservation, determinism, |seen_j| = n_j);
  * agreement with the independent literal transcription oracle/literal.py.
"""
import numpy as np
import pytest

import oracle as O
import synth
from oracle import literal as L

S, E, D, A, SUB = 0, 1, 2, 3, 4


def caps_for(cfg):
    p = O.make_profile(t_gpu=1, t_decode_augment=1, t_augment=1, b_nic=1, b_pcie=1, b_cache=1,
                       b_storage=1, cache_bytes=cfg["cache_bytes"], n_total=cfg["n_total"],
                       s_data=cfg["s_data"], m_num=cfg["m_num"], m_den=cfg["m_den"], nodes=1,
                       gpus_per_node=1)
    na, nd, ne, ns = O.split_counts(p, *cfg["split"])
    return ne, nd, na


def test_config_capacities_match_survey_table():
    # SURVEY §8(d) caps E / D / A (derived from Eqs. 5-7 with the paper's splits)
    assert caps_for(synth.ods_config("toy")) == (80, 11, 11)
    assert caps_for(synth.ods_config("imagenet1k")) == (0, 42_038, 45_541)
    assert caps_for(synth.ods_config("openimages")) == (658_561, 118_731, 0)
    assert caps_for(synth.ods_config("imagenet22k")) == (4_376_846, 0, 0)
    for name in ("toy", "imagenet1k", "openimages", "imagenet22k"):
        assert O.config_capacities(synth.ods_config(name)) == caps_for(synth.ods_config(name))


def test_spec_worked_example():
    """10 samples, A cache = {A,B,C}, job's seen = {A}, request {D,B,E}
    -> response {C,B,E}: C substituted from A, B a hit, E from storage, D deferred."""
    o = O.ODS(10, [3], [1], 0, 0, 3, seed=1)
    tier = np.zeros(10, np.uint8); tier[[0, 1, 2]] = A          # A,B,C = ids 0,1,2
    seen = np.zeros((1, 10), np.uint8); seen[0, 0] = 1           # job has seen A
    o.set_state(tier, seen, np.zeros((1, 10), np.uint8))
    rc, ids, src, lens = o.round([0], requested=[[3, 1, 4]])     # D, B, E
    assert rc == 0 and lens[0] == 3
    assert list(ids[0, :3]) == [2, 1, 4]
    assert list(src[0, :3]) == [A | SUB, A, S]
    t, sn, cn = o.state()
    assert sn[0, 3] == 0                                          # D deferred (unseen)
    assert sn[0, [0, 1, 2, 4]].all()
    # maintain: J = 1 -> threshold 1 -> B and C evicted; refill restores |A| = 3
    assert (t == A).sum() == 3 and t[1] != A and t[2] != A and t[0] == A


def test_all_hits_and_empty_cache_trivia():
    o = O.ODS(20, [4], [1], 20, 0, 0, seed=3)                     # everything encoded-cached
    rc, ids, src, lens = o.round([0], requested=[[5, 9, 1, 0]])
    assert list(ids[0]) == [5, 9, 1, 0] and list(src[0]) == [E] * 4
    o = O.ODS(20, [4], [1], 0, 0, 0, seed=3)                      # empty cache
    rc, ids, src, lens = o.round([0], requested=[[5, 9, 1, 0]])
    assert list(ids[0]) == [5, 9, 1, 0] and list(src[0]) == [S] * 4


def test_protocol_violations():
    o = O.ODS(20, [4], [1], 0, 0, 0, seed=3)
    assert o.round([0], requested=[[5, 5, 1, 0]])[0] == 3         # duplicate -> EPROTO
    assert o.round([0], requested=[[5, 9, 1, 20]])[0] == 3        # out of range
    assert o.round([0], requested=[[5, 9, 1, 0]])[0] == 0
    assert o.round([0], requested=[[5, 2, 3, 4]])[0] == 3         # 5 already seen
    assert o.round([1])[0] == 1                                    # unknown job -> EINVAL


def test_departed_job_is_invalid_state():
    o = O.ODS(8, [8, 4], [1, 2], 0, 0, 2, seed=3)
    o.round([0, 1])                                               # job 0 finishes its only epoch
    assert o.round([0])[0] == 2


def test_threshold_two_evicts_after_both_jobs():
    """threshold 2, a sample served to both jobs is evicted at the round end
    and the A occupancy restored by refill."""
    o = O.ODS(50, [5, 5], [2, 2], 0, 0, 10, seed=4)
    tier0, _, _ = o.state()
    A0 = set(np.flatnonzero(tier0 == A))
    x = sorted(A0)[0]
    rest = [i for i in range(50) if i not in A0][:4]
    o.round([0, 1], requested=[[x] + rest, [x] + rest[::-1]])
    t, _, c = o.state()
    assert t[x] != A and not c[:, x].any()                        # evicted, consumers cleared
    assert (t == A).sum() == 10                                   # refilled to cap_A
    o2 = O.ODS(50, [5, 5], [2, 2], 0, 0, 10, seed=4)
    o2.round([0], requested=[[x] + rest])                         # only one consumer
    t2, _, c2 = o2.state()
    assert t2[x] == A and c2[0, x] == 1 and c2[1, x] == 0


def _check_invariants(o, cfg):
    """I1 (exact-once per job-epoch), I4, I5, I9, I10 on a finished replay."""
    tr = o.transcript()
    st, ev, rf = o.stats()
    N = cfg["n_total"]
    for j in range(len(cfg["batch"])):
        for e in range(cfg["target"][j]):
            row = tr[j, e]
            ids = (row & 0xFFFFFFFF).astype(np.int64)
            assert np.array_equal(np.sort(ids), np.arange(N))      # I1 + I3
            s = st[j, e]
            assert s["served"].sum() == N                          # I5
            srcs = (row >> np.uint64(32)).astype(np.int64)
            for t in range(4):
                assert s["served"][t] == ((srcs & 3) == t).sum()
                assert s["subst"][t] == ((srcs == (t | SUB))).sum()
            digest = 0
            for q in range(N):
                digest = (digest + O.splitmix64((q << 35) | int(row[q]))) & ((1 << 64) - 1)
            assert digest == int(s["digest"])
    t, seen, cons = o.state()
    assert (t == E).sum() <= cfg["cap_e"] and (t == D).sum() <= cfg["cap_d"]
    assert (t == A).sum() <= cfg["cap_a"]                          # I4
    assert (t == A).sum() == cfg["cap_a"] + rf - ev                # A occupancy conservation
    assert (t == E).sum() == cfg["cap_e"] and (t == D).sum() == cfg["cap_d"]   # static E/D (R-O4)


def run_oracle(cfg, transcript=True):
    o = O.ODS(cfg["n_total"], cfg["batch"], cfg["target"], cfg["cap_e"], cfg["cap_d"], cfg["cap_a"],
              cfg["seed"], transcript=transcript)
    return o


def test_toy_config_invariants_and_determinism():
    base = synth.ods_config("toy", seed=1)
    ce, cd, ca = caps_for(base)
    cfg = dict(base, cap_e=ce, cap_d=cd, cap_a=ca)
    o = run_oracle(cfg)
    rounds = o.replay_epochs(3)
    assert rounds == 3 * ((1000 + 31) // 32)
    _check_invariants(o, cfg)
    o2 = run_oracle(cfg)
    o2.replay_epochs(3)
    assert np.array_equal(o.transcript(), o2.transcript())            # I6
    assert np.array_equal(o.stats()[0], o2.stats()[0])


def test_seen_count_tracks_progress_every_round():
    cfg = dict(n_total=300, batch=[7, 16, 32], target=[2, 1, 3], cap_e=40, cap_d=30, cap_a=30, seed=9)
    o = run_oracle(cfg, transcript=False)
    while True:
        c, e, n, act = o.job_state()
        if not act.any():
            break
        _, seen, _ = o.state()
        for j in range(3):
            if act[j]:
                assert seen[j].sum() == n[j]                          # I10
        t, _, _ = o.state()
        assert (t == A).sum() <= 30
        o.replay_rounds(1)


def test_static_tiers_closed_form():
    """cap_A = 0: per job-epoch served[E] + served[D] = cap_E + cap_D exactly and
    served[S] = N - cap_E - cap_D, for any seed (P:L1294 'roughly equal to the
    percentage of cached data')."""
    for seed in (1, 2, 3):
        cfg = dict(n_total=500, batch=[16, 32, 64], target=[2, 2, 2], cap_e=60, cap_d=40, cap_a=0, seed=seed)
        o = run_oracle(cfg)
        o.replay_epochs(2)
        st, ev, rf = o.stats()
        for j in range(3):
            for e in range(2):
                s = st[j, e]
                assert s["served"][E] == 60 and s["served"][D] == 40 and s["served"][S] == 400
        assert ev == 0 and rf == 0
        _check_invariants(o, cfg)


def test_single_job_refill_pays_every_augmented_hit():
    """J = 1 -> threshold 1: every A-served sample is evicted at its round end and
    one storage sample refilled, so storage fetches + refills = delivered, except
    the A-served of the final round (the job departs, no maintain work)."""
    cfg = dict(n_total=1000, batch=[32], target=[2], cap_e=0, cap_d=0, cap_a=200, seed=5)
    o = run_oracle(cfg)
    rounds = o.replay_epochs(2)
    st, ev, rf = o.stats()
    tr = o.transcript()
    delivered = 2 * 1000
    storage = int(st[0, :, ]["served"][:, S].sum())
    last_round = tr[0, 1, 1000 - (1000 % 32 or 32):]
    a_last = int((((last_round >> np.uint64(32)) & np.uint64(3)) == A).sum())
    assert storage + rf == delivered - a_last
    assert ev == rf


def test_cacheless_jobs_decode_everything():
    """4 concurrent jobs, no cache, 1.79 M samples -> 7.16 M decode+augment ops."""
    cfg = dict(n_total=1_790_000, batch=[4096] * 4, target=[1] * 4, cap_e=0, cap_d=0, cap_a=0, seed=2)
    o = run_oracle(cfg, transcript=False)
    o.replay_epochs(1)
    st, _, _ = o.stats()
    ops = int(st["served"][:, 0, S].sum() + st["served"][:, 0, E].sum())   # decode+augment
    assert ops == 7_160_000


def test_ods_uplift_direction():
    """P:L1294 / S:L480: 3 jobs, 20 % cached in A -> stable-epoch hit rate well above
    the cached fraction (the uniform no-evict baseline sits at the fraction)."""
    cfg = dict(n_total=1000, batch=[32] * 3, target=[3] * 3, cap_e=0, cap_d=0, cap_a=200, seed=7)
    o = run_oracle(cfg, transcript=False)
    o.replay_epochs(3)
    st, _, _ = o.stats()
    for j in range(3):
        for e in (1, 2):
            hits = st[j, e]["served"][1:].sum()
            assert hits / 1000 >= 0.30


@pytest.mark.parametrize("block", range(8))
def test_cross_check_with_literal_transcription(block):
    """Agreement with oracle/literal.py on random tiny configs (N <= 64, J <= 3, B <= 8,
    random caps and targets so departures happen mid-replay)."""
    st = synth.Stream(1000 + block)
    for _ in range(60):
        cfg = synth.random_tiny_ods(st)
        o = run_oracle(cfg)
        o.replay_epochs(max(cfg["target"]))
        lit = L.LiteralODS(cfg["n_total"], cfg["batch"], cfg["target"], cfg["cap_e"], cfg["cap_d"],
                           cfg["cap_a"], cfg["seed"])
        lit.replay_all()
        tr = o.transcript()
        for j in range(len(cfg["batch"])):
            for e in range(cfg["target"][j]):
                got = [(int(x) & 0xFFFFFFFF, int(x) >> 32) for x in tr[j, e]]
                assert got == lit.deliveries[j][e], cfg
        t, seen, cons = o.state()
        assert list(t) == lit.tier
        _, ev, rf = o.stats()
        assert (ev, rf) == (lit.evicted, lit.refilled)
        # I2 on the literal side: no A entry served twice to a job between admission and eviction
        _check_invariants(o, cfg)


# ------------------------------------------------------------ evict_tiers = ALL (DESIGN R-O21)
def run_all(cfg, transcript=True):
    return O.ODS(cfg["n_total"], cfg["batch"], cfg["target"], cfg["cap_e"], cfg["cap_d"], cfg["cap_a"],
                 cfg["seed"], transcript=transcript, evict_all=True)


@pytest.mark.parametrize("block", range(8))
def test_evict_all_cross_check_with_literal_transcription(block):
    st = synth.Stream(7000 + block)
    for _ in range(60):
        cfg = synth.random_tiny_ods(st)
        o = run_all(cfg)
        o.replay_epochs(max(cfg["target"]))
        lit = L.LiteralODS(cfg["n_total"], cfg["batch"], cfg["target"], cfg["cap_e"], cfg["cap_d"],
                           cfg["cap_a"], cfg["seed"], evict_all=True)
        lit.replay_all()
        tr = o.transcript()
        for j in range(len(cfg["batch"])):
            for e in range(cfg["target"][j]):
                got = [(int(x) & 0xFFFFFFFF, int(x) >> 32) for x in tr[j, e]]
                assert got == lit.deliveries[j][e], cfg
        t, seen, cons = o.state()
        assert list(t) == lit.tier
        _, ev, rf = o.stats()
        assert (ev, rf) == (lit.evicted, lit.refilled)


def test_evict_all_invariants():
    """I1/I3/I5 per job-epoch, I4 per tier, and cached-occupancy conservation
    |E| + |D| + |A| = caps + refills - evictions, for evict_tiers = ALL."""
    for seed in (1, 2, 3):
        cfg = dict(n_total=600, batch=[16, 40, 9], target=[2, 3, 2], cap_e=70, cap_d=50, cap_a=40, seed=seed)
        o = run_all(cfg)
        o.replay_epochs(3)
        tr = o.transcript()
        st, ev, rf = o.stats()
        for j in range(3):
            for e in range(cfg["target"][j]):
                ids = (tr[j, e] & 0xFFFFFFFF).astype(np.int64)
                assert np.array_equal(np.sort(ids), np.arange(600))
                assert st[j, e]["served"].sum() == 600
        t, _, _ = o.state()
        assert (t == E).sum() <= 70 and (t == D).sum() <= 50 and (t == A).sum() <= 40
        assert (t != S).sum() == 70 + 50 + 40 + rf - ev
        assert ev > 0 and rf > 0


def test_evict_all_single_job_encoded_cache_churns():
    """J = 1 (threshold 1), E-only cache: every E-served sample is evicted at its
    round end and one storage sample refilled into E, so storage fetches +
    refills = delivered, except the E-served of the final round (the job departs:
    no maintain); the E tier is back at cap_E after every round (the storage
    pool is never short here)."""
    cfg = dict(n_total=1000, batch=[32], target=[2], cap_e=200, cap_d=0, cap_a=0, seed=5)
    o = run_all(cfg)
    o.replay_epochs(2)
    st, ev, rf = o.stats()
    tr = o.transcript()
    storage = int(st[0, :]["served"][:, S].sum())
    last_round = tr[0, 1, 1000 - (1000 % 32 or 32):]
    e_last = int((((last_round >> np.uint64(32)) & np.uint64(3)) == E).sum())
    assert storage + rf == 2000 - e_last and ev == rf
    t, _, _ = o.state()
    assert (t == E).sum() == 200 and (t == A).sum() == 0 and (t == D).sum() == 0


def test_evict_all_a_only_mode_is_the_special_case():
    """With no E/D tiers the two modes are the same protocol: identical replays."""
    st = synth.Stream(99)
    for _ in range(40):
        cfg = synth.random_tiny_ods(st)
        cfg = dict(cfg, cap_e=0, cap_d=0)
        a, b = run_oracle(cfg), run_all(cfg)
        a.replay_epochs(max(cfg["target"]))
        b.replay_epochs(max(cfg["target"]))
        assert np.array_equal(a.transcript(), b.transcript())
        assert np.array_equal(a.state()[0], b.state()[0])


def test_evict_all_uplift_on_encoded_only_cache():
    """O4: with static tiers (evict_tiers = A) an E-only cache gives hits exactly
    cap_E per job-epoch whatever the sampler; with evict_tiers = ALL consumed E
    entries are replaced, so 3 concurrent jobs get well above the cached fraction
    (the direction P:L1474-1475 reports for ImageNet-22K at 100-0-0)."""
    cfg = dict(n_total=1000, batch=[32] * 3, target=[3] * 3, cap_e=200, cap_d=0, cap_a=0, seed=7)
    static = run_oracle(cfg, transcript=False)
    static.replay_epochs(3)
    churn = run_all(cfg, transcript=False)
    churn.replay_epochs(3)
    s0, _, _ = static.stats()
    s1, _, _ = churn.stats()
    for j in range(3):
        for e in (1, 2):
            assert s0[j, e]["served"][1:].sum() == 200
            assert s1[j, e]["served"][1:].sum() / 1000 >= 0.30


# ------------------------------------------------------------ NEXT-1: epoch model on top of the replay
def test_epoch_model_preprocessing_ops_pin():
    """P:L428 / S:L396 through the epoch model: 4 cache-less jobs x 1.79 M samples
    -> 7.16 M decode+augment ops, 0 augment-only, hit rate 0."""
    cfg = dict(n_total=1_790_000, batch=[4096] * 4, target=[1] * 4, cap_e=0, cap_d=0, cap_a=0, seed=2)
    o = run_oracle(cfg, transcript=False)
    o.replay_epochs(1)
    st, _, _ = o.stats()
    m = O.epoch_metrics(st, 1_790_000, (2000.0, 2000.0, 2000.0, 1000.0))
    assert int(m["decode_aug_ops"].sum()) == 7_160_000 and int(m["aug_only_ops"].sum()) == 0
    assert np.all(m["hit_rate"] == 0.0)


def test_epoch_model_zero_cache_time_is_n_over_dsi_s():
    """SPEC run example: J = 1, zero cache -> epoch time = N / DSI_S."""
    cfg = dict(n_total=5000, batch=[64], target=[2], cap_e=0, cap_d=0, cap_a=0, seed=3)
    o = run_oracle(cfg, transcript=False)
    o.replay_epochs(2)
    dsi = (2141.58, 2141.58, 2132.0, 1733.7)
    m = O.epoch_metrics(o.stats()[0], 5000, dsi)
    assert np.all(m["epoch_seconds"] == 5000 / 1733.7) and np.all(m["dsi_mix"] == 1733.7)


@pytest.mark.parametrize("server", ["in_house", "aws", "azure"])
def test_epoch_model_static_tiers_equal_eq9(server):
    """With static tiers (cap_A = 0) every job-epoch serves exactly the split's
    counts (served_E = N_E, served_D = N_D, served_S = N_S), so the replayed mix
    evaluated by Eq. 9 is the MDP model's value bit for bit, and the epoch time is
    the tier sum of S:L376 in exact rationals."""
    import json
    import os
    from fractions import Fraction
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table4_nominal_vals.json")))
    g = {k: v for k, v in gold[server].items() if not k.startswith("_")}
    N, split = 20_000, (30, 25, 0)
    p = O.make_profile(**dict(g, model_bytes=0.0, n_total=N, nodes=1, gpus_per_node=1, cache_bytes=10**9))
    na, nd, ne, ns = O.split_counts(p, *split)
    assert na == 0 and nd > 0 and ne > 0 and ns > 0
    cfg = dict(n_total=N, batch=[256, 100], target=[2, 1], cap_e=ne, cap_d=nd, cap_a=0, seed=4)
    o = run_oracle(cfg, transcript=False)
    o.replay_epochs(2)
    st, _, _ = o.stats()
    dsi, _ = O.tiers(p)
    v, _, _ = O.model_eval(p, *split)
    m = O.epoch_metrics(st, N, dsi)
    for j, e in ((0, 0), (0, 1), (1, 0)):
        assert m[j, e]["dsi_mix"] == v
        want = sum(Fraction(int(c)) / Fraction(d) for c, d in
                   zip((st[j, e]["served"][A], st[j, e]["served"][D], st[j, e]["served"][E], st[j, e]["served"][S]),
                       dsi))
        assert abs(Fraction(m[j, e]["epoch_seconds"]) - want) <= want * Fraction(1, 10**14)


# ------------------------------------------------------------ the uniform no-evict baseline sampler (NEXT-3, R-O22)
def run_base(cfg, transcript=True):
    return O.ODS(cfg["n_total"], cfg["batch"], cfg["target"], cfg["cap_e"], cfg["cap_d"], cfg["cap_a"],
                 cfg["seed"], transcript=transcript, baseline=True)


def test_baseline_hit_rate_is_the_cached_fraction_exactly():
    """S:L380 / P:L1294 (MINIO-like): the request stream visits every id once per
    epoch and nothing is substituted or evicted, so every job-epoch hits exactly
    the cached ids: served_E/D/A = cap_E/D/A, served_S = the rest."""
    for seed in (1, 2, 3):
        cfg = dict(n_total=1000, batch=[32, 17, 64], target=[3, 2, 3], cap_e=120, cap_d=50, cap_a=30, seed=seed)
        o = run_base(cfg)
        o.replay_epochs(3)
        st, ev, rf = o.stats()
        assert ev == 0 and rf == 0
        for j in range(3):
            for e in range(cfg["target"][j]):
                s = st[j, e]
                assert list(s["served"]) == [800, 120, 50, 30] and s["subst"].sum() == 0
        tr = o.transcript()
        ids = (tr[0, 0] & 0xFFFFFFFF).astype(np.int64)
        assert np.array_equal(np.sort(ids), np.arange(1000))


@pytest.mark.parametrize("block", range(4))
def test_baseline_cross_check_with_literal_transcription(block):
    st = synth.Stream(11000 + block)
    for _ in range(60):
        cfg = synth.random_tiny_ods(st)
        o = run_base(cfg)
        o.replay_epochs(max(cfg["target"]))
        lit = L.LiteralODS(cfg["n_total"], cfg["batch"], cfg["target"], cfg["cap_e"], cfg["cap_d"],
                           cfg["cap_a"], cfg["seed"], baseline=True)
        lit.replay_all()
        tr = o.transcript()
        for j in range(len(cfg["batch"])):
            for e in range(cfg["target"][j]):
                got = [(int(x) & 0xFFFFFFFF, int(x) >> 32) for x in tr[j, e]]
                assert got == lit.deliveries[j][e], cfg


def test_hit_rate_vs_cache_fraction_ods_above_baseline():
    """The paper's hit-rate experiment (P:L1282-1294, 3 concurrent jobs): with an
    augmented cache ODS serves well above the cached fraction, which the
    no-evict baseline serves exactly (SURVEY [A.7] probe: 0.64 at 20 %, 0.86 at 40 %)."""
    for frac in (0.2, 0.4):
        cap = int(1000 * frac)
        cfg = dict(n_total=1000, batch=[32] * 3, target=[3] * 3, cap_e=0, cap_d=0, cap_a=cap, seed=7)
        ods, base = run_oracle(cfg, transcript=False), run_base(cfg, transcript=False)
        ods.replay_epochs(3)
        base.replay_epochs(3)
        h_ods = ods.stats()[0]["served"][:, 1:, 1:].sum(axis=2) / 1000
        h_base = base.stats()[0]["served"][:, 1:, 1:].sum(axis=2) / 1000
        assert np.all(h_base == frac)
        assert np.all(h_ods >= frac + 0.25)


# ------------------------------------------------------------ job arrivals (NEXT-1 job-arrival traces, R-O23)
def _random_arrivals(st, J):
    return [0 if k == 0 else int(st.u64(1)[0] % 40) for k in range(J)]


@pytest.mark.parametrize("block", range(4))
def test_arrivals_cross_check_with_literal_transcription(block):
    st = synth.Stream(13000 + block)
    for _ in range(60):
        cfg = synth.random_tiny_ods(st)
        arr = _random_arrivals(st, len(cfg["batch"]))
        for evict_all in (False, True):
            o = O.ODS(cfg["n_total"], cfg["batch"], cfg["target"], cfg["cap_e"], cfg["cap_d"], cfg["cap_a"],
                      cfg["seed"], transcript=True, evict_all=evict_all, arrival=arr)
            o.replay_epochs(max(cfg["target"]))
            lit = L.LiteralODS(cfg["n_total"], cfg["batch"], cfg["target"], cfg["cap_e"], cfg["cap_d"],
                               cfg["cap_a"], cfg["seed"], evict_all=evict_all, arrival=arr)
            lit.replay_all()
            tr = o.transcript()
            for j in range(len(cfg["batch"])):
                for e in range(cfg["target"][j]):
                    got = [(int(x) & 0xFFFFFFFF, int(x) >> 32) for x in tr[j, e]]
                    assert got == lit.deliveries[j][e], (cfg, arr)
            assert list(o.state()[0]) == lit.tier
            assert o.r == lit.r


def test_arrivals_makespan_trace():
    """A makespan-style trace (jobs queued, at most two at a time): job
    k arrives when job k-2 departs, computed from the data-independent schedule
    (R-O12).  The replay ends when the last job departs; the round count is the
    makespan in rounds; with a single job at a time the rounds add up exactly."""
    N, B = 2000, 100
    cfg = dict(n_total=N, batch=[B] * 4, target=[2] * 4, cap_e=0, cap_d=0, cap_a=400, seed=8)
    per_job = 2 * ((N + B - 1) // B)                          # rounds a job needs alone: 40
    serial = [0, per_job, 2 * per_job, 3 * per_job]          # one job at a time
    o = O.ODS(N, cfg["batch"], cfg["target"], 0, 0, 400, 8, transcript=True, arrival=serial)
    assert o.replay_epochs(2) == 4 * per_job
    _check_invariants(o, cfg)
    two = [0, 0, per_job, per_job]                            # two at a time
    o2 = O.ODS(N, cfg["batch"], cfg["target"], 0, 0, 400, 8, arrival=two)
    assert o2.replay_epochs(2) == 2 * per_job
    gap = [0, 3 * per_job, 3 * per_job, 3 * per_job]          # idle rounds between the jobs
    o3 = O.ODS(N, cfg["batch"], cfg["target"], 0, 0, 400, 8, arrival=gap)
    assert o3.replay_epochs(2) == 4 * per_job


# ------------------------------------------------------------ cold start (NEXT-2, R-O24)
@pytest.mark.parametrize("block", range(4))
def test_cold_start_cross_check_with_literal_transcription(block):
    st = synth.Stream(15000 + block)
    for _ in range(50):
        cfg = synth.random_tiny_ods(st)
        for evict_all, baseline in ((False, False), (True, False), (False, True)):
            o = O.ODS(cfg["n_total"], cfg["batch"], cfg["target"], cfg["cap_e"], cfg["cap_d"], cfg["cap_a"],
                      cfg["seed"], transcript=True, evict_all=evict_all, baseline=baseline, cold=True)
            o.replay_epochs(max(cfg["target"]))
            lit = L.LiteralODS(cfg["n_total"], cfg["batch"], cfg["target"], cfg["cap_e"], cfg["cap_d"],
                               cfg["cap_a"], cfg["seed"], evict_all=evict_all, baseline=baseline, cold=True)
            lit.replay_all()
            tr = o.transcript()
            for j in range(len(cfg["batch"])):
                for e in range(cfg["target"][j]):
                    got = [(int(x) & 0xFFFFFFFF, int(x) >> 32) for x in tr[j, e]]
                    assert got == lit.deliveries[j][e], cfg
            assert list(o.state()[0]) == lit.tier
            assert o.stats()[1:] == (lit.evicted, lit.refilled)


def test_cold_start_first_vs_stable_epoch():
    """SPEC cold start: the first epoch starts from an empty cache
    and fills it with what it fetches, so it hits less than the stable epochs;
    with one job and no churn (baseline sampler, static once full) the first
    batch is all storage and the cache is full after cap / B rounds."""
    cfg = dict(n_total=2000, batch=[50], target=[3], cap_e=300, cap_d=200, cap_a=0, seed=5)
    o = O.ODS(2000, [50], [3], 300, 200, 0, 5, transcript=True, baseline=True, cold=True)
    o.replay_epochs(3)
    st, ev, rf = o.stats()
    tr = o.transcript()
    first = (tr[0, 0, :50] >> np.uint64(32)) & np.uint64(7)
    assert np.all(first == S)                                  # nothing cached in the first round
    assert rf == 500 and ev == 0                               # 300 + 200 admissions, then static
    hits = st[0, :]["served"][:, 1:].sum(axis=1)
    assert hits[0] < hits[1] and hits[1] == hits[2] == 500     # stable epochs hit exactly the cache
    t, _, _ = o.state()
    assert (t == E).sum() == 300 and (t == D).sum() == 200
    # the same with ODS (A churn after warm-up): first epoch below the stable ones
    o2 = O.ODS(2000, [50] * 3, [3] * 3, 0, 0, 400, 6, cold=True)
    o2.replay_epochs(3)
    s2 = o2.stats()[0]
    for j in range(3):
        h = s2[j, :]["served"][:, 1:].sum(axis=1)
        assert h[0] < h[1] and h[0] < h[2]
