"""GPU parity: the ODS replay through the C-ABI vs the oracle.

Bit-exact for every decision: delivered id and source per position (transcript),
residency / seen / consumer bitmaps, per job-epoch counters and digests,
eviction and refill totals.  Sizes: the toy config and random tiny configs in
full; N/64-scaled versions of every config in full; the full-size configs for a
prefix of rounds (oracle one by one) and, where tests/golden holds the oracle's
full replay (written by tests/golden/make_oracle_golden.py, oracle only), the
whole replay."""
import glob
import hashlib
import json
import os

import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2511_13724_b200 as P  # noqa: E402
from paper_2511_13724_b200 import seneca as S  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def caps_of(c):
    """The oracle's own capacities (oracle.config_capacities); the product's
    seneca_split_capacities must agree (checked here and in tests/test_abi.py)."""
    caps = O.config_capacities(c)
    prod = S.split_capacities(c["n_total"], c["s_data"], c["m_num"], c["m_den"], c["cache_bytes"], *c["split"])
    assert tuple(prod[:3]) == tuple(caps), (prod, caps)
    return caps


def make_pair(n, batch, target, ce, cd, ca, seed, transcript=True, evict_all=False, baseline=False):
    o = O.ODS(n, batch, target, ce, cd, ca, seed, transcript=transcript, evict_all=evict_all, baseline=baseline)
    g = P.ODSContext(n, batch, target, ce, cd, ca, seed, evict_tiers=int(evict_all), sampler=int(baseline))
    return o, g


def compare_state(o, g, check_transcript=None):
    st_o, ev_o, rf_o = o.stats()
    st_g, ev_g, rf_g = g.stats()
    assert (ev_g, rf_g) == (ev_o, rf_o)
    assert st_g.tobytes() == st_o.tobytes()
    t_o, s_o, c_o = o.state()
    t_g, s_g, c_g = g.state()
    np.testing.assert_array_equal(t_g, t_o)
    np.testing.assert_array_equal(s_g, s_o)
    np.testing.assert_array_equal(c_g, c_o)
    if check_transcript is not None:
        tr_o = o.transcript()
        tr_g = check_transcript.cpu().numpy().view(np.uint64)
        if not np.array_equal(tr_g, tr_o):
            j, e, q = np.argwhere(tr_g != tr_o)[0]
            raise AssertionError(f"first transcript mismatch job {j} epoch {e} pos {q}: "
                                 f"gpu {int(tr_g[j, e, q]):#x} oracle {int(tr_o[j, e, q]):#x}")
    g.sync()


def replay_pair(n, batch, target, ce, cd, ca, seed, evict_all=False, baseline=False):
    o, g = make_pair(n, batch, target, ce, cd, ca, seed, evict_all=evict_all, baseline=baseline)
    tr = g.new_transcript()
    r_g = g.replay_epochs(max(target), tr)
    r_o = o.replay_epochs(max(target))
    torch.cuda.synchronize()
    assert r_g == r_o
    compare_state(o, g, tr)
    return o, g


@pytest.mark.parametrize("seed", synth.PARITY_SEEDS)
def test_toy_config(seed):
    c = synth.ods_config("toy", seed=seed)
    ce, cd, ca = caps_of(c)
    assert (ce, cd, ca) == (80, 11, 11)
    replay_pair(c["n_total"], c["batch"], c["target"], ce, cd, ca, seed)


@pytest.mark.parametrize("block", range(6))
def test_random_tiny_configs(block):
    st = synth.Stream(5000 + block)
    for _ in range(50):
        c = synth.random_tiny_ods(st)
        replay_pair(c["n_total"], c["batch"], c["target"], c["cap_e"], c["cap_d"], c["cap_a"], c["seed"])


@pytest.mark.parametrize("name", ["imagenet1k", "openimages", "imagenet22k"])
def test_scaled_configs_full_replay(name):
    """N/64 with split 34-33-33: every tier populated, A churn, mixed batches (OI),
    ragged tails, several superblocks."""
    c = synth.ods_config(name, scale=64, seed=1)
    ce, cd, ca = caps_of(c)
    replay_pair(c["n_total"], c["batch"], c["target"], ce, cd, ca, 1)


def test_ragged_and_edge_shapes():
    cases = [
        (1, [1], [3], 0, 0, 1),            # single sample
        (33, [33], [2], 0, 0, 33),         # whole dataset in A, one batch per epoch
        (1025, [1024, 7], [2, 3], 100, 100, 100),
        (32768 + 5, [4096, 1000], [1, 2], 2000, 1000, 3000),   # superblock boundary, max batch
        (5000, [17, 33, 64], [1, 1, 1], 0, 0, 0),               # no cache at all
        (5000, [17, 33, 64], [2, 1, 1], 5000, 0, 0),            # everything encoded-cached
    ]
    for n, b, t, ce, cd, ca in cases:
        replay_pair(n, b, t, ce, cd, ca, 7)


@pytest.mark.parametrize("name,rounds", [("imagenet1k", 400), ("openimages", 300), ("imagenet22k", 120)])
def test_full_size_prefix(name, rounds):
    """Full-size configs, first rounds, in the launch configuration bench.py times."""
    seed = synth.PERF_SEED
    c = synth.ods_config(name, seed=seed)
    ce, cd, ca = caps_of(c)
    o, g = make_pair(c["n_total"], c["batch"], c["target"], ce, cd, ca, seed, transcript=False)
    assert g.replay_rounds(rounds) == rounds
    assert o.replay_rounds(rounds) == rounds
    torch.cuda.synchronize()
    compare_state(o, g)


@pytest.mark.parametrize("name,split", [("imagenet1k", None), ("openimages", (52, 48, 0)), ("imagenet22k", (100, 0, 0))])
def test_replay_in_launches_of_random_length(name, split):
    """A replay cut into launches of random length (1..300 rounds, epochs ending
    inside and at the edges of launches) equals the oracle's: the per job-epoch
    counters and digests the round kernel keeps in shared memory across rounds
    are added to memory at every epoch end and launch end.  Coupled (ImageNet-1K's
    A churn) and uncoupled (the paper's OpenImages / ImageNet-22K splits) kernels."""
    c = synth.ods_config(name, scale=64, seed=3)
    if split is not None:
        c["split"] = split
    ce, cd, ca = caps_of(c)
    o, g = make_pair(c["n_total"], c["batch"], c["target"], ce, cd, ca, 3)
    tr = g.new_transcript()
    st = synth.Stream(4242)
    total = 0
    while True:
        k = int(st.u64(1)[0] % np.uint64(300)) + 1
        done = g.replay_rounds(k, tr)
        total += done
        if done < k or g.view().active_mask == 0:
            break
    torch.cuda.synchronize()
    assert total == o.replay_epochs(max(c["target"]))
    compare_state(o, g, tr)


def _golden_files():
    return sorted(glob.glob(os.path.join(HERE, "golden", "oracle_*_seed*.json")))


@pytest.mark.parametrize("path", _golden_files(), ids=lambda p: os.path.basename(p))
def test_full_replay_against_oracle_golden(path):
    gold = json.load(open(path))
    c = synth.ods_config(gold["config"].split("/")[0], seed=gold["seed"])
    ce, cd, ca = caps_of(c)
    assert [ce, cd, ca] == gold["caps"]
    g = P.ODSContext(c["n_total"], c["batch"], c["target"], ce, cd, ca, gold["seed"],
                     evict_tiers=gold.get("evict_tiers", 0))
    rounds = g.replay_epochs(max(c["target"]))
    torch.cuda.synchronize()
    g.sync()
    assert rounds == gold["rounds"]
    st, ev, rf = g.stats()
    assert (ev, rf) == (gold["evicted"], gold["refilled"])
    for j, row in enumerate(gold["stats"]):
        for e, s in enumerate(row):
            assert [int(v) for v in st[j, e]["served"]] == s["served"]
            assert [int(v) for v in st[j, e]["subst"]] == s["subst"]
            assert [int(v) for v in st[j, e]["req_hits"]] == s["req_hits"]
            assert int(st[j, e]["digest"]) == int(s["digest"])
    tier, seen, cons = g.state()
    h = hashlib.sha256()
    h.update(tier.tobytes()); h.update(seen.tobytes()); h.update(cons.tobytes())
    assert h.hexdigest() == gold["state_sha256"]


def test_next_batch_subsets_of_jobs():
    """seneca_ods_next_batch with changing job subsets (R-O11) vs oracle rounds."""
    n, batch, target = 700, [16, 40, 9], [2, 2, 3]
    o, g = make_pair(n, batch, target, 60, 50, 90, 11, transcript=False)
    st = synth.Stream(77)
    for _ in range(150):
        _, _, _, act = o.job_state()
        live = [j for j in range(3) if act[j]]
        if not live:
            break
        pick = [j for j in live if st.uniform(1)[0] < 0.7] or live[:1]
        rc, ids_o, src_o, lens_o = o.round(pick)
        assert rc == 0
        ids_g, src_g, lens_g = g.next_batch(pick)
        torch.cuda.synchronize()
        assert list(lens_o) == lens_g
        for x, L_ in enumerate(lens_g):
            assert np.array_equal(ids_g[x, :L_].cpu().numpy().view(np.uint32), ids_o[x, :L_])
            assert np.array_equal(src_g[x, :L_].cpu().numpy(), src_o[x, :L_])
    compare_state(o, g)


def test_caller_supplied_requests():
    """request_mode 1 (R-O20): ids chosen by the caller; the SPEC request_batch path."""
    n, batch, target = 400, [12, 20], [2, 2]
    o = O.ODS(n, batch, target, 40, 30, 50, 5)
    g = P.ODSContext(n, batch, target, 40, 30, 50, 5, request_mode=1)
    st = synth.Stream(8)
    for _ in range(80):
        _, _, _, act = o.job_state()
        live = [j for j in range(2) if act[j]]
        if not live:
            break
        _, seen, _ = o.state()
        reqs = []
        for j in live:
            unseen = np.flatnonzero(seen[j] == 0)
            need = o.need(j)
            order = np.argsort(st.u64(len(unseen)))
            reqs.append([int(v) for v in unseen[order[:need]]])
        rc, ids_o, src_o, lens_o = o.round(live, requested=reqs)
        assert rc == 0
        ids_g, src_g, lens_g = g.next_batch(live, requested=reqs)
        torch.cuda.synchronize()
        for x, L_ in enumerate(lens_g):
            assert np.array_equal(ids_g[x, :L_].cpu().numpy().view(np.uint32), ids_o[x, :L_])
            assert np.array_equal(src_g[x, :L_].cpu().numpy(), src_o[x, :L_])
    compare_state(o, g)


def test_protocol_violations_and_state_errors():
    g = P.ODSContext(100, [4, 4], [1, 1], 10, 10, 10, 3, request_mode=1)
    with pytest.raises(S.SenecaError) as ei:
        g.next_batch([0], requested=[[1, 1, 2, 3]])          # duplicate
    assert ei.value.status == S.EPROTO
    with pytest.raises(S.SenecaError) as ei:
        g.next_batch([0], requested=[[1, 2, 3, 100]])        # out of range
    assert ei.value.status == S.EPROTO
    ids, src, lens = g.next_batch([0, 1], requested=[[1, 2, 3, 4], [1, 2, 3, 4]])  # same ids, two jobs: fine
    delivered = int(ids[0, 0].item())                           # seen by job 0 now (a replaced miss is not)
    fresh = [i for i in range(100) if i not in ids[0, :4].tolist() and i not in (1, 2, 3, 4)][:3]
    with pytest.raises(S.SenecaError) as ei:
        g.next_batch([0], requested=[[delivered] + fresh])      # already seen by job 0
    assert ei.value.status == S.EPROTO
    with pytest.raises(S.SenecaError) as ei:
        g.next_batch([0, 0], requested=[[5, 6, 7, 8], [9, 10, 11, 12]])
    assert ei.value.status == S.EINVAL
    h = P.ODSContext(8, [8, 4], [1, 2], 0, 0, 2, 3)
    h.next_batch([0, 1])
    with pytest.raises(S.SenecaError) as ei:
        h.next_batch([0])                                    # job 0 departed
    assert ei.value.status == S.ESTATE
    g.sync()
    h.sync()


def test_determinism_and_launch_count():
    c = synth.ods_config("imagenet1k", scale=64, seed=2)
    ce, cd, ca = caps_of(c)
    outs = []
    for _ in range(2):
        g = P.ODSContext(c["n_total"], c["batch"], c["target"], ce, cd, ca, 2)
        g.replay_epochs(2)
        torch.cuda.synchronize()
        outs.append(g.stats()[0].tobytes())
        assert g.launches() > 0
    assert outs[0] == outs[1]


# ---------------------------------------------------------------- replicas
def compare_replica(o, g, k, tr_k=None):
    st_o, ev_o, rf_o = o.stats()
    st_g, ev_g, rf_g = g.stats(k)
    assert (ev_g, rf_g) == (ev_o, rf_o), k
    assert st_g.tobytes() == st_o.tobytes(), k
    for a, b in zip(g.state(k), o.state()):
        np.testing.assert_array_equal(a, b)
    if tr_k is not None:
        assert np.array_equal(tr_k.cpu().numpy().view(np.uint64), o.transcript()), k


@pytest.mark.parametrize("name,scale,R", [("toy", 1, 48), ("toy", 1, 64), ("imagenet1k", 64, 4),
                                          ("openimages", 64, 3), ("imagenet1k", 64, 40)])
def test_replicas_match_independent_oracles(name, scale, R):
    """R replicas in one context == R independent oracle replays with seeds
    seed + k (every decision, bitmap and counter), including launches that fill
    the GPU with round CTAs: toy 48 x 3 CTAs (one 512-thread CTA per SM), toy
    64 x 3 and ImageNet-1K/64 40 x 5 (two 256-thread CTAs per SM)."""
    seed = 3
    c = synth.ods_config(name, scale=scale, seed=seed)
    ce, cd, ca = caps_of(c)
    g = P.ODSContext(c["n_total"], c["batch"], c["target"], ce, cd, ca, seed, replicas=R)
    tr = g.new_transcript()
    rounds = g.replay_epochs(max(c["target"]), tr)
    torch.cuda.synchronize()
    g.sync()
    for k in range(R):
        o = O.ODS(c["n_total"], c["batch"], c["target"], ce, cd, ca, seed + k, transcript=True)
        assert o.replay_epochs(max(c["target"])) == rounds
        compare_replica(o, g, k, tr[k])


@pytest.mark.parametrize("name,split,R", [("imagenet22k", (100, 0, 0), 4), ("openimages", (52, 48, 0), 8),
                                          ("openimages", (52, 48, 0), 20)])
def test_replicas_uncoupled(name, split, R):
    """Replicas of the uncoupled instantiation (no tracked tier: the paper's own
    OpenImages / ImageNet-22K splits): 512-thread CTAs (22K), 256-thread CTAs one
    per SM (OpenImages x 8: its longest round chain has batch 128) and two per SM
    (OpenImages x 20) -- each replica equals its independent oracle replay."""
    seed = 5
    c = synth.ods_config(name, scale=64, seed=seed)
    c["split"] = split
    ce, cd, ca = caps_of(c)
    assert ca == 0
    g = P.ODSContext(c["n_total"], c["batch"], c["target"], ce, cd, ca, seed, replicas=R)
    tr = g.new_transcript()
    rounds = g.replay_epochs(max(c["target"]), tr)
    torch.cuda.synchronize()
    g.sync()
    for k in range(R):
        o = O.ODS(c["n_total"], c["batch"], c["target"], ce, cd, ca, seed + k, transcript=True)
        assert o.replay_epochs(max(c["target"])) == rounds
        compare_replica(o, g, k, tr[k])


def test_replicas_next_batch():
    n, batch, target, R = 600, [16, 40, 9], [2, 1, 2], 3
    g = P.ODSContext(n, batch, target, 60, 50, 90, 21, replicas=R)
    oracles = [O.ODS(n, batch, target, 60, 50, 90, 21 + k, transcript=False) for k in range(R)]
    st = synth.Stream(5)
    for _ in range(120):
        _, _, _, act = oracles[0].job_state()
        live = [j for j in range(3) if act[j]]
        if not live:
            break
        pick = [j for j in live if st.uniform(1)[0] < 0.6] or live[-1:]
        ids_g, src_g, lens_g = g.next_batch(pick)
        torch.cuda.synchronize()
        assert ids_g.shape == (R, len(pick), max(batch))
        for k, o in enumerate(oracles):
            rc, ids_o, src_o, lens_o = o.round(pick)
            assert rc == 0 and list(lens_o) == lens_g
            for x, L_ in enumerate(lens_g):
                assert np.array_equal(ids_g[k, x, :L_].cpu().numpy().view(np.uint32), ids_o[x, :L_])
                assert np.array_equal(src_g[k, x, :L_].cpu().numpy(), src_o[x, :L_])
    for k, o in enumerate(oracles):
        compare_replica(o, g, k)


def test_replicas_that_cannot_be_co_resident_are_rejected():
    with pytest.raises(S.SenecaError) as ei:
        P.ODSContext(1000, [32] * 8, [1] * 8, 10, 10, 10, 1, replicas=64)      # 64 x 9 CTAs > 2 x 148
    assert ei.value.status == S.EINVAL


# ---------------------------------------------------------------- evict_tiers = ALL (R-O21)
@pytest.mark.parametrize("block", range(4))
def test_evict_all_random_tiny_configs(block):
    st = synth.Stream(9000 + block)
    for _ in range(50):
        c = synth.random_tiny_ods(st)
        replay_pair(c["n_total"], c["batch"], c["target"], c["cap_e"], c["cap_d"], c["cap_a"], c["seed"],
                    evict_all=True)


@pytest.mark.parametrize("name", ["toy", "imagenet1k", "openimages", "imagenet22k"])
def test_evict_all_scaled_configs_full_replay(name):
    """SURVEY 8(d) parity variant: every config scaled down (N/64) with split
    34-33-33 in the second eviction mode; the toy config at its own size."""
    scale = 1 if name == "toy" else 64
    c = synth.ods_config(name, scale=scale, seed=2)
    ce, cd, ca = caps_of(c)
    o, g = replay_pair(c["n_total"], c["batch"], c["target"], ce, cd, ca, 2, evict_all=True)
    assert o.stats()[1] > 0                                      # evictions happened


def test_evict_all_imagenet22k_full_size_prefix():
    """ImageNet-22K additionally runs with evict_tiers = ALL (O4):
    full size, its own 100-0-0 split (E churns), first rounds vs the oracle."""
    seed = synth.PERF_SEED
    c = synth.ods_config("imagenet22k", seed=seed)
    ce, cd, ca = caps_of(c)
    o, g = make_pair(c["n_total"], c["batch"], c["target"], ce, cd, ca, seed, transcript=False, evict_all=True)
    assert g.replay_rounds(60) == 60
    assert o.replay_rounds(60) == 60
    torch.cuda.synchronize()
    compare_state(o, g)


def test_evict_all_imagenet22k_own_split_scaled_full_replay():
    """ImageNet-22K shape at its own 100-0-0 split (an E-only cache), N/64, whole
    replay under evict_tiers = ALL: E entries consumed by all 8 jobs churn."""
    c = synth.ods_config("imagenet22k", scale=64, seed=5)
    c["split"] = (100, 0, 0)
    ce, cd, ca = caps_of(c)
    assert cd == 0 and ca == 0 and ce > 0
    o, g = replay_pair(c["n_total"], c["batch"], c["target"], ce, cd, ca, 5, evict_all=True)
    assert o.stats()[1] > 0


def test_evict_all_next_batch_and_replicas():
    n, batch, target, R = 500, [16, 40, 9], [2, 1, 2], 3
    g = P.ODSContext(n, batch, target, 60, 50, 40, 31, replicas=R, evict_tiers=1)
    oracles = [O.ODS(n, batch, target, 60, 50, 40, 31 + k, evict_all=True) for k in range(R)]
    st = synth.Stream(6)
    for _ in range(100):
        _, _, _, act = oracles[0].job_state()
        live = [j for j in range(3) if act[j]]
        if not live:
            break
        pick = [j for j in live if st.uniform(1)[0] < 0.7] or live[:1]
        ids_g, src_g, lens_g = g.next_batch(pick)
        torch.cuda.synchronize()
        for k, o in enumerate(oracles):
            rc, ids_o, src_o, lens_o = o.round(pick)
            assert rc == 0 and list(lens_o) == lens_g
            for x, L_ in enumerate(lens_g):
                assert np.array_equal(ids_g[k, x, :L_].cpu().numpy().view(np.uint32), ids_o[x, :L_])
                assert np.array_equal(src_g[k, x, :L_].cpu().numpy(), src_o[x, :L_])
    for k, o in enumerate(oracles):
        compare_replica(o, g, k)


# ---------------------------------------------------------------- NEXT-1 epoch model
@pytest.mark.parametrize("name,scale", [("toy", 1), ("imagenet1k", 64), ("openimages", 64)])
def test_epoch_model_matches_oracle(name, scale):
    c = synth.ods_config(name, scale=scale, seed=3)
    ce, cd, ca = caps_of(c)
    o, g = make_pair(c["n_total"], c["batch"], c["target"], ce, cd, ca, 3, transcript=False)
    g.replay_epochs(max(c["target"]))
    o.replay_epochs(max(c["target"]))
    torch.cuda.synchronize()
    dsi = (8014.245267534, 6424.75, 9783.0, 2735.52905131)
    got = g.epoch_model(dsi)
    want = O.epoch_metrics(o.stats()[0], c["n_total"], dsi)
    for f in ("epoch_seconds", "dsi_mix", "hit_rate"):
        assert np.array_equal(got[f].view(np.uint64), want[f].view(np.uint64)), f
    for f in ("decode_aug_ops", "aug_only_ops"):
        assert np.array_equal(got[f], want[f]), f
    with pytest.raises(S.SenecaError):
        g.epoch_model((1.0, 0.0, 1.0, 1.0))


# ---------------------------------------------------------------- uniform no-evict baseline sampler (R-O22)
def test_baseline_sampler_random_tiny_and_scaled():
    st = synth.Stream(12000)
    for _ in range(60):
        c = synth.random_tiny_ods(st)
        replay_pair(c["n_total"], c["batch"], c["target"], c["cap_e"], c["cap_d"], c["cap_a"], c["seed"],
                    baseline=True)
    for name in ("toy", "imagenet1k", "openimages"):
        c = synth.ods_config(name, scale=1 if name == "toy" else 64, seed=4)
        ce, cd, ca = caps_of(c)
        o, g = replay_pair(c["n_total"], c["batch"], c["target"], ce, cd, ca, 4, baseline=True)
        st_g, ev, rf = g.stats()
        assert ev == 0 and rf == 0
        assert np.all(st_g["served"][:, :, 1:].sum(axis=2) == ce + cd + ca)     # hit rate = cached fraction


@pytest.mark.parametrize("evict_all", [False, True])
def test_thirty_two_jobs(evict_all):
    """The maximum job count (a full 32-bit active mask, 33 round CTAs), mixed
    batches and targets (staggered departures), every tier populated."""
    batch = [1 + (7 * j) % 32 for j in range(32)]
    target = [1 + j % 3 for j in range(32)]
    replay_pair(3000, batch, target, 300, 200, 400, 17, evict_all=evict_all)


def test_replay_epoch_alias():
    """seneca_replay_epoch (the north_star name) is seneca_replay_epochs."""
    import ctypes
    c = synth.ods_config("toy", seed=6)
    ce, cd, ca = caps_of(c)
    a = P.ODSContext(c["n_total"], c["batch"], c["target"], ce, cd, ca, 6)
    b = P.ODSContext(c["n_total"], c["batch"], c["target"], ce, cd, ca, 6)
    ra = a.replay_epochs(3)
    rb = ctypes.c_uint64()
    assert S.lib().seneca_replay_epoch(b.ctx, 3, None, ctypes.byref(rb),
                                       torch.cuda.current_stream().cuda_stream) == 0
    torch.cuda.synchronize()
    assert ra == rb.value and a.stats()[0].tobytes() == b.stats()[0].tobytes()


# ---------------------------------------------------------------- job arrivals (R-O23)
@pytest.mark.parametrize("block", range(3))
def test_arrivals_random_tiny_configs(block):
    st = synth.Stream(14000 + block)
    for _ in range(40):
        c = synth.random_tiny_ods(st)
        J = len(c["batch"])
        arr = [0 if k == 0 else int(st.u64(1)[0] % 40) for k in range(J)]
        for evict_all in (False, True):
            o = O.ODS(c["n_total"], c["batch"], c["target"], c["cap_e"], c["cap_d"], c["cap_a"], c["seed"],
                      transcript=True, evict_all=evict_all, arrival=arr)
            g = P.ODSContext(c["n_total"], c["batch"], c["target"], c["cap_e"], c["cap_d"], c["cap_a"], c["seed"],
                             evict_tiers=int(evict_all), arrival=arr)
            tr = g.new_transcript()
            rg = g.replay_epochs(max(c["target"]), tr)
            ro = o.replay_epochs(max(c["target"]))
            torch.cuda.synchronize()
            assert rg == ro, (c, arr)
            compare_state(o, g, tr)


def test_arrivals_makespan_trace_and_replicas():
    """Two-at-a-time makespan trace on ImageNet-1K/64 (A churn), 3 replicas."""
    c = synth.ods_config("imagenet1k", scale=64, seed=9)
    ce, cd, ca = caps_of(c)
    per_job = c["target"][0] * -(-c["n_total"] // c["batch"][0])
    arr = [0, 0, per_job, per_job]
    R = 3
    g = P.ODSContext(c["n_total"], c["batch"], c["target"], ce, cd, ca, 9, replicas=R, arrival=arr)
    tr = g.new_transcript()
    rounds = g.replay_epochs(max(c["target"]), tr)
    torch.cuda.synchronize()
    assert rounds == 2 * per_job
    for k in range(R):
        o = O.ODS(c["n_total"], c["batch"], c["target"], ce, cd, ca, 9 + k, transcript=True, arrival=arr)
        assert o.replay_epochs(max(c["target"])) == rounds
        compare_replica(o, g, k, tr[k])


def test_arrivals_next_batch():
    n, batch, target = 500, [16, 40, 9], [2, 1, 2]
    arr = [0, 12, 30]
    o = O.ODS(n, batch, target, 60, 50, 40, 3, arrival=arr)
    g = P.ODSContext(n, batch, target, 60, 50, 40, 3, arrival=arr)
    with pytest.raises(S.SenecaError) as ei:
        g.next_batch([1])                                     # job 1 arrives at round 12
    assert ei.value.status == S.ESTATE
    st = synth.Stream(4)
    for _ in range(200):
        _, e, _, _ = o.job_state()
        if all(int(e[j]) >= target[j] for j in range(3)):
            break
        live = [j for j in range(3) if arr[j] <= o.r and int(e[j]) < target[j]]
        if not live:                                         # idle round on both sides
            assert o.replay_rounds(1) == 1 and g.replay_rounds(1) == 1
            continue
        pick = [j for j in live if st.uniform(1)[0] < 0.7] or live[:1]
        rc, ids_o, src_o, lens_o = o.round(pick)
        assert rc == 0
        ids_g, src_g, lens_g = g.next_batch(pick)
        torch.cuda.synchronize()
        assert list(lens_o) == lens_g
        for x, L_ in enumerate(lens_g):
            assert np.array_equal(ids_g[x, :L_].cpu().numpy().view(np.uint32), ids_o[x, :L_])
            assert np.array_equal(src_g[x, :L_].cpu().numpy(), src_o[x, :L_])
    compare_state(o, g)


# ---------------------------------------------------------------- cold start (R-O24)
def test_cold_start_random_tiny_configs():
    st = synth.Stream(16000)
    for _ in range(50):
        c = synth.random_tiny_ods(st)
        for evict_all, baseline in ((False, False), (True, False), (False, True)):
            o = O.ODS(c["n_total"], c["batch"], c["target"], c["cap_e"], c["cap_d"], c["cap_a"], c["seed"],
                      transcript=True, evict_all=evict_all, baseline=baseline, cold=True)
            g = P.ODSContext(c["n_total"], c["batch"], c["target"], c["cap_e"], c["cap_d"], c["cap_a"], c["seed"],
                             evict_tiers=int(evict_all), sampler=int(baseline), cold_start=1)
            tr = g.new_transcript()
            assert g.replay_epochs(max(c["target"]), tr) == o.replay_epochs(max(c["target"]))
            torch.cuda.synchronize()
            compare_state(o, g, tr)


@pytest.mark.parametrize("name,evict_all", [("toy", False), ("imagenet1k", False), ("imagenet1k", True),
                                            ("openimages", False)])
def test_cold_start_scaled_configs(name, evict_all):
    scale = 1 if name == "toy" else 64
    c = synth.ods_config(name, scale=scale, seed=12)
    ce, cd, ca = caps_of(c)
    o = O.ODS(c["n_total"], c["batch"], c["target"], ce, cd, ca, 12, transcript=True, evict_all=evict_all,
              cold=True)
    g = P.ODSContext(c["n_total"], c["batch"], c["target"], ce, cd, ca, 12, evict_tiers=int(evict_all),
                     cold_start=1, replicas=2)
    tr = g.new_transcript()
    assert g.replay_epochs(max(c["target"]), tr) == o.replay_epochs(max(c["target"]))
    torch.cuda.synchronize()
    compare_replica(o, g, 0, tr[0])
    o1 = O.ODS(c["n_total"], c["batch"], c["target"], ce, cd, ca, 13, transcript=True, evict_all=evict_all,
               cold=True)
    o1.replay_epochs(max(c["target"]))
    compare_replica(o1, g, 1, tr[1])


def test_cold_start_next_batch_and_arrivals():
    n, batch, target, arr = 600, [16, 40, 9], [2, 1, 2], [0, 5, 20]
    o = O.ODS(n, batch, target, 60, 50, 40, 7, cold=True, arrival=arr)
    g = P.ODSContext(n, batch, target, 60, 50, 40, 7, cold_start=1, arrival=arr)
    st = synth.Stream(8)
    for _ in range(200):
        _, e, _, _ = o.job_state()
        if all(int(e[j]) >= target[j] for j in range(3)):
            break
        live = [j for j in range(3) if arr[j] <= o.r and int(e[j]) < target[j]]
        if not live:
            assert o.replay_rounds(1) == 1 and g.replay_rounds(1) == 1
            continue
        pick = [j for j in live if st.uniform(1)[0] < 0.7] or live[-1:]
        rc, ids_o, src_o, lens_o = o.round(pick)
        ids_g, src_g, lens_g = g.next_batch(pick)
        torch.cuda.synchronize()
        for x, L_ in enumerate(lens_g):
            assert np.array_equal(ids_g[x, :L_].cpu().numpy().view(np.uint32), ids_o[x, :L_])
            assert np.array_equal(src_g[x, :L_].cpu().numpy(), src_o[x, :L_])
    compare_state(o, g)


# ---------------------------------------------------------------- permutation ring
@pytest.mark.parametrize("evict_all,R", [(False, 1), (True, 1), (False, 3), (True, 3)])
def test_permutation_ring_jobs_at_different_epochs(evict_all, R):
    """Mixed batches and target epochs (7, 3, 5, 1): the jobs cross epoch
    boundaries at different rounds.  One replica: the 2-slot ring of each job is
    refilled DURING the launch by the concurrent generator (ods_perm_ring);
    replicas: launches stop where a job would enter an epoch that is not in its
    ring.  Every decision equals the oracle's (transcripts), also with the replay
    cut into random-length launches on top."""
    n = 5003
    batch, target = [64, 512, 200, 1000], [7, 3, 5, 1]
    ce, cd, ca = 700, 400, 600
    g = P.ODSContext(n, batch, target, ce, cd, ca, 9, replicas=R, evict_tiers=int(evict_all))
    tr = g.new_transcript()
    st = synth.Stream(99)
    total = 0
    while g.view().active_mask:
        k = int(st.u64(1)[0] % np.uint64(97)) + 1
        done = g.replay_rounds(k, tr)
        total += done
        if done < k:
            break
    torch.cuda.synchronize()
    g.sync()
    for k in range(R):
        o = O.ODS(n, batch, target, ce, cd, ca, 9 + k, transcript=True, evict_all=evict_all)
        assert total == o.replay_epochs(max(target))
        compare_replica(o, g, k, tr if R == 1 else tr[k])


def test_permutation_ring_replicas_many_epochs():
    """Replicas generate their ring on the caller's stream between launches: 12
    replicas x 12 epochs of ImageNet-1K/64, each equal to its oracle replay."""
    seed = 4
    c = synth.ods_config("imagenet1k", scale=64, seed=seed)
    c["target"] = [12, 11, 12, 9]
    ce, cd, ca = caps_of(c)
    R = 12
    g = P.ODSContext(c["n_total"], c["batch"], c["target"], ce, cd, ca, seed, replicas=R)
    rounds = g.replay_epochs(max(c["target"]))
    torch.cuda.synchronize()
    g.sync()
    for k in (0, 5, 11):
        o = O.ODS(c["n_total"], c["batch"], c["target"], ce, cd, ca, seed + k)
        assert o.replay_epochs(max(c["target"])) == rounds
        compare_replica(o, g, k)


def test_workspace_above_2gib_per_replica():
    """a replica slice above 2 GiB (32 jobs x 14.2 M samples: rings and
    lap lists of 3.6 GB each) -- the per-launch signal reset and the status read
    use the contiguous control block, so two such replicas replay and report OK;
    replica 1 equals its oracle replay for the rounds played."""
    c = synth.ods_config("imagenet22k", seed=6)
    ce, cd, ca = caps_of(c)
    J = 32
    batch, target = [128] * J, [2] * J
    g = P.ODSContext(c["n_total"], batch, target, ce, cd, ca, 6, replicas=2)
    v = g.view()
    assert v.replica_stride > 2 ** 31
    assert g.replay_rounds(3) == 3
    torch.cuda.synchronize()
    g.sync()
    o = O.ODS(c["n_total"], batch, target, ce, cd, ca, 7)
    o.replay_rounds(3)
    compare_replica(o, g, 1)
    g.close()


@pytest.mark.parametrize("env", [{}, {"SENECA_ROUND_CLUSTER": "0"}, {"SENECA_DSMEM_SIGNALS": "0"}])
def test_coupled_signal_paths(env):
    """The three signal paths of a coupled replay: the J + 1 CTAs as
    one cluster with DSMEM signals (default), the plain cooperative launch with
    global-memory signals (SENECA_ROUND_CLUSTER=0, also what runs under ncu), and
    the cluster launch with global signals (SENECA_DSMEM_SIGNALS=0) -- A churn,
    evict-all and cold start in launches of random length, vs the oracle (the
    knobs are read once per process, hence a subprocess)."""
    import subprocess
    import sys
    out = subprocess.run([sys.executable, os.path.join(os.path.dirname(HERE), "tools", "signal_paths.py")],
                         capture_output=True, text=True, timeout=600, env=dict(os.environ, **env))
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-3000:]
    assert "signal paths ok" in out.stdout


# ---------------------------------------------------------------- sample-ID-range sharding
def sharded_replay(c, ce, cd, ca, seed, G, evict_all=False, cold=False, arrival=None, rounds=None):
    g = P.ODSContext(c["n_total"], c["batch"], c["target"], ce, cd, ca, seed, shards=G,
                     evict_tiers=int(evict_all), cold_start=int(cold), arrival=arrival)
    tr = g.new_transcript()
    r = g.replay_rounds(rounds, tr) if rounds else g.replay_epochs(max(c["target"]), tr)
    torch.cuda.synchronize()
    g.sync()
    return g, tr, r


@pytest.mark.parametrize("name,scale", [("toy", 1), ("imagenet1k", 64), ("openimages", 64), ("imagenet22k", 64)])
def test_sharded_replay_identical_for_every_G(name, scale):
    """Invariant I8: one replay partitioned by sample-ID range over
    G = 1, 2, 4, 8 shards (all shards in one launch on this device, exchanging
    pool sizes and resolved ids through their mailboxes every round) delivers
    exactly the oracle's transcript on EVERY shard, with identical bitmaps and
    counters.  Toy (one superblock: shards 1.. own nothing), N/64 configs with
    A churn (ImageNet-1K), mixed batches (OpenImages) and 55 superblocks (22K)."""
    seed = 12
    c = synth.ods_config(name, scale=scale, seed=seed)
    ce, cd, ca = caps_of(c)
    o = O.ODS(c["n_total"], c["batch"], c["target"], ce, cd, ca, seed, transcript=True)
    ro = o.replay_epochs(max(c["target"]))
    for G in (1, 2, 4, 8):
        try:
            g, tr, r = sharded_replay(c, ce, cd, ca, seed, G)
        except Exception as e:
            raise AssertionError(f"G = {G}: {e}")
        assert r == ro
        for k in range(G):
            compare_replica(o, g, k, tr if G == 1 else tr[k])
        g.close()


@pytest.mark.parametrize("mode", ["evict_all", "cold", "arrivals"])
def test_sharded_replay_variants(mode):
    """Sharding under evict_tiers = ALL (E/D churn through the exchange), cold start
    (admissions replicated, counts per shard) and job arrivals (pools rebuilt per
    shard at arrival), G = 3 and 8, against the oracle."""
    seed = 13
    c = synth.ods_config("imagenet1k", scale=64, seed=seed)
    ce, cd, ca = caps_of(c)
    kw = dict(evict_all=mode == "evict_all", cold=mode == "cold")
    arr = None
    if mode == "arrivals":
        per_job = c["target"][0] * -(-c["n_total"] // c["batch"][0])
        arr = [0, 0, per_job // 3, per_job]
    o = O.ODS(c["n_total"], c["batch"], c["target"], ce, cd, ca, seed, transcript=True, arrival=arr, **kw)
    ro = o.replay_epochs(max(c["target"]))
    for G in (3, 8):
        g, tr, r = sharded_replay(c, ce, cd, ca, seed, G, arrival=arr, **kw)
        assert r == ro
        for k in range(G):
            compare_replica(o, g, k, tr[k])
        g.close()


def test_sharded_full_size_prefix_22k():
    """The full ImageNet-22K config (3,467 superblocks) split over 8 shards, first
    160 rounds, every shard against the oracle (bitmaps and counters)."""
    seed = synth.PERF_SEED
    c = synth.ods_config("imagenet22k", seed=seed)
    ce, cd, ca = caps_of(c)
    g = P.ODSContext(c["n_total"], c["batch"], c["target"], ce, cd, ca, seed, shards=8)
    assert g.replay_rounds(160) == 160
    torch.cuda.synchronize()
    g.sync()
    o = O.ODS(c["n_total"], c["batch"], c["target"], ce, cd, ca, seed)
    o.replay_rounds(160)
    for k in (0, 7):
        compare_replica(o, g, k)


@pytest.mark.parametrize("block", range(2))
def test_sharded_late_mode_random_static_configs(block):
    """Sharded replays with static tiers: once a job's pools are empty GLOBALLY
    (the sizes every shard learns in C1, less the round's substitutes) every
    shard enters the storage-list walk in the same round, skips C1/C2 and the
    classification gathers, and decides the rest of the epoch with the late bulk
    until the epoch-start recount resumes the exchange.  Random
    static configs, G = 2 / 3 / 5, replays cut into launches of random length
    (the late state and the stamps persist across launches), every shard vs the
    oracle transcript, bitmaps and counters."""
    st = synth.Stream(9900 + block)
    for it in range(6):
        n = int(st.choice(1, [1000, 16385, 40000, 70000])[0])
        J = int(st.choice(1, [1, 2, 3])[0])
        batch = [int(x) for x in st.choice(J, [7, 64, 100, 512])]
        target = [int(x) for x in st.choice(J, [1, 2, 3])]
        ce = int(n * float(st.uniform(1)[0]) * 0.6)
        cd = int((n - ce) * float(st.uniform(1)[0]) * 0.5) if it % 2 else 0
        G = (2, 3, 5)[it % 3]
        seed = int(st.u64(1)[0])
        o = O.ODS(n, batch, target, ce, cd, 0, seed, transcript=True)
        g = P.ODSContext(n, batch, target, ce, cd, 0, seed, shards=G)
        tr = g.new_transcript()
        total = 0
        while g.view().active_mask:
            k = int(st.u64(1)[0] % np.uint64(400)) + 1
            done = g.replay_rounds(k, tr)
            total += done
            if done < k:
                break
        torch.cuda.synchronize()
        g.sync()
        assert total == o.replay_epochs(max(target)), (n, batch, target, ce, cd, G)
        for k in range(G):
            compare_replica(o, g, k, tr[k])
        g.close()


@pytest.mark.parametrize("G,name,scale", [(2, "toy", 1), (4, "imagenet1k", 64), (2, "openimages", 64),
                                          (3, "imagenet22k", 64)])
def test_sharded_one_context_per_shard(G, name, scale):
    """shard_mode 1 (one shard per context, peers attached by mailbox address, as
    one process per GPU runs it): G contexts on this device replay concurrently
    on G streams and every shard equals the oracle (subprocess under a timeout:
    a missing peer would spin)."""
    import subprocess
    import sys
    out = subprocess.run([sys.executable, os.path.join(os.path.dirname(HERE), "tools", "shard_contexts.py"),
                          str(G), name, str(scale)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-3000:]
    assert "ok" in out.stdout


@pytest.mark.parametrize("args", [["2"], ["2", "openimages", "256"], ["3", "imagenet22k", "1024"]])
def test_sharded_across_processes_cuda_ipc(args):
    """PROCESSES, one shard each (the one-process-per-GPU layout, all on this
    device): mailboxes mapped by CUDA IPC through dist.attach_shard_peers (handles
    all-gathered over gloo); each rank's transcript equals the oracle's.  Without
    MPS the processes time-slice the device, so only small replays are run: the
    toy (A churn) and two static-tier configs (tracked sizes and late mode across
    processes)."""
    import subprocess
    import sys
    out = subprocess.run([sys.executable, os.path.join(os.path.dirname(HERE), "tools", "shard_ranks.py"), *args],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-3000:]
    assert "all ranks ok" in out.stdout


# ---------------------------------------------------------------- storage-list walk (static tiers)
@pytest.mark.parametrize("block", range(3))
def test_storage_list_walk_random_static_configs(block):
    """Static tiers (no A tier, ODS sampler, one replica): once all of a job's pools
    are empty the kernel walks the epoch's storage-list segments and the lap
    lists without seen tests (Cfg.late).  Random tiny and small
    configs (N up to 70,000: several 16 K-position generation chunks, empty
    segments when everything is cached), mixed batches and epochs, replays cut
    into random-length launches (the late state persists across launches), vs
    the oracle transcript."""
    st = synth.Stream(9100 + block)
    for it in range(12):
        n = int(st.choice(1, [40, 1000, 16384, 16385, 40000, 70000])[0])
        J = int(st.choice(1, [1, 2, 3, 4])[0])
        batch = [int(x) for x in st.choice(J, [7, 64, 100, 512])]
        target = [int(x) for x in st.choice(J, [1, 2, 3])]
        frac_e, frac_d = float(st.uniform(1)[0]), float(st.uniform(1)[0])
        ce = int(n * frac_e * 0.6)
        cd = int((n - ce) * frac_d * 0.5) if it % 3 else 0
        if it % 5 == 4:
            ce, cd = n, 0                                 # everything cached: empty storage segments
        seed = int(st.u64(1)[0])
        o, g = make_pair(n, batch, target, ce, cd, 0, seed)
        tr = g.new_transcript()
        total = 0
        while g.view().active_mask:
            k = int(st.u64(1)[0] % np.uint64(400)) + 1
            done = g.replay_rounds(k, tr)
            total += done
            if done < k:
                break
        torch.cuda.synchronize()
        assert total == o.replay_epochs(max(target)), (n, batch, target, ce, cd)
        compare_state(o, g, tr)


@pytest.mark.parametrize("block", range(2))
def test_late_bulk_with_arrivals_departures_and_launch_cuts(block):
    """The late bulk: an uncoupled job's late rounds decided in one
    pass while warp 0 advances the schedule in closed form.  Static tiers (so the
    bulk applies), jobs arriving at random rounds and departing after different
    epoch counts (spans of the closed-form skip cut at arrivals, departures inside
    them), mixed batches, replays cut into launches of random length (bulk spans
    end at launch edges), vs the oracle transcript, counters and state."""
    st = synth.Stream(9700 + block)
    for it in range(10):
        n = int(st.choice(1, [300, 1000, 16385, 40000])[0])
        J = int(st.choice(1, [2, 3, 4])[0])
        batch = [int(x) for x in st.choice(J, [7, 32, 100, 256])]
        target = [int(x) for x in st.choice(J, [1, 2, 3])]
        ce = int(n * float(st.uniform(1)[0]) * 0.5)
        cd = int((n - ce) * float(st.uniform(1)[0]) * 0.3) if it % 2 else 0
        arr = [0] + [int(st.u64(1)[0] % np.uint64(60)) for _ in range(J - 1)]
        seed = int(st.u64(1)[0])
        o = O.ODS(n, batch, target, ce, cd, 0, seed, transcript=True, arrival=arr)
        g = P.ODSContext(n, batch, target, ce, cd, 0, seed, arrival=arr)
        tr = g.new_transcript()
        total = 0
        while True:                                       # (pending arrivals are not in active_mask)
            k = int(st.u64(1)[0] % np.uint64(300)) + 1
            try:
                done = g.replay_rounds(k, tr)
            except S.SenecaError as ex:                   # the last launch ended exactly at the end
                assert ex.status == S.ESTATE
                break
            total += done
            if done < k:
                break
        torch.cuda.synchronize()
        assert total == o.replay_epochs(max(target)), (n, batch, target, ce, cd, arr)
        compare_state(o, g, tr)
