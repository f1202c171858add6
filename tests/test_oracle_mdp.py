"""Pins for the oracle's MDP evaluator: the DSI model (Eqs. 1-9, §5.1,
P:L465-664) and the brute-force split search."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
import synth
from tests import mdp_exact

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table4_nominal_vals.json")))
CACHE, NIC, PCIE, CPU_AUG, CPU_DEC_AUG, GPU, STORAGE = range(7)


def prof(server, **over):
    g = {k: v for k, v in GOLD[server].items() if not k.startswith("_")}
    kw = dict(g, model_bytes=0.0, n_total=1_300_000, nodes=1, gpus_per_node=1)
    kw.update(over)
    return O.make_profile(**kw)


# ------------------------------------------------------------ Eq. 1-4 with Table 4 values
def test_in_house_dsi_e_is_cpu_bound_2132():
    # T_{D+A} = 2132 binds Eq. 3 (B_cache/S = 10965 > 2132)
    d, l = O.tiers(prof("in_house"))
    assert d[2] == 2132.0 and l[2] == CPU_DEC_AUG
    # Eq. 4: B_storage/S = 500e6/114e3 = 4386 > 2132 -> DSI_S = DSI_E
    assert d[3] == 2132.0 and l[3] == CPU_DEC_AUG


def test_in_house_dsi_a_cache_bound():
    # Eq. 1: B_cache/(M S) = 1.25e9/(5.12*114e3) = 1.25e9/583680 (ties with NIC -> first term)
    d, l = O.tiers(prof("in_house"))
    assert d[0] == 1.25e9 / 583680.0 and l[0] == CACHE
    assert abs(d[0] - 2141.5844298245) < 1e-9
    # Eq. 2: T_A = 4050 does not bind -> DSI_D == DSI_A exactly
    assert d[1] == d[0] and l[1] == CACHE


def test_azure_9139_rows():
    p = prof("azure", s_data=91_390, n_total=14_000_000)
    d, l = O.tiers(p)
    assert d[2] == 9783.0 and l[2] == CPU_DEC_AUG                 # Eq. 3
    assert d[3] == 250e6 / 91390.0 and l[3] == STORAGE             # Eq. 4 storage-bound
    assert abs(d[3] - 2735.5290513185) < 1e-9
    assert d[0] == 3.75e9 / 467916.8 and l[0] == CACHE             # Eq. 1 (SPEC's "8013" is a slip)
    assert abs(d[0] - 8014.2452675347) < 1e-9


def test_degeneracies_eq2_eq4():
    p = prof("in_house", t_augment=1e300)
    d, l = O.tiers(p)
    assert d[1] == d[0] and l[1] == l[0]                           # Eq. 2 -> Eq. 1
    p = prof("azure", b_storage=1e300)
    d, l = O.tiers(p)
    assert d[3] == d[2] and l[3] == l[2]                           # Eq. 4 -> Eq. 3
    p = prof("in_house", t_gpu=1000.0, b_cache=1e300, b_nic=1e300, b_pcie=1e300,
             t_augment=1e300, t_decode_augment=1e300, b_storage=1e300)
    d, l = O.tiers(p)
    assert d == [1000.0] * 4 and l == [GPU] * 4


# ------------------------------------------------------------ A1: comm overhead
def test_comm_overhead_closed_form():
    assert O.comm_overhead(1, 100e6) == 0.0
    assert O.comm_overhead(4, 100e6) == 150e6
    assert O.comm_overhead(2, 0.0) == 0.0
    assert O.comm_overhead(8, 8e6) == 14e6


def test_comm_mapping_and_nvlink_zeroing():
    # 4 nodes x 2 GPUs, 100 MB model.  mapping 0: C_nw = C(4) = 150 MB on the NIC term.
    base = dict(model_bytes=100e6, nodes=4, gpus_per_node=2, b_cache=1e300, t_gpu=1e300,
                t_decode_augment=1e300, t_augment=1e300)
    d0, l0 = O.tiers(prof("in_house", **base))
    ms = 583680.0
    assert d0[0] == min(4 * 1.25e9 / (ms + 150e6), 4 * 32e9 / (ms + 100e6))
    # mapping 1 (literal P:L529 text): C_nw = C(2) = 100 MB, C_PCIe = C(4) = 150 MB
    d1, _ = O.tiers(prof("in_house", comm_mapping=1, **base))
    assert d1[0] == min(4 * 1.25e9 / (ms + 100e6), 4 * 32e9 / (ms + 150e6))
    # inter-node NVLink zeroes both terms
    d2, _ = O.tiers(prof("in_house", nvlink_inter=1, **base))
    assert d2[0] == min(4 * 1.25e9 / ms, 4 * 32e9 / ms)
    # intra-node NVLink zeroes only C_PCIe
    d3, _ = O.tiers(prof("in_house", nvlink_intra=1, **base))
    assert d3[0] == min(4 * 1.25e9 / (ms + 150e6), 4 * 32e9 / ms)


# ------------------------------------------------------------ Eqs. 5-8
def test_counts_in1k_64gb_encoded_only():
    p = prof("in_house", n_total=1_300_000, s_data=114_620)
    # floor(64e9 / 114620) = 558366 (SPEC's 558,367 is a slip; R-M14)
    assert O.split_counts(p, 100, 0, 0) == [0, 0, 558_366, 741_634]
    assert O.split_counts(p, 0, 0, 0) == [0, 0, 0, 1_300_000]


def test_counts_full_fit_and_partition_identity():
    p = prof("in_house", n_total=1000, s_data=1000, cache_bytes=10**9)
    assert O.split_counts(p, 0, 0, 100) == [1000, 0, 0, 0]
    st = synth.Stream(5)
    for _ in range(200):
        n = int(st.u64(1)[0] % 10**7) + 1
        s = int(st.u64(1)[0] % 10**6) + 1
        cache = int(st.u64(1)[0] % 10**13)
        a = int(st.u64(1)[0] % 101); b = int(st.u64(1)[0] % (101 - a)); e = 100 - a - b
        p = prof("aws", n_total=n, s_data=s, cache_bytes=cache)
        c = O.split_counts(p, e, b, a)
        assert sum(c) == n and min(c) >= 0
        assert tuple(c) == mdp_exact.counts(n, s, cache, 128, 25, e, b, a)


# ------------------------------------------------------------ Eq. 9 degeneracies
def test_eq9_degenerate_identities():
    p = prof("azure", n_total=1_300_000, s_data=114_620)
    v, r, c = O.model_eval(p, 0, 0, 0)
    assert v == r.dsi_s                        # all storage -> DSI_S bit-exactly
    p = prof("azure", n_total=1000, s_data=1000, cache_bytes=10**9)
    v, r, c = O.model_eval(p, 0, 0, 100)
    assert v == r.dsi_a                        # full A fit -> DSI_A bit-exactly
    p = prof("in_house", n_total=1_300_000, s_data=114_620)
    v, r, c = O.model_eval(p, 100, 0, 0)       # DSI_E == DSI_S == 2132 -> weighting invariant
    assert abs(v - 2132.0) <= 2132.0 * 2 ** -51


def test_homogeneity_degree_one():
    # scaling every rate by 2 is exact in binary64 -> V doubles bit-exactly, counts fixed
    st = synth.Stream(9)
    cols = synth.mdp_profiles(50, seed=9)
    arr = O.profiles_from_columns(cols)
    arr2 = arr.copy()
    for f in ("t_gpu", "t_decode_augment", "t_augment", "b_nic", "b_pcie", "b_cache", "b_storage"):
        arr2[f] *= 2.0
    arr2["model_bytes"] *= 1.0
    for i in range(50):
        p, q = O.profile_row(arr, i), O.profile_row(arr2, i)
        for pe, pd, pa in [(100, 0, 0), (30, 30, 40), (0, 0, 100), (10, 85, 5)]:
            v1, _, c1 = O.model_eval(p, pe, pd, pa)
            v2, _, c2 = O.model_eval(q, pe, pd, pa)
            assert c1 == c2 and v2 == 2.0 * v1


def test_hardware_monotonicity():
    cols = synth.mdp_profiles(40, seed=10)
    arr = O.profiles_from_columns(cols)
    for f in ("t_gpu", "t_decode_augment", "t_augment", "b_nic", "b_pcie", "b_cache", "b_storage"):
        up = arr.copy()
        up[f] *= 1.5
        for i in range(40):
            for split in [(100, 0, 0), (50, 25, 25), (0, 100, 0), (0, 0, 100)]:
                assert O.model_eval(O.profile_row(up, i), *split)[0] >= O.model_eval(O.profile_row(arr, i), *split)[0]


# ------------------------------------------------------------ grid + argmax
def test_grid_sizes():
    assert O.num_splits(1) == 5151 and O.num_splits(10) == 66 and O.num_splits(100) == 3


@pytest.mark.parametrize("server,cache", [("azure", 64), ("azure", 115), ("azure", 400),
                                          ("aws", 64), ("aws", 400)])
def test_imagenet22k_rows_reproduce_100_0_0(server, cache):
    # tab:dataset_characteristics P:L976: ImageNet-22K -> 100-0-0 (reproducible rows, R-M16)
    p = prof(server, n_total=14_000_000, s_data=91_390, cache_bytes=cache * 10**9)
    arr = np.frombuffer(bytes(p), dtype=O.PROFILE_DTYPE).copy()
    res, _ = O.mdp_sweep(arr, 1)
    assert (res[0]["p_e"], res[0]["p_d"], res[0]["p_a"]) == (100, 0, 0)


def test_imagenet22k_azure_value():
    p = prof("azure", n_total=14_000_000, s_data=91_390)
    arr = np.frombuffer(bytes(p), dtype=O.PROFILE_DTYPE).copy()
    res, grid = O.mdp_sweep(arr, 1, want_grid=True)
    assert res[0]["v"] == 3088.051099033303 and grid.shape == (1, 5151)
    # the value is the exact-rational Eq. 9 rounded (single profile, unique max)
    ex = mdp_exact.exact_values(dict(n_total=14_000_000, s_data=91_390, cache_bytes=64 * 10**9,
                                     m_num=128, m_den=25),
                                [res[0]["dsi_a"], res[0]["dsi_d"], res[0]["dsi_e"], res[0]["dsi_s"]], 1)
    assert abs(float(max(ex)) - res[0]["v"]) <= 1e-12 * res[0]["v"]


def test_zero_cache_ties_break_to_100_0_0():
    p = prof("in_house", cache_bytes=0)
    arr = np.frombuffer(bytes(p), dtype=O.PROFILE_DTYPE).copy()
    res, grid = O.mdp_sweep(arr, 1, want_grid=True)
    assert (res[0]["p_e"], res[0]["p_d"], res[0]["p_a"]) == (100, 0, 0)
    assert np.all(grid[0] == res[0]["dsi_s"])


def test_full_fit_prefers_augmented():
    # dataset fits in A only at x_A = 100 (cache = N M S exactly) and DSI_A (GPU-bound
    # 14301) > DSI_E (CPU-bound 9783) -> x_A = 100 is the unique optimum
    p = prof("azure", n_total=1000, s_data=1000, cache_bytes=5_120_000)
    arr = np.frombuffer(bytes(p), dtype=O.PROFILE_DTYPE).copy()
    res, _ = O.mdp_sweep(arr, 1)
    assert (res[0]["p_e"], res[0]["p_d"], res[0]["p_a"]) == (0, 0, 100)
    assert res[0]["v"] == res[0]["dsi_a"] == 14301.0
    # with a larger cache every x_A >= 1 fits: exact tie, broken to the highest x_E
    p = prof("azure", n_total=1000, s_data=1000, cache_bytes=10**9)
    arr = np.frombuffer(bytes(p), dtype=O.PROFILE_DTYPE).copy()
    res, _ = O.mdp_sweep(arr, 1)
    assert (res[0]["p_e"], res[0]["p_d"], res[0]["p_a"]) == (99, 0, 1) and res[0]["v"] == 14301.0


def test_argmax_against_exact_rationals():
    """Brute force in exact rationals over random synthetic profiles (5 % grid)."""
    cols = synth.mdp_profiles(120, seed=12345)
    arr = O.profiles_from_columns(cols)
    res, grid = O.mdp_sweep(arr, 5, want_grid=True)
    sp = list(mdp_exact.splits(5))
    for i in range(len(arr)):
        r = res[i]
        pr = dict(n_total=int(cols["n_total"][i]), s_data=int(cols["s_data"][i]),
                  cache_bytes=int(cols["cache_bytes"][i]), m_num=128, m_den=25)
        ex = mdp_exact.exact_values(pr, [r["dsi_a"], r["dsi_d"], r["dsi_e"], r["dsi_s"]], 5)
        # every FP64 grid value is the exact value up to a few roundings
        for k in range(len(sp)):
            assert abs(float(ex[k]) - grid[i, k]) <= 8 * 2 ** -52 * abs(float(ex[k]))
        exmax = max(ex)
        assert float(exmax - Fraction(r["v"])) <= 1e-12 * float(exmax)
        order = sorted(range(len(ex)), key=lambda k: (-ex[k], k))
        if ex[order[0]] - ex[order[1]] > Fraction(1, 10**12) * exmax:
            assert sp[order[0]] == (r["p_e"], r["p_d"], r["p_a"])
        # the reported split's own grid value is the max of the grid, first index on ties
        k = sp.index((r["p_e"], r["p_d"], r["p_a"]))
        assert grid[i, k] == grid[i].max() and k == int(np.argmax(grid[i]))


def test_metadata_bytes_pin():
    assert O.metadata_bytes(1_300_000, 8) == 2_600_000      # P:L710 "2.6MB"
    assert O.metadata_bytes(8, 1) == 9 and O.metadata_bytes(1000, 0) == 1000


def test_cache_monotonicity_soft():
    # the optimum is non-decreasing in cache size up to grid rounding (R-M17)
    cols = synth.mdp_profiles(30, seed=77)
    arr = O.profiles_from_columns(cols)
    big = arr.copy()
    big["cache_bytes"] = big["cache_bytes"] * 2
    r1, _ = O.mdp_sweep(arr, 1)
    r2, _ = O.mdp_sweep(big, 1)
    assert np.all(r2["v"] >= r1["v"] * (1 - 1e-9))


# ------------------------------------------------------------ NEXT-4: dataset-size curves (Fig. 7)
def _sizes():
    """Dataset sizes 8 GB .. 512 GB at S_data = 114 KB (the Fig. 7 axis), plus
    tiny and huge datasets so both the full-fit and neither-fits regimes occur."""
    gb = [0.001, 0.01, 0.1, 1, 2, 4, 8, 16, 32, 64, 128, 256, 327.68, 512, 1024, 4096, 65536]
    return [max(1, int(x * 1e9 / 114_000)) for x in gb]


@pytest.mark.parametrize("server", ["in_house", "aws", "azure"])
def test_single_tier_curves_move_toward_dsi_s(server):
    """for a fixed split V(N) = DSI_S + sum_t f_t(N)(DSI_t - DSI_S)
    with non-increasing f_t, so a single-tier curve moves monotonically toward
    DSI_S as the dataset grows; at full fit it IS DSI_t (N_t/N = 1 exactly) and
    beyond it equals (cap/N) DSI_t + ((N - cap)/N) DSI_S."""
    for split in ((100, 0, 0), (0, 100, 0), (0, 0, 100)):
        dist = []
        for n in _sizes():
            p = prof(server, n_total=n)
            v, _, _ = O.model_eval(p, *split)
            d, _ = O.tiers(p)
            na, nd, ne, ns = O.split_counts(p, *split)
            t = 2 if split[0] else (1 if split[1] else 0)            # dsi index: 0 A, 1 D, 2 E
            cap = {0: na, 1: nd, 2: ne}[t]
            if ns == 0:
                assert v == d[t]                                     # full fit: exactly DSI_t
            want = Fraction(cap, n) * Fraction(d[t]) + Fraction(n - cap, n) * Fraction(d[3])
            assert abs(Fraction(v) - want) <= abs(want) * Fraction(1, 10**14)
            dist.append(abs(v - d[3]))
        for a, b in zip(dist, dist[1:]):
            assert b <= a * (1 + 1e-12) + 1e-12


@pytest.mark.parametrize("server,b_cache", [("in_house", None), ("aws", None), ("azure", None),
                                            ("azure", 30e9)])
def test_a_only_vs_e_only_crossing_rule(server, b_cache):
    """M15(ii): the A-only and E-only curves cross iff sign(DSI_A - DSI_E) (both fit)
    differs from sign((DSI_A - DSI_S) - M'(DSI_E - DSI_S)) (neither fits, M' =
    cap_E / cap_A, the E tier's sample-count advantage).  Azure with B_cache read
    as 30 GB/s is the profile SURVEY [A.4] names as crossing exactly once."""
    over = {} if b_cache is None else dict(b_cache=b_cache)
    diffs = []
    for n in _sizes():
        p = prof(server, n_total=n, **over)
        va, _, _ = O.model_eval(p, 0, 0, 100)
        ve, _, _ = O.model_eval(p, 100, 0, 0)
        diffs.append(va - ve)
    p = prof(server, n_total=_sizes()[-1], **over)
    d, _ = O.tiers(p)
    na, _, _, _ = O.split_counts(p, 0, 0, 100)
    _, _, ne, _ = O.split_counts(p, 100, 0, 0)
    small = np.sign(d[0] - d[2])
    large = np.sign((d[0] - d[3]) * na - (d[2] - d[3]) * ne)
    s = [np.sign(x) for x in diffs if x != 0]
    changes = sum(1 for a, b in zip(s, s[1:]) if a != b)
    assert s[0] == small and s[-1] == large
    assert changes == (1 if small != large else 0)
    if b_cache == 30e9:
        assert changes == 1
