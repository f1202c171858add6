"""GPU parity: seneca_mdp_sweep (C-ABI) vs the oracle, bit-exact.

north_star tolerance for FP64 throughputs is 1e-9 relative; the kernel is
bit-identical by construction (explicit round-to-nearest ops in the oracle's
order, R-M7), so every value is compared with ==.  Argmax splits and limiting
factors are exact integers."""
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

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table4_nominal_vals.json")))


def to_dev_rows(oracle_rows):
    """The two sides define their profile structs independently; convert by field name."""
    out = np.zeros(len(oracle_rows), S.PROFILE_DTYPE)
    for f in O.PROFILE_FIELDS:
        out[f] = oracle_rows[f]
    return out


def run_gpu(rows, g, grid=True):
    d_res, d_grid = P.mdp_sweep_device(to_dev_rows(rows), g, want_grid=grid)
    torch.cuda.synchronize()
    res = P.results_to_numpy(d_res)
    return res, (d_grid.cpu().numpy() if grid else None)


def assert_same(res, ores, grid=None, ogrid=None):
    assert np.all(res["status"] == 0)
    for a, b in [("p_e", "p_e"), ("p_d", "p_d"), ("p_a", "p_a"), ("lim_a", "lim_a"), ("lim_d", "lim_d"),
                 ("lim_e", "lim_e"), ("lim_s", "lim_s")]:
        np.testing.assert_array_equal(res[a], ores[b], err_msg=a)
    for a, b in [("v_best", "v"), ("dsi_a", "dsi_a"), ("dsi_d", "dsi_d"), ("dsi_e", "dsi_e"), ("dsi_s", "dsi_s")]:
        assert np.array_equal(res[a].view(np.uint64), ores[b].view(np.uint64)), a      # bit-exact
    if grid is not None:
        assert np.array_equal(grid.view(np.uint64), ogrid.view(np.uint64))


def table4_rows():
    rows = []
    for server in ("in_house", "aws", "azure"):
        g = {k: v for k, v in GOLD[server].items() if not k.startswith("_")}
        for ds in ("imagenet1k", "openimages", "imagenet22k"):
            for nodes in (1, 2):
                for cache in (64, 115, 400):
                    kw = dict(g, model_bytes=102.4e6, nodes=nodes, gpus_per_node=4, cache_bytes=cache * 10**9,
                              **GOLD["datasets"][ds])
                    rows.append(kw)
    arr = np.zeros(len(rows), O.PROFILE_DTYPE)
    for i, kw in enumerate(rows):
        for k, v in kw.items():
            arr[i][k] = v
    return arr


@pytest.mark.parametrize("g", [1, 2, 5, 10, 20, 25, 50, 100])
def test_table4_profiles_all_grids(g):
    rows = table4_rows()
    ores, ogrid = O.mdp_sweep(rows, g, want_grid=True)
    res, grid = run_gpu(rows, g)
    assert_same(res, ores, grid, ogrid)


def test_imagenet22k_azure_pin_on_device():
    rows = table4_rows()
    g = {k: v for k, v in GOLD["azure"].items() if not k.startswith("_")}
    one = np.zeros(1, O.PROFILE_DTYPE)
    for k, v in dict(g, model_bytes=0.0, nodes=1, gpus_per_node=1, n_total=14_000_000, s_data=91_390).items():
        one[0][k] = v
    res, _ = run_gpu(one, 1, grid=False)
    assert (res[0]["p_e"], res[0]["p_d"], res[0]["p_a"]) == (100, 0, 0)
    assert res[0]["v_best"] == 3088.051099033303


def test_synthetic_10k_profiles_1pct_full_grid():
    """BASELINE.json configs[4]: 10,000 profiles x 5151 splits, every value."""
    cols = synth.mdp_profiles(10_000, seed=synth.PERF_SEED)
    rows = O.profiles_from_columns(cols)
    ores, ogrid = O.mdp_sweep(rows, 1, want_grid=True)
    res, grid = run_gpu(rows, 1)
    assert_same(res, ores, grid, ogrid)


@pytest.mark.parametrize("seed", synth.PARITY_SEEDS)
def test_synthetic_profiles_toy_grid(seed):
    cols = synth.mdp_profiles(3000, seed=seed)
    rows = O.profiles_from_columns(cols)
    for g in (10, 1):
        ores, ogrid = O.mdp_sweep(rows, g, want_grid=True)
        res, grid = run_gpu(rows, g)
        assert_same(res, ores, grid, ogrid)


def test_edge_profiles():
    """Zero cache (all ties), tiny datasets (full fit everywhere), huge model (comm-bound),
    both comm mappings, NVLink flags."""
    cols = synth.mdp_profiles(600, seed=99)
    rows = O.profiles_from_columns(cols)
    rows["cache_bytes"][:100] = 0
    rows["n_total"][100:200] = np.arange(1, 101)
    rows["model_bytes"][200:300] = 5e11
    rows["comm_mapping"][300:400] = 1
    rows["nvlink_inter"][400:500] = 1
    rows["cache_bytes"][500:600] = np.uint64(10**15)
    for g in (1, 4):
        ores, ogrid = O.mdp_sweep(rows, g, want_grid=True)
        res, grid = run_gpu(rows, g)
        assert_same(res, ores, grid, ogrid)


def test_invalid_profiles_flagged():
    cols = synth.mdp_profiles(8, seed=3)
    rows = to_dev_rows(O.profiles_from_columns(cols))
    rows["t_gpu"][0] = 0.0
    rows["b_cache"][1] = np.inf
    rows["n_total"][2] = 0
    rows["m_num"][3] = 1              # M < 1
    rows["cache_bytes"][4] = np.uint64(2**62)
    rows["model_bytes"][5] = -1.0
    d_res, _ = P.mdp_sweep_device(rows, 1)
    res = P.results_to_numpy(d_res)
    assert list(res["status"]) == [1, 1, 1, 1, 1, 1, 0, 0]


def test_results_without_grid_match():
    cols = synth.mdp_profiles(2000, seed=5)
    rows = O.profiles_from_columns(cols)
    ores, _ = O.mdp_sweep(rows, 1)
    res, _ = run_gpu(rows, 1, grid=False)
    assert_same(res, ores)


def test_wide_counts_paths():
    """N >= 2^31 (64-bit split path), N >= 2^53 (__ddiv_rn tables) and capacities
    near N: every path of the kernel against the oracle."""
    cols = synth.mdp_profiles(400, seed=77)
    rows = O.profiles_from_columns(cols)
    big = [2**31 - 1, 2**31, 2**31 + 12345, 3 * 2**32 + 7, 2**52 + 1, 2**53 + 3, 2**60 + 11, 2**63 + 5]
    for k in range(len(rows)):
        rows["n_total"][k] = big[k % len(big)]
        rows["s_data"][k] = 1 + (k % 3)                     # capacities comparable to N
        lim = (2**64 - 1) // 100 // int(rows["m_den"][k])      # the ABI's overflow bound (EINVAL above it)
        rows["cache_bytes"][k] = np.uint64(min(int(rows["n_total"][k]) // (1 + k % 5), lim))
    for g in (1, 5):
        ores, ogrid = O.mdp_sweep(rows, g, want_grid=True)
        res, grid = run_gpu(rows, g)
        assert_same(res, ores, grid, ogrid)


def test_capacity_floor_boundaries():
    """Eqs. 5-7 floors at exact multiples and +-1 (mdp.cu floor_div: a reciprocal
    estimate and one integer correction), for small divisors, divisors near the
    2^62 fast-path limit and above it (the u64 division fallback)."""
    cols = synth.mdp_profiles(270, seed=1234)
    rows = O.profiles_from_columns(cols)
    sd = [1, 7, 114620, 2**33 + 5, 2**45 - 1, 2**53 + 1, 2**55 + 3, 2**56 + 3, 2**57 - 1]
    lim = (2**64 - 1) // 100                      # 100 * cache_bytes * m_den < 2^64 (m_den = 1)
    for k in range(len(rows)):
        s = sd[k % len(sd)]
        t = 1 + (k // len(sd)) % 10
        d = (k // (len(sd) * 10)) % 3 - 1
        base = 100 * (2**24 + 1) if s == 1 else t * s
        rows["s_data"][k] = s
        rows["m_num"][k] = 1
        rows["m_den"][k] = 1
        rows["n_total"][k] = 2**31 - 1
        rows["cache_bytes"][k] = np.uint64(max(0, min(base * (t if s == 1 else 1) + d, lim)))
    for g in (1, 3):
        if 100 % g:
            continue
        ores, ogrid = O.mdp_sweep(rows, g, want_grid=True)
        res, grid = run_gpu(rows, g)
        assert_same(res, ores, grid, ogrid)


def test_every_grid_step():
    """Every divisor of 100: one to several row items and partial sweep chunks."""
    rows = O.profiles_from_columns(synth.mdp_profiles(700, seed=31))
    for g in (1, 2, 4, 5, 10, 20, 25, 50, 100):
        ores, ogrid = O.mdp_sweep(rows, g, want_grid=True)
        res, grid = run_gpu(rows, g)
        assert_same(res, ores, grid, ogrid)


def test_invalid_profiles_interleaved():
    """Invalid rows scattered through a long list (several profiles per CTA, the
    double-buffered tables meet invalid neighbours): status 1 for those, the
    oracle's results for the rest."""
    rows = O.profiles_from_columns(synth.mdp_profiles(5000, seed=12))
    bad = np.arange(0, 5000, 7)
    dev = to_dev_rows(rows)
    dev["t_gpu"][bad] = 0.0
    d_res, d_grid = P.mdp_sweep_device(dev, 1, want_grid=True)
    torch.cuda.synchronize()
    res = P.results_to_numpy(d_res)
    good = np.setdiff1d(np.arange(5000), bad)
    assert np.all(res["status"][bad] == 1) and np.all(res["status"][good] == 0)
    ores, ogrid = O.mdp_sweep(rows[good], 1, want_grid=True)
    assert_same(res[good], ores, d_grid.cpu().numpy()[good], ogrid)


# ------------------------------------------------------------ seneca_mdp_eval (SPEC evaluate, NEXT-4 size curves)
def _oracle_eval(rows, splits):
    vals = np.zeros((len(rows), len(splits)))
    cnts = np.zeros((len(rows), len(splits), 4), np.uint64)
    for i in range(len(rows)):
        p = O.profile_row(rows, i)
        for s, (e, d, a) in enumerate(splits):
            v, _, c = O.model_eval(p, e, d, a)
            vals[i, s] = v
            na, nd, ne, ns = O.split_counts(p, e, d, a)
            cnts[i, s] = (na, nd, ne, ns)
    return vals, cnts


def test_eval_random_splits_bit_exact():
    rows = O.profiles_from_columns(synth.mdp_profiles(300, seed=41))
    st = synth.Stream(9)
    splits = []
    for _ in range(97):
        e = int(st.u64(1)[0] % 101); d = int(st.u64(1)[0] % (101 - e))
        splits.append((e, d, 100 - e - d))
    splits += [(100, 0, 0), (0, 100, 0), (0, 0, 100), (0, 0, 100)]
    d_val, d_cnt, d_tiers = P.mdp_eval_device(to_dev_rows(rows), splits, want_counts=True)
    torch.cuda.synchronize()
    ov, oc = _oracle_eval(rows, splits)
    assert np.array_equal(d_val.cpu().numpy().view(np.uint64), ov.view(np.uint64))
    assert np.array_equal(d_cnt.cpu().numpy().view(np.uint64), oc)
    tiers = P.results_to_numpy(d_tiers)
    ores, _ = O.mdp_sweep(rows, 10)
    for f in ("dsi_a", "dsi_d", "dsi_e", "dsi_s"):
        assert np.array_equal(tiers[f].view(np.uint64), ores[f].view(np.uint64))
    assert np.all(tiers["status"] == 0)


def test_eval_fig7_dataset_size_curves():
    """NEXT-4: A-only and E-only curves over dataset sizes 8-512 GB at a 64 GB
    cache for the three Table-4 servers (Fig. 7 axis), bit-exact; the
    crossing rule of the oracle pins (test_oracle_mdp) then holds on the device."""
    sizes = [int(x * 1e9 / 114_000) for x in (8, 16, 32, 64, 128, 256, 512)]
    rows = []
    for server in ("in_house", "aws", "azure"):
        g = {k: v for k, v in GOLD[server].items() if not k.startswith("_")}
        for n in sizes:
            rows.append(dict(g, model_bytes=0.0, n_total=n, nodes=1, gpus_per_node=1))
    arr = np.zeros(len(rows), O.PROFILE_DTYPE)
    for i, kw in enumerate(rows):
        for k, v in kw.items():
            arr[i][k] = v
    splits = [(0, 0, 100), (100, 0, 0), (0, 100, 0), (52, 48, 0)]
    d_val, _, _ = P.mdp_eval_device(to_dev_rows(arr), splits)
    torch.cuda.synchronize()
    ov, _ = _oracle_eval(arr, splits)
    got = d_val.cpu().numpy()
    assert np.array_equal(got.view(np.uint64), ov.view(np.uint64))
    a_minus_e = (got[:, 0] - got[:, 1]).reshape(3, len(sizes))
    assert np.all(a_minus_e[0] > 0) and np.all(a_minus_e[1] < 0) and np.all(a_minus_e[2] < 0)   # [A.4]


def test_eval_invalid_profile_and_arguments():
    rows = to_dev_rows(O.profiles_from_columns(synth.mdp_profiles(4, seed=2)))
    rows["t_gpu"][1] = 0.0
    d_val, d_cnt, d_tiers = P.mdp_eval_device(rows, [(10, 20, 70)], want_counts=True)
    torch.cuda.synchronize()
    v = d_val.cpu().numpy()[:, 0]
    assert np.isnan(v[1]) and not np.isnan(v[[0, 2, 3]]).any()
    assert list(P.results_to_numpy(d_tiers)["status"]) == [0, 1, 0, 0]
    for bad in ([(10, 20, 71)], [(50, 50, 0)] * 4097, []):
        with pytest.raises(S.SenecaError) as ei:
            P.mdp_eval_device(rows, bad)
        assert ei.value.status == S.EINVAL
