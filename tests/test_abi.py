"""CPU checks of the boundary: libseneca.so loads, exports every function that
include/seneca.h declares, and its host-only helpers agree with the oracle.
No device compute is called here."""
import ctypes
import os
import re

import pytest

import oracle as O
import synth
from paper_2511_13724_b200 import seneca as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "seneca.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(seneca_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2511_13724_b200 import build
    build.build()
    return S.lib()


def test_every_declared_symbol_is_exported(lib):
    names = declared_functions()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(S.EXPORTED) == names


def test_struct_sizes_match_header(lib):
    assert S.PROFILE_DTYPE.itemsize == 112
    assert S.RESULT_DTYPE.itemsize == 48
    assert S.STATS_DTYPE.itemsize == 104


def test_metadata_bytes_paper_pin(lib):
    assert S.metadata_bytes(1_300_000, 8) == 2_600_000
    assert S.metadata_bytes(8, 1) == 9


def test_split_capacities_match_oracle(lib):
    st = synth.Stream(21)
    for _ in range(300):
        n = int(st.u64(1)[0] % 10**8) + 1
        s = int(st.u64(1)[0] % 10**6) + 1
        cache = int(st.u64(1)[0] % 10**13)
        a = int(st.u64(1)[0] % 101); b = int(st.u64(1)[0] % (101 - a)); e = 100 - a - b
        caps = S.split_capacities(n, s, 128, 25, cache, e, b, a)
        p = O.make_profile(t_gpu=1, t_decode_augment=1, t_augment=1, b_nic=1, b_pcie=1, b_cache=1,
                           b_storage=1, cache_bytes=cache, n_total=n, s_data=s, m_num=128, m_den=25,
                           nodes=1, gpus_per_node=1)
        na, nd, ne, ns = O.split_counts(p, e, b, a)
        assert caps == [ne, nd, na, ns]


def test_config_capacities(lib):
    for name, want in [("toy", (80, 11, 11)), ("imagenet1k", (0, 42_038, 45_541)),
                       ("openimages", (658_561, 118_731, 0)), ("imagenet22k", (4_376_846, 0, 0))]:
        c = synth.ods_config(name)
        caps = S.split_capacities(c["n_total"], c["s_data"], c["m_num"], c["m_den"], c["cache_bytes"], *c["split"])
        assert tuple(caps[:3]) == want


def test_invalid_arguments_rejected_on_host(lib):
    with pytest.raises(S.SenecaError) as ei:
        S.split_capacities(10, 10, 128, 25, 10**9, 50, 50, 1)
    assert ei.value.status == S.EINVAL
    with pytest.raises(S.SenecaError) as ei:
        S.mdp_sweep(1, 1, 7, 1, None, 0)                    # 7 does not divide 100
    assert ei.value.status == S.EINVAL
    assert S.mdp_num_splits(1) == 5151 and S.mdp_num_splits(10) == 66 and S.mdp_num_splits(7) == 0
    for splits in ([(10, 20, 71)], [(50, 50, 0)] * 4097, []):    # host-side checks, before any launch
        with pytest.raises(S.SenecaError) as ei:
            S.mdp_eval(1, 1, splits, 1, stream=0)
        assert ei.value.status == S.EINVAL
    bad = [dict(n_total=0), dict(n_total=2**31), dict(batch=[0]), dict(batch=[5000]),
           dict(cap_e=600, cap_d=600), dict(target=[0])]
    for over in bad:
        kw = dict(n_total=1000, batch=[32], target=[1], cap_e=10, cap_d=10, cap_a=10, seed=1)
        kw.update(over)
        cfg = S.make_config(kw["n_total"], kw["batch"], kw["target"], kw["cap_e"], kw["cap_d"],
                            kw["cap_a"], kw["seed"])
        with pytest.raises(S.SenecaError):
            S.state_bytes(cfg)


def test_state_bytes_scale(lib):
    c = synth.ods_config("imagenet22k")
    caps = S.split_capacities(c["n_total"], c["s_data"], c["m_num"], c["m_den"], c["cache_bytes"], *c["split"])
    cfg = S.make_config(c["n_total"], c["batch"], c["target"], caps[0], caps[1], caps[2], 1)
    nbytes = S.state_bytes(cfg)
    # 3 + 2J bitmaps (R-O14), the 2-slot permutation ring, the storage-id segments of the
    # late walk (one u32 per ring position) and the lap lists per job dominate; fits easily in 180 GB
    assert 2.0e9 < nbytes < 3.2e9


def test_ctypes_layouts_match_c_header(lib, tmp_path):
    """sizeof/offsetof of every C-ABI struct as gcc sees include/seneca.h ==
    the ctypes mirror the binding passes across the boundary."""
    import subprocess
    probe = tmp_path / "probe.c"
    structs = {"seneca_cache_config": S.CacheConfig, "seneca_state_view": S.StateView,
               "seneca_job_epoch_stats": S.JobEpochStats, "seneca_mdp_profile": S.MdpProfile,
               "seneca_mdp_result": S.MdpResult, "seneca_kernel_stat": S.KernelStat, "seneca_split": S.Split,
               "seneca_epoch_metrics": S.EpochMetrics}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "seneca.h"', "int main(void) {"]
    for cname, ct in structs.items():
        lines.append(f'printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for f in ct._fields_:
            if f[0].startswith("_pad"):
                continue
            lines.append(f'printf("{cname} {f[0]} %zu\\n", offsetof({cname}, {f[0]}));')
    lines.append("return 0; }")
    probe.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(probe), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l}
    for cname, ct in structs.items():
        assert got[(cname, "sizeof")] == ctypes.sizeof(ct), cname
        for f in ct._fields_:
            if not f[0].startswith("_pad"):
                assert got[(cname, f[0])] == getattr(ct, f[0]).offset, (cname, f[0])


def test_replicas_workspace_and_arguments(lib):
    c = synth.ods_config("toy")
    caps = S.split_capacities(c["n_total"], c["s_data"], c["m_num"], c["m_den"], c["cache_bytes"], *c["split"])
    one = S.state_bytes(S.make_config(c["n_total"], c["batch"], c["target"], caps[0], caps[1], caps[2], 1))
    two = S.state_bytes(S.make_config(c["n_total"], c["batch"], c["target"], caps[0], caps[1], caps[2], 1,
                                      replicas=2))
    slice_ = two - one                                         # one 256-aligned slice per replica
    ctl = one - slice_                                         # + a control block, 64 B per replica
    assert slice_ % 256 == 0 and ctl == 256
    for r in (0, 1, 2, 7, 64):
        cfg = S.make_config(c["n_total"], c["batch"], c["target"], caps[0], caps[1], caps[2], 1, replicas=r)
        R = max(r, 1)
        assert S.state_bytes(cfg) == R * slice_ + -(-R * 64 // 256) * 256
    for r, mode in ((65, 0), (2, 1)):                          # too many; caller-supplied requests need R = 1
        cfg = S.make_config(c["n_total"], c["batch"], c["target"], caps[0], caps[1], caps[2], 1, mode, replicas=r)
        with pytest.raises(S.SenecaError) as ei:
            S.state_bytes(cfg)
        assert ei.value.status == S.EINVAL


def test_epoch_model_host_checks(lib):
    for dsi in ((1.0, 0.0, 1.0, 1.0), (1.0, float("inf"), 1.0, 1.0), (1.0, 1.0, float("nan"), 1.0)):
        with pytest.raises(S.SenecaError) as ei:
            S.epoch_model(1, 1, 10, dsi, 1, stream=0)
        assert ei.value.status == S.EINVAL
    with pytest.raises(S.SenecaError):
        S.epoch_model(1, 0, 10, (1.0,) * 4, 1, stream=0)


def test_mode_fields_validated(lib):
    c = synth.ods_config("toy")
    caps = S.split_capacities(c["n_total"], c["s_data"], c["m_num"], c["m_den"], c["cache_bytes"], *c["split"])
    args = (c["n_total"], c["batch"], c["target"], caps[0], caps[1], caps[2], 1)
    base = S.state_bytes(S.make_config(*args))
    for kw in (dict(evict_tiers=1), dict(sampler=1), dict(cold_start=1), dict(arrival=[0, 7])):
        assert S.state_bytes(S.make_config(*args, **kw)) >= base       # valid modes
    for kw in (dict(evict_tiers=2), dict(sampler=2), dict(cold_start=2)):
        with pytest.raises(S.SenecaError) as ei:
            S.state_bytes(S.make_config(*args, **kw))
        assert ei.value.status == S.EINVAL


def test_workspace_is_independent_of_target_epochs(lib):
    """The permutation ring (K = min(epochs, 2) slots per job) keeps the workspace
    flat in the number of epochs: only the per job-epoch counters (104 B) and the
    per job-epoch ready/progress flags (8 B) grow.  ImageNet-22K x 50 epochs fits
    in a few GB (it needed 22.7 GB when every epoch was materialised)."""
    c = synth.ods_config("imagenet22k")
    caps = S.split_capacities(c["n_total"], c["s_data"], c["m_num"], c["m_den"], c["cache_bytes"], *c["split"])
    J = len(c["batch"])
    sizes = {}
    for T in (2, 3, 50, 250):
        cfg = S.make_config(c["n_total"], c["batch"], [T] * J, caps[0], caps[1], caps[2], 1)
        sizes[T] = S.state_bytes(cfg)
    for T in (3, 50, 250):
        grow = sizes[T] - sizes[2]
        assert 0 <= grow <= J * (T - 2) * (104 + 8) + 3 * 256, (T, grow)
    assert sizes[250] < 4 * 2**30
    one = S.make_config(c["n_total"], c["batch"], [1] * J, caps[0], caps[1], caps[2], 1)
    assert S.state_bytes(one) < sizes[2]          # one epoch: a one-slot ring


def test_sharding_arguments_and_workspace(lib):
    """sample-ID-range sharding: G slices of the replicated state +
    a mailbox each in emulation; EINVAL for G > 8, replicas or caller-supplied
    requests with G > 1, a bad shard_mode / shard_rank."""
    c = synth.ods_config("toy")
    caps = S.split_capacities(c["n_total"], c["s_data"], c["m_num"], c["m_den"], c["cache_bytes"], *c["split"])
    mk = lambda **kw: S.make_config(c["n_total"], c["batch"], c["target"], caps[0], caps[1], caps[2], 1, **kw)
    one = S.state_bytes(mk())
    for G in (2, 4, 8):
        b = S.state_bytes(mk(shards=G))
        assert G * (one - 256) <= b <= G * (one - 256) + 256 + G * 8192, (G, b)
        assert S.state_bytes(mk(shards=G, shard_mode=1, shard_rank=G - 1)) < b
    for kw in (dict(shards=9), dict(shards=2, replicas=2), dict(shards=2, request_mode=1),
               dict(shards=2, shard_mode=2), dict(shards=4, shard_mode=1, shard_rank=4)):
        with pytest.raises(S.SenecaError) as ei:
            S.state_bytes(mk(**kw))
        assert ei.value.status == S.EINVAL, kw
