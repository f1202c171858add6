"""The bench.py contract on CPU: the reference arm (the oracle) prints one JSON
line with the keys the driver reads; the GPU arm's keys are checked by the GPU
pass (profiles/r1/bench_*.json)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "toy",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("toy")


def test_committed_bench_lines_have_the_contract_keys():
    """The committed round-2 bench lines (profiles/r2, the pass its README names)
    carry the driver's keys, a roofline with its latency floor, bit-exact parity
    gates on every workload, replica and shard count, and the reference arm
    loads nothing but the oracle."""
    import re
    readme = open(os.path.join(ROOT, "profiles", "r2", "README.md")).read()
    tag = re.search(r"Current pass: \*\*(r2[a-z]?)\*\*", readme).group(1)
    d = json.loads(open(os.path.join(ROOT, "profiles", "r2", f"bench_{tag}.json")).read().strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "clocks", "gpu_launches",
              "cpu_baseline"):
        assert k in d, k
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert 0 < r["latency"]["frac"] <= 1 and r["latency"]["floor_us_per_round"] > 0
    assert d["config"]["workload"].startswith("imagenet22k")
    assert d["steps"] >= 1 and d["warmup"] >= 3 and d["gpu_launches"] > 0
    assert d["parity"]["ods_vs_oracle_golden"] == "bit-exact"
    assert d["parity"]["mdp_vs_oracle_first_200_profiles"] == "bit-exact"
    for w in ("imagenet1k", "openimages"):
        assert d["workloads"][w]["parity"] == "bit-exact", w
    assert all(v == "bit-exact" or v is True for v in d["replicas"]["parity"].values())
    assert all(run["parity"] == "bit-exact" for run in d["sharded"]["runs"])
    assert not set(d["clocks"]["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    ref = json.loads(open(os.path.join(ROOT, "profiles", "r2", f"bench_reference_{tag}.json")).read().strip())
    assert ref["impl"] == "reference" and ref["so_loaded"] == ["oracle/liboracle.so"]


def test_pass_equivalent_matches_the_survey_sizes():
    """bench.pass_equivalent restates SURVEY §8(a) row a4 / §8(d) target 1; pin it to
    the sizes the survey prints: 22K 2 x 1,774,644 B per job-round (seen + E),
    IN1K 4 x 160,148 B per job-round (seen, D, A, cons) + 3 x 160,148 B storage
    pool per round, OpenImages 3 x 217,500 B per job-round."""
    sys.path.insert(0, ROOT)
    import bench
    import synth
    W = {"imagenet22k": 443661, "imagenet1k": 40037, "openimages": 54375}
    split_caps = {"imagenet22k": (4376846, 0, 0), "imagenet1k": (0, 42038, 45541),
                  "openimages": (658561, 118731, 0)}
    for name, words in W.items():
        c = synth.ods_config(name, seed=synth.PERF_SEED)
        pe = bench.pass_equivalent(c, split_caps[name], words, ods_s=1.0, steps=1, world=1, hbm_peak=1000.0)
        jr = sum(t * -(-c["n_total"] // b) for t, b in zip(c["target"], c["batch"]))
        if name == "imagenet22k":
            assert jr == 8 * 2 * 27729                          # 8 jobs x 2 epochs x ceil(14,197,122 / 512)
            per_round_8jobs = 8 * 2 * 4 * words
            assert per_round_8jobs == 28394304                  # SURVEY: 28.4 MB per round
            assert pe["bytes_per_replay"] == 2 * 4 * words * jr + 4 * words * 16
        elif name == "imagenet1k":
            rounds = 10 * -(-c["n_total"] // 256)
            assert 4 * 4 * words * 4 + 3 * 4 * words == 3042812   # SURVEY: 2.56 MB + 0.48 MB per round
            assert pe["bytes_per_replay"] == 4 * 4 * words * jr + 3 * 4 * words * rounds + 4 * words * 40
        else:
            assert 8 * 3 * 4 * words == 5220000                 # SURVEY: 5.22 MB per round
            assert pe["bytes_per_replay"] == 3 * 4 * words * jr + 4 * words * 40
        assert abs(pe["frac"] - pe["achieved"] / pe["peak"]) < 1e-12
        assert abs(pe["achieved"] - pe["bytes_per_replay"] / 1e9) < 1e-6


def test_all_cores_oracle_baselines():
    """bench.py's all-host-cores oracle figures: one process per core,
    the MDP oracle on profile slices and independent ODS oracle replays (seed + k)."""
    import types
    sys.path.insert(0, ROOT)
    import bench
    import synth
    args = types.SimpleNamespace(mdp_grid_step=10, evict_tiers=0)
    v, cores, done, dt = bench.oracle_mdp_all_cores(args, per_core=20)
    assert cores >= 1 and done == 20 * cores and v > 0 and dt > 0
    c = synth.ods_config("toy", seed=synth.PERF_SEED)
    v, cores, dec, dt = bench.oracle_ods_all_cores(args, c, bench.oracle_caps(c), 10)
    assert dec == cores * 10 * sum(c["batch"])          # every replay plays 10 full rounds of both jobs
    assert v > 0


def test_latency_floor_model():
    """bench.latency_floor (DESIGN.md 7.1 "latency roofline"): per job-round
    floor = dependent L2 trips x 300 cycles + scattered accesses x 1 cycle +
    substituting share x the perm_apply chain (1,790 cycles), from the replay's
    own counters.  Pinned on hand-computed cases: one job, 1,000 samples, batch
    100 (10 job-rounds), 400 requested hits and 300 substitutes over the epoch;
    static tiers (E only: only the rounds with non-empty pools test their
    requests) and with an A tier (every request tested, maintain trips)."""
    import numpy as np
    sys.path.insert(0, ROOT)
    import bench
    c = dict(n_total=1000, batch=[100], target=[1])
    st = np.zeros((1, 1), dtype=[("served", "<u8", 4), ("subst", "<u8", 4), ("req_hits", "<u8", 4), ("digest", "<u8")])
    st["served"][0, 0] = [300, 700, 0, 0]            # storage 300, E 700 (= 400 hits + 300 substitutes)
    st["subst"][0, 0] = [0, 300, 0, 0]
    st["req_hits"][0, 0] = [0, 400, 0, 0]
    jr, req, hits, subs = 10, 1000.0, 400.0, 300.0
    sub_rounds = min(jr, subs / ((req - hits) / jr))                    # 5
    # static: 5 of 10 rounds test their 100 requests
    lf = bench.latency_floor(c, (500, 0, 0), st, 10, 0, 0, 2000.0)
    rt = sub_rounds * req / jr                                          # 500 tested requests
    scattered = rt / 4 + rt + rt * 1 + rt + hits + subs + 2 * subs + 2 * subs + subs
    dep = sub_rounds * 3 + 2 * sub_rounds
    cyc = dep * 300 + scattered + sub_rounds * 1790
    assert lf["static_tiers"] is True
    assert abs(lf["cycles_per_job_round"] - cyc / jr) < 1e-9
    assert abs(lf["floor_us_per_round"] - cyc / jr / 2000.0) < 1e-12
    assert abs(lf["substituting_job_round_share"] - 0.5) < 1e-12
    # with an A tier (the same counters, caps E 400 / A 100): every request tested
    lf = bench.latency_floor(c, (400, 0, 100), st, 10, 0, 0, 2000.0)
    positions = req + subs
    scattered = positions / 4 + positions + req * 2 + req + hits + subs + 2 * subs + 2 * subs + subs
    dep = jr * 3 + 2 * sub_rounds + jr * 3
    cyc = dep * 300 + scattered + sub_rounds * 1790
    assert lf["static_tiers"] is False
    assert abs(lf["cycles_per_job_round"] - cyc / jr) < 1e-9
