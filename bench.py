#!/usr/bin/env python3
"""Benchmark of Seneca's hot path on B200 (BASELINE.json metric:
"ODS sample decisions/sec & MDP split evals/sec (1/2/4/8 B200), % of HBM roofline").

A step = one pass of the whole hot path over one
batch of synthetic input:
  * ODS: init_cache + the full trace-driven replay of the workload (default
    BASELINE configs[3] on one GPU, the ImageNet-22K-shaped trace the north_star's
    roofline target names: 14,197,122 samples, 8 jobs x 512, cache 400 GB at
    split 100-0-0, 2 epochs = 55,458 rounds, 227.15 M sample decisions) -- the
    headline `value` (decisions/s).  The ImageNet-1K and OpenImages traces
    (configs[1], configs[2]) are timed in the same run under `workloads`, each
    gated by its oracle golden;
  * MDP: the sweep over 10,000 synthetic hardware profiles x 5,151 splits (1 %
    grid, configs[4]) with the full grid written to HBM -- reported in `mdp`.

    python bench.py [--gpus N --steps K --warmup W] [--workload imagenet1k]
    python bench.py --impl reference      # the oracle (CPU) as the reference arm

N > 1 (torchrun, one process per GPU): every rank replays its own instance
(seed + rank) and sweeps its own 10,000 profiles -- the path partitions into
independent problems, so there is no data-path collective (weak scaling).

`replicas`: the same workload as R independent replays in ONE
context (replica k: seed + k), one cooperative launch filling the GPU with
R x (J + 1) round CTAs; reported beside the single-replay headline.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "ODS sample decisions/sec & MDP split evals/sec (1/2/4/8 B200), % of HBM roofline"
WORKLOADS = {
    "imagenet1k": "ImageNet-1K-shaped trace (BASELINE configs[1])",
    "openimages": "OpenImages-shaped trace (BASELINE configs[2])",
    "imagenet22k": "ImageNet-22K-shaped trace (BASELINE configs[3], one GPU)",
    "toy": "toy trace (BASELINE configs[0])",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="imagenet22k", choices=sorted(WORKLOADS))
    ap.add_argument("--extra-workloads", default="imagenet1k,openimages",
                    help="comma list of further workloads timed in the same run ('' : none)")
    ap.add_argument("--mdp-profiles", type=int, default=10_000)
    ap.add_argument("--mdp-grid-step", type=int, default=1)
    ap.add_argument("--mdp-large", type=int, default=100_000,
                    help="also time one MDP sweep of this many profiles with the grid written (0: skip)")
    ap.add_argument("--no-grid", action="store_true", help="MDP argmax only (no grid write)")
    ap.add_argument("--no-profile", action="store_true", help="no CUDA-event kernel timing in the timed steps")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target oracle sample duration")
    ap.add_argument("--evict-tiers", type=int, default=0, choices=[0, 1],
                    help="0: A only (SPEC default, the headline); 1: every cached tier (R-O21)")
    ap.add_argument("--shards", default="2,4,8",
                    help="N = 1: shard counts of the emulated sample-ID-range-sharded replay ('' : none)")
    ap.add_argument("--no-shard-replay", action="store_true",
                    help="N > 1: skip the replay sharded across the ranks (one shard per GPU)")
    ap.add_argument("--replicas", type=int, default=-1,
                    help="also time R independent replays in one context (-1: as many as fit the GPU, 0: skip)")
    return ap.parse_args()


def dist_env():
    """(rank, world, local_rank) from the torchrun environment (read here, so the
    reference arm imports nothing from the product package)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def oracle_caps(c):
    """The oracle's own capacities (Eqs. 5-7 in oracle/): every oracle leg uses these."""
    import oracle as O
    return tuple(O.config_capacities(c))


def caps_of(c):
    """The product's capacities (seneca_split_capacities), checked against the oracle's."""
    from paper_2511_13724_b200 import seneca as S
    caps = S.split_capacities(c["n_total"], c["s_data"], c["m_num"], c["m_den"], c["cache_bytes"], *c["split"])
    caps = (caps[0], caps[1], caps[2])
    assert caps == oracle_caps(c), (caps, oracle_caps(c))
    return caps


def decisions_of(c):
    return sum(c["n_total"] * e for e in c["target"])


def workload_config(c, name, extra):
    return dict(workload=f"{name}: {WORKLOADS[name]}", n_total=c["n_total"], jobs=len(c["batch"]),
                batch=c["batch"] if len(set(c["batch"])) > 1 else c["batch"][0],
                epochs=c["target"][0], split="-".join(map(str, c["split"])), seed=hex(c["seed"]), **extra)


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if not self.proc:
            return dict(sm_mhz=None, sm_max_mhz=None, reasons=["nvidia-smi unavailable"], samples=0)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = self.rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[3 + k].lower() == "active"})

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[0]) for r in rows if num(r[0]) is not None]
        mx = [num(r[1]) for r in rows if num(r[1]) is not None]
        return dict(sm_mhz=float(np.median(sm)) if sm else None, sm_max_mhz=max(mx) if mx else None,
                    reasons=reasons, samples=len(rows))


# --------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    """The oracle (plain single-threaded C, oracle/) timed on the host cores, as it
    stands, on the same workload: each step replays a bounded prefix of rounds."""
    if rank != 0:
        return 0
    import oracle as O
    c = synth.ods_config(args.workload, seed=synth.PERF_SEED)
    ce, cd, ca = oracle_caps(c)
    rounds_per_step = {"toy": 96, "imagenet1k": 800, "openimages": 500, "imagenet22k": 40}[args.workload]
    decisions = 0
    t_tot = 0.0
    for s in range(args.warmup + args.steps):
        o = O.ODS(c["n_total"], c["batch"], c["target"], ce, cd, ca, c["seed"], evict_all=bool(args.evict_tiers))
        t0 = time.perf_counter()
        done = o.replay_rounds(rounds_per_step)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            _, e, n, _ = o.job_state()
            decisions += int(sum(int(e[j]) * c["n_total"] + int(n[j]) for j in range(len(c["batch"]))))
            t_tot += dt
    val = decisions / t_tot
    sample = f"first {rounds_per_step} rounds of the {args.workload} replay per step (oracle, 1 thread)"
    line = dict(metric=METRIC, value=val, unit="decisions/s", impl="reference", n_gpus=args.gpus,
                steps=args.steps, warmup=args.warmup, ms_per_step=1e3 * t_tot / args.steps,
                higher_is_better=True, scaling="weak", vs_baseline=None, dtype="u32", data="synthetic",
                config=workload_config(c, args.workload, dict(note="reference arm = the CPU oracle")),
                cpu_baseline=dict(value=val, unit="decisions/s", cores=1, kind="oracle", sample=sample),
                e2e=dict(value=val, unit="decisions/s", h2d_bytes_per_step=0, d2h_bytes_per_step=0),
                so_loaded=repo_so_loaded())
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- cpu baseline
def _oracle_mdp_slice(job):
    """One worker of the all-cores MDP oracle run (a process: the oracle is
    single-threaded C)."""
    rows, g = job
    import oracle as O
    O.mdp_sweep(rows, g, want_grid=False)
    return len(rows)


def oracle_mdp_all_cores(args, per_core=1000):
    """the MDP oracle also on all host cores -- profiles striped over
    one process per core, each running the unmodified oracle on its slice."""
    import multiprocessing as mp
    import oracle as O
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    rows = O.profiles_from_columns(synth.mdp_profiles(per_core * cores, seed=synth.PERF_SEED))
    jobs = [(rows[k * per_core:(k + 1) * per_core], args.mdp_grid_step) for k in range(cores)]
    with mp.get_context("fork").Pool(cores) as pool:
        pool.map(_oracle_mdp_slice, [(rows[:1], args.mdp_grid_step)] * cores)     # start the workers
        t0 = time.perf_counter()
        done = sum(pool.map(_oracle_mdp_slice, jobs, chunksize=1))
        dt = time.perf_counter() - t0
    return done * O.num_splits(args.mdp_grid_step) / dt, cores, done, dt


def _oracle_ods_prefix(job):
    """One worker of the all-cores ODS oracle run: replica k's replay (seed + k) for a
    fixed number of rounds; returns the decisions it made."""
    c, caps, k, rounds, evict_all = job
    import oracle as O
    ce, cd, ca = caps
    o = O.ODS(c["n_total"], c["batch"], c["target"], ce, cd, ca, c["seed"] + k, evict_all=evict_all)
    o.replay_rounds(rounds)
    _, e, n, _ = o.job_state()
    return int(sum(int(e[j]) * c["n_total"] + int(n[j]) for j in range(len(c["batch"]))))


def oracle_ods_all_cores(args, c, caps, rounds):
    """"with R replicas, R processes spread over host cores" -- one
    independent oracle replay (seed + k) per core, each a fixed prefix of rounds;
    the counterpart of the GPU replicas line."""
    import multiprocessing as mp
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    jobs = [(c, caps, k, rounds, bool(args.evict_tiers)) for k in range(cores)]
    with mp.get_context("fork").Pool(cores) as pool:
        t0 = time.perf_counter()
        dec = sum(pool.map(_oracle_ods_prefix, jobs, chunksize=1))
        dt = time.perf_counter() - t0
    return dec / dt, cores, dec, dt


def cpu_baseline(args, c, caps):
    import oracle as O
    ce, cd, ca = caps
    # calibrate: a short run, then scale to ~args.cpu_seconds
    o = O.ODS(c["n_total"], c["batch"], c["target"], ce, cd, ca, c["seed"], evict_all=bool(args.evict_tiers))
    t0 = time.perf_counter()
    o.replay_rounds(50)
    per = (time.perf_counter() - t0) / 50
    rounds = max(50, int(args.cpu_seconds / max(per, 1e-6)))
    o = O.ODS(c["n_total"], c["batch"], c["target"], ce, cd, ca, c["seed"], evict_all=bool(args.evict_tiers))
    t0 = time.perf_counter()
    done = o.replay_rounds(rounds)
    dt = time.perf_counter() - t0
    _, e, n, _ = o.job_state()
    dec = int(sum(int(e[j]) * c["n_total"] + int(n[j]) for j in range(len(c["batch"]))))
    # MDP oracle on a profile sample
    rows = O.profiles_from_columns(synth.mdp_profiles(1000, seed=synth.PERF_SEED))
    t1 = time.perf_counter()
    O.mdp_sweep(rows, args.mdp_grid_step, want_grid=False)
    dm = time.perf_counter() - t1
    ns = O.num_splits(args.mdp_grid_step)
    mdp_all, mcores, mdone, mdt = oracle_mdp_all_cores(args)
    ods_all, ocores, odec, odt = oracle_ods_all_cores(args, c, caps, max(10, done // 4))
    return dict(value=dec / dt, unit="decisions/s", cores=1, kind="oracle",
                sample=f"oracle replay of the first {done} rounds ({dec} decisions, {dt:.1f} s) of the same "
                       f"workload (the ODS oracle is a sequential protocol: 1 core); MDP oracle 1,000 profiles x "
                       f"{ns} splits in {dm:.2f} s on 1 core, {mdone:,} profiles in {mdt:.2f} s on {mcores} cores",
                mdp_value=1000 * ns / dm, mdp_unit="split-evals/s",
                replicas_value_all_cores=ods_all, replicas_cores_all=ocores,
                replicas_sample=f"{ocores} independent oracle replays (seed + k), {max(10, done // 4)} rounds each "
                                f"({odec} decisions in {odt:.1f} s), one process per core",
                mdp_value_all_cores=mdp_all, mdp_cores_all=mcores,
                mdp_cores_note="processes launched = the affinity count; a CPU quota can leave fewer effective cores")


# --------------------------------------------------------------------------- roofline models
def algorithmic_bytes(name, info):
    """Algorithmic (logical) bytes one launch of `name` must move.
    info: per-step workload facts (rounds, decisions, substitutes, bitmap words...)."""
    W4 = info["words"] * 4                          # bytes of one bitmap
    J = info["jobs"]
    if name == "mdp_sweep":
        return info["mdp_profiles"] * (112 + 48) + (8 * info["mdp_profiles"] * info["mdp_splits"]
                                                   if info["mdp_grid"] else 0)
    if name == "ods_rounds":
        # per requested sample: list entry 4 + seen word 4 + residency words (<= 3) 12 + consumer word 4
        #   + seen RMW 8 = 32 B
        # per substitute: 32-B block-count row + one 16-B vector of each of <= 3 bitmaps 48 + seen/consumer
        #   RMW 16 + block-count RMW 8 = 104 B
        # per A-served sample: consumer-count RMW 8 B; per eviction: residency + J consumer RMW 8(J+1)
        # per refill: count row 32 + 3 bitmap vectors 48 + residency RMW 8 + J seen words 4J
        # per job-epoch: seen clear W4 + recount (residency x3 + consumers + seen) 5 W4
        return (32 * info["decisions"] + 104 * info["substitutes"] + 8 * info["a_served"]
                + 8 * (J + 1) * info["refilled"] + (88 + 4 * J) * info["refilled"]
                + 6 * W4 * info["job_epochs"])
    if name == "ods_perm_all":
        return 4 * info["n_total"] * info["job_epochs"]     # ALU-bound (Philox); bytes written
    if name == "ods_recount_all":
        # the init bitmap pass: 3 residency + J seen + J consumer bitmaps (DRAM reads; the
        # residency re-reads per job hit L2); per pool
        # (3J + 1) one u8 count per 128 ids and one u32 per 4096 ids written
        return (3 + 2 * J) * W4 + (3 * J + 1) * (W4 // 16 + W4 // 512 * 4)
    if name == "ods_init_tiers":
        return 4 * info["cache_entries"]
    return 0


NCU_TRAFFIC = os.path.join(ROOT, "profiles", "r2", "ncu_traffic.json")


def repo_so_loaded():
    """The shared objects of this repository mapped into this process (evidence of
    which native code ran: the reference arm must show only oracle/liboracle.so)."""
    try:
        maps = open("/proc/self/maps").read().split("\n")
    except OSError:
        return None
    return sorted({os.path.relpath(l.split()[-1], ROOT) for l in maps
                   if l.strip().endswith(".so") and l.split()[-1].startswith(ROOT)})
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12      # nominal B200 FP64 (non-tensor), ~37.2 TFLOP/s


def pass_equivalent(c, caps, words, ods_s, steps, world, hbm_peak, replicas=None):
    """SURVEY §8(d) "How the targets are measured", item 1: the logical bytes a
    full-pass design moves for this replay -- per job-round one pass over seen_j,
    every non-empty tier bitmap and (with A) cons_j, i.e. (1 + #tiers + [A]) N/8 B
    (SURVEY §8(a) row a4); per round with A one storage-pool pass over the three
    residency bitmaps (3 N/8 B); per job-epoch one seen reset (N/8 B, row a8) --
    divided by the replay's measured time.  ods_rounds maintains the pool counts
    incrementally and moves far fewer bytes; this is the rate a
    pass-based replay would have to sustain to match it, as a fraction of peak."""
    W = words * 4
    ce, cd, ca = caps[0], caps[1], caps[2]
    tiers = (ce > 0) + (cd > 0) + (ca > 0)
    per_job_round = (1 + tiers + (1 if ca > 0 else 0)) * W
    job_rounds = sum(t * -(-c["n_total"] // b) for t, b in zip(c["target"], c["batch"]))
    rounds = max(t * -(-c["n_total"] // b) for t, b in zip(c["target"], c["batch"]))
    total = per_job_round * job_rounds + (3 * W * rounds if ca > 0 else 0) + W * sum(c["target"])
    rate = total * steps * world / ods_s / 1e9
    out = dict(bytes_per_replay=int(total), job_rounds=int(job_rounds), achieved=rate, peak=hbm_peak,
               unit="GB/s", frac=rate / hbm_peak,
               note="full-pass logical bytes (SURVEY 8(d) target 1) / measured replay time; not DRAM traffic "
                    "(ods_rounds keeps pool counts incrementally, see roofline.traffic)")
    if replicas is not None:
        rr = replicas["value"] / decisions_of(c)      # replays per second, all ranks
        out["replicas"] = dict(R=replicas["R"], achieved=total * rr / 1e9, frac=total * rr / 1e9 / hbm_peak)
    return out


def ncu_traffic(key):
    """DRAM bytes (read + write) of one launch, from the committed `ncu --set full`
    capture of the same launch (tools/measure.sh -> tools/ncu_summary.py), or None."""
    try:
        t = json.load(open(NCU_TRAFFIC))
    except (OSError, ValueError):
        return None
    e = t.get(key)
    return None if e is None else e["dram_bytes_per_launch"]


def roofline_for(name, k, info, hbm_peak, peak_src, traffic=None):
    bpl = algorithmic_bytes(name, info)
    avg_s = (k["avg_us"] or 0.0) / 1e6
    ach = bpl / avg_s / 1e9 if avg_s > 0 else 0.0
    return dict(kernel=name, bound="hbm", achieved=ach, peak=hbm_peak, unit="GB/s",
                frac=ach / hbm_peak, traffic=traffic, bytes_per_launch=bpl, avg_launch_us=k["avg_us"],
                peak_source=peak_src)


# --------------------------------------------------------------------------- latency floor of ods_rounds
# Inputs measured on B200 (profiles/r1/microbench.md, tools/micro): a dependent
# ld.global.cg chain costs 267-358 cycles per step (median ~300); one CTA issues
# ~1 scattered global access (wavefront) per cycle; perm_apply (4 Philox-10 on
# Z_a x Z_b) takes ~1,790 cycles per call with 512 threads.
L2_DEP_CYCLES = 300
PERM_CYCLES = 1790


def latency_floor(c, caps, st, rounds, evicted, refilled, sm_mhz):
    """Per-round floor of the round chain of one job CTA (DESIGN.md §7.1 "latency
    roofline"): dependent L2 round trips x the measured dependent latency +
    scattered global accesses at one per cycle + the substitution-rank ALU
    chain (perm_apply) in rounds that substitute -- each summed per job-round
    from the replay's own counters, averaged over job-rounds, and compared with
    the measured microseconds per round of the whole replay (rounds run in
    lock-step across jobs).

    Static tiers (no A tier): a job-round whose pools are empty needs no seen
    test, no residency gather and no seen mark (its requests are the next
    storage ids in permutation order, DESIGN.md 7.1 "late rounds"), so only the
    rounds with non-empty pools -- estimated as the substituting ones -- carry
    per-request scattered accesses; the late rounds are counted at zero (most of
    them are not on the round chain at all: the late bulk decides them in one
    pass per stretch)."""
    ce, cd, ca = caps
    J = len(c["batch"])
    N = c["n_total"]
    tiers = (ce > 0) + (cd > 0) + (ca > 0)
    job_rounds = sum(t * -(-N // b) for t, b in zip(c["target"], c["batch"]))
    req = float(st["served"].sum())                        # delivered decisions = requests
    hits = float(st["req_hits"].sum())
    sub = st["subst"].sum(axis=(0, 1)).astype(float)       # by tier code S0 E1 D2 A3
    subs = float(sub.sum())
    a_served = float(st["served"][:, :, 3].sum())
    # substituting job-rounds (not counted by the kernel): substitutes / mean misses
    # per job-round -- a lower bound, since a substituting round replaces at most
    # its misses (so the floor below stays a floor)
    sub_rounds = min(job_rounds, subs / max(1.0, (req - hits) / job_rounds))
    static = ca == 0
    # requests that needed the seen test / residency gather: all of them with an
    # A tier; with static tiers those of the rounds whose pools were non-empty
    req_tested = req if not static else min(req, sub_rounds * req / job_rounds)
    # walk: positions examined = tested requests + deferred re-requests (R-O1)
    positions = req_tested + (0.0 if static else subs)
    scattered = (positions / 4 + positions          # list vectors + per-position seen chunk copies
                 + req_tested * max(1, tiers)       # residency word gathers (classify)
                 + req_tested                       # seen RMW (respond)
                 + hits + subs                      # pool block-count RMW
                 + 2 * subs                         # 32-B count row (two 16-B loads)
                 + 2 * sub[1] + 2 * sub[2] + 3 * sub[3]   # bitmap vectors of the selected block
                 + subs                             # deferral-list store
                 + 2 * a_served                     # consumer-set RMW + consumer-count RMW
                 + J * 2 * refilled)                # refill intake: seen gather + count RMW per job
    tested_rounds = job_rounds if not static else sub_rounds
    dep = tested_rounds * 3 + 2 * sub_rounds        # walk prefetch wait, classify, respond RMW; + select
    if ca > 0:
        dep += job_rounds * 3                       # maintain: signal, eviction/refill apply, release
    cyc = dep * L2_DEP_CYCLES + scattered + sub_rounds * PERM_CYCLES
    floor_us = cyc / job_rounds / sm_mhz
    return dict(floor_us_per_round=floor_us, cycles_per_job_round=cyc / job_rounds,
                dependent_trips_per_job_round=dep / job_rounds, scattered_per_job_round=scattered / job_rounds,
                substituting_job_round_share=sub_rounds / job_rounds, static_tiers=static,
                inputs=dict(l2_dependent_cycles=L2_DEP_CYCLES, perm_apply_cycles=PERM_CYCLES,
                            scattered_per_cycle=1, sm_mhz=sm_mhz, source="profiles/r2/microbench.md"))


def golden_gate(name, seed, evict_tiers, st_raw, evicted=None, refilled=None):
    """Per job-epoch counters + digests (and eviction/refill totals) of a full replay
    against the oracle's golden file (tests/golden/, written by oracle/ only)."""
    path = os.path.join(ROOT, "tests", "golden", f"oracle_{name}_seed{seed}{'_evictall' if evict_tiers else ''}.json")
    if not os.path.exists(path):
        return "n/a (no golden for this seed)"
    gold = json.load(open(path))
    ok = all(int(st_raw[j, e]["digest"]) == int(s_["digest"]) and
             [int(x) for x in st_raw[j, e]["served"]] == s_["served"] and
             [int(x) for x in st_raw[j, e]["subst"]] == s_["subst"]
             for j, row in enumerate(gold["stats"]) for e, s_ in enumerate(row))
    if evicted is not None:
        ok = ok and (evicted, refilled) == (gold["evicted"], gold["refilled"])
    return "bit-exact" if ok else "MISMATCH"


def prefix_gate(c, seed, replicas, ks, rounds, evict_tiers, stream):
    """The launch configuration bench.py times (same workload, same replica count,
    hence the same kernel variant and grid), replayed for `rounds` rounds; replica
    k's residency/seen/consumer bitmaps and counters vs an oracle replay of seed + k
    (oracle capacities) for the same rounds.  Returns {k: bool}."""
    import torch
    import oracle as O
    import paper_2511_13724_b200 as P
    ce, cd, ca = caps_of(c)
    oc = oracle_caps(c)
    g = P.ODSContext(c["n_total"], c["batch"], c["target"], ce, cd, ca, seed, replicas=replicas,
                     evict_tiers=evict_tiers, stream=stream)
    g.replay_rounds(rounds)
    torch.cuda.synchronize()
    g.sync()
    out = {}
    for k in ks:
        o = O.ODS(c["n_total"], c["batch"], c["target"], *oc, (seed + k) & 0xFFFFFFFFFFFFFFFF,
                  evict_all=bool(evict_tiers))
        o.replay_rounds(rounds)
        st_o, ev_o, rf_o = o.stats()
        st_g, ev_g, rf_g = g.stats(k)
        ok = st_g.tobytes() == st_o.tobytes() and (ev_g, rf_g) == (ev_o, rf_o)
        if ok:
            for a, b in zip(g.state(k), o.state()):
                ok = ok and np.array_equal(a, b)
        out[k] = bool(ok)
        del o
    g.close()
    return out


PREFIX_ROUNDS = {"toy": 96, "imagenet1k": 256, "openimages": 200, "imagenet22k": 48}


def read_stats(S, ws, ctx, c, k=0):
    v = S.read_state(ctx)
    nst = len(c["batch"]) * v.max_target * S.STATS_DTYPE.itemsize
    off = v.d_stats + k * v.replica_stride - ws.data_ptr()
    st = ws[off:off + nst].cpu().numpy().view(S.STATS_DTYPE).reshape(len(c["batch"]), v.max_target).copy()
    o_ev = v.d_evicted + k * v.replica_stride - ws.data_ptr()
    o_rf = v.d_refilled + k * v.replica_stride - ws.data_ptr()
    ev = int(ws[o_ev:o_ev + 8].cpu().numpy().view(np.uint64)[0])
    rf = int(ws[o_rf:o_rf + 8].cpu().numpy().view(np.uint64)[0])
    return st, ev, rf


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    from paper_2511_13724_b200 import seneca as S
    from paper_2511_13724_b200 import dist as D

    # One process per GPU over NCCL.  SENECA_DIST_BACKEND=gloo (test only) runs the
    # multi-rank host logic with several ranks sharing the GPUs there are
    # (ranks map to local_rank mod device_count; timings reduce on the CPU).
    backend = os.environ.get("SENECA_DIST_BACKEND", "nccl")
    local_dev = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        import torch.distributed as dist
        import datetime
        tmo = datetime.timedelta(minutes=5)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev, timeout=tmo)
        else:
            dist.init_process_group(backend, timeout=tmo)
    red_dev = dev if backend == "nccl" else None
    stream = torch.cuda.current_stream(dev)

    seed = D.rank_seed(synth.PERF_SEED, rank)
    c = synth.ods_config(args.workload, seed=seed)
    caps = caps_of(c)
    ce, cd, ca = caps
    dec_per_step = decisions_of(c)

    # ---- inputs resident in HBM before timing
    mdp_cols = synth.mdp_profiles(args.mdp_profiles, seed=seed)
    prof_host = S.profiles_from_columns(mdp_cols)
    d_prof = torch.from_numpy(prof_host.view(np.uint8).copy()).to(dev)
    nsplit = S.mdp_num_splits(args.mdp_grid_step)
    d_res = torch.empty(args.mdp_profiles * S.RESULT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    d_grid = None if args.no_grid else torch.empty((args.mdp_profiles, nsplit), dtype=torch.float64, device=dev)
    cfg = S.make_config(c["n_total"], c["batch"], c["target"], ce, cd, ca, c["seed"], evict_tiers=args.evict_tiers)
    ws_bytes = S.state_bytes(cfg)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)      # > 126 MB L2

    fill_ms = []                                                     # the flush's fill_: a pure 512 MiB write

    def l2_flush(v):
        # evict L2 by writing 512 MiB, then read the first 256 MiB of it back so that
        # the flush's own dirty lines are written back here, not inside the next timed
        # region (where they would compete with the kernel's own DRAM writes)
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        flush.view(torch.float64).fill_(float(v & 0xFF))              # 8-B elements: full-width stores
        f1.record(stream)
        flush[: 256 << 20].max()
        f1.synchronize()
        fill_ms.append(f0.elapsed_time(f1))

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def one_step(profile=False, ev=None):
        # MDP first: its launch is queued behind a short device sleep so the
        # host's enqueue latency is not inside its events; the replay follows
        # (with profiling on, its launches are host-synchronised).
        if ev is not None:
            torch.cuda._sleep(200_000)                              # ~0.1 ms, before the first event
            ev[0].record(stream)
        S.mdp_sweep(d_prof, args.mdp_profiles, args.mdp_grid_step, d_res, d_grid, stream)
        if ev is not None:
            ev[1].record(stream)
        ctx = S.init_cache(cfg, ws, ws_bytes, stream)
        if profile:
            S.profile(ctx, 1)                                      # event-timed launches only
        rounds = S.replay_epochs(ctx, max(c["target"]), None, stream)
        return ctx, rounds

    # ---- warm-up
    for _ in range(max(args.warmup, 0)):
        ctx, _ = one_step()
        torch.cuda.synchronize(dev)
        S.destroy(ctx)

    # ---- timed steps (device time, CUDA events on the launch stream)
    clocks = ClockSampler(local_dev)
    clocks.start()
    ods_ms, mdp_ms, launches, rounds_tot = [], [], 0, 0
    kstats = {}
    last_ctx = None
    for s in range(args.steps):
        l2_flush(s & 0xFF)                                      # evict L2 between steps
        barrier()
        torch.cuda.synchronize(dev)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ctx, rounds = one_step(not args.no_profile, ev)
        ev[2].record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        mdp_ms.append(ev[0].elapsed_time(ev[1]))
        ods_ms.append(ev[1].elapsed_time(ev[2]))
        launches += S.launch_count(ctx) + 1
        rounds_tot += rounds
        for k, v in S.profile_read(ctx).items():
            a = kstats.setdefault(k, dict(launches=0, sampled=0, sampled_ms=0.0))
            for f in a:
                a[f] += v[f]
        if last_ctx:
            S.destroy(last_ctx)
        last_ctx = ctx
    clk = clocks.stop()

    # ---- parity gates (outside the timed region)
    parity = {}
    S.sync_status(last_ctx, stream)
    v = S.read_state(last_ctx)
    st_raw, ev_tot, rf_tot = read_stats(S, ws, last_ctx, c)
    parity["ods_served_per_job_epoch_equals_N"] = bool(np.all(st_raw["served"].sum(axis=2) == c["n_total"]))
    parity["ods_vs_oracle_golden"] = golden_gate(args.workload, c["seed"], args.evict_tiers, st_raw, ev_tot, rf_tot)
    if parity["ods_vs_oracle_golden"] == "n/a (no golden for this seed)":
        # rank > 0 (seed + rank): the same launch configuration for a prefix of
        # rounds against an oracle replay of this rank's seed
        pg = prefix_gate(c, c["seed"], 1, [0], PREFIX_ROUNDS[args.workload], args.evict_tiers, stream)
        parity["ods_vs_oracle_prefix"] = "bit-exact" if pg[0] else "MISMATCH"
    try:
        import oracle as O
        k = min(200, args.mdp_profiles)
        orow = O.profiles_from_columns({f: mdp_cols[f][:k] for f in mdp_cols})
        ores, ogrid = O.mdp_sweep(orow, args.mdp_grid_step, want_grid=d_grid is not None)
        res = d_res.cpu().numpy().view(S.RESULT_DTYPE)[:k]
        ok = np.array_equal(res["v_best"].view(np.uint64), ores["v"].view(np.uint64)) and \
            all(np.array_equal(res[f], ores[f]) for f in ("p_e", "p_d", "p_a"))
        if d_grid is not None:
            ok = ok and np.array_equal(d_grid[:k].cpu().numpy().view(np.uint64), ogrid.view(np.uint64))
        parity["mdp_vs_oracle_first_200_profiles"] = "bit-exact" if ok else "MISMATCH"
    except Exception as e:  # the oracle is only a checker; report, do not fall back
        parity["mdp_vs_oracle_first_200_profiles"] = f"unchecked: {e}"

    # ---- MDP at scale ("also measure 10^5-10^6 profiles or grid-dump
    #      mode"): 100,000 profiles x 5,151 splits, 4.1 GB of grid written; median of 3
    #      event-timed sweeps after a warm-up, L2 flushed before each; parity on the
    #      first and last 50 profiles
    mdp_large = None
    if args.mdp_large > 0 and not args.no_grid:
        import oracle as O
        nl = args.mdp_large
        cols_l = synth.mdp_profiles(nl, seed=seed + 1)
        d_prof_l = torch.from_numpy(S.profiles_from_columns(cols_l).view(np.uint8).copy()).to(dev)
        d_res_l = torch.empty(nl * S.RESULT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        d_grid_l = torch.empty((nl, nsplit), dtype=torch.float64, device=dev)
        S.mdp_sweep(d_prof_l, nl, args.mdp_grid_step, d_res_l, d_grid_l, stream)
        times = []
        for _ in range(3):
            l2_flush(3)
            torch.cuda.synchronize(dev)
            e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            torch.cuda._sleep(200_000)
            e[0].record(stream)
            S.mdp_sweep(d_prof_l, nl, args.mdp_grid_step, d_res_l, d_grid_l, stream)
            e[1].record(stream)
            torch.cuda.synchronize(dev)
            times.append(e[0].elapsed_time(e[1]))
        ms_l = float(np.median(times))
        idx = np.r_[0:50, nl - 50:nl]
        orow = O.profiles_from_columns({f: cols_l[f][idx] for f in cols_l})
        ores, ogrid = O.mdp_sweep(orow, args.mdp_grid_step, want_grid=True)
        res = d_res_l.cpu().numpy().view(S.RESULT_DTYPE)[idx]
        ok = np.array_equal(res["v_best"].view(np.uint64), ores["v"].view(np.uint64)) and \
            all(np.array_equal(res[f], ores[f]) for f in ("p_e", "p_d", "p_a")) and \
            np.array_equal(d_grid_l[torch.from_numpy(idx).to(dev)].cpu().numpy().view(np.uint64), ogrid.view(np.uint64))
        bytes_l = nl * (112 + 48) + 8 * nl * nsplit
        mdp_large = dict(profiles=nl, splits=nsplit, ms=ms_l, value=nl * nsplit / (ms_l / 1e3), unit="split-evals/s",
                         grid_bytes=8 * nl * nsplit,
                         roofline=dict(bound="hbm", achieved=bytes_l / (ms_l / 1e3) / 1e9, unit="GB/s"),
                         parity="bit-exact (first and last 50 profiles, results and grid rows)" if ok else "MISMATCH")
        del d_prof_l, d_res_l, d_grid_l

    # ---- the other ODS workloads of BASELINE.json, timed the same way (init_cache +
    #      full replay, L2 flushed, one warm-up), each gated by its oracle golden
    extra = {}
    for name in [w for w in args.extra_workloads.split(",") if w and w != args.workload]:
        cx = synth.ods_config(name, seed=seed)
        cex, cdx, cax = caps_of(cx)
        cfgx = S.make_config(cx["n_total"], cx["batch"], cx["target"], cex, cdx, cax, cx["seed"],
                             evict_tiers=args.evict_tiers)
        wbx = S.state_bytes(cfgx)
        wsx = torch.empty(wbx, dtype=torch.uint8, device=dev)
        msx, ctxx, rx = [], None, 0
        for s in range(1 + args.steps):
            l2_flush(s & 0xFF)
            barrier()
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctxx = S.init_cache(cfgx, wsx, wbx, stream)
            rx = S.replay_epochs(ctxx, max(cx["target"]), None, stream)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            barrier()
            if s >= 1:
                msx.append(e0.elapsed_time(e1))
            if s < args.steps:
                S.destroy(ctxx)
        S.sync_status(ctxx, stream)
        stx, evx, rfx = read_stats(S, wsx, ctxx, cx)
        gate = golden_gate(name, cx["seed"], args.evict_tiers, stx, evx, rfx)
        if gate == "n/a (no golden for this seed)":
            pg = prefix_gate(cx, cx["seed"], 1, [0], PREFIX_ROUNDS[name], args.evict_tiers, stream)
            gate = "bit-exact (oracle prefix)" if pg[0] else "MISMATCH"
        S.destroy(ctxx)
        del wsx
        (sx,) = D.reduce_times([sum(msx) / 1e3], device=red_dev)
        decx = decisions_of(cx)
        extra[name] = dict(value=decx * args.steps * world / sx, unit="decisions/s", ms_per_step=1e3 * sx / args.steps,
                           rounds=rx, us_per_round=1e3 * sx / args.steps / rx * 1e3,
                           config=workload_config(cx, name, dict(rounds_per_step=rx, decisions_per_step=decx)),
                           parity=gate)

    # ---- R independent replays in one context (untimed warm-up, then timed steps).
    #      Candidates: the most replicas with one 512-thread round CTA per SM, and
    #      with two 256-thread CTAs per SM (the library picks the kernel variant);
    #      the line reports the faster, both are listed.  Gates: replica 0 (seed =
    #      the golden's at rank 0) digests vs the oracle golden; replicas 1 and 2 of
    #      the same launch configuration vs oracle replays of seed + 1, seed + 2 for a
    #      prefix of rounds.
    rep_line = None
    if args.replicas != 0:
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        J1 = len(c["batch"]) + 1
        cands = [args.replicas] if args.replicas > 0 else sorted({min(64, sms // J1), min(64, 2 * sms // J1)})
        rseed = (synth.PERF_SEED + 64 * rank) & 0xFFFFFFFFFFFFFFFF
        tried = []
        for R in cands:
            rcfg = S.make_config(c["n_total"], c["batch"], c["target"], ce, cd, ca, rseed, replicas=R,
                                 evict_tiers=args.evict_tiers)
            rbytes = S.state_bytes(rcfg)
            ws_r = torch.empty(rbytes, dtype=torch.uint8, device=dev)
            rep_ms = []
            for s in range(1 + args.steps):
                l2_flush(s & 0xFF)
                barrier()
                torch.cuda.synchronize(dev)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                rctx = S.init_cache(rcfg, ws_r, rbytes, stream)
                S.replay_epochs(rctx, max(c["target"]), None, stream)
                e1.record(stream)
                torch.cuda.synchronize(dev)
                barrier()
                if s >= 1:
                    rep_ms.append(e0.elapsed_time(e1))
                    launches_rep = S.launch_count(rctx)
                if s < args.steps:
                    S.destroy(rctx)
            S.sync_status(rctx, stream)
            served_all = True
            for k in range(R):
                stk, _, _ = read_stats(S, ws_r, rctx, c, k)
                served_all &= bool(np.all(stk["served"].sum(axis=2) == c["n_total"]))
            st0, ev0, rf0 = read_stats(S, ws_r, rctx, c, 0)
            gate0 = golden_gate(args.workload, rseed, args.evict_tiers, st0, ev0, rf0)
            S.destroy(rctx)
            del ws_r
            gates = prefix_gate(c, rseed, R, [1, 2] if R > 2 else list(range(R)), PREFIX_ROUNDS[args.workload],
                                args.evict_tiers, stream)
            (rep_s,) = D.reduce_times([sum(rep_ms) / 1e3], device=red_dev)
            tried.append(dict(R=R, value=R * dec_per_step * args.steps * world / rep_s, unit="decisions/s",
                              ms_per_step=1e3 * rep_s / args.steps,
                              per_replica_value=dec_per_step * args.steps / rep_s,
                              round_ctas=R * J1, ctas_per_sm=1 if R * J1 <= sms else 2,
                              launches_per_step=launches_rep, served_ok=served_all,
                              parity=dict(replica0_vs_oracle_golden=gate0,
                                          **{f"replica{k}_vs_oracle_first_{PREFIX_ROUNDS[args.workload]}_rounds":
                                             "bit-exact" if ok else "MISMATCH" for k, ok in gates.items()})))
        best = max(tried, key=lambda t: t["value"])
        rep_line = dict(best, seeds=f"{hex(rseed)} + k, k < R",
                        candidates=[{k: t[k] for k in ("R", "value", "per_replica_value", "ctas_per_sm", "parity")}
                                    for t in tried],
                        note="init_cache + replay_epochs of R independent instances of the workload in one "
                             "context (one cooperative launch); L2 flushed between steps")
        rep_line["parity"] = dict(best["parity"],
                                  every_replica_served_each_sample_once_per_job_epoch=all(t["served_ok"] for t in tried))
        rep_line.pop("served_ok", None)

    # ---- e2e through the public API with host buffers (pinned), copies inside
    pin_prof = torch.from_numpy(prof_host.view(np.uint8).copy()).pin_memory()
    pin_res = torch.empty(d_res.numel(), dtype=torch.uint8).pin_memory()
    nst = len(c["batch"]) * v.max_target * S.STATS_DTYPE.itemsize
    pin_stats = torch.empty(nst, dtype=torch.uint8).pin_memory()
    e2e_ods, e2e_mdp = [], []
    for s in range(args.steps):
        l2_flush(s & 0xFF)
        barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        ctx = S.init_cache(cfg, ws, ws_bytes, stream)
        S.replay_epochs(ctx, max(c["target"]), None, stream)
        vv = S.read_state(ctx)
        o2 = vv.d_stats - ws.data_ptr()
        pin_stats.copy_(ws[o2:o2 + nst], non_blocking=True)
        torch.cuda.synchronize(dev)
        t1 = time.perf_counter()
        d_prof.copy_(pin_prof, non_blocking=True)
        S.mdp_sweep(d_prof, args.mdp_profiles, args.mdp_grid_step, d_res, d_grid, stream)
        pin_res.copy_(d_res, non_blocking=True)
        torch.cuda.synchronize(dev)
        t2 = time.perf_counter()
        e2e_ods.append(t1 - t0)
        e2e_mdp.append(t2 - t1)
        S.destroy(ctx)

    # ---- phase split of the round kernel: one more, untimed replay with the
    #      in-kernel phase counters on (they cost clock reads, so never timed)
    ctx = S.init_cache(cfg, ws, ws_bytes, stream)
    S.profile(ctx, 3)
    S.replay_epochs(ctx, max(c["target"]), None, stream)
    torch.cuda.synchronize(dev)
    vp = S.read_state(ctx)
    ph = ws[vp.d_phase_cycles - ws.data_ptr():vp.d_phase_cycles - ws.data_ptr() + 256].cpu().numpy().view(np.uint64)
    ph_names = {0: "job_epoch_start", 1: "job_classify", 8: "job_subst_prefix", 9: "job_subst_ranks_locate",
                2: "job_subst_apply", 10: "job_storage_deferral", 11: "job_respond_loop", 3: "job_respond_stats",
                4: "job_wait_maint", 5: "job_advance", 12: "job_walk_prefetched_step", 13: "job_walk_rest",
                14: "job_prefetch_issue", 6: "job_late_bulk",
                16: "maint_spec_prefix", 17: "maint_spec_refill_ranks", 18: "maint_barrier1_wait",
                19: "maint_evict_decide", 20: "maint_apply", 21: "maint_barrier2_wait"}
    phase_share = {}
    for base in (0, 16):
        keys = [k for k in ph_names if base <= k < base + 16]
        tot = float(sum(ph[k] for k in keys))
        for k in keys:
            phase_share[ph_names[k]] = round(float(ph[k]) / tot, 4) if tot else None
    phase_share["walk_steps_per_round"] = round(float(ph[7]) / max(1, rounds_tot / args.steps), 3)
    # rounds of job 0 decided by the late bulk pass (DESIGN.md 7.1 "late bulk") / all its rounds
    rounds_job0 = int(c["target"][0]) * -(-int(c["n_total"]) // int(c["batch"][0]))
    phase_share["late_bulk_round_share_job0"] = round(float(ph[15]) / max(1, rounds_job0), 4)
    S.destroy(ctx)

    # ---- aggregate over ranks (max time)
    ods_s = sum(ods_ms) / 1e3
    mdp_s = sum(mdp_ms) / 1e3
    e2e_s = sum(e2e_ods)
    e2e_m = sum(e2e_mdp)
    ods_s, mdp_s, e2e_s, e2e_m = D.reduce_times([ods_s, mdp_s, e2e_s, e2e_m], device=red_dev)   # max over ranks
    total_dec = dec_per_step * args.steps * world
    total_evals = args.mdp_profiles * nsplit * args.steps * world
    parity_ok = [1.0 if all(str(x).startswith(("bit-exact", "n/a")) or x is True for x in parity.values()) else 0.0]
    (parity_all,) = D.reduce_sum(parity_ok, device=red_dev)
    parity["all_ranks_bit_exact"] = f"{int(parity_all)}/{world}"

    # ---- roofline of the dominant kernel (sampled CUDA-event durations)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    if mdp_large:
        mdp_large["roofline"].update(peak=hbm_peak, frac=mdp_large["roofline"]["achieved"] / hbm_peak)
    peak_src = "MEASURED_PEAKS.json hbm_gbs (measured copy)" if "hbm_gbs" in peaks else "fallback 6.65 TB/s"
    kernels = {}
    for name, kv in kstats.items():
        if kv["launches"] == 0:
            continue
        avg = kv["sampled_ms"] / kv["sampled"] if kv["sampled"] else None
        kernels[name] = dict(launches_per_step=kv["launches"] / args.steps,
                             avg_us=None if avg is None else 1e3 * avg,
                             est_ms_per_step=None if avg is None else avg * kv["launches"] / args.steps)
    mdp_ms_step = mdp_s * 1e3 / args.steps
    kernels["mdp_sweep"] = dict(launches_per_step=1, avg_us=1e3 * mdp_ms_step, est_ms_per_step=mdp_ms_step)
    dom = max(kernels, key=lambda k: kernels[k]["est_ms_per_step"] or 0.0)
    info = dict(words=v.words, blocks=(c["n_total"] + 1023) // 1024,
                superblocks=(c["n_total"] + 32767) // 32768, jobs=len(c["batch"]), n_total=c["n_total"],
                rounds=rounds_tot / args.steps, decisions=dec_per_step,
                substitutes=int(st_raw["subst"].sum()), a_served=int(st_raw["served"][:, :, 3].sum()),
                refilled=rf_tot, cache_entries=ce + cd + ca, mdp_profiles=args.mdp_profiles, mdp_splits=nsplit,
                job_epochs=sum(c["target"]), mdp_grid=d_grid is not None)
    tkey = {"ods_rounds": f"ods_rounds@{args.workload}{'-evictall' if args.evict_tiers else ''}",
            "mdp_sweep": f"mdp_sweep@{args.mdp_profiles}x{nsplit}{'' if d_grid is not None else '-nogrid'}"}
    roof = roofline_for(dom, kernels[dom], info, hbm_peak, peak_src, ncu_traffic(tkey.get(dom, dom)))
    if dom == "ods_rounds":
        sm_mhz = clk.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
        lf = latency_floor(c, caps, st_raw, rounds_tot / args.steps, ev_tot, rf_tot, sm_mhz)
        ach_us = kernels["ods_rounds"]["avg_us"] / (rounds_tot / args.steps) if kernels["ods_rounds"]["avg_us"] else \
            1e6 * ods_s / args.steps / (rounds_tot / args.steps)
        roof["latency"] = dict(bound="latency (dependent round chain on one SM per job)",
                               achieved_us_per_round=ach_us, frac=lf["floor_us_per_round"] / ach_us, **lf,
                               note="frac = floor / achieved; the HBM fraction above counts the method's own "
                                    "bytes (DESIGN.md 7.1)")
    mdp_roof = roofline_for("mdp_sweep", kernels["mdp_sweep"], info, hbm_peak, peak_src,
                            ncu_traffic(tkey["mdp_sweep"]))
    if fill_ms:
        # context: the sweep's own bytes are almost all grid writes; a pure write on this GPU
        # (the L2 flush's 512 MiB fill_, timed live, best of the run) is the write-only ceiling
        wr_gbs = (512 << 20) / (min(fill_ms) / 1e3) / 1e9
        mdp_roof["write_only_ceiling"] = dict(gbs=wr_gbs, frac=mdp_roof["achieved"] / wr_gbs,
                                              source="torch fill_ of the 512 MiB L2-flush buffer, CUDA events")
        if mdp_large:
            mdp_large["roofline"]["write_only_ceiling"] = dict(gbs=wr_gbs, frac=mdp_large["roofline"]["achieved"] / wr_gbs)
    for name in kernels:
        kernels[name]["algorithmic_bytes_per_launch"] = algorithmic_bytes(name, info)

    # ---- (last of the device work, so that nothing else depends on it)
    # ---- ONE replay partitioned by sample-ID range, timed like the
    #      headline (init_cache + the full replay, L2 flushed, one warm-up) and gated
    #      by the golden digests on every shard.  N = 1: G shards emulated on this
    #      device (one launch of G x (J + 1) CTAs exchanging through device
    #      mailboxes); N > 1: rank r is shard r of one replay (mailboxes mapped into
    #      every rank over NVLink by CUDA IPC, the kernels store into their peers'),
    #      strong scaling of one replay -- reported beside the headline.
    sharded = None
    shard_counts = ([int(x) for x in args.shards.split(",") if x] if world == 1 else
                    ([] if args.no_shard_replay else [world]))
    if shard_counts:
        import paper_2511_13724_b200 as P
        us1 = 1e6 * (sum(ods_ms) / 1e3) / rounds_tot            # the unsharded headline, this rank
        sharded = dict(mode="emulated on one device" if world == 1 else "one shard per GPU (CUDA IPC mailboxes)",
                       workload=args.workload, unsharded_us_per_round=us1, runs=[],
                       note="exchange_us_per_round = us_per_round - unsharded_us_per_round: the cost of the two "
                            "per-round exchanges (pool sizes, resolved ids) and the replicated work, DESIGN.md 8")
        c_sh = synth.ods_config(args.workload, seed=synth.PERF_SEED)
        for G in shard_counts:
            try:
                ms_g, rr_g, gate = [], 0, "bit-exact"
                for s_ in range(2):
                    l2_flush(s_ & 0xFF)
                    barrier()
                    torch.cuda.synchronize(dev)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    kw = dict(shards=G) if world == 1 else dict(shards=G, shard_rank=rank, shard_mode=1)
                    if world > 1:
                        gsh = P.ODSContext(c_sh["n_total"], c_sh["batch"], c_sh["target"], ce, cd, ca, c_sh["seed"],
                                           evict_tiers=args.evict_tiers, stream=stream, **kw)
                        D.attach_shard_peers(gsh)
                        torch.cuda.synchronize(dev)
                        barrier()
                        e0.record(stream)
                    else:
                        e0.record(stream)
                        gsh = P.ODSContext(c_sh["n_total"], c_sh["batch"], c_sh["target"], ce, cd, ca, c_sh["seed"],
                                           evict_tiers=args.evict_tiers, stream=stream, **kw)
                    rr_g = gsh.replay_epochs(max(c_sh["target"]))
                    e1.record(stream)
                    torch.cuda.synchronize(dev)
                    barrier()
                    if s_ == 1:
                        ms_g.append(e0.elapsed_time(e1))
                        gsh.sync()
                        for k in range(gsh.R):
                            stk, evk, rfk = gsh.stats(k)
                            gk = golden_gate(args.workload, c_sh["seed"], args.evict_tiers, stk, evk, rfk)
                            if gk != "bit-exact":
                                gate = f"shard {k}: {gk}"
                    gsh.close()
                (t_g,) = D.reduce_times([sum(ms_g) / 1e3], device=red_dev)
                sharded["runs"].append(dict(shards=G, ms=1e3 * t_g, rounds=rr_g,
                                            us_per_round=1e6 * t_g / rr_g,
                                            exchange_us_per_round=1e6 * t_g / rr_g - us1,
                                            value=dec_per_step / t_g, unit="decisions/s (one replay)",
                                            parity=gate))
            except Exception as ex:  # report; the headline stands
                sharded["runs"].append(dict(shards=G, error=f"{type(ex).__name__}: {ex}"[:300]))

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, synth.ods_config(args.workload, seed=synth.PERF_SEED),
                           oracle_caps(synth.ods_config(args.workload, seed=synth.PERF_SEED)))
    if rank == 0:
        ms_per_step = 1e3 * (ods_s + mdp_s) / args.steps
        line = dict(
            metric=METRIC, value=total_dec / ods_s, unit="decisions/s", n_gpus=world, steps=args.steps,
            warmup=args.warmup, ms_per_step=ms_per_step, higher_is_better=True, scaling="weak",
            vs_baseline=None, dtype="u32", data="synthetic",
            config=workload_config(c, args.workload, dict(
                rounds_per_step=rounds_tot // args.steps, decisions_per_step=dec_per_step,
                us_per_round=1e6 * ods_s / args.steps / (rounds_tot / args.steps),
                evict_tiers="all" if args.evict_tiers else "A",
                mdp_profiles=args.mdp_profiles, mdp_grid_step_pct=args.mdp_grid_step,
                mdp_grid_written=d_grid is not None,
                parallelism=f"{world} independent replays (seed+rank) + {world} independent MDP profile sets",
                l2="flushed between timed steps (512 MiB write, then a 256 MiB read-back so the flush's dirty lines leave L2 before the timed region)")),
            e2e=dict(value=total_dec / e2e_s, unit="decisions/s",
                     h2d_bytes_per_step=int(pin_prof.numel()), d2h_bytes_per_step=int(nst + pin_res.numel()),
                     mdp_value=total_evals / e2e_m, mdp_unit="split-evals/s",
                     note="public API from Python: init_cache + replay_epochs + stats D2H; MDP profiles "
                          "H2D from pinned memory + sweep + results D2H; host wall clock"),
            roofline=roof,
            pass_equivalent=dict(pass_equivalent(c, caps, v.words, ods_s, args.steps, world, hbm_peak, rep_line),
                                 caveat="NOT a roofline: bytes a pass-based design would stream, which this "
                                        "kernel never moves; see roofline (own bytes) and roofline.latency"),
            workloads=extra,
            mdp=dict(value=total_evals / mdp_s, unit="split-evals/s", dtype="f64", ms_per_step=mdp_ms_step,
                     roofline=mdp_roof, large=mdp_large,
                     fp64=dict(flops_per_split=11, achieved_tflops=total_evals * 11 / mdp_s / 1e12,
                               peak_tflops=FP64_PEAK_TFLOPS, frac=total_evals * 11 / mdp_s / 1e12 / FP64_PEAK_TFLOPS,
                               note="SURVEY 8(d): Eq. 9 is 4 div + 4 mul + 3 add per split (a division counted "
                                    "once; hardware expands it to ~9-10 FP64-pipe instructions); peak = 148 SMs x "
                                    "64 FP64 FMA/clk x 2 x 1.965 GHz, nominal (MEASURED_PEAKS.json has no FP64 "
                                    "figure); the kernel is issue-bound, DESIGN.md 7.3")),
            replicas=rep_line,
            sharded=sharded,
            cpu_baseline=cpu,
            clocks=clk,
            gpu_launches=int(launches),
            kernels=kernels,
            ods_round_phase_share=phase_share,
            parity=parity,
            so_loaded=repo_so_loaded(),
        )
        print(json.dumps(line), flush=True)
    S.destroy(last_ctx)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
