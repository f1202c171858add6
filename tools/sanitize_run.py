"""Small invocations of every libseneca kernel instantiation, for compute-sanitizer
(tests/test_gpu_sanitizers.py runs this under memcheck, racecheck, synccheck and
initcheck).  Each case is also checked against the oracle (counters bit-exact),
so a run that finishes with 0 sanitizer errors also produced correct results.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py [case ...]

Cases (the round-kernel instantiations chosen at init_cache):
  coupled       toy (A tier): 512-thread ods_rounds<., kCoupled>, maintain CTA, signals
  uncoupled     E/D only, batch 300: 512-thread uncoupled ods_rounds
  half          E/D only, batch 32: ods_rounds_half (256 threads, 1 CTA / SM)
  x2            64 toy replicas: ods_rounds_x2 (256 threads, 2 CTAs / SM)
  evict_all     toy with evict_tiers = ALL
  cold          toy cold start
  arrivals      toy with a late job (makespan trace)
  next_batch    generated requests, one round per launch, changing job subsets
  supplied      caller-supplied requests (ods_validate_requests)
  baseline      the uniform no-evict sampler
  ring          jobs at different epochs: launches bounded by the permutation ring
  mdp           mdp_sweep (grid written) + mdp_eval + epoch_model
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2511_13724_b200 as P  # noqa: E402
import synth  # noqa: E402


def replay(n, batch, target, ce, cd, ca, seed, R=1, **kw):
    okw = dict(evict_all=bool(kw.get("evict_tiers", 0)), baseline=bool(kw.get("sampler", 0)),
               arrival=kw.get("arrival"), cold=bool(kw.get("cold_start", 0)))
    g = P.ODSContext(n, batch, target, ce, cd, ca, seed, replicas=R, **kw)
    rounds = g.replay_epochs(max(target))
    torch.cuda.synchronize()
    g.sync()
    for k in sorted({0, R - 1}):
        o = O.ODS(n, batch, target, ce, cd, ca, seed + k, **okw)
        assert o.replay_epochs(max(target)) == rounds
        assert g.stats(k)[0].tobytes() == o.stats()[0].tobytes(), k
    g.close()


def case(name):
    toy = synth.ods_config("toy", seed=1)
    ce, cd, ca = O.config_capacities(toy)
    N, B, T = toy["n_total"], toy["batch"], toy["target"]
    if name == "coupled":
        replay(N, B, T, ce, cd, ca, 1)
    elif name == "uncoupled":
        replay(3000, [300, 300], [2, 2], 500, 400, 0, 2)
    elif name == "half":
        replay(N, B, T, 150, 100, 0, 3)
    elif name == "x2":
        replay(N, B, T, ce, cd, ca, 4, R=64)
    elif name == "evict_all":
        replay(N, B, T, ce, cd, ca, 5, evict_tiers=1)
    elif name == "cold":
        replay(N, B, T, ce, cd, ca, 6, cold_start=1)
    elif name == "arrivals":
        replay(N, B + [16], T + [2], ce, cd, ca, 7, arrival=[0, 0, 40])
    elif name == "baseline":
        replay(N, B, T, ce, cd, ca, 8, sampler=1)
    elif name == "ring":
        replay(997, [64, 300, 100], [5, 2, 3], 100, 80, 120, 9)
    elif name == "next_batch":
        o = O.ODS(N, B, T, ce, cd, ca, 10)
        g = P.ODSContext(N, B, T, ce, cd, ca, 10)
        for r in range(60):
            pick = [0, 1] if r % 3 else [r % 2]
            rc, ids_o, src_o, lens_o = o.round(pick)
            ids_g, src_g, lens_g = g.next_batch(pick)
            torch.cuda.synchronize()
            for x, L_ in enumerate(lens_g):
                assert np.array_equal(ids_g[x, :L_].cpu().numpy().view(np.uint32), ids_o[x, :L_])
        g.sync()
    elif name == "supplied":
        g = P.ODSContext(400, [12, 20], [2, 2], 40, 30, 50, 5, request_mode=1)
        g.next_batch([0, 1], requested=[list(range(12)), list(range(100, 120))])
        try:
            g.next_batch([0], requested=[[200] * 12])          # duplicates: EPROTO
            raise AssertionError("EPROTO expected")
        except P.SenecaError:
            pass
        torch.cuda.synchronize()
        unseen = [int(i) for i in np.flatnonzero(g.state()[1][1] == 0)[:20]]
        g.next_batch([1], requested=[unseen])
        torch.cuda.synchronize()
        g.sync()
    elif name == "mdp":
        cols = synth.mdp_profiles(96, seed=3)
        d_res, d_grid = P.mdp_sweep_device(P.seneca.profiles_from_columns(cols), 1, want_grid=True)
        torch.cuda.synchronize()
        ores, ogrid = O.mdp_sweep(O.profiles_from_columns(cols), 1, want_grid=True)
        assert np.array_equal(d_grid.cpu().numpy().view(np.uint64), ogrid.view(np.uint64))
        vals, cnt, _ = P.mdp_eval_device(P.seneca.profiles_from_columns(cols), [(100, 0, 0), (20, 30, 50)], True)
        g = P.ODSContext(N, B, T, ce, cd, ca, 11)
        g.replay_epochs(max(T))
        g.epoch_model((1.0, 2.0, 3.0, 4.0))
        torch.cuda.synchronize()
    else:
        raise KeyError(name)


ALL = ["coupled", "uncoupled", "half", "x2", "evict_all", "cold", "arrivals", "baseline", "ring", "next_batch",
       "supplied", "mdp"]

if __name__ == "__main__":
    for name in sys.argv[1:] or ALL:
        case(name)
        print(f"case {name} ok", flush=True)
