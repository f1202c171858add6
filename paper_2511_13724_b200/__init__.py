"""paper_2511_13724_b200 -- Seneca's hot path (ODS replay + MDP sweep) on B200.

The compute lives in libseneca.so (CUDA, sm_100a; C-ABI in include/seneca.h).
``seneca`` is the ctypes binding with the C names; the helpers below only own
device memory (torch tensors) and read results back.  No CPU fallback exists.
"""
from __future__ import annotations

import numpy as np

from . import seneca
from .seneca import (PROFILE_DTYPE, RESULT_DTYPE, STATS_DTYPE, SenecaError, mdp_num_splits,
                     metadata_bytes, split_capacities)

__all__ = ["seneca", "ODSContext", "mdp_sweep_device", "SenecaError", "PROFILE_DTYPE",
           "RESULT_DTYPE", "STATS_DTYPE", "split_capacities", "metadata_bytes", "mdp_num_splits"]


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2511_13724_b200 needs a CUDA device (there is no CPU fallback)")
    return torch


def mdp_sweep_device(profiles: np.ndarray, grid_step_pct: int = 1, want_grid: bool = False,
                     device="cuda", stream=None):
    """Copy PROFILE_DTYPE rows to the device, run seneca_mdp_sweep, return device tensors
    (results as uint8 bytes [n, 48], grid float64 [n, splits] or None)."""
    torch = _torch()
    n = len(profiles)
    d_prof = torch.from_numpy(np.ascontiguousarray(profiles).view(np.uint8)).to(device)
    d_res = torch.empty(n * RESULT_DTYPE.itemsize, dtype=torch.uint8, device=device)
    d_grid = (torch.empty((n, mdp_num_splits(grid_step_pct)), dtype=torch.float64, device=device)
              if want_grid else None)
    seneca.mdp_sweep(d_prof, n, grid_step_pct, d_res, d_grid, stream)
    return d_res, d_grid


def mdp_eval_device(profiles: np.ndarray, splits, want_counts: bool = False, device="cuda", stream=None):
    """DSI_overall of every profile at the given (p_e, p_d, p_a) splits on the
    device: (values float64 [n, s], counts uint64 [n, s, 4] or None, tier rows
    as RESULT_DTYPE bytes [n, 48])."""
    torch = _torch()
    n, ns = len(profiles), len(splits)
    d_prof = torch.from_numpy(np.ascontiguousarray(profiles).view(np.uint8)).to(device)
    d_val = torch.empty((n, ns), dtype=torch.float64, device=device)
    d_cnt = torch.empty((n, ns, 4), dtype=torch.int64, device=device) if want_counts else None
    d_tiers = torch.empty(n * RESULT_DTYPE.itemsize, dtype=torch.uint8, device=device)
    seneca.mdp_eval(d_prof, n, splits, d_val, d_cnt, d_tiers, stream)
    return d_val, d_cnt, d_tiers


def results_to_numpy(d_res) -> np.ndarray:
    return d_res.cpu().numpy().view(RESULT_DTYPE)


class ODSContext:
    """A torch-owned workspace + a libseneca context: `replicas` independent
    replay instances (replica k uses seed + k), played by the same launches.
    Readback methods take the replica index (default 0)."""

    def __init__(self, n_total, batch, target, cap_e, cap_d, cap_a, seed, request_mode=0,
                 device="cuda", stream=None, replicas=1, evict_tiers=0, sampler=0, arrival=None, cold_start=0,
                 shards=1, shard_rank=0, shard_mode=0):
        """shards > 1: ONE replay partitioned by sample-ID range; with
        shard_mode 0 all shards run in this context (slice k = shard k, each with
        the replicated state; readback index = shard)."""
        torch = _torch()
        self.torch = torch
        self.cfg = seneca.make_config(int(n_total), list(batch), list(target), int(cap_e), int(cap_d),
                                      int(cap_a), int(seed), request_mode, int(replicas), int(evict_tiers),
                                      int(sampler), arrival, int(cold_start), int(shards), int(shard_rank),
                                      int(shard_mode))
        self.R = int(shards) if int(shards) > 1 and int(shard_mode) == 0 else int(replicas)
        self.N, self.J = int(n_total), len(batch)
        self.bmax = max(batch)
        self.max_target = max(target)
        self.nbytes = seneca.state_bytes(self.cfg)
        self.ws = torch.empty(self.nbytes, dtype=torch.uint8, device=device)
        self.device = device
        self.stream = stream
        self.ctx = seneca.init_cache(self.cfg, self.ws, self.nbytes, stream)

    def close(self):
        if getattr(self, "ctx", None):
            seneca.destroy(self.ctx)
            self.ctx = None

    __del__ = close

    # -- driving
    def replay_epochs(self, n_epochs, transcript=None):
        return seneca.replay_epochs(self.ctx, n_epochs, transcript, self.stream)

    def replay_rounds(self, n_rounds, transcript=None):
        return seneca.replay_rounds(self.ctx, n_rounds, transcript, self.stream)

    def new_transcript(self):
        """[J][max_target][N] (one replica) or [R][J][max_target][N] int64 zeros."""
        shape = (self.J, self.max_target, self.N) if self.R == 1 else (self.R, self.J, self.max_target, self.N)
        return self.torch.zeros(shape, dtype=self.torch.int64, device=self.device)

    def next_batch(self, jobs, requested=None):
        """One round; ids/src are [n][Bmax] (one replica) or [R][n][Bmax]."""
        torch = self.torch
        n = len(jobs)
        shape = (n, self.bmax) if self.R == 1 else (self.R, n, self.bmax)
        ids = torch.zeros(shape, dtype=torch.int32, device=self.device)
        src = torch.zeros(shape, dtype=torch.uint8, device=self.device)
        req = None
        if requested is not None:
            r = np.zeros((n, self.bmax), np.uint32)
            for x, row in enumerate(requested):
                r[x, :len(row)] = row
            req = torch.from_numpy(r.view(np.int32)).to(self.device)
        lens = seneca.ods_next_batch(self.ctx, jobs, req, ids, src, self.stream)
        return ids, src, lens

    def sync(self):
        seneca.sync_status(self.ctx, self.stream)

    def launches(self):
        return seneca.launch_count(self.ctx)

    def profile(self, flags: int = 3):
        """bit 0: event-timed launches; bit 1: in-kernel phase counters."""
        seneca.profile(self.ctx, flags)

    def phase_cycles(self, k=0):
        v = self.view()
        return self._slice(self._rep(v, v.d_phase_cycles, k), 256).cpu().numpy().view(np.uint64).copy()

    def profile_read(self) -> dict:
        return seneca.profile_read(self.ctx)

    # -- readback
    def _slice(self, ptr, nbytes):
        off = ptr - self.ws.data_ptr()
        return self.ws[off:off + nbytes]

    def view(self):
        return seneca.read_state(self.ctx)

    @staticmethod
    def _rep(v, ptr, k):
        if not 0 <= k < v.replicas:
            raise IndexError(f"replica {k} of {v.replicas}")
        return ptr + k * v.replica_stride

    def state(self, k=0):
        """Replica k: (tier codes uint8[N], seen uint8[J][N], cons uint8[J][N]) as numpy."""
        v = self.view()
        W = v.words

        def bits(ptr, rows):
            ptr = self._rep(v, ptr, k)
            raw = self._slice(ptr, rows * W * 4).cpu().numpy().view(np.uint32).reshape(rows, W)
            b = np.unpackbits(raw.view(np.uint8).reshape(rows, W * 4), axis=1, bitorder="little")
            return b[:, :self.N]

        e, d, a = bits(v.d_tier_e, 1)[0], bits(v.d_tier_d, 1)[0], bits(v.d_tier_a, 1)[0]
        tier = np.zeros(self.N, np.uint8)
        tier[e == 1] = 1
        tier[d == 1] = 2
        tier[a == 1] = 3
        return tier, bits(v.d_seen, self.J), bits(v.d_cons, self.J)

    def epoch_model(self, dsi, k=0) -> np.ndarray:
        """Replica k's per job-epoch model metrics (NEXT-1) on the device:
        EPOCH_DTYPE [J][max_target]; dsi = (DSI_A, DSI_D, DSI_E, DSI_S)."""
        v = self.view()
        n = self.J * v.max_target
        out = self.torch.empty(n * seneca.EPOCH_DTYPE.itemsize, dtype=self.torch.uint8, device=self.device)
        seneca.epoch_model(self._rep(v, v.d_stats, k), n, self.N, dsi, out, self.stream)
        return out.cpu().numpy().view(seneca.EPOCH_DTYPE).reshape(self.J, v.max_target)

    def stats(self, k=0):
        """Replica k: (per job-epoch STATS_DTYPE [J][max_target], evicted, refilled)."""
        v = self.view()
        raw = self._slice(self._rep(v, v.d_stats, k), self.J * v.max_target * STATS_DTYPE.itemsize).cpu().numpy()
        st = raw.view(STATS_DTYPE).reshape(self.J, v.max_target)
        ev = int(self._slice(self._rep(v, v.d_evicted, k), 8).cpu().numpy().view(np.uint64)[0])
        rf = int(self._slice(self._rep(v, v.d_refilled, k), 8).cpu().numpy().view(np.uint64)[0])
        return st, ev, rf
