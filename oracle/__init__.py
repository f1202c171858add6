"""oracle -- TEST INFRASTRUCTURE ONLY.

ctypes binding for ``oracle/oracle.c``: the plain single-threaded CPU
implementation of Seneca's hot path (arXiv 2511.13724) written from the paper.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this package.  It
imports nothing from ``paper_2511_13724_b200`` and the product imports nothing
from here.

The library is compiled on first use (or by ``__graft_entry__.build()``) with
``gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math`` so that its binary64
arithmetic rounds once per written operation, like the CUDA path's explicit
``__d*_rn`` intrinsics.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC"]


def build(force: bool = False) -> str:
    """Compile liboracle.so next to oracle.c (the checker, not the product)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _declare(_lib)
    return _lib


class Profile(C.Structure):
    """oracle_profile: one row of tab:model_vars."""
    _fields_ = [
        ("t_gpu", C.c_double), ("t_decode_augment", C.c_double), ("t_augment", C.c_double),
        ("b_nic", C.c_double), ("b_pcie", C.c_double), ("b_cache", C.c_double),
        ("b_storage", C.c_double), ("model_bytes", C.c_double),
        ("cache_bytes", C.c_uint64), ("n_total", C.c_uint64), ("s_data", C.c_uint64),
        ("m_num", C.c_uint32), ("m_den", C.c_uint32), ("nodes", C.c_uint32),
        ("gpus_per_node", C.c_uint32),
        ("nvlink_intra", C.c_uint8), ("nvlink_inter", C.c_uint8), ("comm_mapping", C.c_uint8),
        ("pad", C.c_uint8 * 5),
    ]


class Result(C.Structure):
    _fields_ = [
        ("p_e", C.c_uint8), ("p_d", C.c_uint8), ("p_a", C.c_uint8),
        ("lim_a", C.c_uint8), ("lim_d", C.c_uint8), ("lim_e", C.c_uint8), ("lim_s", C.c_uint8),
        ("pad", C.c_uint8),
        ("v", C.c_double), ("dsi_a", C.c_double), ("dsi_d", C.c_double),
        ("dsi_e", C.c_double), ("dsi_s", C.c_double),
    ]


class Stats(C.Structure):
    _fields_ = [("served", C.c_uint64 * 4), ("subst", C.c_uint64 * 4),
                ("req_hits", C.c_uint64 * 4), ("digest", C.c_uint64)]


STATS_DTYPE = np.dtype([("served", "<u8", 4), ("subst", "<u8", 4),
                        ("req_hits", "<u8", 4), ("digest", "<u8")])

PROFILE_FIELDS = [f for f, _ in Profile._fields_ if f != "pad"]


def _declare(L):
    u32p = np.ctypeslib.ndpointer(np.uint32, flags="C")
    u8p = np.ctypeslib.ndpointer(np.uint8, flags="C")
    u64p = np.ctypeslib.ndpointer(np.uint64, flags="C")
    L.oracle_philox4x32_10.argtypes = [u32p, u32p, u32p]
    L.oracle_splitmix64.argtypes = [C.c_uint64]; L.oracle_splitmix64.restype = C.c_uint64
    L.oracle_key.argtypes = [C.c_uint64] * 5; L.oracle_key.restype = C.c_uint64
    L.oracle_perm.argtypes = [C.c_uint64] * 3; L.oracle_perm.restype = C.c_uint64
    L.oracle_perm_block.argtypes = [C.c_uint64] * 4 + [u32p]; L.oracle_perm_block.restype = None
    L.oracle_comm_overhead.argtypes = [C.c_uint64, C.c_double]; L.oracle_comm_overhead.restype = C.c_double
    L.oracle_tiers.argtypes = [C.POINTER(Profile), C.POINTER(C.c_double), C.POINTER(C.c_uint8)]
    L.oracle_split_counts.argtypes = [C.POINTER(Profile), C.c_uint32, C.c_uint32, C.c_uint32, u64p]
    L.oracle_model_eval.argtypes = [C.POINTER(Profile), C.c_uint32, C.c_uint32, C.c_uint32,
                                    C.POINTER(Result), C.c_void_p]
    L.oracle_model_eval.restype = C.c_double
    L.oracle_num_splits.argtypes = [C.c_uint32]; L.oracle_num_splits.restype = C.c_uint64
    L.oracle_mdp_sweep.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p, C.c_void_p]
    L.oracle_mdp_sweep.restype = C.c_int
    L.oracle_metadata_bytes.argtypes = [C.c_uint64, C.c_uint32]; L.oracle_metadata_bytes.restype = C.c_uint64
    L.oracle_epoch_metrics.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.POINTER(C.c_double), C.c_void_p]
    L.oracle_epoch_metrics.restype = None
    L.oracle_ods_create.argtypes = [C.c_uint64, C.c_uint32, u32p, u32p, C.c_uint64, C.c_uint64,
                                    C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_int]
    L.oracle_ods_create.restype = C.c_void_p
    L.oracle_ods_set_arrivals.argtypes = [C.c_void_p, u32p]
    L.oracle_ods_set_arrivals.restype = None
    L.oracle_ods_set_cold.argtypes = [C.c_void_p]
    L.oracle_ods_set_cold.restype = None
    L.oracle_ods_destroy.argtypes = [C.c_void_p]
    L.oracle_ods_need.argtypes = [C.c_void_p, C.c_uint32]; L.oracle_ods_need.restype = C.c_uint64
    L.oracle_ods_round.argtypes = [C.c_void_p, u32p, C.c_uint32, C.c_void_p, C.c_uint32, u32p, u8p, u32p]
    L.oracle_ods_round.restype = C.c_int
    L.oracle_ods_replay_rounds.argtypes = [C.c_void_p, C.c_uint64]; L.oracle_ods_replay_rounds.restype = C.c_uint64
    L.oracle_ods_replay_epochs.argtypes = [C.c_void_p, C.c_uint32]; L.oracle_ods_replay_epochs.restype = C.c_uint64
    L.oracle_ods_round_index.argtypes = [C.c_void_p]; L.oracle_ods_round_index.restype = C.c_uint64
    L.oracle_ods_max_target.argtypes = [C.c_void_p]; L.oracle_ods_max_target.restype = C.c_uint32
    L.oracle_ods_job_state.argtypes = [C.c_void_p, u64p, u64p, u64p, np.ctypeslib.ndpointer(np.int32, flags="C")]
    L.oracle_ods_set_state.argtypes = [C.c_void_p, u8p, C.c_void_p, C.c_void_p]
    L.oracle_ods_read_state.argtypes = [C.c_void_p, u8p, C.c_void_p, C.c_void_p]
    L.oracle_ods_read_stats.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
    L.oracle_ods_read_transcript.argtypes = [C.c_void_p, u64p]; L.oracle_ods_read_transcript.restype = C.c_int


# --------------------------------------------------------------------------- PRNG
def philox4x32_10(ctr, key):
    out = np.zeros(4, np.uint32)
    lib().oracle_philox4x32_10(np.asarray(ctr, np.uint32), np.asarray(key, np.uint32), out)
    return out


def splitmix64(x: int) -> int:
    return lib().oracle_splitmix64(x)


def key(seed, purpose, a=0, b=0, c=0) -> int:
    return lib().oracle_key(seed, purpose, a, b, c)


def perm(K: int, n: int, x: int) -> int:
    return lib().oracle_perm(K, n, x)


def perm_block(K: int, n: int, x0: int = 0, count: int | None = None) -> np.ndarray:
    """[perm(K, n, x) for x in x0 .. x0 + count - 1] as uint32 (default: all of [0, n))."""
    count = n - x0 if count is None else count
    out = np.zeros(count, np.uint32)
    lib().oracle_perm_block(K, n, x0, count, out)
    return out


# --------------------------------------------------------------------------- MDP
def make_profile(**kw) -> Profile:
    p = Profile()
    for k, v in kw.items():
        setattr(p, k, v)
    return p


PROFILE_DTYPE = np.dtype(Profile)
RESULT_DTYPE = np.dtype(Result)


def profiles_from_columns(cols: dict) -> np.ndarray:
    """Pack a dict of equal-length columns (synth.mdp_profiles) into oracle_profile rows."""
    n = len(cols["t_gpu"])
    arr = np.zeros(n, PROFILE_DTYPE)
    for f in PROFILE_FIELDS:
        arr[f] = cols[f]
    return arr


def profile_row(arr: np.ndarray, i: int) -> Profile:
    return Profile.from_buffer_copy(arr[i:i + 1].tobytes())


def comm_overhead(participants: int, model_bytes: float) -> float:
    return lib().oracle_comm_overhead(participants, model_bytes)


def tiers(p: Profile):
    d = (C.c_double * 4)(); l = (C.c_uint8 * 4)()
    lib().oracle_tiers(C.byref(p), d, l)
    return list(d), list(l)


def split_counts(p: Profile, pe, pd, pa):
    out = np.zeros(4, np.uint64)
    lib().oracle_split_counts(C.byref(p), pe, pd, pa, out)
    return [int(x) for x in out]


def capacities(n_total, s_data, m_num, m_den, cache_bytes, pe, pd, pa):
    """(cap_E, cap_D, cap_A) of a split (Eqs. 5-7, exact floors R-M6),
    computed by the oracle's own split_counts: the capacities every oracle call
    site uses (never the product's)."""
    p = make_profile(t_gpu=1, t_decode_augment=1, t_augment=1, b_nic=1, b_pcie=1, b_cache=1, b_storage=1,
                     cache_bytes=int(cache_bytes), n_total=int(n_total), s_data=int(s_data),
                     m_num=int(m_num), m_den=int(m_den), nodes=1, gpus_per_node=1)
    na, nd, ne, _ = split_counts(p, int(pe), int(pd), int(pa))
    return ne, nd, na


def config_capacities(c: dict):
    """capacities() of a synth.ods_config workload description."""
    return capacities(c["n_total"], c["s_data"], c["m_num"], c["m_den"], c["cache_bytes"], *c["split"])


def model_eval(p: Profile, pe, pd, pa):
    r = Result(); cnt = np.zeros(4, np.uint64)
    v = lib().oracle_model_eval(C.byref(p), pe, pd, pa, C.byref(r), cnt.ctypes.data)
    return v, r, [int(x) for x in cnt]


def num_splits(g: int) -> int:
    return lib().oracle_num_splits(g)


def mdp_sweep(profiles: np.ndarray, g: int, want_grid: bool = False):
    """profiles: PROFILE_DTYPE array.  Returns (RESULT_DTYPE array, grid or None)."""
    profiles = np.ascontiguousarray(profiles, PROFILE_DTYPE)
    n = len(profiles)
    res = np.zeros(n, RESULT_DTYPE)
    grid = np.zeros((n, num_splits(g)), np.float64) if want_grid else None
    rc = lib().oracle_mdp_sweep(profiles.ctypes.data, n, g, res.ctypes.data,
                                grid.ctypes.data if grid is not None else None)
    if rc != 0:
        raise ValueError(f"oracle_mdp_sweep rc={rc}")
    return res, grid


EPOCH_DTYPE = np.dtype([("epoch_seconds", "<f8"), ("dsi_mix", "<f8"), ("decode_aug_ops", "<u8"),
                        ("aug_only_ops", "<u8"), ("hit_rate", "<f8")])


def epoch_metrics(stats: np.ndarray, n_total: int, dsi) -> np.ndarray:
    """Per job-epoch model metrics (NEXT-1) from oracle stats rows (any shape);
    dsi = (DSI_A, DSI_D, DSI_E, DSI_S)."""
    st = np.ascontiguousarray(stats).reshape(-1)
    out = np.zeros(len(st), EPOCH_DTYPE)
    d = (C.c_double * 4)(*[float(x) for x in dsi])
    lib().oracle_epoch_metrics(st.ctypes.data, len(st), int(n_total), d, out.ctypes.data)
    return out.reshape(stats.shape)


def metadata_bytes(n_total: int, n_jobs: int) -> int:
    return lib().oracle_metadata_bytes(n_total, n_jobs)


# --------------------------------------------------------------------------- ODS
class ODS:
    """One oracle replay instance (R-O1..R-O24 of DESIGN.md §3); evict_all selects
    evict_tiers = ALL (R-O21), baseline the uniform no-evict sampler (R-O22),
    arrival the job arrival rounds (R-O23), cold the cold start (R-O24)."""

    def __init__(self, n_total, batch, target, cap_e, cap_d, cap_a, seed, transcript=False, evict_all=False,
                 baseline=False, arrival=None, cold=False):
        self.N = int(n_total)
        self.batch = np.ascontiguousarray(batch, np.uint32)
        self.target = np.ascontiguousarray(target, np.uint32)
        self.J = len(self.batch)
        self.bmax = int(self.batch.max())
        self.h = lib().oracle_ods_create(self.N, self.J, self.batch, self.target,
                                         int(cap_e), int(cap_d), int(cap_a), int(seed), int(transcript),
                                         int(bool(evict_all)), int(bool(baseline)))
        if not self.h:
            raise ValueError("oracle_ods_create rejected the configuration")
        if cold:                                                    # R-O24
            lib().oracle_ods_set_cold(self.h)
        if arrival is not None:                                     # R-O23
            self._arrival = np.ascontiguousarray(arrival, np.uint32)
            lib().oracle_ods_set_arrivals(self.h, self._arrival)
        self.max_target = lib().oracle_ods_max_target(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().oracle_ods_destroy(self.h)
            self.h = None

    def need(self, j):
        return lib().oracle_ods_need(self.h, j)

    def round(self, jobs, requested=None):
        jobs = np.ascontiguousarray(jobs, np.uint32)
        n = len(jobs)
        ids = np.zeros((n, self.bmax), np.uint32)
        src = np.zeros((n, self.bmax), np.uint8)
        lens = np.zeros(n, np.uint32)
        req = None
        if requested is not None:
            req = np.zeros((n, self.bmax), np.uint32)
            for x, row in enumerate(requested):
                req[x, :len(row)] = row
        rc = lib().oracle_ods_round(self.h, jobs, n, req.ctypes.data if req is not None else None,
                                    self.bmax, ids, src, lens)
        return rc, ids, src, lens

    def replay_rounds(self, n):
        return lib().oracle_ods_replay_rounds(self.h, n)

    def replay_epochs(self, n):
        return lib().oracle_ods_replay_epochs(self.h, n)

    @property
    def r(self):
        return lib().oracle_ods_round_index(self.h)

    def job_state(self):
        c = np.zeros(self.J, np.uint64); e = np.zeros(self.J, np.uint64)
        n = np.zeros(self.J, np.uint64); a = np.zeros(self.J, np.int32)
        lib().oracle_ods_job_state(self.h, c, e, n, a)
        return c, e, n, a

    def set_state(self, tier, seen=None, cons=None):
        tier = np.ascontiguousarray(tier, np.uint8)
        s = None if seen is None else np.ascontiguousarray(seen, np.uint8)
        c = None if cons is None else np.ascontiguousarray(cons, np.uint8)
        lib().oracle_ods_set_state(self.h, tier, s.ctypes.data if s is not None else None,
                                   c.ctypes.data if c is not None else None)

    def state(self):
        tier = np.zeros(self.N, np.uint8)
        seen = np.zeros((self.J, self.N), np.uint8)
        cons = np.zeros((self.J, self.N), np.uint8)
        lib().oracle_ods_read_state(self.h, tier, seen.ctypes.data, cons.ctypes.data)
        return tier, seen, cons

    def stats(self):
        out = np.zeros((self.J, self.max_target), STATS_DTYPE)
        ev = C.c_uint64(); rf = C.c_uint64()
        lib().oracle_ods_read_stats(self.h, out.ctypes.data, C.byref(ev), C.byref(rf))
        return out, ev.value, rf.value

    def transcript(self):
        out = np.zeros((self.J, self.max_target, self.N), np.uint64)
        if not lib().oracle_ods_read_transcript(self.h, out):
            return None
        return out
