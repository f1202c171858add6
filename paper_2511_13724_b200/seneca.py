"""ctypes binding of libseneca.so (include/seneca.h) -- argument marshalling only.

Every function here forwards to the C-ABI with the same name (minus the
``seneca_`` prefix); device buffers are torch tensors (or raw device pointers)
and every step of the hot path runs in the library's CUDA kernels.  There is no
CPU fallback: if the extension is missing this module raises on import of the
library.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SENECA_LIB") or os.path.join(_HERE, "libseneca.so")   # override: experiments only

OK, EINVAL, ESTATE, EPROTO, ECUDA, ENOSPC = 0, 1, 2, 3, 4, 6
_NAMES = {0: "OK", 1: "EINVAL", 2: "ESTATE", 3: "EPROTO", 4: "ECUDA", 6: "ENOSPC"}


class SenecaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_NAMES.get(status, status)}: {msg}")
        self.status = status


class MdpProfile(C.Structure):
    _fields_ = [
        ("t_gpu", C.c_double), ("t_decode_augment", C.c_double), ("t_augment", C.c_double),
        ("b_nic", C.c_double), ("b_pcie", C.c_double), ("b_cache", C.c_double),
        ("b_storage", C.c_double), ("model_bytes", C.c_double),
        ("cache_bytes", C.c_uint64), ("n_total", C.c_uint64), ("s_data", C.c_uint64),
        ("m_num", C.c_uint32), ("m_den", C.c_uint32), ("nodes", C.c_uint32),
        ("gpus_per_node", C.c_uint32),
        ("nvlink_intra", C.c_uint8), ("nvlink_inter", C.c_uint8), ("comm_mapping", C.c_uint8),
        ("_pad", C.c_uint8 * 5),
    ]


class MdpResult(C.Structure):
    _fields_ = [
        ("p_e", C.c_uint8), ("p_d", C.c_uint8), ("p_a", C.c_uint8),
        ("lim_a", C.c_uint8), ("lim_d", C.c_uint8), ("lim_e", C.c_uint8), ("lim_s", C.c_uint8),
        ("status", C.c_uint8),
        ("v_best", C.c_double), ("dsi_a", C.c_double), ("dsi_d", C.c_double),
        ("dsi_e", C.c_double), ("dsi_s", C.c_double),
    ]


class Split(C.Structure):
    _fields_ = [("p_e", C.c_uint8), ("p_d", C.c_uint8), ("p_a", C.c_uint8), ("_pad", C.c_uint8)]


class CacheConfig(C.Structure):
    _fields_ = [
        ("n_total", C.c_uint64), ("n_jobs", C.c_uint32), ("request_mode", C.c_uint32),
        ("batch_size", C.POINTER(C.c_uint32)), ("target_epochs", C.POINTER(C.c_uint32)),
        ("cap_e", C.c_uint64), ("cap_d", C.c_uint64), ("cap_a", C.c_uint64), ("seed", C.c_uint64),
        ("replicas", C.c_uint32), ("evict_tiers", C.c_uint32), ("sampler", C.c_uint32), ("_pad0", C.c_uint32),
        ("arrival_round", C.POINTER(C.c_uint32)), ("cold_start", C.c_uint32), ("_pad1", C.c_uint32),
        ("shards", C.c_uint32), ("shard_rank", C.c_uint32), ("shard_mode", C.c_uint32), ("_pad2", C.c_uint32),
    ]


class JobEpochStats(C.Structure):
    _fields_ = [("served", C.c_uint64 * 4), ("subst", C.c_uint64 * 4),
                ("req_hits", C.c_uint64 * 4), ("digest", C.c_uint64)]


class StateView(C.Structure):
    _fields_ = [
        ("n_total", C.c_uint64), ("n_jobs", C.c_uint32), ("max_target", C.c_uint32),
        ("words", C.c_uint64),
        ("d_tier_e", C.c_void_p), ("d_tier_d", C.c_void_p), ("d_tier_a", C.c_void_p),
        ("d_seen", C.c_void_p), ("d_cons", C.c_void_p), ("d_stats", C.c_void_p),
        ("d_evicted", C.c_void_p), ("d_refilled", C.c_void_p), ("d_phase_cycles", C.c_void_p),
        ("round", C.c_uint64), ("epoch", C.c_uint64 * 32), ("consumed", C.c_uint64 * 32),
        ("active_mask", C.c_uint32), ("replicas", C.c_uint32), ("replica_stride", C.c_uint64),
    ]


class KernelStat(C.Structure):
    _fields_ = [("name", C.c_char_p), ("launches", C.c_uint64), ("sampled", C.c_uint64),
                ("sampled_ms", C.c_double)]


PROFILE_DTYPE = np.dtype(MdpProfile)
RESULT_DTYPE = np.dtype(MdpResult)
STATS_DTYPE = np.dtype(JobEpochStats)
assert PROFILE_DTYPE.itemsize == 112 and RESULT_DTYPE.itemsize == 48 and STATS_DTYPE.itemsize == 104

_lib = None


def lib() -> C.CDLL:
    """Load libseneca.so; raises if it has not been built (no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2511_13724_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, u32, u64 = C.c_void_p, C.c_uint32, C.c_uint64
        L.seneca_mdp_num_splits.argtypes = [u32]; L.seneca_mdp_num_splits.restype = u64
        L.seneca_mdp_sweep.argtypes = [vp, u32, u32, vp, vp, vp]; L.seneca_mdp_sweep.restype = C.c_int
        L.seneca_mdp_eval.argtypes = [vp, u32, C.POINTER(Split), u32, vp, vp, vp, vp]
        L.seneca_mdp_eval.restype = C.c_int
        L.seneca_epoch_model.argtypes = [vp, u32, u64, C.POINTER(C.c_double), vp, vp]
        L.seneca_epoch_model.restype = C.c_int
        L.seneca_split_capacities.argtypes = [u64, u64, u32, u32, u64, u32, u32, u32, C.POINTER(u64)]
        L.seneca_split_capacities.restype = C.c_int
        L.seneca_metadata_bytes.argtypes = [u64, u32]; L.seneca_metadata_bytes.restype = u64
        L.seneca_state_bytes.argtypes = [C.POINTER(CacheConfig), C.POINTER(C.c_size_t)]
        L.seneca_state_bytes.restype = C.c_int
        L.seneca_init_cache.argtypes = [C.POINTER(CacheConfig), vp, C.c_size_t, vp, C.POINTER(vp)]
        L.seneca_init_cache.restype = C.c_int
        L.seneca_ods_next_batch.argtypes = [vp, C.POINTER(u32), u32, vp, vp, vp, C.POINTER(u32), vp]
        L.seneca_ods_next_batch.restype = C.c_int
        L.seneca_replay_epochs.argtypes = [vp, u32, vp, C.POINTER(u64), vp]
        L.seneca_replay_epochs.restype = C.c_int
        L.seneca_replay_epoch.argtypes = [vp, u32, vp, C.POINTER(u64), vp]
        L.seneca_replay_epoch.restype = C.c_int
        L.seneca_replay_rounds.argtypes = [vp, u64, vp, C.POINTER(u64), vp]
        L.seneca_replay_rounds.restype = C.c_int
        L.seneca_read_state.argtypes = [vp, C.POINTER(StateView)]; L.seneca_read_state.restype = C.c_int
        L.seneca_sync_status.argtypes = [vp, vp]; L.seneca_sync_status.restype = C.c_int
        L.seneca_shard_mailbox.argtypes = [vp, C.POINTER(vp), C.POINTER(C.c_size_t)]
        L.seneca_shard_mailbox.restype = C.c_int
        L.seneca_shard_attach.argtypes = [vp, C.POINTER(vp)]; L.seneca_shard_attach.restype = C.c_int
        L.seneca_launch_count.argtypes = [vp]; L.seneca_launch_count.restype = u64
        L.seneca_profile.argtypes = [vp, u32]; L.seneca_profile.restype = C.c_int
        L.seneca_profile_read.argtypes = [vp, C.POINTER(KernelStat), u32, C.POINTER(u32)]
        L.seneca_profile_read.restype = C.c_int
        L.seneca_destroy.argtypes = [vp]; L.seneca_destroy.restype = None
        L.seneca_last_error.argtypes = []; L.seneca_last_error.restype = C.c_char_p
        _lib = L
    return _lib


EXPORTED = ["seneca_mdp_num_splits", "seneca_mdp_sweep", "seneca_mdp_eval", "seneca_epoch_model",
            "seneca_split_capacities",
            "seneca_metadata_bytes", "seneca_state_bytes", "seneca_init_cache",
            "seneca_ods_next_batch", "seneca_replay_epochs", "seneca_replay_epoch", "seneca_replay_rounds",
            "seneca_read_state", "seneca_sync_status", "seneca_launch_count", "seneca_destroy",
            "seneca_shard_mailbox", "seneca_shard_attach",
            "seneca_last_error", "seneca_profile", "seneca_profile_read"]


def _check(status: int):
    if status != OK:
        raise SenecaError(status, lib().seneca_last_error().decode())


def _ptr(x) -> int | None:
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()


def _stream(stream) -> int | None:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return stream if isinstance(stream, int) else stream.cuda_stream


# ------------------------------------------------------------------ MDP
def mdp_num_splits(grid_step_pct: int) -> int:
    return lib().seneca_mdp_num_splits(grid_step_pct)


def mdp_sweep(d_profiles, n_profiles: int, grid_step_pct: int, d_results, d_grid=None, stream=None):
    _check(lib().seneca_mdp_sweep(_ptr(d_profiles), n_profiles, grid_step_pct, _ptr(d_results),
                                  _ptr(d_grid), _stream(stream)))


def mdp_eval(d_profiles, n_profiles: int, splits, d_values, d_counts=None, d_tiers=None, stream=None):
    """splits: sequence of (p_e, p_d, p_a) integer percents summing to 100."""
    splits = list(splits)
    arr = (Split * len(splits))(*[Split(int(e), int(d), int(a), 0) for e, d, a in splits])
    _check(lib().seneca_mdp_eval(_ptr(d_profiles), n_profiles, arr, len(splits), _ptr(d_values), _ptr(d_counts),
                                 _ptr(d_tiers), _stream(stream)))


EPOCH_DTYPE = np.dtype([("epoch_seconds", "<f8"), ("dsi_mix", "<f8"), ("decode_aug_ops", "<u8"),
                        ("aug_only_ops", "<u8"), ("hit_rate", "<f8")])


class EpochMetrics(C.Structure):
    _fields_ = [("epoch_seconds", C.c_double), ("dsi_mix", C.c_double), ("decode_aug_ops", C.c_uint64),
                ("aug_only_ops", C.c_uint64), ("hit_rate", C.c_double)]


def epoch_model(d_stats, n_rows: int, n_total: int, dsi, d_out, stream=None):
    """dsi = (DSI_A, DSI_D, DSI_E, DSI_S); d_out: device [n_rows] EPOCH_DTYPE rows."""
    d = (C.c_double * 4)(*[float(x) for x in dsi])
    _check(lib().seneca_epoch_model(_ptr(d_stats), n_rows, n_total, d, _ptr(d_out), _stream(stream)))


def split_capacities(n_total, s_data, m_num, m_den, cache_bytes, p_e, p_d, p_a):
    caps = (C.c_uint64 * 4)()
    _check(lib().seneca_split_capacities(n_total, s_data, m_num, m_den, cache_bytes, p_e, p_d, p_a, caps))
    return [int(v) for v in caps]


def metadata_bytes(n_total: int, n_jobs: int) -> int:
    return lib().seneca_metadata_bytes(n_total, n_jobs)


def profiles_from_columns(cols: dict) -> np.ndarray:
    arr = np.zeros(len(cols["t_gpu"]), PROFILE_DTYPE)
    for name, _ in MdpProfile._fields_:
        if name != "_pad":
            arr[name] = cols[name]
    return arr


# ------------------------------------------------------------------ ODS
def make_config(n_total, batch, target, cap_e, cap_d, cap_a, seed, request_mode=0, replicas=1, evict_tiers=0,
                sampler=0, arrival=None, cold_start=0, shards=1, shard_rank=0, shard_mode=0):
    b = (C.c_uint32 * len(batch))(*batch)
    t = (C.c_uint32 * len(target))(*target)
    arr = (C.c_uint32 * len(batch))(*arrival) if arrival is not None else None
    cfg = CacheConfig(n_total=n_total, n_jobs=len(batch), request_mode=request_mode,
                      batch_size=b, target_epochs=t, cap_e=cap_e, cap_d=cap_d, cap_a=cap_a, seed=seed,
                      replicas=replicas, evict_tiers=evict_tiers, sampler=sampler,
                      arrival_round=C.cast(arr, C.POINTER(C.c_uint32)) if arr is not None else None,
                      cold_start=cold_start, shards=shards, shard_rank=shard_rank, shard_mode=shard_mode)
    cfg._keep = (b, t, arr)
    return cfg


def state_bytes(cfg: CacheConfig) -> int:
    n = C.c_size_t()
    _check(lib().seneca_state_bytes(C.byref(cfg), C.byref(n)))
    return n.value


def init_cache(cfg: CacheConfig, d_workspace, workspace_bytes: int, stream=None) -> int:
    h = C.c_void_p()
    _check(lib().seneca_init_cache(C.byref(cfg), _ptr(d_workspace), workspace_bytes, _stream(stream),
                                   C.byref(h)))
    return h.value


def ods_next_batch(ctx: int, jobs, d_requested, d_out_ids, d_out_src, stream=None):
    jobs = list(jobs)
    hj = (C.c_uint32 * len(jobs))(*jobs)
    lens = (C.c_uint32 * len(jobs))()
    _check(lib().seneca_ods_next_batch(ctx, hj, len(jobs), _ptr(d_requested), _ptr(d_out_ids),
                                       _ptr(d_out_src), lens, _stream(stream)))
    return list(lens)


def replay_epochs(ctx: int, n_epochs: int, d_transcript=None, stream=None) -> int:
    r = C.c_uint64()
    _check(lib().seneca_replay_epochs(ctx, n_epochs, _ptr(d_transcript), C.byref(r), _stream(stream)))
    return r.value


def replay_rounds(ctx: int, n_rounds: int, d_transcript=None, stream=None) -> int:
    r = C.c_uint64()
    _check(lib().seneca_replay_rounds(ctx, n_rounds, _ptr(d_transcript), C.byref(r), _stream(stream)))
    return r.value


def read_state(ctx: int) -> StateView:
    v = StateView()
    _check(lib().seneca_read_state(ctx, C.byref(v)))
    return v


def shard_mailbox(ctx: int):
    """(device pointer, bytes) of this shard's mailbox (shard_mode 1)."""
    p, n = C.c_void_p(), C.c_size_t()
    _check(lib().seneca_shard_mailbox(ctx, C.byref(p), C.byref(n)))
    return p.value, n.value


def shard_attach(ctx: int, peer_mailboxes):
    """peer_mailboxes: [shards] device pointers (None for this shard's own)."""
    arr = (C.c_void_p * len(peer_mailboxes))(*[p if p else None for p in peer_mailboxes])
    _check(lib().seneca_shard_attach(ctx, arr))


def sync_status(ctx: int, stream=None):
    _check(lib().seneca_sync_status(ctx, _stream(stream)))


def launch_count(ctx: int) -> int:
    return lib().seneca_launch_count(ctx)


def profile(ctx: int, enable: int):
    _check(lib().seneca_profile(ctx, enable))


def profile_read(ctx: int) -> dict:
    out = (KernelStat * 16)()
    n = C.c_uint32()
    _check(lib().seneca_profile_read(ctx, out, 16, C.byref(n)))
    return {out[k].name.decode(): dict(launches=out[k].launches, sampled=out[k].sampled,
                                       sampled_ms=out[k].sampled_ms) for k in range(min(n.value, 16))}


def destroy(ctx: int):
    lib().seneca_destroy(ctx)


def last_error() -> str:
    return lib().seneca_last_error().decode()
