"""ctypes binding of libdooly_b200.so (include/dooly_b200.h).

The library is built in-tree (``make -C paper_2605_07985_b200/csrc``, or
``__graft_entry__.build()``).  There is no fallback: if the shared object is
missing or no CUDA device is present, every hot-path call raises.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

import torch

from .errors import DeviceError, raise_for_status

import os as _os

# DOOLY_LIB_PATH: load an alternative build (tuning experiments in tools/)
LIB_PATH = Path(_os.environ.get("DOOLY_LIB_PATH") or
                Path(__file__).resolve().parent / "_lib" / "libdooly_b200.so")

KIND_AFFINE = 0
KIND_ATTN = 1
KIND_ATTN_PACKED = 2   # predict-only 96-B rows (dooly_attn_pack), see include/dooly_b200.h
PACK_MAGIC = 0x66504144   # "DAPf": folded coefficients (include/dooly_b200.h)
FEAT_NUM_TOKS, FEAT_NUM_SEQS, FEAT_ATTN, FEAT_COMM = 0, 1, 2, 3
MAX_OPS = 64
IT_FEATS = 5
AFFINE_ROW_BYTES = 32
ATTN_ROW_BYTES = 128
ATTN96_ROW_BYTES = 96
ROW_BYTES = {KIND_AFFINE: AFFINE_ROW_BYTES, KIND_ATTN: ATTN_ROW_BYTES,
             KIND_ATTN_PACKED: ATTN96_ROW_BYTES}
PLANES = {KIND_AFFINE: 1, KIND_ATTN: 3, KIND_ATTN_PACKED: 3}


class OpList(C.Structure):
    _fields_ = [
        ("n_ops", C.c_int32),
        ("tp", C.c_int32),
        ("comm_alpha", C.c_double),
        ("comm_beta", C.c_double),
        ("feat", C.c_int32 * MAX_OPS),
        ("row", C.c_int32 * MAX_OPS),
        ("repeat", C.c_int32 * MAX_OPS),
        ("window_slot", C.c_int32 * MAX_OPS),
        ("bytes_per_tok", C.c_int64 * MAX_OPS),
    ]


SWEEP_MAX = 16
OP_CODES = {"reshape": 0, "linear": 1, "embedding": 2, "rms_norm": 3, "rotary_embedding": 4,
            "silu_and_mul": 5, "topk_softmax": 6, "fused_moe": 7, "attention": 8}


class SweepDesc(C.Structure):
    _fields_ = [
        ("op", C.c_int32),
        ("feature", C.c_int32),
        ("dim", C.c_int64 * 4),
        ("window", C.c_int32),
        ("dtype_bytes", C.c_int32),
        ("max_context", C.c_int64),
        ("mult", C.c_double * 2),
    ]


class SweepGrid(C.Structure):
    _fields_ = [
        ("n_tok", C.c_int32), ("n_req", C.c_int32), ("n_kv", C.c_int32), ("pad_", C.c_int32),
        ("chunk", C.c_int64), ("max_batch", C.c_int64),
        ("tok", C.c_uint32 * SWEEP_MAX), ("req", C.c_uint32 * SWEEP_MAX),
        ("kv", C.c_uint32 * SWEEP_MAX),
        ("peak_flops", C.c_double), ("mem_bw", C.c_double), ("overhead", C.c_double),
    ]


class Sched(C.Structure):
    _fields_ = [
        ("chunk", C.c_int32),
        ("max_batch", C.c_int32),
        ("window", C.c_int32),
        ("pad_", C.c_int32),
        ("kv_bytes_per_token", C.c_int64),
        ("kv_capacity_bytes", C.c_int64),
        ("max_iterations", C.c_int64),
    ]


MAX_PEERS = 7


class GridPeers(C.Structure):
    """dooly_grid_peers: the other ranks' buffers for dooly_fit_grid_bcast."""
    _fields_ = [
        ("n_peers", C.c_int32),
        ("pad_", C.c_int32),
        ("row0", C.c_int64),
        ("table", C.c_void_p * MAX_PEERS),
        ("fit_err", C.c_void_p * MAX_PEERS),
        ("status", C.c_void_p * MAX_PEERS),
        ("flag", C.c_void_p * MAX_PEERS),
    ]


class DigestPeers(C.Structure):
    """dooly_digest_peers: the other ranks' gathered digest arrays."""
    _fields_ = [
        ("n_peers", C.c_int32),
        ("pad_", C.c_int32),
        ("row0", C.c_int64),
        ("digest", C.c_void_p * MAX_PEERS),
        ("flag", C.c_void_p * MAX_PEERS),
    ]


_P = C.c_void_p
_I64 = C.c_int64
_SIGS = {
    "dooly_version": (C.c_int, []),
    "dooly_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "dooly_ctx_destroy": (None, [_P]),
    "dooly_last_error": (C.c_char_p, [_P]),
    "dooly_launch_count": (_I64, [_P]),
    "dooly_sha256_records": (C.c_int, [_P, _P, _P, _I64, _P, _P, _I64, _P, _P, _I64, _P, _I64,
                                       _P, _P]),
    "dooly_sha256_messages": (C.c_int, [_P, _P, _P, _I64, _P, _P]),
    "dooly_sha256_records_bcast": (C.c_int, [_P, _P, _P, _I64, _P, _P, _I64, _P, _P, _I64, _P,
                                             _I64, _P, C.POINTER(DigestPeers), _P, C.c_uint32, _P,
                                             _P]),
    "dooly_dedup_workspace_size": (C.c_size_t, [_I64, _I64]),
    "dooly_dedup_digests": (C.c_int, [_P, _P, _I64, _P, _I64, _P, _P, _P, _P, _P, _P,
                                      C.c_size_t, _P]),
    "dooly_fit_workspace_size": (C.c_size_t, [C.c_int, _I64]),
    "dooly_fit": (C.c_int, [_P, C.c_int, _P, _I64, _P, _P, _I64, _P, _P, _P, _P, C.c_size_t,
                            _P]),
    "dooly_predict": (C.c_int, [_P, C.c_int, _P, _I64, _P, _P, _I64, _P, _P, _P, _P]),
    "dooly_attn_pack_bytes": (C.c_size_t, [_I64]),
    "dooly_fit_grid_workspace_size": (C.c_size_t, [C.c_int, _I64]),
    "dooly_dedup": (C.c_int, [_P, _P, _P, _I64, _P, _P, _I64, _P, _P, _I64, _P, _I64, _P, _I64,
                              _P, _P, _P, _P, _P, _P, _P, C.c_size_t, _P]),
    "dooly_sim_eval": (C.c_int, [_P, C.POINTER(OpList), _P, _I64, _P, _I64, _P, _P, _P, _I64, _I64, _P, _P, _P,
                                 _P, _I64, _P, _P, _P, _P, _P, _P, _P]),
    "dooly_fit_grid": (C.c_int, [_P, C.c_int, _P, _I64, _P, _I64, _P, _P, _P, _P, C.c_size_t, _P]),
    "dooly_fit_grid_packed": (C.c_int, [_P, _P, _I64, _P, _I64, _P, _P, _P, _P, _P, C.c_size_t,
                                        _P]),
    "dooly_fit_grid_bcast": (C.c_int, [_P, C.c_int, _P, _I64, _P, _I64, _P, _P, _P,
                                       C.POINTER(GridPeers), _P, C.c_uint32, _P, _P, C.c_size_t,
                                       _P]),
    "dooly_attn_pack": (C.c_int, [_P, _P, _I64, _P, _P]),
    "dooly_iter_eval": (C.c_int, [_P, C.POINTER(OpList), _P, _I64, _P, _I64, _P, _I64, _P, _P,
                                  _P]),
    "dooly_profile_fit": (C.c_int, [_P, C.c_int, _P, _I64, C.POINTER(SweepGrid), _P, _P, _P, _P,
                                    _P, _P, _I64, _P]),
    "dooly_sim_workspace_size": (C.c_size_t, [C.POINTER(Sched), _I64, _I64]),
    "dooly_sim_run": (C.c_int, [_P, C.POINTER(OpList), C.POINTER(Sched), _P, _I64, _P, _I64,
                                _P, _P, _P, _P, _P, _I64, _P, _P, _P, _P, _P, _P, _P, _I64, _P,
                                C.c_size_t, _P]),
    "dooly_enable_peer_access": (C.c_int, [_P, C.c_int]),
    "dooly_route_workspace_size": (C.c_size_t, [_I64, C.c_int]),
    "dooly_route_plan": (C.c_int, [_P, _P, _I64, C.c_int, _I64, _P, _P, _P, _P, _P, C.c_size_t,
                                   _P]),
    "dooly_dedup_firsts": (C.c_int, [_P, _I64, _I64, _P, _P, _P, C.c_size_t, _P]),
    "dooly_route_reply": (C.c_int, [_P, _P, _P, _P, _P, _I64, _P, _I64, C.c_int, _P, _P]),
    "dooly_route_finish": (C.c_int, [_P, _P, _P, _I64, _P, _P, _P, _P, _P]),
    "dooly_comm_unique_id": (C.c_int, [_P]),
    "dooly_comm_init_rank": (C.c_int, [C.c_int, _P, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "dooly_comm_create": (C.c_int, [C.c_int, _P, C.POINTER(C.c_void_p)]),
    "dooly_comm_destroy": (None, [_P]),
    "dooly_comm_last_error": (C.c_char_p, [_P]),
    "dooly_comm_size": (C.c_int, [_P, _P, _P, _P]),
    "dooly_allgather": (C.c_int, [_P, _P, C.c_size_t, _P]),
    "dooly_alltoallv": (C.c_int, [_P, _P, _P, _P, _P, C.c_size_t, _P]),
}
EXPORTS = tuple(_SIGS)
COMM_ID_BYTES = 128

_lock = threading.Lock()
_lib = None
_tls = threading.local()


def load_library() -> C.CDLL:
    """Load and prototype the shared object (no CUDA device needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise DeviceError(
                    f"{LIB_PATH} is missing: build it with `make -C paper_2605_07985_b200/csrc` "
                    "(there is no CPU fallback)")
            lib = C.CDLL(str(LIB_PATH))
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
        return _lib


def ctx_for(device: torch.device) -> C.c_void_p:
    """This thread's dooly_ctx for ``device``, created on first use.

    A dooly_ctx is not thread-safe (include/dooly_b200.h) and ctypes releases
    the GIL during the call, so every host thread gets its own context."""
    if device.type != "cuda":
        raise DeviceError(f"libdooly_b200 runs on CUDA devices only (got {device})")
    idx = device.index if device.index is not None else torch.cuda.current_device()
    ctxs = getattr(_tls, "ctx", None)
    if ctxs is None:
        ctxs = _tls.ctx = {}
    if idx not in ctxs:
        lib = load_library()
        h = C.c_void_p()
        rc = lib.dooly_ctx_create(idx, C.byref(h))
        if rc != 0:
            raise DeviceError(f"dooly_ctx_create({idx}) failed with status {rc}")
        ctxs[idx] = h
    return ctxs[idx]


def check(rc: int, ctx) -> None:
    if rc:
        msg = load_library().dooly_last_error(ctx)
        raise_for_status(rc, msg.decode() if msg else f"status {rc}")


def check_comm(rc: int, comm) -> None:
    if rc:
        msg = load_library().dooly_comm_last_error(comm)
        raise_for_status(rc, msg.decode() if msg else f"status {rc}")


def launch_count(device: torch.device) -> int:
    return int(load_library().dooly_launch_count(ctx_for(device)))


def stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t) -> int:
    return 0 if t is None else t.data_ptr()
