"""Regression-backed serving simulation: the drop-in for the reference's
`dooly.sim` (module absent from pkg/src).

    fit(db)                 -> Regressors        K2
    predict(regs, sig, x)   -> seconds           K3
    iter_latency(batch, calltree, regs)          K4a
    run(workload, model, backend, hw, regs, sched) -> Metrics   K4b
    mape(pred, truth)                            (host utility)

Every scalar form is a one-element call of the batch form (``fit_tables``,
``predict_batch``, ``iter_latency_batch``, ``run_shards``), which launch the
sm_100a kernels of libdooly_b200 on the current stream.  There is no CPU
fallback: without the library or a CUDA device these raise.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from .errors import (InsufficientData, LengthMismatch, NonTermination, UnknownSignature,
                     ValidationError, ZeroTruth)
from .modelir import BackendSpec, HardwareSpec, ModelConfig, Request
from .profiler import LatencyDB, _device, DeviceRecords, hash_records
from .records import pack_entries, runnable_entries

NEED = {_lib.KIND_AFFINE: 4, _lib.KIND_ATTN: 11}          # max(4, p + 1), App. A.8
FEATURE_NAMES = {_lib.KIND_AFFINE: ("num_toks",),
                 _lib.KIND_ATTN: ("prefill_toks", "batch_size", "kv_tokens")}
AFFINE_ROW = np.dtype([("c", "<f8", 2), ("inv", "<f8", 1), ("lo", "<u4", 1), ("hi", "<u4", 1)])
ATTN_ROW = np.dtype([("c", "<f8", 10), ("inv", "<f8", 3), ("lo", "<u4", 3), ("hi", "<u4", 3)])
ROW_DTYPE = {_lib.KIND_AFFINE: AFFINE_ROW, _lib.KIND_ATTN: ATTN_ROW}
PERCENTILES = (25, 50, 75, 90, 95, 99)


# ------------------------------------------------------------------------ fit


@dataclass
class FitResult:
    kind: int
    table: torch.Tensor        # (n_sig, row_bytes) u8 on device
    fit_err: torch.Tensor      # (n_sig,) f64
    status: torch.Tensor       # (n_sig,) u8 (0 ok, 1 insufficient)

    def rows(self) -> np.ndarray:
        return self.table.cpu().numpy().view(ROW_DTYPE[self.kind]).reshape(-1)


_FIT_WS: dict = {}


def _ws_key(device, tag) -> tuple:
    """Scratch is cached per (device, stream, use): fits enqueued on different
    streams may run concurrently and must not share a workspace."""
    return (str(device), torch.cuda.current_stream(device).cuda_stream, tag)


def _fit_workspace(kind: int, n_sig: int, device) -> torch.Tensor:
    """Cached device scratch for the attention fit's moment buffers."""
    need = int(_lib.load_library().dooly_fit_workspace_size(kind, n_sig))
    key = _ws_key(device, kind)
    buf = _FIT_WS.get(key)
    if buf is None or buf.numel() < need:
        buf = torch.empty(max(need, 256), dtype=torch.uint8, device=device)
        _FIT_WS[key] = buf
    return buf


def fit_tables(kind: int, x: torch.Tensor, y: torch.Tensor, pt_off: torch.Tensor,
               out: Optional[FitResult] = None, fused: bool = False) -> FitResult:
    """Batch fit (K2) of n_sig signatures whose points are CSR-ranged by pt_off.

    x: (P, n_pts) int32/uint32 device tensor (P = 1 affine, 3 attention),
    y: (n_pts,) f64, pt_off: (n_sig + 1,) i64.  Asynchronous; no exceptions
    for per-signature shortfalls (see ``status``).  ``fused`` forces the
    single-kernel attention path (no workspace)."""
    dev = y.device
    n_sig = pt_off.numel() - 1
    n_pts = y.numel()
    if x.shape != (_lib.PLANES[kind], n_pts):
        raise ValueError(f"x must have shape ({_lib.PLANES[kind]}, {n_pts}), got {tuple(x.shape)}")
    if out is None:
        out = FitResult(kind, torch.empty((n_sig, _lib.ROW_BYTES[kind]), dtype=torch.uint8,
                                          device=dev),
                        torch.empty(n_sig, dtype=torch.float64, device=dev),
                        torch.empty(n_sig, dtype=torch.uint8, device=dev))
    ws = None if (fused or kind == _lib.KIND_AFFINE) else _fit_workspace(kind, n_sig, dev)
    ctx = _lib.ctx_for(dev)
    _lib.check(_lib.load_library().dooly_fit(
        ctx, kind, x.data_ptr(), n_pts, y.data_ptr(), pt_off.data_ptr(), n_sig,
        out.table.data_ptr(), out.fit_err.data_ptr(), out.status.data_ptr(),
        _lib.ptr(ws), 0 if ws is None else ws.numel(), _lib.stream_ptr(dev)), ctx)
    return out


@dataclass
class Regressor:
    """Host view of one fitted regressor."""

    signature_hash: bytes
    feature_names: tuple
    coefficients: tuple          # scaled basis
    inv_scale: tuple
    box: tuple                   # ((lo, hi), ...) training box
    fit_error: float


@dataclass
class Regressors:
    """All fitted signatures: one device table per regression kind plus the
    digest -> (kind, row) index."""

    tables: dict                  # kind -> FitResult
    index: dict                   # digest -> (kind, row)
    device: torch.device

    def n(self, kind: int) -> int:
        fr = self.tables.get(kind)
        return 0 if fr is None else fr.table.shape[0]

    def table_ptr(self, kind: int) -> int:
        fr = self.tables.get(kind)
        return 0 if fr is None or fr.table.numel() == 0 else fr.table.data_ptr()

    def regressor(self, digest: bytes) -> Regressor:
        if digest not in self.index:
            raise UnknownSignature(digest.hex())
        kind, row = self.index[digest]
        # one row crosses the link, not the table
        r = self.tables[kind].table[row].cpu().numpy().view(ROW_DTYPE[kind])[0]
        return Regressor(digest, FEATURE_NAMES[kind], tuple(np.atleast_1d(r["c"]).tolist()),
                         tuple(np.atleast_1d(r["inv"]).tolist()),
                         tuple(zip(np.atleast_1d(r["lo"]).tolist(), np.atleast_1d(r["hi"]).tolist())),
                         float(self.tables[kind].fit_err[row].item()))

    def __contains__(self, digest: bytes) -> bool:
        return digest in self.index


def _csr(items: Sequence, planes: int):
    """[(x (P, n_i), y (n_i,))] -> (x (P, N) u32, y (N,), off (n+1,))."""
    off = np.zeros(len(items) + 1, dtype=np.int64)
    if items:
        off[1:] = np.cumsum([it[1].shape[0] for it in items])
    x = np.zeros((planes, int(off[-1])), dtype=np.uint32)
    y = np.zeros(int(off[-1]), dtype=np.float64)
    for i, (xi, yi) in enumerate(items):
        x[:, off[i]:off[i + 1]] = np.asarray(xi, dtype=np.uint32).reshape(planes, -1)
        y[off[i]:off[i + 1]] = yi
    return x, y, off


GRID_GROUP_MIN = 8   # signatures sharing one sweep grid before fit() takes the grid path


def _grid_groups(items: Sequence, planes: int):
    """Partition signatures by their exact training points: {x bytes: [i, ...]}."""
    groups: dict = {}
    for i, (x, _) in enumerate(items):
        xa = np.ascontiguousarray(np.asarray(x, dtype=np.uint32).reshape(planes, -1))
        groups.setdefault(xa.tobytes(), []).append(i)
    return groups


def fit(db: LatencyDB, device=None, strict: bool = True) -> Regressors:
    """One least-squares regressor per measured signature.

    Signatures swept over the same points (one sweep grid per model/backend,
    SPEC.md:466-474) are fitted together by the shared-grid kernel
    (``fit_grid``: the Gram and its factor once per group); the rest go through
    the per-signature CSR kernel (``fit_tables``).  Both meet the same result
    contract, so the grouping is invisible to callers.

    Raises InsufficientData(signature, have, need) for the first signature with
    fewer than max(4, p + 1) measurements (App. A.8) when ``strict``."""
    dev = _device(device)
    tables, index = {}, {}
    for kind in (_lib.KIND_AFFINE, _lib.KIND_ATTN):
        sigs = [s for s in db.signatures if s.kind == kind and s.digest in db.measurements]
        items = [db.measurements[s.digest] for s in sigs]
        if strict:
            for s, (_, y) in zip(sigs, items):
                if y.shape[0] < NEED[kind]:
                    raise InsufficientData(s.digest.hex(), int(y.shape[0]), NEED[kind])
        planes = _lib.PLANES[kind]
        grids = [g for g in _grid_groups(items, planes).values() if len(g) >= GRID_GROUP_MIN]
        in_grid = {i for g in grids for i in g}
        rest = [i for i in range(len(items)) if i not in in_grid]
        order = [i for g in grids for i in g] + rest
        n = len(order)
        fr = FitResult(kind, torch.empty((n, _lib.ROW_BYTES[kind]), dtype=torch.uint8, device=dev),
                       torch.empty(n, dtype=torch.float64, device=dev),
                       torch.empty(n, dtype=torch.uint8, device=dev))
        r0 = 0
        for g in grids:
            xg = np.asarray(items[g[0]][0], dtype=np.uint32).reshape(planes, -1)
            yg = np.stack([np.asarray(items[i][1], dtype=np.float64) for i in g])
            r1 = r0 + len(g)
            fit_grid(kind, torch.from_numpy(np.ascontiguousarray(xg).view(np.int32)).to(dev),
                     torch.from_numpy(yg).to(dev),
                     FitResult(kind, fr.table[r0:r1], fr.fit_err[r0:r1], fr.status[r0:r1]))
            r0 = r1
        if rest:
            x, y, off = _csr([items[i] for i in rest], planes)
            fit_tables(kind, torch.from_numpy(x.view(np.int32)).to(dev),
                       torch.from_numpy(y).to(dev), torch.from_numpy(off).to(dev),
                       FitResult(kind, fr.table[r0:], fr.fit_err[r0:], fr.status[r0:]))
        tables[kind] = fr
        for row, i in enumerate(order):
            index[sigs[i].digest] = (kind, row)
    torch.cuda.synchronize(dev)
    return Regressors(tables, index, dev)


def fit_cached(db: LatencyDB, db_path, device=None, strict: bool = True) -> Regressors:
    """cmd_simulate's lazy fit ("fit runs lazily and caches
    regressors alongside the db"): reuse the regressor file beside ``db_path``
    when every measured signature's fingerprint still matches its
    measurements, else fit on the GPU and rewrite the file."""
    from .store import load_regressors, save_regressors

    regs = load_regressors(db_path, db, device)
    if regs is not None:
        return regs
    regs = fit(db, device, strict)
    save_regressors(db_path, regs, db)
    return regs


# -------------------------------------------------------------------- predict


def fit_grid(kind: int, x: torch.Tensor, y: torch.Tensor,
             out: Optional[FitResult] = None, packed: Optional[torch.Tensor] = None) -> FitResult:
    """Shared-grid batch fit (dooly_fit_grid): every signature was swept over the
    same points.  x: (P, n_pts) int32/uint32 device tensor, y: (n_sig, n_pts) f64.
    Same result contract as ``fit_tables`` with x repeated per signature; the
    Gram matrix and its factor are built once for the whole batch.

    ``packed`` (attention only; (n_sig + 1, 96) u8): the fit epilogue also
    writes the 96-B serving table, byte-identical to ``pack_attn(table)``
    (dooly_fit_grid_packed)."""
    dev = y.device
    if y.dim() != 2:
        raise ValueError("y must be (n_sig, n_pts)")
    n_sig, n_pts = y.shape
    if x.shape != (_lib.PLANES[kind], n_pts):
        raise ValueError(f"x must have shape ({_lib.PLANES[kind]}, {n_pts}), got {tuple(x.shape)}")
    x, y = x.contiguous(), y.contiguous()
    if out is None:
        out = FitResult(kind, torch.empty((n_sig, _lib.ROW_BYTES[kind]), dtype=torch.uint8,
                                          device=dev),
                        torch.empty(n_sig, dtype=torch.float64, device=dev),
                        torch.empty(n_sig, dtype=torch.uint8, device=dev))
    lib = _lib.load_library()
    ws = _grid_workspace(dev, kind, n_pts)
    ctx = _lib.ctx_for(dev)
    if packed is not None:
        if kind != _lib.KIND_ATTN or packed.shape != (n_sig + 1, 96) or \
                packed.dtype != torch.uint8 or not packed.is_contiguous():
            raise ValueError("packed must be a contiguous (n_sig + 1, 96) uint8 tensor "
                             "(attention kind)")
        _lib.check(lib.dooly_fit_grid_packed(
            ctx, x.data_ptr() if x.numel() else 0, n_pts, y.data_ptr() if y.numel() else 0,
            n_sig, out.table.data_ptr() if n_sig else 0, out.fit_err.data_ptr() if n_sig else 0,
            out.status.data_ptr() if n_sig else 0, packed.data_ptr(), ws.data_ptr(), ws.numel(),
            _lib.stream_ptr(dev)), ctx)
        return out
    _lib.check(lib.dooly_fit_grid(
        ctx, kind, x.data_ptr() if x.numel() else 0, n_pts, y.data_ptr() if y.numel() else 0,
        n_sig, out.table.data_ptr() if n_sig else 0, out.fit_err.data_ptr() if n_sig else 0,
        out.status.data_ptr() if n_sig else 0, ws.data_ptr(), ws.numel(), _lib.stream_ptr(dev)),
        ctx)
    return out


def _grid_workspace(dev: torch.device, kind: int, n_pts: int) -> torch.Tensor:
    need = int(_lib.load_library().dooly_fit_grid_workspace_size(kind, n_pts))
    key = _ws_key(dev, "grid")
    ws = _FIT_WS.get(key)
    if ws is None or ws.numel() < need:
        ws = torch.empty(max(need, 256), dtype=torch.uint8, device=dev)
        _FIT_WS[key] = ws
    return ws


PACK_HEADER = np.dtype([("magic", "<u4"), ("ok", "<u4"), ("width", "<u4", 3), ("max_hi", "<u4", 3),
                        ("bad_inv", "<u4"), ("pad_", "<u4"), ("n_sig", "<i8"),
                        ("reserved", "u1", 48)])


def pack_attn(table: torch.Tensor, out: Optional[torch.Tensor] = None,
              check: bool = True) -> torch.Tensor:
    """Attention table (n_sig, 128) u8 -> packed serving table (n_sig + 1, 96) u8
    (``KIND_ATTN_PACKED``: 3 sectors per row, coefficients folded into
    raw-feature space with the row's inv_scale = 1/hi, box bit-packed;
    include/dooly_b200.h).  Served by the cooperative 3-lanes-per-row kernel
    with the folded 3-way evaluation tree (oracle/sim.py predict_packed is its
    bit-exact CPU form; it differs from the 128-B row's evaluation by rounding
    only, <= 1e-12 relative in the tests).  ``check``
    syncs and raises ValueError when the table is not representable (box widths
    over 64 bits, or an inv_scale that is not 1/hi); unchecked, a bad header
    makes predict flag every query unknown."""
    if table.dim() != 2 or table.shape[1] != _lib.ATTN_ROW_BYTES:
        raise ValueError(f"expected an (n_sig, {_lib.ATTN_ROW_BYTES}) attention table")
    dev = table.device
    n_sig = table.shape[0]
    if out is None:
        out = torch.empty((n_sig + 1, _lib.ATTN96_ROW_BYTES), dtype=torch.uint8, device=dev)
    ctx = _lib.ctx_for(dev)
    _lib.check(_lib.load_library().dooly_attn_pack(
        ctx, table.data_ptr() if n_sig else 0, n_sig, out.data_ptr(), _lib.stream_ptr(dev)), ctx)
    if check:
        h = out[0].cpu().numpy().view(PACK_HEADER)[0]
        if int(h["ok"]) != 1:
            raise ValueError(f"attention table not packable: widths {list(h['width'])}, "
                             f"{int(h['bad_inv'])} rows with inv_scale != 1/hi")
    return out


def predict_batch(kind: int, table: torch.Tensor, sig: torch.Tensor, x: torch.Tensor,
                  out: Optional[torch.Tensor] = None, flags: Optional[torch.Tensor] = None,
                  err_first: Optional[torch.Tensor] = None, want_flags: bool = True):
    """K3 over n_q queries: sig (n_q,) i32 rows of ``table`` (n_sig, row_bytes) u8
    (or a ``pack_attn`` table for ``KIND_ATTN_PACKED``),
    x (P, n_q) i32/u32 features.  Returns (out f64 (n_q,), flag bits (2, ceil(n_q/32))
    i32 or None, err_first i64 (1,): INT64_MAX unless some query hit an unknown row)."""
    dev = sig.device
    n_q = sig.numel()
    n_sig = table.shape[0] - (1 if kind == _lib.KIND_ATTN_PACKED else 0)
    if out is None:
        out = torch.empty(n_q, dtype=torch.float64, device=dev)
    if flags is None and want_flags:
        flags = torch.empty((2, (n_q + 31) // 32), dtype=torch.int32, device=dev)
    if err_first is None:
        err_first = torch.full((1,), torch.iinfo(torch.int64).max, dtype=torch.int64, device=dev)
    ctx = _lib.ctx_for(dev)
    _lib.check(_lib.load_library().dooly_predict(
        ctx, kind, table.data_ptr() if table.numel() else 0, n_sig, sig.data_ptr(), x.data_ptr(),
        n_q, out.data_ptr(), _lib.ptr(flags), err_first.data_ptr(), _lib.stream_ptr(dev)), ctx)
    return out, flags, err_first


class Prediction(float):
    """A latency (seconds) that also carries the SPEC.md:569 flags."""

    def __new__(cls, value: float, extrapolated: bool = False, clamped: bool = False):
        obj = float.__new__(cls, value)
        obj.extrapolated = extrapolated
        obj.clamped = clamped
        return obj


def predict(regs: Regressors, signature_hash: bytes, features: Sequence[int]) -> Prediction:
    """Scalar predict: clamped at 1e-7 s, flags extrapolation."""
    if signature_hash not in regs.index:
        raise UnknownSignature(signature_hash.hex())
    kind, row = regs.index[signature_hash]
    feats = list(features)
    if len(feats) != _lib.PLANES[kind]:
        raise ValueError(f"expected {_lib.PLANES[kind]} features {FEATURE_NAMES[kind]}")
    dev = regs.device
    sig = torch.tensor([row], dtype=torch.int32, device=dev)
    x = torch.tensor(np.asarray(feats, dtype=np.uint32).view(np.int32).reshape(-1, 1), device=dev)
    out, flags, err = predict_batch(kind, regs.tables[kind].table, sig, x)
    if int(err.item()) != torch.iinfo(torch.int64).max:
        raise UnknownSignature(f"{signature_hash.hex()} has no fitted regressor")
    f = flags.cpu().numpy()
    return Prediction(float(out.item()), bool(f[0, 0] & 1), bool(f[1, 0] & 1))


# ---------------------------------------------------------------- call graph


@dataclass
class CallTree:
    """The op list the simulator walks per iteration."""

    entries: list                 # RunnableEntry, list order = evaluation order
    oplist: _lib.OpList
    window: int                   # sliding window of the windowed kv plane (0 = none)

    @property
    def n_ops(self) -> int:
        return int(self.oplist.n_ops)


def build_calltree(model: ModelConfig, backend: BackendSpec, regs: Regressors,
                   hw: Optional[HardwareSpec] = None, tp: int = 1,
                   entries: Optional[list] = None) -> CallTree:
    """Map a (model, backend, tp) runnable set onto regressor rows (digests are
    computed by the GPU hash kernel) and append the TP all-reduces: 2 per
    layer of num_toks * hidden * dtype bytes (App. A.16)."""
    entries = runnable_entries(model, backend, tp) if entries is None else list(entries)
    recs = DeviceRecords.from_packed(pack_entries(entries), regs.device)
    digs = hash_records(recs).cpu().numpy()
    ol = _lib.OpList()
    windows = {e.window for e in entries if e.feature == "attention" and e.window}
    if len(windows) > 1:
        raise ValidationError("model.layer_attention", "at most one sliding-window size supported")
    window = windows.pop() if windows else 0
    n = 0
    for i, e in enumerate(entries):
        d = bytes(digs[i])
        if d not in regs.index:
            raise UnknownSignature(f"{e.name} ({d.hex()[:12]}) has no fitted regressor; "
                                   "profile it first")
        kind, row = regs.index[d]
        ol.feat[n] = {"num_toks": _lib.FEAT_NUM_TOKS, "num_seqs": _lib.FEAT_NUM_SEQS,
                      "attention": _lib.FEAT_ATTN}[e.feature]
        ol.row[n] = row
        ol.repeat[n] = e.repeat_count
        ol.window_slot[n] = 1 if (e.feature == "attention" and e.window) else 0
        n += 1
    ol.tp = tp
    if tp > 1:
        if hw is None:
            raise ValueError("tp > 1 needs the hardware spec for comm_latency")
        ol.comm_alpha, ol.comm_beta = hw.comm_alpha, hw.comm_beta
        ol.feat[n] = _lib.FEAT_COMM
        ol.repeat[n] = 2 * model.num_layers
        ol.bytes_per_tok[n] = model.hidden_dim * model.dtype_bytes
        n += 1
    if n > _lib.MAX_OPS:
        raise ValidationError("calltree", f"{n} entries exceed {_lib.MAX_OPS}")
    ol.n_ops = n
    return CallTree(entries, ol, window)


@dataclass(frozen=True)
class IterationBatch:
    """Features of one scheduled iteration (App. A.6)."""

    num_toks: int
    prefill_toks: int
    batch_size: int
    kv_tokens: int
    kv_tokens_window: int = 0

    def as_row(self) -> list:
        return [self.num_toks, self.prefill_toks, self.batch_size, self.kv_tokens,
                self.kv_tokens_window]


def iter_latency_batch(features: torch.Tensor, calltree: CallTree, regs: Regressors,
                       out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """K4a: latency of n iterations; features (5, n) i32 device tensor."""
    dev = features.device
    n_it = features.shape[1]
    if out is None:
        out = torch.empty(n_it, dtype=torch.float64, device=dev)
    err = torch.full((1,), torch.iinfo(torch.int64).max, dtype=torch.int64, device=dev)
    ctx = _lib.ctx_for(dev)
    _lib.check(_lib.load_library().dooly_iter_eval(
        ctx, C.byref(calltree.oplist), regs.table_ptr(_lib.KIND_AFFINE), regs.n(_lib.KIND_AFFINE),
        regs.table_ptr(_lib.KIND_ATTN), regs.n(_lib.KIND_ATTN), features.data_ptr(), n_it,
        out.data_ptr(), err.data_ptr(), _lib.stream_ptr(dev)), ctx)
    return out


def iter_latency(batch: IterationBatch, calltree: CallTree, regs: Regressors) -> float:
    """Sum over the call graph of repeat x predict (+ comm) for one iteration."""
    f = torch.tensor(np.asarray(batch.as_row(), dtype=np.uint32).view(np.int32).reshape(5, 1),
                     device=regs.device)
    return float(iter_latency_batch(f, calltree, regs).item())


def sim_eval(calltree: CallTree, regs: Regressors, it_feat: torch.Tensor,
             arrival: torch.Tensor, first_it: torch.Tensor, last_it: torch.Tensor,
             out_tok: torch.Tensor, it_start: Optional[torch.Tensor] = None,
             it_off: Optional[torch.Tensor] = None):
    """Host-scheduled evaluation (dooly_sim_eval): an external scheduler's
    iterations (5, n_it) i32 -> (it_lat, clock, ttft, tpot) f64 device tensors.
    clock[i] = max(clock[i-1], it_start[i]) + it_lat[i] per shard (it_off), the
    event loop's clock bit for bit; first_it / last_it are the global iterations
    that produced a request's first / last token (-1 = never)."""
    dev = it_feat.device
    n_it = it_feat.shape[1]
    n_req = arrival.numel()
    n_shards = 0 if it_off is None else it_off.numel() - 1
    it_lat = torch.empty(n_it, dtype=torch.float64, device=dev)
    clock = torch.empty(n_it, dtype=torch.float64, device=dev)
    ttft = torch.empty(n_req, dtype=torch.float64, device=dev)
    tpot = torch.empty(n_req, dtype=torch.float64, device=dev)
    errs = torch.full((2,), torch.iinfo(torch.int64).max, dtype=torch.int64, device=dev)
    ctx = _lib.ctx_for(dev)
    _lib.check(_lib.load_library().dooly_sim_eval(
        ctx, C.byref(calltree.oplist), regs.table_ptr(_lib.KIND_AFFINE), regs.n(_lib.KIND_AFFINE),
        regs.table_ptr(_lib.KIND_ATTN), regs.n(_lib.KIND_ATTN), _lib.ptr(it_feat),
        _lib.ptr(it_start), _lib.ptr(it_off), n_shards, n_it, _lib.ptr(arrival),
        _lib.ptr(first_it), _lib.ptr(last_it), _lib.ptr(out_tok), n_req,
        _lib.ptr(it_lat), _lib.ptr(clock), _lib.ptr(ttft), _lib.ptr(tpot),
        errs.data_ptr(), errs.data_ptr() + 8, _lib.stream_ptr(dev)), ctx)
    e = errs.cpu().numpy()
    if e[0] != np.iinfo(np.int64).max:
        raise UnknownSignature(f"iteration {int(e[0])} evaluates an unfitted regressor row")
    if e[1] != np.iinfo(np.int64).max:
        raise ValueError(f"request {int(e[1])}: first/last iteration index out of range")
    return it_lat, clock, ttft, tpot


# ----------------------------------------------------------------------- run


@dataclass(frozen=True)
class SchedConfig:
    """Continuous batching + chunked prefill."""

    chunk: int = 8192
    max_batch: int = 256
    max_kv_memory: Optional[float] = None   # bytes; default tp*capacity - weights (App. A.13)
    max_iterations: int = 50_000_000


@dataclass
class Metrics:
    ttft: np.ndarray                  # per request, input order (s)
    tpot: np.ndarray                  # NaN where output_tokens < 2
    n_iterations: np.ndarray          # per shard
    final_clock: np.ndarray           # per shard
    percentiles: dict = field(default_factory=dict)

    @staticmethod
    def summarize(ttft, tpot, n_it, clock) -> "Metrics":
        m = Metrics(ttft, tpot, n_it, clock)
        for name, arr in (("ttft", ttft), ("tpot", tpot)):
            v = arr[~np.isnan(arr)]
            m.percentiles[name] = {f"p{p}": (float(np.percentile(v, p)) if v.size else math.nan)
                                   for p in PERCENTILES}
        return m


def kv_capacity(model: ModelConfig, hw: HardwareSpec, tp: int, sched: SchedConfig) -> int:
    if sched.max_kv_memory is not None:
        return int(sched.max_kv_memory)
    cap = int(tp * hw.memory_capacity) - model.weight_bytes()
    if cap <= 0:
        raise ValidationError("hardware.memory_capacity",
                              f"{model.name} weights do not fit tp={tp} x {hw.memory_capacity:.3g} B")
    return cap


def make_sched(model: ModelConfig, hw: HardwareSpec, tp: int, sched: SchedConfig,
               calltree: CallTree) -> _lib.Sched:
    if sched.chunk < sched.max_batch:
        raise ValidationError("sched.chunk", "chunk must be >= max_batch (decodes count, D1)")
    if sched.max_batch > 1024:
        raise ValidationError("sched.max_batch", "at most 1024 running requests per replica")
    s = _lib.Sched()
    s.chunk, s.max_batch, s.window = sched.chunk, sched.max_batch, calltree.window
    s.kv_bytes_per_token = model.kv_bytes_per_token()
    s.kv_capacity_bytes = kv_capacity(model, hw, tp, sched)
    s.max_iterations = sched.max_iterations
    return s


@dataclass
class ShardedTrace:
    """Requests regrouped into S replica shards (request i -> shard i mod S, App. A.14)."""

    arrival: torch.Tensor
    prompt: torch.Tensor
    output: torch.Tensor
    cached: torch.Tensor
    shard_off: torch.Tensor
    order: np.ndarray            # position in the sharded layout -> original request index
    n_shards: int

    @staticmethod
    def build(requests: Sequence[Request], n_shards: int, device) -> "ShardedTrace":
        n = len(requests)
        arr = np.fromiter((r.arrival_s for r in requests), dtype=np.float64, count=n)
        pr = np.fromiter((r.prompt_tokens for r in requests), dtype=np.uint32, count=n)
        ou = np.fromiter((r.output_tokens for r in requests), dtype=np.uint32, count=n)
        ca = np.fromiter((r.cached_tokens for r in requests), dtype=np.uint32, count=n)
        return ShardedTrace.from_arrays(arr, pr, ou, ca, n_shards, device)

    @staticmethod
    def from_arrays(arr, pr, ou, ca, n_shards: int, device) -> "ShardedTrace":
        n = arr.shape[0]
        if n and np.any(np.diff(arr) < 0):
            raise ValidationError("workload", "requests must be sorted by arrival")
        if np.any(ou < 1) or np.any(ca > pr):
            raise ValidationError("workload", "need output_tokens >= 1 and cached <= prompt")
        idx = np.arange(n)
        order = np.concatenate([idx[s::n_shards] for s in range(n_shards)]) if n else idx
        counts = np.array([len(range(s, n, n_shards)) for s in range(n_shards)], dtype=np.int64)
        off = np.zeros(n_shards + 1, dtype=np.int64)
        off[1:] = np.cumsum(counts)
        dev = torch.device(device)

        def t(a):
            return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

        return ShardedTrace(t(arr[order]), t(pr[order].view(np.int32)), t(ou[order].view(np.int32)),
                            t(ca[order].view(np.int32)), t(off), order, n_shards)


@dataclass
class SimOutputs:
    ttft: torch.Tensor
    tpot: torch.Tensor
    n_iter: torch.Tensor
    clock: torch.Tensor
    status: torch.Tensor
    log_feat: Optional[torch.Tensor] = None
    log_lat: Optional[torch.Tensor] = None


def run_sharded(trace: ShardedTrace, calltree: CallTree, sched: _lib.Sched, regs: Regressors,
                log_cap: int = 0, out: Optional[SimOutputs] = None) -> SimOutputs:
    """K4b: device-resident event loop over every shard (asynchronous)."""
    dev = trace.arrival.device
    n = trace.arrival.numel()
    S = trace.n_shards
    if out is None:
        out = SimOutputs(torch.full((n,), math.nan, dtype=torch.float64, device=dev),
                         torch.full((n,), math.nan, dtype=torch.float64, device=dev),
                         torch.zeros(S, dtype=torch.int64, device=dev),
                         torch.zeros(S, dtype=torch.float64, device=dev),
                         torch.zeros(S, dtype=torch.int32, device=dev))
        if log_cap:
            out.log_feat = torch.zeros((S, log_cap, _lib.IT_FEATS), dtype=torch.int32, device=dev)
            out.log_lat = torch.zeros((S, log_cap), dtype=torch.float64, device=dev)
    ctx = _lib.ctx_for(dev)
    _lib.check(_lib.load_library().dooly_sim_run(
        ctx, C.byref(calltree.oplist), C.byref(sched), regs.table_ptr(_lib.KIND_AFFINE),
        regs.n(_lib.KIND_AFFINE), regs.table_ptr(_lib.KIND_ATTN), regs.n(_lib.KIND_ATTN),
        _lib.ptr(trace.arrival), _lib.ptr(trace.prompt), _lib.ptr(trace.output),
        _lib.ptr(trace.cached), trace.shard_off.data_ptr(), S, _lib.ptr(out.ttft),
        _lib.ptr(out.tpot), out.n_iter.data_ptr(), out.clock.data_ptr(), out.status.data_ptr(),
        _lib.ptr(out.log_feat), _lib.ptr(out.log_lat), log_cap, 0, 0, _lib.stream_ptr(dev)), ctx)
    return out


def collect(trace: ShardedTrace, res: SimOutputs) -> Metrics:
    """Sync, raise the reference's errors, and restore input order."""
    status = res.status.cpu().numpy()
    if np.any(status == 5):
        raise NonTermination(f"shard {int(np.argmax(status == 5))} hit the iteration cap")
    if np.any(status == 3):
        raise UnknownSignature("call graph references an unfitted regressor row")
    if np.any(status != 0):
        raise ValidationError("workload", "a request can never fit the KV-memory capacity")
    n = trace.order.shape[0]
    ttft = np.empty(n)
    tpot = np.empty(n)
    ttft[trace.order] = res.ttft.cpu().numpy()
    tpot[trace.order] = res.tpot.cpu().numpy()
    return Metrics.summarize(ttft, tpot, res.n_iter.cpu().numpy(), res.clock.cpu().numpy())


def run_shards(workload: Sequence[Request], n_shards: int, model: ModelConfig,
               backend: BackendSpec, hw: HardwareSpec, regs: Regressors, sched: SchedConfig,
               tp: int = 1, calltree: Optional[CallTree] = None) -> Metrics:
    """S independent replicas (request i -> shard i mod S); identical results for
    any device count because S is fixed."""
    ct = calltree or build_calltree(model, backend, regs, hw, tp)
    cfg = make_sched(model, hw, tp, sched, ct)
    trace = ShardedTrace.build(workload, n_shards, regs.device)
    return collect(trace, run_sharded(trace, ct, cfg, regs))


def run(workload: Sequence[Request], model: ModelConfig, backend: BackendSpec,
        hw: HardwareSpec, regs: Regressors, sched: SchedConfig, tp: int = 1) -> Metrics:
    """End-to-end event loop of one serving replica."""
    return run_shards(workload, 1, model, backend, hw, regs, sched, tp)


def mape(pred: Sequence[float], truth: Sequence[float]) -> float:
    """mean(|p - t| / t)."""
    p = np.asarray(pred, dtype=np.float64)
    t = np.asarray(truth, dtype=np.float64)
    if p.shape != t.shape:
        raise LengthMismatch(f"{p.shape} vs {t.shape}")
    if np.any(t == 0):
        raise ZeroTruth("truth series contains 0")
    return float(np.mean(np.abs(p - t) / t)) if t.size else 0.0


def predict_host(kind: int, table: torch.Tensor, sig: torch.Tensor, x: torch.Tensor,
                 out: torch.Tensor, flags: Optional[torch.Tensor] = None, chunk: int = 1 << 23,
                 n_streams: int = 3) -> torch.Tensor:
    """Host-buffer entry point of K3: pinned host sig (n,) i32 and x (P, n) i32 in,
    pinned host f64 latencies out and, when ``flags`` is given, the SPEC.md:569
    flag bit-planes (2, ceil(n/32)) i32 (extrapolated, clamped; bit q % 32 of
    word q // 32) — see ``predict_host_many``; returns ``out``."""
    predict_host_many([(kind, table, sig, x, out, flags)], chunk, n_streams)
    return out


def predict_host_many(batches: Sequence, chunk: int = 1 << 23, n_streams: int = 3) -> None:
    """Several host-buffer query batches ``(kind, table, sig, x, out[, flags])``
    (pinned host tensors; tables on the device; ``flags`` None or a pinned
    (2, ceil(n/32)) i32 tensor receiving the extrapolation / clamp bit-planes)
    through one copy/compute pipeline.  Chunks of all batches are interleaved
    over ``n_streams`` CUDA streams, so the H2D copy engine, the kernels and the
    D2H copy engine overlap.  Mixing kinds also balances the link: attention
    queries are H2D-heavy (16 B in, 8 B out), affine ones symmetric (8 B in,
    8 B out).  Synchronises; raises UnknownSignature if any query hit an
    unfitted row."""
    if not batches:
        return
    batches = [tuple(b) + (None,) * (6 - len(b)) for b in batches]
    dev = batches[0][1].device
    cur = torch.cuda.current_stream(dev)
    streams = [torch.cuda.Stream(dev) for _ in range(max(1, n_streams))]
    pmax = max(b[3].shape[0] for b in batches)
    c = min(chunk, max(max(b[2].numel() for b in batches), 1))
    c = -(-c // 32) * 32                       # chunk starts stay on flag-word boundaries
    cw = c // 32
    bufs = [(torch.empty(c, dtype=torch.int32, device=dev),
             torch.empty((pmax, c), dtype=torch.int32, device=dev),
             torch.empty(c, dtype=torch.float64, device=dev),
             torch.empty(2 * cw, dtype=torch.int32, device=dev),
             torch.full((1,), torch.iinfo(torch.int64).max, dtype=torch.int64, device=dev))
            for _ in streams]
    for s in streams:
        s.wait_stream(cur)
    work = []                                  # round-robin chunks of every batch
    cursors = [0] * len(batches)
    while any(cursors[i] < batches[i][2].numel() for i in range(len(batches))):
        for i, bt in enumerate(batches):
            n = bt[2].numel()
            if cursors[i] < n:
                work.append((i, cursors[i], min(n, cursors[i] + c)))
                cursors[i] += c
    for j, (i, q0, q1) in enumerate(work):
        kind, table, sig, x, out, hflags = batches[i]
        P = x.shape[0]
        m = q1 - q0
        w = (m + 31) // 32
        s = streams[j % len(streams)]
        d_sig, d_x, d_out, d_flags, d_err = bufs[j % len(streams)]
        with torch.cuda.stream(s):
            d_sig[:m].copy_(sig[q0:q1], non_blocking=True)
            xs = d_x[:P, :m] if m == c else torch.empty((P, m), dtype=torch.int32, device=dev)
            for p in range(P):
                xs[p].copy_(x[p, q0:q1], non_blocking=True)
            fl = d_flags[:2 * w].view(2, w) if hflags is not None else None
            predict_batch(kind, table, d_sig[:m], xs, d_out[:m], fl, d_err,
                          want_flags=hflags is not None)
            out[q0:q1].copy_(d_out[:m], non_blocking=True)
            if hflags is not None:
                for p in range(2):
                    hflags[p, q0 // 32:q0 // 32 + w].copy_(fl[p], non_blocking=True)
    for s in streams:
        s.synchronize()
    if any(int(b[4].item()) != torch.iinfo(torch.int64).max for b in bufs):
        raise UnknownSignature("a query references an unfitted regressor row")
