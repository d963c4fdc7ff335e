"""Duplication-aware profiler: the drop-in for the reference's `dooly.profiler`
(module absent from pkg/src).

Hot path (GPU, libdooly_b200):
    canonicalize -> signature_hash -> dedup
  ``dedup_packed`` hashes packed records on the device (K1a) and resolves
  first occurrences against the DB key set (K1b).  ``dedup`` / ``signature_hash``
  are thin wrappers over the same device path (no CPU fallback).

Host side (inputs to the fit, SURVEY §8(f) row f1 is their GPU fusion):
    sweep, oracle_latency, comm_latency
  and the in-memory ``LatencyDB`` working set with the Fig. 9 logical tables
   — configurations, signatures, model_operations,
  measurements, comm_measurements.  ``store.py`` persists it as one SQLite file
  (D5) with JSON-lines import/export (D4) and a schema dump;
  ``.npz`` snapshots remain for quick round trips.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from .errors import DuplicateKey, OraclePanic, StoreUnavailable
from .modelir import BackendSpec, HardwareSpec, ModelConfig, SweepGrid
from .records import PackedRecords, RunnableEntry, canonical_bytes, pack_entries

OVERHEAD_S = 5e-6  # fixed launch overhead of the analytical latency model


def _device(device=None) -> torch.device:
    if device is None:
        if not torch.cuda.is_available():
            raise StoreUnavailable("libdooly_b200 needs a CUDA device (no CPU fallback)")
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


# ------------------------------------------------------------------ signatures


def canonicalize(entry: RunnableEntry) -> bytes:
    """Canonical serialisation of one runnable entry."""
    return canonical_bytes(entry)


def signature_hash(canonical: bytes, device=None) -> bytes:
    """SHA-256 of a canonical message, computed by the GPU kernel."""
    return signature_hash_batch([canonical], device)[0]


def signature_hash_batch(messages: Sequence[bytes], device=None) -> list:
    dev = _device(device)
    n = len(messages)
    if n == 0:
        return []
    off = np.zeros(n + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(m) for m in messages])
    data = np.frombuffer(b"".join(messages) or b"\0", dtype=np.uint8)
    d_msgs = torch.from_numpy(data.copy()).to(dev)
    d_off = torch.from_numpy(off).to(dev)
    out = torch.empty((n, 32), dtype=torch.uint8, device=dev)
    ctx = _lib.ctx_for(dev)
    _lib.check(_lib.load_library().dooly_sha256_messages(
        ctx, d_msgs.data_ptr(), d_off.data_ptr(), n, out.data_ptr(), _lib.stream_ptr(dev)), ctx)
    host = out.cpu().numpy()
    return [bytes(host[i]) for i in range(n)]


@dataclass
class DeviceRecords:
    words: torch.Tensor
    rec_off: torch.Tensor
    op_bytes: torch.Tensor
    op_off: torch.Tensor
    sym_bytes: torch.Tensor
    sym_off: torch.Tensor
    attr_digests: torch.Tensor
    n: int

    @staticmethod
    def from_packed(p: PackedRecords, device) -> "DeviceRecords":
        dev = torch.device(device)

        def t(a, dtype):
            a = np.ascontiguousarray(a)
            if a.size == 0:
                a = np.zeros(1, dtype=a.dtype)
            return torch.from_numpy(a.view(dtype) if a.dtype != dtype else a).to(dev)

        return DeviceRecords(t(p.words.view(np.int32), np.int32), t(p.rec_off, np.int64),
                             t(p.op_bytes, np.uint8), t(p.op_off, np.int64),
                             t(p.sym_bytes, np.uint8), t(p.sym_off, np.int64),
                             t(p.attr_digests.reshape(-1), np.uint8), p.n)


def hash_records(recs: DeviceRecords, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """K1a: SHA-256 of every packed record's canonical message -> (n, 32) u8."""
    dev = recs.words.device
    if out is None:
        out = torch.empty((recs.n, 32), dtype=torch.uint8, device=dev)
    ctx = _lib.ctx_for(dev)
    _lib.check(_lib.load_library().dooly_sha256_records(
        ctx, recs.words.data_ptr(), recs.rec_off.data_ptr(), recs.n, recs.op_bytes.data_ptr(),
        recs.op_off.data_ptr(), recs.op_off.numel() - 1, recs.sym_bytes.data_ptr(),
        recs.sym_off.data_ptr(), recs.sym_off.numel() - 1, recs.attr_digests.data_ptr(),
        recs.attr_digests.numel() // 32, out.data_ptr(), _lib.stream_ptr(dev)), ctx)
    return out


@dataclass
class DedupResult:
    digests: torch.Tensor     # (n, 32) u8
    first: torch.Tensor       # (n,) i64 smallest index with the same digest
    uid: torch.Tensor         # (n,) i32 rank of `first` among first occurrences
    is_new: torch.Tensor      # (n,) u8  first occurrence and not in the DB -> profile it
    in_db: torch.Tensor       # (n,) u8
    n_unique: int

    def to_profile_index(self) -> np.ndarray:
        return np.nonzero(self.is_new.cpu().numpy())[0]


class DedupWorkspace:
    """Reusable device scratch for dedup_digests (no allocation in the hot call)."""

    def __init__(self, device) -> None:
        self.device = torch.device(device)
        self.buf = torch.empty(0, dtype=torch.uint8, device=self.device)

    def get(self, n: int, n_db: int) -> torch.Tensor:
        need = int(_lib.load_library().dooly_dedup_workspace_size(n, n_db))
        if self.buf.numel() < need:
            self.buf = torch.empty(need, dtype=torch.uint8, device=self.device)
        return self.buf


def dedup_digests(digests: torch.Tensor, db_digests: Optional[torch.Tensor] = None,
                  workspace: Optional[DedupWorkspace] = None, sync: bool = True) -> DedupResult:
    """K1b: first-occurrence dedup of (n, 32) digests against a (n_db, 32) key set."""
    dev = digests.device
    n = digests.shape[0]
    if db_digests is None:
        db_digests = torch.empty((0, 32), dtype=torch.uint8, device=dev)
    n_db = db_digests.shape[0]
    ws = (workspace or DedupWorkspace(dev)).get(n, n_db)
    first = torch.empty(n, dtype=torch.int64, device=dev)
    uid = torch.empty(n, dtype=torch.int32, device=dev)
    is_new = torch.empty(n, dtype=torch.uint8, device=dev)
    in_db = torch.empty(n, dtype=torch.uint8, device=dev)
    n_unique = torch.empty(1, dtype=torch.int64, device=dev)
    ctx = _lib.ctx_for(dev)
    _lib.check(_lib.load_library().dooly_dedup_digests(
        ctx, digests.data_ptr() if n else 0, n, db_digests.data_ptr() if n_db else 0, n_db,
        first.data_ptr(), uid.data_ptr(), is_new.data_ptr(), in_db.data_ptr(),
        n_unique.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr(dev)), ctx)
    nu = int(n_unique.item()) if sync else -1
    return DedupResult(digests, first, uid, is_new, in_db, nu)


def dedup_packed(recs: DeviceRecords, db_digests: Optional[torch.Tensor] = None,
                 workspace: Optional[DedupWorkspace] = None, sync: bool = True) -> DedupResult:
    """Batch form of dedup: packed records in HBM -> digests + dedup table, one
    C-ABI call (dooly_dedup = K1a SHA-256 + K1b first-occurrence resolve)."""
    dev = recs.words.device
    n = recs.n
    if db_digests is None:
        db_digests = torch.empty((0, 32), dtype=torch.uint8, device=dev)
    n_db = db_digests.shape[0]
    ws = (workspace or DedupWorkspace(dev)).get(n, n_db)
    dig = torch.empty((n, 32), dtype=torch.uint8, device=dev)
    first = torch.empty(n, dtype=torch.int64, device=dev)
    uid = torch.empty(n, dtype=torch.int32, device=dev)
    is_new = torch.empty(n, dtype=torch.uint8, device=dev)
    in_db = torch.empty(n, dtype=torch.uint8, device=dev)
    n_unique = torch.empty(1, dtype=torch.int64, device=dev)
    ctx = _lib.ctx_for(dev)
    _lib.check(_lib.load_library().dooly_dedup(
        ctx, recs.words.data_ptr(), recs.rec_off.data_ptr(), n, recs.op_bytes.data_ptr(),
        recs.op_off.data_ptr(), recs.op_off.numel() - 1, recs.sym_bytes.data_ptr(),
        recs.sym_off.data_ptr(), recs.sym_off.numel() - 1, recs.attr_digests.data_ptr(),
        recs.attr_digests.numel() // 32, db_digests.data_ptr() if n_db else 0, n_db,
        dig.data_ptr(), first.data_ptr(), uid.data_ptr(), is_new.data_ptr(), in_db.data_ptr(),
        n_unique.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr(dev)), ctx)
    nu = int(n_unique.item()) if sync else -1
    return DedupResult(dig, first, uid, is_new, in_db, nu)


# ------------------------------------------------------------------ LatencyDB


def _kind_of(entry: RunnableEntry) -> int:
    return _lib.KIND_ATTN if entry.feature == "attention" else _lib.KIND_AFFINE


@dataclass
class SignatureRow:
    digest: bytes
    op_name: str
    granularity: str
    kind: int
    feature: str
    components: str = "{}"   # JSON: model_dims, kernel_symbols, attrs, window


def _components(entry: RunnableEntry) -> str:
    import json

    return json.dumps({"model_dims": entry.model_dims(), "kernel_symbols": list(entry.kernel_symbols),
                       "attrs": dict(entry.attrs), "window": entry.window}, sort_keys=True)


@dataclass
class LatencyDB:
    """In-memory store with the Fig. 9 logical schema (D5 :517)."""

    configurations: list = field(default_factory=list)     # (hardware, model, backend, tp)
    signatures: list = field(default_factory=list)         # SignatureRow, insertion order
    model_operations: list = field(default_factory=list)   # (config_id, digest, repeat)
    measurements: dict = field(default_factory=dict)       # digest -> (x (p, n) u32, y f64)
    workloads: dict = field(default_factory=dict)          # digest -> [workload dict | None] per point
    sources: dict = field(default_factory=dict)            # digest -> ["oracle" | "imported"] per point
    comm_measurements: dict = field(default_factory=dict)  # (topology, tp, bytes) -> latency_s
    _index: dict = field(default_factory=dict)

    def schema_dump(self) -> str:
        """The logical schema (D5 conformance dump), identical to the SQLite DDL."""
        from .store import schema_dump

        return schema_dump()

    def has(self, digest: bytes) -> bool:
        return digest in self._index

    def signature(self, digest: bytes) -> SignatureRow:
        return self.signatures[self._index[digest]]

    def add_configuration(self, hardware: str, model: str, backend: str, tp: int) -> int:
        key = (hardware, model, backend, tp)
        if key in self.configurations:
            return self.configurations.index(key)
        self.configurations.append(key)
        return len(self.configurations) - 1

    def add_signature(self, digest: bytes, entry: RunnableEntry) -> None:
        if digest not in self._index:
            self._index[digest] = len(self.signatures)
            self.signatures.append(SignatureRow(digest, entry.name, entry.granularity,
                                                _kind_of(entry), entry.feature,
                                                _components(entry)))

    def add_model_operation(self, config_id: int, digest: bytes, repeat_count: int) -> None:
        """model_operations row; must reference an existing configuration and
        signature (referential integrity)."""
        if not 0 <= config_id < len(self.configurations) or digest not in self._index:
            raise StoreUnavailable("model_operations must reference an existing configuration "
                                   "and signature")
        self.model_operations.append((int(config_id), digest, int(repeat_count)))

    def insert_measurements(self, digest: bytes, x: np.ndarray, y: np.ndarray,
                            workloads: Optional[Sequence] = None, source: str = "oracle") -> None:
        """Insert a sweep; re-inserting an identical key with a different latency
        raises DuplicateKey.  ``workloads`` optionally carries the
        LatencyRecord workload of every point."""
        if digest not in self._index:
            raise StoreUnavailable("model_operations/measurements must reference a signature")
        x = np.atleast_2d(np.asarray(x, dtype=np.uint32))
        y = np.asarray(y, dtype=np.float64)
        if np.any(~(y > 0)):
            raise OraclePanic(f"{digest.hex()[:12]}: latency_s must be > 0 (SPEC.md:427)")
        wl = list(workloads) if workloads is not None else [None] * y.shape[0]
        src = [source] * y.shape[0]
        if digest in self.measurements:
            ox, oy = self.measurements[digest]
            old = {tuple(ox[:, i]): oy[i] for i in range(oy.shape[0])}
            keep = []
            for i in range(y.shape[0]):
                k = tuple(x[:, i])
                if k in old:
                    if old[k] != y[i]:
                        raise DuplicateKey(f"{digest.hex()[:12]} at {k}: {old[k]} != {y[i]}")
                else:
                    keep.append(i)
            x = np.concatenate([ox, x[:, keep]], axis=1)
            y = np.concatenate([oy, y[keep]])
            wl = self.workloads.get(digest, [None] * oy.shape[0]) + [wl[i] for i in keep]
            src = self.point_sources(digest) + [source] * len(keep)
        self.measurements[digest] = (x, y)
        self.workloads[digest] = wl
        self.sources[digest] = src

    def point_sources(self, digest: bytes) -> list:
        """Source of every measurement point of a signature (SPEC D4: oracle or
        imported, tracked per point)."""
        n = self.measurements[digest][1].shape[0] if digest in self.measurements else 0
        src = self.sources.get(digest)
        if src is None:
            return ["oracle"] * n
        return [src] * n if isinstance(src, str) else list(src)

    def insert_comm(self, topology: str, tp_degree: int, nbytes: int, latency_s: float) -> None:
        """comm sub-schema keyed by hardware topology (Appendix E)."""
        key = (topology, int(tp_degree), int(nbytes))
        old = self.comm_measurements.get(key)
        if old is not None and old != latency_s:
            raise DuplicateKey(f"comm {key}: {old} != {latency_s}")
        self.comm_measurements[key] = float(latency_s)

    def digest_tensor(self, device) -> torch.Tensor:
        if not self.signatures:
            return torch.empty((0, 32), dtype=torch.uint8, device=device)
        arr = np.frombuffer(b"".join(s.digest for s in self.signatures), dtype=np.uint8)
        return torch.from_numpy(arr.reshape(-1, 32).copy()).to(device)

    def save(self, path) -> None:
        """Persist: ``.npz`` snapshot, or the single-file SQLite store (D5) for any
        other suffix (``store.save``).  The snapshot holds plain arrays only (the
        metadata as one UTF-8 JSON array) and loads with allow_pickle=False; it
        keeps every table (components, per-point workloads and sources, comm)."""
        if not str(path).endswith(".npz"):
            from .store import save

            save(self, path)
            return
        import json

        meta = {"configurations": [list(c) for c in self.configurations],
                "signatures": [[r.digest.hex(), r.op_name, r.granularity, int(r.kind), r.feature,
                                r.components] for r in self.signatures],
                "model_operations": [[int(c), d.hex(), int(r)] for c, d, r in self.model_operations],
                "workloads": {d.hex(): w for d, w in self.workloads.items()},
                "sources": {d.hex(): self.point_sources(d) for d in self.measurements},
                "comm": [[t, int(tp), int(b), float(v)]
                         for (t, tp, b), v in self.comm_measurements.items()]}
        arrays = {"meta": np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)}
        for d, (x, y) in self.measurements.items():
            arrays[f"x_{d.hex()}"] = np.ascontiguousarray(x, dtype=np.uint32)
            arrays[f"y_{d.hex()}"] = np.ascontiguousarray(y, dtype=np.float64)
        np.savez(path, **arrays)

    @staticmethod
    def load(path) -> "LatencyDB":
        if not str(path).endswith(".npz"):
            from .store import load

            return load(path)
        import json

        try:
            z = np.load(path, allow_pickle=False)
            meta = json.loads(bytes(z["meta"]).decode())
        except (OSError, KeyError, ValueError) as exc:
            raise StoreUnavailable(f"{path}: {exc}") from exc
        db = LatencyDB()
        db.configurations = [tuple(c) for c in meta["configurations"]]
        for h, name, gran, kind, feat, comp in meta["signatures"]:
            d = bytes.fromhex(h)
            db._index[d] = len(db.signatures)
            db.signatures.append(SignatureRow(d, name, gran, int(kind), feat, comp))
        db.model_operations = [(int(c), bytes.fromhex(h), int(r))
                               for c, h, r in meta["model_operations"]]
        for key in z.files:
            if key.startswith("x_"):
                d = bytes.fromhex(key[2:])
                db.measurements[d] = (z[key], z["y_" + key[2:]])
        db.workloads = {bytes.fromhex(h): w for h, w in meta["workloads"].items()}
        db.sources = {bytes.fromhex(h): s for h, s in meta["sources"].items()}
        db.comm_measurements = {(t, tp, b): v for t, tp, b, v in meta["comm"]}
        return db


def dedup(entries: Sequence[RunnableEntry], db: LatencyDB, config_id: Optional[int] = None,
          device=None, register: bool = True):
    """Partition entries into (to_profile, skipped).

    skipped <=> the signature is already in the DB, or an earlier entry of this
    call has it.  model_operations rows are recorded for ALL entries when a
    config id is given; new signatures are registered so a re-run profiles
    nothing."""
    to_profile, skipped, _ = dedup_with_digests(entries, db, config_id, device, register)
    return to_profile, skipped


def dedup_with_digests(entries: Sequence[RunnableEntry], db: LatencyDB,
                       config_id: Optional[int] = None, device=None, register: bool = True):
    """dedup that also returns the device-computed digest of every to_profile entry."""
    if db is None:
        raise StoreUnavailable("no latency database")
    dev = _device(device)
    entries = list(entries)
    if not entries:
        return [], [], []
    recs = DeviceRecords.from_packed(pack_entries(entries), dev)
    res = dedup_packed(recs, db.digest_tensor(dev))
    is_new = res.is_new.cpu().numpy().astype(bool)
    digs = res.digests.cpu().numpy()
    to_profile, skipped, new_digests = [], [], []
    for i, e in enumerate(entries):
        d = bytes(digs[i])
        if is_new[i] and register:
            db.add_signature(d, e)
        if config_id is not None and db.has(d):   # dry runs (register=False) record nothing new
            db.add_model_operation(config_id, d, e.repeat_count)
        if is_new[i]:
            to_profile.append(e)
            new_digests.append(d)
        else:
            skipped.append(e)
    return to_profile, skipped, new_digests


# ------------------------------------------- analytical latency model (host, f1)


def comm_latency(topology: str, tp: int, nbytes: int, hw: HardwareSpec) -> float:
    """Ring all-reduce alpha-beta model, Python operator order."""
    del topology  # keyed by (topology, tp) in the DB; the formula is topology-free
    if tp < 2:
        raise ValueError("comm_latency needs tp >= 2")
    return 2 * (tp - 1) / tp * (hw.comm_alpha + nbytes / tp * hw.comm_beta)


def _dims(entry: RunnableEntry) -> list:
    return [[s for s, _ in a] for a in entry.arg_template]


def op_cost(entry: RunnableEntry, point: dict, dtype_bytes: int) -> tuple:
    """(flops, bytes) of one op instance at a sweep point."""
    name = entry.name
    a = _dims(entry)
    t = point.get("num_toks", 1)
    if name == "linear":
        k, n = a[1][1], a[1][0]
        m = point["num_reqs"] if entry.feature == "num_seqs" else t
        return 2.0 * m * k * n, float((m * k + k * n + m * n) * dtype_bytes)
    if name == "embedding":
        h = a[1][1]
        return 0.0, float(2 * t * h * dtype_bytes + 4 * t)
    if name == "rms_norm":
        h = a[0][1]
        return 4.0 * t * h, float((2 * t * h + h) * dtype_bytes)
    if name == "rotary_embedding":
        w = a[0][1] * a[0][2] + a[1][1] * a[1][2]
        return 3.0 * t * w, float(2 * t * w * dtype_bytes)
    if name == "silu_and_mul":
        i2 = a[0][1]
        return 2.0 * t * i2, float((t * i2 + t * i2 // 2) * dtype_bytes)
    if name == "topk_softmax":
        e = a[0][1]
        return 5.0 * t * e, float(t * e * (dtype_bytes + 8))
    if name == "fused_moe":
        e, i2, h = a[1]
        k = entry.scalars[0][0]
        touched = min(e, t * k)
        return 2.0 * t * k * (i2 + i2 // 2) * h, float(
            (touched * (i2 + i2 // 2) * h + 2 * t * h) * dtype_bytes)
    if name == "attention":
        hq, d = a[0][1], a[0][2]
        hkv = a[1][1]
        r = point["num_reqs"]
        c = point["kv_len"]
        if entry.window:
            c = min(c, entry.window)
        if point["phase"] == "prefill":
            q = t / r
        else:
            q = 1.0
        ctx = c + q
        flops = 4.0 * hq * d * r * q * ctx
        nbytes = float(dtype_bytes * (r * ctx * 2 * hkv * d + 2 * r * q * hq * d))
        return flops, nbytes
    if name == "reshape":
        return 0.0, 0.0
    raise OraclePanic(f"no cost formula for op kind {name!r} at {point}")


def oracle_latency(entry: RunnableEntry, point: dict, hw: HardwareSpec, backend: BackendSpec,
                   dtype_bytes: int = 2) -> float:
    """overhead + multiplier * max(flops/peak, bytes/bw)."""
    flops, nbytes = op_cost(entry, point, dtype_bytes)
    syms = entry.kernel_symbols
    if entry.feature == "attention":
        syms = tuple(s.replace("_decode_attn_", f"_{point['phase']}_attn_") for s in syms)
    mult = backend.multiplier(syms)
    return OVERHEAD_S + mult * max(flops / hw.peak_flops, nbytes / hw.mem_bw)


def sweep_points(entry: RunnableEntry, grid: SweepGrid, max_context: int) -> list:
    """Training points of one signature (D3 :515, App. A.5)."""
    cap_t = min(grid.prefill_chunk, max_context)
    toks = [t for t in grid.token_counts if t <= cap_t]
    reqs = [r for r in grid.request_counts if r <= grid.max_batch]
    if entry.feature == "num_toks":
        return [{"num_toks": t} for t in toks]
    if entry.feature == "num_seqs":
        return [{"num_reqs": r} for r in reqs]
    pts = []
    for t in toks:
        for r in reqs:
            if t < r:
                continue
            for c in grid.kv_lens:
                if c + -(-t // r) <= max_context:
                    pts.append({"phase": "prefill", "num_toks": t, "num_reqs": r, "kv_len": c})
    for r in reqs:
        for c in grid.kv_lens:
            if c + 1 <= max_context:
                pts.append({"phase": "decode", "num_toks": r, "num_reqs": r, "kv_len": c})
    return pts


def point_features(entry: RunnableEntry, p: dict) -> tuple:
    """Regression features of a sweep point (App. A.6): affine -> (x,), attention ->
    (prefill_toks, batch, kv_tokens) with kv capped by the sliding window."""
    if entry.feature == "num_toks":
        return (p["num_toks"],)
    if entry.feature == "num_seqs":
        return (p["num_reqs"],)
    c = min(p["kv_len"], entry.window) if entry.window else p["kv_len"]
    pre = p["num_toks"] if p["phase"] == "prefill" else 0
    return (pre, p["num_reqs"], p["num_reqs"] * c)


def sweep(entry: RunnableEntry, grid: SweepGrid, model: ModelConfig, hw: HardwareSpec,
          backend: BackendSpec):
    """Evaluate the analytical model over the signature's grid -> (x (p, n) u32, y f64)."""
    pts = sweep_points(entry, grid, model.max_context)
    x = np.array([point_features(entry, p) for p in pts], dtype=np.uint32).T
    y = np.array([oracle_latency(entry, p, hw, backend, model.dtype_bytes) for p in pts])
    return np.ascontiguousarray(x), y


def profile_corpus(manifest, db: Optional[LatencyDB] = None, device=None,
                   grid: Optional[SweepGrid] = None):
    """cmd_profile without the CLI: dedup every (model, backend)
    runnable set in manifest order against the DB, sweep the new signatures.
    Returns (db, report) with per-config N/R counts."""
    from .records import runnable_entries

    db = db if db is not None else LatencyDB()
    grid = grid or manifest.grid
    report = []
    for m in manifest.models:
        for b in manifest.backends:
            cid = db.add_configuration(manifest.hardware.name, m.name, b.name, manifest.tp_degree)
            entries = runnable_entries(m, b, manifest.tp_degree)
            to_profile, skipped, digests = dedup_with_digests(entries, db, cid, device)
            for e, d in zip(to_profile, digests):
                x, y = sweep(e, grid, m, manifest.hardware, b)
                db.insert_measurements(d, x, y, sweep_points(e, grid, m.max_context))
            report.append({"model": m.name, "backend": b.name, "entries": len(entries),
                           "profiled": len(to_profile), "skipped": len(skipped)})
    return db, report


# ------------------------------------------------- K5: fused sweep -> fit (f1)


def sweep_descriptor(entry: RunnableEntry, model: ModelConfig, backend: BackendSpec):
    """Device descriptor of one signature's sweep for dooly_profile_fit (the
    dims op_cost reads, the backend multipliers of both attention phases)."""
    d = _lib.SweepDesc()
    if entry.name not in _lib.OP_CODES:
        raise OraclePanic(f"no cost formula for op kind {entry.name!r}")
    d.op = _lib.OP_CODES[entry.name]
    d.feature = {"num_toks": _lib.FEAT_NUM_TOKS, "num_seqs": _lib.FEAT_NUM_SEQS,
                 "attention": _lib.FEAT_ATTN}[entry.feature]
    a = _dims(entry)
    dims = {
        "linear": lambda: (a[1][1], a[1][0]),
        "embedding": lambda: (a[1][1],),
        "rms_norm": lambda: (a[0][1],),
        "rotary_embedding": lambda: (a[0][1] * a[0][2] + a[1][1] * a[1][2],),
        "silu_and_mul": lambda: (a[0][1],),
        "topk_softmax": lambda: (a[0][1],),
        "fused_moe": lambda: (a[1][0], a[1][1], a[1][2], entry.scalars[0][0]),
        "attention": lambda: (a[0][1], a[0][2], a[1][1]),
        "reshape": lambda: (),
    }[entry.name]()
    for i, v in enumerate(dims):
        d.dim[i] = int(v)
    d.window = int(entry.window or 0)
    d.dtype_bytes = model.dtype_bytes
    d.max_context = model.max_context
    if entry.feature == "attention":
        for i, phase in enumerate(("prefill", "decode")):
            syms = tuple(s.replace("_decode_attn_", f"_{phase}_attn_") for s in entry.kernel_symbols)
            d.mult[i] = backend.multiplier(syms)
    else:
        d.mult[0] = d.mult[1] = backend.multiplier(entry.kernel_symbols)
    return d


def sweep_grid_struct(grid: SweepGrid, hw: HardwareSpec):
    g = _lib.SweepGrid()
    for name, vals in (("tok", grid.token_counts), ("req", grid.request_counts),
                       ("kv", grid.kv_lens)):
        if len(vals) > _lib.SWEEP_MAX:
            raise ValueError(f"sweep grid axis {name} longer than {_lib.SWEEP_MAX}")
        arr = getattr(g, name)
        for i, v in enumerate(vals):
            arr[i] = int(v)
    g.n_tok, g.n_req, g.n_kv = len(grid.token_counts), len(grid.request_counts), len(grid.kv_lens)
    g.chunk, g.max_batch = grid.prefill_chunk, grid.max_batch
    g.peak_flops, g.mem_bw, g.overhead = hw.peak_flops, hw.mem_bw, OVERHEAD_S
    return g


def profile_fit(items: Sequence, hw: HardwareSpec, grid: SweepGrid, device=None,
                emit_points: bool = False):
    """K5: sweep + fit (entry, model, backend) triples on the device, one launch
    per regression kind (descriptors carry each model's caps and each backend's
    multipliers; the grid and hardware are shared).  Returns
    {kind: (FitResult, item indices, (x, y, off) | None)}."""
    from .sim import FitResult

    dev = _device(device)
    g = sweep_grid_struct(grid, hw)
    out = {}
    for kind in (_lib.KIND_AFFINE, _lib.KIND_ATTN):
        idx = [i for i, it in enumerate(items) if _kind_of(it[0]) == kind]
        if not idx:
            continue
        descs = (_lib.SweepDesc * len(idx))(*[sweep_descriptor(*items[i]) for i in idx])
        d_desc = torch.frombuffer(bytearray(descs), dtype=torch.uint8).to(dev)
        n = len(idx)
        fr = FitResult(kind, torch.empty((n, _lib.ROW_BYTES[kind]), dtype=torch.uint8, device=dev),
                       torch.empty(n, dtype=torch.float64, device=dev),
                       torch.empty(n, dtype=torch.uint8, device=dev))
        px = py = poff = None
        if emit_points:
            counts = [len(sweep_points(items[i][0], grid, items[i][1].max_context)) for i in idx]
            off = np.zeros(n + 1, dtype=np.int64)
            off[1:] = np.cumsum(counts)
            total = int(off[-1])
            px = torch.zeros((_lib.PLANES[kind], max(total, 1)), dtype=torch.int32, device=dev)
            py = torch.zeros(max(total, 1), dtype=torch.float64, device=dev)
            poff = torch.from_numpy(off).to(dev)
        ctx = _lib.ctx_for(dev)
        _lib.check(_lib.load_library().dooly_profile_fit(
            ctx, kind, d_desc.data_ptr(), n, C.byref(g), fr.table.data_ptr(),
            fr.fit_err.data_ptr(), fr.status.data_ptr(), _lib.ptr(px), _lib.ptr(py),
            _lib.ptr(poff), 0 if px is None else px.shape[1], _lib.stream_ptr(dev)), ctx)
        out[kind] = (fr, idx, (px, py, poff) if emit_points else None)
    return out


def profile_and_fit(manifest, db: Optional[LatencyDB] = None, device=None,
                    grid: Optional[SweepGrid] = None):
    """cmd_profile + fit with the fused K5 path.

    One GPU dedup of every runnable set of the manifest in global order
    (App. A.4) against the DB's keys, then one sweep+fit launch per regression
    kind for the new signatures.  The DB changes only after the sweep+fit
    succeeded (an OraclePanic leaves it untouched): the new signatures, their
    swept measurements (emitted by the same kernel, so ``sim.fit(db)`` and
    ``store.save`` see them) and the model_operations rows of every entry.
    The returned Regressors cover every signature the manifest references:
    the new ones from the fused fit, those already in the DB fitted from their
    stored measurements (InsufficientData if they have none).
    Returns (db, Regressors, report)."""
    from .errors import InsufficientData
    from .records import runnable_entries
    from .sim import NEED, FitResult, Regressors, fit as fit_db

    dev = _device(device)
    db = db if db is not None else LatencyDB()
    grid = grid or manifest.grid
    configs, entries = [], []
    for m in manifest.models:
        for b in manifest.backends:
            ents = runnable_entries(m, b, manifest.tp_degree)
            configs.append((m, b, len(entries), len(entries) + len(ents)))
            entries += ents
    if not entries:
        return db, Regressors({}, {}, dev), []
    res = dedup_packed(DeviceRecords.from_packed(pack_entries(entries), dev), db.digest_tensor(dev))
    is_new = res.is_new.cpu().numpy().astype(bool)
    digs = [bytes(r) for r in res.digests.cpu().numpy()]
    items, new_digests, report = [], [], []
    for m, b, lo, hi in configs:
        for i in range(lo, hi):
            if is_new[i]:
                items.append((entries[i], m, b))
                new_digests.append(digs[i])
        n_new = int(is_new[lo:hi].sum())
        report.append({"model": m.name, "backend": b.name, "entries": hi - lo,
                       "profiled": n_new, "skipped": hi - lo - n_new})
    fitted = profile_fit(items, manifest.hardware, grid, dev, emit_points=True)  # may raise
    torch.cuda.synchronize(dev)
    # ---- commit to the DB (nothing above touched it)
    for (e, _, _), d in zip(items, new_digests):
        db.add_signature(d, e)
    tables, index = {}, {}
    for kind, (fr, idx, (px, py, poff)) in fitted.items():
        tables[kind] = fr
        x, y, off = px.cpu().numpy().view(np.uint32), py.cpu().numpy(), poff.cpu().numpy()
        for row, i in enumerate(idx):
            e, m, _ = items[i]
            a, z = int(off[row]), int(off[row + 1])
            db.insert_measurements(new_digests[i], x[:, a:z], y[a:z],
                                   sweep_points(e, grid, m.max_context))
            index[new_digests[i]] = (kind, row)
    for (m, b, lo, hi) in configs:
        cid = db.add_configuration(manifest.hardware.name, m.name, b.name, manifest.tp_degree)
        for i in range(lo, hi):
            db.add_model_operation(cid, digs[i], entries[i].repeat_count)
    # ---- signatures the manifest shares with what the DB already held
    old = [d for d in dict.fromkeys(digs) if d not in index]
    if old:
        sub = LatencyDB()
        for d in old:
            row = db.signature(d)
            if d not in db.measurements:
                raise InsufficientData(d.hex(), 0, NEED[row.kind])
            sub._index[d] = len(sub.signatures)
            sub.signatures.append(row)
            sub.measurements[d] = db.measurements[d]
        prev = fit_db(sub, dev)
        for kind, fr in prev.tables.items():
            base = tables[kind].table.shape[0] if kind in tables else 0
            if kind in tables:
                t = tables[kind]
                tables[kind] = FitResult(kind, torch.cat([t.table, fr.table]),
                                         torch.cat([t.fit_err, fr.fit_err]),
                                         torch.cat([t.status, fr.status]))
            else:
                tables[kind] = fr
            for d, (k, r) in prev.index.items():
                if k == kind:
                    index[d] = (kind, base + r)
    torch.cuda.synchronize(dev)
    return db, Regressors(tables, index, dev), report
