"""Single-file latency database (SURVEY §8(f) row f3; SPEC.md:430-435, :496-504,
D4/D5 :516-517, External Interfaces :522).

The GPU path works on the in-memory ``profiler.LatencyDB``.  This module
persists it as one SQLite file with the Fig. 9 logical schema, and adds the
other store operations the SPEC names:

* ``save`` / ``load`` are atomic.  The file is written beside the target and
  then renamed.  Foreign keys enforce referential integrity:
  model_operations and measurements must reference an existing signature.
* ``export_jsonl`` / ``import_jsonl`` carry measurements as JSON lines
  ``{sig, workload, latency_s, source}`` (D4).  Imported rows get
  ``source = "imported"``.  Re-importing a key with a different latency raises
  ``DuplicateKey``.
* ``query`` looks up one signature's records, either by exact workload
  features or by a feature range (db_query).
* ``schema_dump`` returns the logical schema text for conformance checking
  (D5).

Python's stdlib sqlite3 is the storage engine.  The SPEC leaves the engine to
the implementation.
"""

from __future__ import annotations

import json
import os
import sqlite3
from types import SimpleNamespace
from typing import Iterable, Optional, Sequence

import numpy as np

from .errors import StoreUnavailable

STORE_VERSION = 1

DDL = (
    "CREATE TABLE meta(key TEXT PRIMARY KEY, value TEXT NOT NULL);",
    "CREATE TABLE configurations(\n"
    "  id INTEGER PRIMARY KEY, hardware TEXT NOT NULL, model TEXT NOT NULL,\n"
    "  backend TEXT NOT NULL, tp_degree INTEGER NOT NULL,\n"
    "  UNIQUE(hardware, model, backend, tp_degree));",
    "CREATE TABLE signatures(\n"
    "  hash BLOB PRIMARY KEY CHECK(length(hash) = 32), op_name TEXT NOT NULL,\n"
    "  granularity TEXT NOT NULL, kind INTEGER NOT NULL, feature TEXT NOT NULL,\n"
    "  components TEXT NOT NULL, ord INTEGER NOT NULL);",
    "CREATE TABLE model_operations(\n"
    "  config_id INTEGER NOT NULL REFERENCES configurations(id),\n"
    "  signature_hash BLOB NOT NULL REFERENCES signatures(hash),\n"
    "  repeat_count INTEGER NOT NULL, seq INTEGER NOT NULL);",
    "CREATE TABLE measurements(\n"
    "  signature_hash BLOB NOT NULL REFERENCES signatures(hash),\n"
    "  f0 INTEGER NOT NULL, f1 INTEGER NOT NULL, f2 INTEGER NOT NULL,  -- regression features\n"
    "  workload TEXT, latency_s REAL NOT NULL CHECK(latency_s > 0),\n"
    "  source TEXT NOT NULL, seq INTEGER NOT NULL,\n"
    "  PRIMARY KEY(signature_hash, seq), UNIQUE(signature_hash, workload));",
    "CREATE INDEX measurements_by_features ON measurements(signature_hash, f0, f1, f2);",
    "CREATE TABLE comm_measurements(\n"
    "  topology TEXT NOT NULL, tp_degree INTEGER NOT NULL, bytes INTEGER NOT NULL,\n"
    "  latency_s REAL NOT NULL CHECK(latency_s > 0),\n"
    "  PRIMARY KEY(topology, tp_degree, bytes));",
)


def schema_dump() -> str:
    """Logical schema of the store (the ``schema-dump`` output, D5 SPEC.md:517)."""
    return f"-- dooly latency database, store version {STORE_VERSION}\n" + "\n".join(DDL) + "\n"


def _connect(path, create: bool) -> sqlite3.Connection:
    if not create and not os.path.exists(path):
        raise StoreUnavailable(f"no latency database at {path}")
    try:
        con = sqlite3.connect(str(path))
        con.execute("PRAGMA foreign_keys = ON")
        return con
    except sqlite3.Error as exc:
        raise StoreUnavailable(str(exc)) from exc


def _features(x: np.ndarray, i: int) -> tuple:
    f = [int(v) for v in x[:, i]]
    return tuple(f + [0] * (3 - len(f)))


def save(db, path) -> None:
    """Write ``db`` to ``path`` atomically (temp file + rename), one transaction."""
    path = str(path)
    tmp = path + ".tmp"
    if os.path.exists(tmp):
        os.remove(tmp)
    con = _connect(tmp, create=True)
    try:
        with con:
            for stmt in DDL:
                con.execute(stmt)
            con.execute("INSERT INTO meta VALUES ('store_version', ?)", (str(STORE_VERSION),))
            con.executemany("INSERT INTO configurations VALUES (?, ?, ?, ?, ?)",
                            [(i, *c) for i, c in enumerate(db.configurations)])
            con.executemany("INSERT INTO signatures VALUES (?, ?, ?, ?, ?, ?, ?)",
                            [(s.digest, s.op_name, s.granularity, int(s.kind), s.feature,
                              s.components, i) for i, s in enumerate(db.signatures)])
            con.executemany("INSERT INTO model_operations VALUES (?, ?, ?, ?)",
                            [(int(c), d, int(r), i) for i, (c, d, r) in enumerate(db.model_operations)])
            rows = []
            for d, (x, y) in db.measurements.items():
                wl = db.workloads.get(d) or [None] * y.shape[0]
                src = db.point_sources(d)
                for i in range(y.shape[0]):
                    rows.append((d, *_features(x, i), None if wl[i] is None else json.dumps(wl[i]),
                                 float(y[i]), src[i], i))
            con.executemany("INSERT INTO measurements VALUES (?, ?, ?, ?, ?, ?, ?, ?)", rows)
            con.executemany("INSERT INTO comm_measurements VALUES (?, ?, ?, ?)",
                            [(*k, v) for k, v in db.comm_measurements.items()])
    except sqlite3.IntegrityError as exc:
        con.close()
        os.remove(tmp)
        raise StoreUnavailable(f"referential integrity: {exc}") from exc
    con.close()
    os.replace(tmp, path)


def load(path):
    """Read a store written by ``save`` back into a ``profiler.LatencyDB``."""
    from .profiler import LatencyDB, SignatureRow
    from . import _lib

    con = _connect(path, create=False)
    try:
        ver = con.execute("SELECT value FROM meta WHERE key = 'store_version'").fetchone()
        if ver is None or int(ver[0]) != STORE_VERSION:
            raise StoreUnavailable(f"{path}: store version {ver} != {STORE_VERSION}")
        db = LatencyDB()
        db.configurations = [tuple(r) for r in con.execute(
            "SELECT hardware, model, backend, tp_degree FROM configurations ORDER BY id")]
        for h, name, gran, kind, feat, comp in con.execute(
                "SELECT hash, op_name, granularity, kind, feature, components FROM signatures "
                "ORDER BY ord"):
            d = bytes(h)
            db._index[d] = len(db.signatures)
            db.signatures.append(SignatureRow(d, name, gran, int(kind), feat, comp))
        db.model_operations = [(int(c), bytes(h), int(r)) for c, h, r in con.execute(
            "SELECT config_id, signature_hash, repeat_count FROM model_operations ORDER BY seq")]
        cur = con.execute("SELECT signature_hash, f0, f1, f2, workload, latency_s, source "
                          "FROM measurements ORDER BY signature_hash, seq")
        groups: dict = {}
        for h, f0, f1, f2, wl, lat, src in cur:
            groups.setdefault(bytes(h), []).append((f0, f1, f2, wl, lat, src))
        for d, rows in groups.items():
            P = _lib.PLANES[db.signature(d).kind]
            x = np.array([r[:P] for r in rows], dtype=np.uint32).T.reshape(P, -1)
            db.measurements[d] = (np.ascontiguousarray(x), np.array([r[4] for r in rows]))
            db.workloads[d] = [None if r[3] is None else json.loads(r[3]) for r in rows]
            db.sources[d] = [r[5] for r in rows]
        db.comm_measurements = {(t, int(tp), int(b)): float(v) for t, tp, b, v in con.execute(
            "SELECT topology, tp_degree, bytes, latency_s FROM comm_measurements")}
        return db
    except sqlite3.Error as exc:
        raise StoreUnavailable(str(exc)) from exc
    finally:
        con.close()


def export_jsonl(db, path) -> int:
    """One JSON line per measurement: {sig, workload, features, latency_s, source} (D4)."""
    n = 0
    with open(path, "w") as f:
        for d, (x, y) in db.measurements.items():
            wl = db.workloads.get(d) or [None] * y.shape[0]
            src = db.point_sources(d)
            for i in range(y.shape[0]):
                rec = {"sig": d.hex(), "workload": wl[i],
                       "features": [int(v) for v in x[:, i]],
                       "latency_s": float(y[i]), "source": src[i]}
                f.write(json.dumps(rec, sort_keys=True) + "\n")
                n += 1
    return n


def _features_of(db, digest: bytes, rec: dict) -> tuple:
    """Regression features of a JSON-lines record: given, or derived from the
    workload exactly as the sweep derives them (profiler.point_features)."""
    from .profiler import point_features

    if rec.get("features") is not None:
        return tuple(int(v) for v in rec["features"])
    wl = rec.get("workload")
    if not isinstance(wl, dict):
        raise StoreUnavailable(f"record for {digest.hex()[:12]} has neither features nor workload")
    row = db.signature(digest)
    comp = json.loads(row.components or "{}")
    entry = SimpleNamespace(feature=row.feature, window=comp.get("window"))
    return tuple(int(v) for v in point_features(entry, wl))


def import_jsonl(db, lines: Iterable[str] | str, source: str = "imported") -> int:
    """Import measurements (D4).  Every record must name a signature already in
    the DB (referential integrity); a key re-imported with a different latency
    raises DuplicateKey.  Returns the number of records read."""
    if isinstance(lines, (str, os.PathLike)):
        with open(lines) as f:
            return import_jsonl(db, f.readlines(), source)
    per_sig: dict = {}
    n = 0
    for ln in lines:
        ln = ln.strip()
        if not ln:
            continue
        rec = json.loads(ln)
        d = bytes.fromhex(rec["sig"])
        if not db.has(d):
            raise StoreUnavailable(f"measurement references unknown signature {rec['sig'][:12]}")
        lat = float(rec["latency_s"])
        per_sig.setdefault(d, []).append((_features_of(db, d, rec), lat, rec.get("workload")))
        n += 1
    for d, rows in per_sig.items():
        x = np.array([r[0] for r in rows], dtype=np.uint32).T
        db.insert_measurements(d, x, np.array([r[1] for r in rows]), [r[2] for r in rows],
                               source=source)
    return n


def query(db, digest: bytes, features: Optional[Sequence[int]] = None,
          lo: Optional[Sequence[int]] = None, hi: Optional[Sequence[int]] = None) -> list:
    """db_query: records of one signature, all of them, the one
    at exact ``features``, or those inside the box [lo, hi].  Unknown hash -> []."""
    if digest not in db.measurements:
        return []
    x, y = db.measurements[digest]
    out = []
    for i in range(y.shape[0]):
        f = tuple(int(v) for v in x[:, i])
        if features is not None and f != tuple(features):
            continue
        if lo is not None and any(a < b for a, b in zip(f, lo)):
            continue
        if hi is not None and any(a > b for a, b in zip(f, hi)):
            continue
        out.append((f, float(y[i])))
    return out


# ------------------------------------------------- regressors beside the DB


REG_DDL = (
    "CREATE TABLE meta(key TEXT PRIMARY KEY, value TEXT NOT NULL);",
    "CREATE TABLE regressors(\n"
    "  signature_hash BLOB PRIMARY KEY CHECK(length(signature_hash) = 32),\n"
    "  kind INTEGER NOT NULL, ord INTEGER NOT NULL, row BLOB NOT NULL,\n"
    "  fit_error REAL, status INTEGER NOT NULL, fingerprint BLOB NOT NULL);",
)


def regressor_path(db_path) -> str:
    """The regressor cache that lives beside a DB file."""
    return str(db_path) + ".regressors"


def measurement_fingerprint(x: np.ndarray, y: np.ndarray) -> bytes:
    """SHA-256 of a signature's training points: a cached regressor is valid
    only for exactly the measurements it was fitted on."""
    import hashlib

    h = hashlib.sha256(np.ascontiguousarray(x, dtype=np.uint32).tobytes())
    h.update(np.ascontiguousarray(y, dtype=np.float64).tobytes())
    return h.digest()


def save_regressors(db_path, regs, db) -> None:
    """Write every fitted row (the exact device bytes), its fit_error, status and
    the fingerprint of the measurements it came from, atomically."""
    path = regressor_path(db_path)
    tmp = path + ".tmp"
    if os.path.exists(tmp):
        os.remove(tmp)
    host = {k: (fr.table.cpu().numpy(), fr.fit_err.cpu().numpy(), fr.status.cpu().numpy())
            for k, fr in regs.tables.items()}
    rows = []
    for d, (kind, row) in regs.index.items():
        t, fe, st = host[kind]
        x, y = db.measurements[d]
        rows.append((d, int(kind), int(row), t[row].tobytes(), float(fe[row]), int(st[row]),
                     measurement_fingerprint(x, y)))
    con = _connect(tmp, create=True)
    with con:
        for stmt in REG_DDL:
            con.execute(stmt)
        con.execute("INSERT INTO meta VALUES ('store_version', ?)", (str(STORE_VERSION),))
        con.executemany("INSERT INTO regressors VALUES (?, ?, ?, ?, ?, ?, ?)", rows)
    con.close()
    os.replace(tmp, path)


def load_regressors(db_path, db, device=None):
    """The cached Regressors for ``db``, or None when the cache is missing,
    lacks a measured signature, or any fingerprint is stale."""
    import torch

    from . import _lib
    from .profiler import _device
    from .sim import FitResult, Regressors

    path = regressor_path(db_path)
    if not os.path.exists(path):
        return None
    con = _connect(path, create=False)
    try:
        rows = con.execute("SELECT signature_hash, kind, ord, row, fit_error, status, fingerprint "
                           "FROM regressors ORDER BY kind, ord").fetchall()
    except sqlite3.Error:
        return None
    finally:
        con.close()
    have = {bytes(r[0]): r for r in rows}
    if set(have) != set(db.measurements):
        return None
    for d, (x, y) in db.measurements.items():
        if bytes(have[d][6]) != measurement_fingerprint(x, y):
            return None
    dev = _device(device)
    tables, index = {}, {}
    for kind in sorted({int(r[1]) for r in rows}):
        ks = [r for r in rows if int(r[1]) == kind]
        if [int(r[2]) for r in ks] != list(range(len(ks))):
            return None
        tab = np.frombuffer(b"".join(bytes(r[3]) for r in ks), dtype=np.uint8)
        tab = tab.reshape(len(ks), _lib.ROW_BYTES[kind])
        fe = np.array([np.nan if r[4] is None else r[4] for r in ks], dtype=np.float64)
        st = np.array([r[5] for r in ks], dtype=np.uint8)
        tables[kind] = FitResult(kind, torch.from_numpy(tab.copy()).to(dev),
                                 torch.from_numpy(fe).to(dev), torch.from_numpy(st).to(dev))
        for r in ks:
            index[bytes(r[0])] = (kind, int(r[2]))
    return Regressors(tables, index, dev)
