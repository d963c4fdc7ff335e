"""Single-file latency database (store.py, D4/D5 :516-517).

CPU-only: the store is host code.  Signatures are registered with synthetic
digests so no GPU hashing is needed."""

from __future__ import annotations

import json
import sqlite3

import numpy as np
import pytest

from paper_2605_07985_b200 import store
from paper_2605_07985_b200.errors import DuplicateKey, StoreUnavailable
from paper_2605_07985_b200.profiler import (LatencyDB, point_features, sweep, sweep_points)
from paper_2605_07985_b200.records import synthesize_entries


def _db(corpus, n_models=2):
    """A DB shaped like profile_corpus output, built without the GPU dedup."""
    db = LatencyDB()
    model, backend = corpus.models[0], corpus.backends[0]
    cid = db.add_configuration(corpus.hardware.name, model.name, backend.name, 1)
    ents = synthesize_entries(model, backend, 1)
    for i, e in enumerate(ents):
        d = bytes([i + 1]) * 32
        db.add_signature(d, e)
        db.add_model_operation(cid, d, e.repeat_count)
        x, y = sweep(e, corpus.grid, model, corpus.hardware, backend)
        db.insert_measurements(d, x, y, sweep_points(e, corpus.grid, model.max_context))
    db.insert_comm("nvlink-like", 2, 1 << 20, 7.62144e-6)   # SPEC.md:489-493 golden
    return db, ents


def _same(a: LatencyDB, b: LatencyDB):
    assert a.configurations == b.configurations
    assert [(s.digest, s.op_name, s.granularity, s.kind, s.feature, s.components)
            for s in a.signatures] == [(s.digest, s.op_name, s.granularity, s.kind, s.feature,
                                        s.components) for s in b.signatures]
    assert a.model_operations == b.model_operations
    assert set(a.measurements) == set(b.measurements)
    for d in a.measurements:
        ka = sorted(zip(map(tuple, a.measurements[d][0].T.tolist()), a.measurements[d][1]))
        kb = sorted(zip(map(tuple, b.measurements[d][0].T.tolist()), b.measurements[d][1]))
        assert ka == kb                              # exact f64 round trip
    assert a.comm_measurements == b.comm_measurements


def test_sqlite_roundtrip_is_exact(corpus, tmp_path):
    db, _ = _db(corpus)
    p = tmp_path / "latency.db"
    db.save(p)
    assert not (tmp_path / "latency.db.tmp").exists()       # atomic rename
    back = LatencyDB.load(p)
    _same(db, back)
    d = db.signatures[0].digest
    assert back.workloads[d] == db.workloads[d]
    assert back.sources[d] == ["oracle"] * db.measurements[d][1].shape[0]
    con = sqlite3.connect(str(p))
    tabs = {r[0] for r in con.execute("SELECT name FROM sqlite_master WHERE type='table'")}
    assert {"configurations", "signatures", "model_operations", "measurements",
            "comm_measurements"} <= tabs
    n = con.execute("SELECT COUNT(*) FROM measurements").fetchone()[0]
    assert n == sum(y.shape[0] for _, y in db.measurements.values())
    con.close()


def test_schema_dump_matches_store(tmp_path):
    text = store.schema_dump()
    for t in ("configurations", "signatures", "model_operations", "measurements",
              "comm_measurements"):
        assert f"CREATE TABLE {t}(" in text
    assert "REFERENCES signatures(hash)" in text and "UNIQUE(signature_hash, workload)" in text
    assert LatencyDB().schema_dump() == text


def test_jsonl_export_import_roundtrip(corpus, tmp_path):
    db, ents = _db(corpus)
    p = tmp_path / "m.jsonl"
    n = store.export_jsonl(db, p)
    lines = p.read_text().splitlines()
    assert n == len(lines) == sum(y.shape[0] for _, y in db.measurements.values())
    rec = json.loads(lines[0])
    assert set(rec) == {"sig", "workload", "features", "latency_s", "source"}
    # import into a DB holding only the signatures: identical measurements, source=imported
    fresh = LatencyDB()
    for s in db.signatures:
        fresh._index[s.digest] = len(fresh.signatures)
        fresh.signatures.append(s)
    assert store.import_jsonl(fresh, p) == n
    for d, (x, y) in db.measurements.items():
        assert np.array_equal(fresh.measurements[d][0], x)
        assert np.array_equal(fresh.measurements[d][1], y)
        assert fresh.point_sources(d) == ["imported"] * y.shape[0]
    # records carrying only the workload derive the features like the sweep does
    att = [i for i, e in enumerate(ents) if e.feature == "attention"][0]
    d = db.signatures[att].digest
    wl_only = [json.dumps({"sig": d.hex(), "workload": w, "latency_s": float(yv)})
               for w, yv in zip(db.workloads[d], db.measurements[d][1])]
    fresh2 = LatencyDB()
    fresh2._index[d] = 0
    fresh2.signatures.append(db.signatures[att])
    store.import_jsonl(fresh2, wl_only)
    assert np.array_equal(fresh2.measurements[d][0], db.measurements[d][0])
    assert tuple(fresh2.measurements[d][0][:, 0]) == point_features(ents[att], db.workloads[d][0])


def test_import_rejects_conflicts_and_dangling(corpus, tmp_path):
    db, _ = _db(corpus)
    d = db.signatures[0].digest
    x, y = db.measurements[d]
    same = json.dumps({"sig": d.hex(), "features": [int(v) for v in x[:, 0]], "latency_s": float(y[0])})
    store.import_jsonl(db, [same])                                   # identical key+value: ok
    bad = json.dumps({"sig": d.hex(), "features": [int(v) for v in x[:, 0]],
                      "latency_s": float(y[0]) * 2})
    with pytest.raises(DuplicateKey):
        store.import_jsonl(db, [bad])
    dangling = json.dumps({"sig": "ab" * 32, "features": [1], "latency_s": 1e-5})
    with pytest.raises(StoreUnavailable):                            # referential integrity
        store.import_jsonl(db, [dangling])
    with pytest.raises(StoreUnavailable):
        db.add_model_operation(0, b"\xee" * 32, 1)
    with pytest.raises(StoreUnavailable):
        db.add_model_operation(7, d, 1)
    with pytest.raises(DuplicateKey):
        db.insert_comm("nvlink-like", 2, 1 << 20, 8e-6)


def test_query_exact_range_and_unknown(corpus):
    db, ents = _db(corpus)
    lin = [i for i, e in enumerate(ents) if e.name == "linear"][0]
    d = db.signatures[lin].digest
    rows = store.query(db, d)
    assert len(rows) == db.measurements[d][1].shape[0]
    f0, y0 = rows[2]
    assert store.query(db, d, features=f0) == [(f0, y0)]
    inside = store.query(db, d, lo=(16,), hi=(512,))
    assert [f[0] for f, _ in inside] == [16, 128, 512]
    assert store.query(db, b"\x00" * 32) == []


def test_load_missing_or_foreign_file(tmp_path):
    with pytest.raises(StoreUnavailable):
        LatencyDB.load(tmp_path / "nope.db")
    other = tmp_path / "other.db"
    con = sqlite3.connect(str(other))
    con.execute("CREATE TABLE meta(key TEXT, value TEXT)")
    con.commit()
    con.close()
    with pytest.raises(StoreUnavailable):
        LatencyDB.load(other)


def test_sources_are_per_point_and_survive_every_format(corpus, tmp_path):
    """SPEC D4: imported rows merged into a signature that has oracle rows keep
    source=imported per row through save/load, the npz snapshot and JSON lines."""
    db, ents = _db(corpus)
    lin = [i for i, e in enumerate(ents) if e.name == "linear"][0]
    d = db.signatures[lin].digest
    n0 = db.measurements[d][1].shape[0]
    new = json.dumps({"sig": d.hex(), "features": [3], "latency_s": 4.2e-5})
    store.import_jsonl(db, [new])
    want = ["oracle"] * n0 + ["imported"]
    assert db.point_sources(d) == want
    for path in (tmp_path / "a.db", tmp_path / "a.npz"):
        db.save(path)
        back = LatencyDB.load(path)
        _same(db, back)
        assert back.point_sources(d) == want
        assert back.workloads == db.workloads
        assert [s.components for s in back.signatures] == [s.components for s in db.signatures]
    p = tmp_path / "m.jsonl"
    store.export_jsonl(db, p)
    srcs = [json.loads(ln)["source"] for ln in p.read_text().splitlines()
            if json.loads(ln)["sig"] == d.hex()]
    assert srcs == want


def test_npz_snapshot_loads_without_pickle(corpus, tmp_path):
    db, _ = _db(corpus)
    p = tmp_path / "s.npz"
    db.save(p)
    z = np.load(p, allow_pickle=False)                   # no object arrays anywhere
    assert all(z[k].dtype != object for k in z.files)
    _same(db, LatencyDB.load(p))
