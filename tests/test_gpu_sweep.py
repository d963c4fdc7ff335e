"""K5 fused sweep -> fit vs the ORACLE sweep (oracle/profiler.py
op_cost / oracle_latency) + oracle fit."""

from __future__ import annotations

import numpy as np
import pytest

from helpers import oracle_sweep, rows_to_table
from oracle import sim as osim

pytestmark = pytest.mark.gpu


def _unique_entries(manifest):
    from paper_2605_07985_b200.records import canonical_bytes, synthesize_entries

    seen, out = set(), []
    for m in manifest.models:
        for b in manifest.backends:
            for e in synthesize_entries(m, b, manifest.tp_degree):
                key = canonical_bytes(e)
                if key not in seen:
                    seen.add(key)
                    out.append((m, b, e))
    return out


@pytest.mark.parametrize("name", ["corpus12", "mixtral", "fixtures", "llama70b"])
def test_profile_fit_matches_host_sweep_and_oracle(name, dev):
    from paper_2605_07985_b200 import modelir, profiler

    man = modelir.load_manifest(modelir.builtin_manifest_path(name))
    items = _unique_entries(man)
    checked = 0
    # one launch per (model, backend) group: descriptors carry the model caps
    groups: dict = {}
    for m, b, e in items:
        groups.setdefault((m.name, b.name), (m, b, []))[2].append(e)
    for (mname, bname), (m, b, ents) in groups.items():
        res = profiler.profile_fit([(e, m, b) for e in ents], man.hardware, man.grid, dev,
                                   emit_points=True)
        for kind, (fr, idx, (px, py, poff)) in res.items():
            off = poff.cpu().numpy()
            gx = px.cpu().numpy().view(np.uint32)
            gy = py.cpu().numpy()
            rows = rows_to_table(kind, fr.rows())
            for j, i in enumerate(idx):
                x, y = oracle_sweep(ents[i], man.grid, m, man.hardware, b)
                a, z = off[j], off[j + 1]
                assert np.array_equal(gx[:, a:z], x), (ents[i].name, j)
                assert np.array_equal(gy[a:z], y), ents[i].name       # bit-identical latencies
                ref = osim.fit(kind, x, y, np.array([0, y.shape[0]], dtype=np.int64))
                if ref["status"][0]:
                    assert fr.status.cpu().numpy()[j] == 1
                    continue
                c = rows["coef"][j]
                assert np.max(np.abs(c - ref["coef"][0])) <= 1e-9 * np.max(np.abs(ref["coef"][0]))
                fe = fr.fit_err.cpu().numpy()[j]
                assert abs(fe - ref["fit_err"][0]) <= 1e-9 * ref["fit_err"][0] + 1e-12
                checked += 1
    assert checked >= 10


def test_profile_and_fit_equals_db_fit(corpus, dev):
    """The fused path produces the same regressors as host sweep -> LatencyDB -> K2."""
    from paper_2605_07985_b200.profiler import profile_and_fit, profile_corpus
    from paper_2605_07985_b200.sim import fit

    db_a, regs_a, rep_a = profile_and_fit(corpus, device=dev)
    db_b, rep_b = profile_corpus(corpus, device=dev)
    regs_b = fit(db_b, dev)
    assert rep_a == rep_b and set(regs_a.index) == set(regs_b.index)
    for d in regs_a.index:
        ca = np.array(regs_a.regressor(d).coefficients)
        cb = np.array(regs_b.regressor(d).coefficients)
        assert np.max(np.abs(ca - cb)) <= 1e-9 * np.max(np.abs(cb))
        assert regs_a.regressor(d).box == regs_b.regressor(d).box


def test_profile_and_fit_with_prepopulated_db(corpus, dev):
    """a second profile_and_fit over a manifest sharing signatures
    with the DB returns regressors for EVERY referenced signature, writes the
    swept measurements of the new ones (so sim.fit(db) covers them), and
    records model_operations for all entries."""
    from paper_2605_07985_b200 import modelir
    from paper_2605_07985_b200.profiler import profile_and_fit
    from paper_2605_07985_b200.records import runnable_entries, canonical_bytes
    from paper_2605_07985_b200.sim import fit

    first = modelir.CorpusManifest(corpus.models[:2], corpus.backends, corpus.hardware, 1,
                                   corpus.grid)
    db, regs1, _ = profile_and_fit(first, device=dev)
    n_sig1 = len(db.signatures)
    db, regs2, rep = profile_and_fit(corpus, db=db, device=dev)
    assert sum(r["profiled"] for r in rep) == len(db.signatures) - n_sig1
    assert set(db.measurements) == {s.digest for s in db.signatures}
    referenced = {d for _, d, _ in db.model_operations}
    assert referenced <= set(regs2.index)
    assert len(db.model_operations) == sum(len(runnable_entries(m, b, 1))
                                           for m in first.models + corpus.models
                                           for b in corpus.backends)
    ref = fit(db, dev)
    for d in referenced:
        a = np.array(regs2.regressor(d).coefficients)
        b = np.array(ref.regressor(d).coefficients)
        assert np.max(np.abs(a - b)) <= 1e-9 * np.max(np.abs(b))
        assert regs2.regressor(d).box == ref.regressor(d).box


def test_profile_and_fit_failure_leaves_db_untouched(fixtures_manifest, dev, monkeypatch):
    from paper_2605_07985_b200 import records
    from paper_2605_07985_b200.errors import OraclePanic
    from paper_2605_07985_b200.profiler import LatencyDB, profile_and_fit

    real = records.runnable_entries

    def with_unknown_op(m, b, tp=1, producer="trace"):
        ents = real(m, b, tp, producer)
        e = ents[-1]
        return ents + [records.RunnableEntry("operator", "mystery_op", e.arg_template,
                                             kernel_symbols=("k",))]

    monkeypatch.setattr(records, "runnable_entries", with_unknown_op)
    db = LatencyDB()
    with pytest.raises(OraclePanic):
        profile_and_fit(fixtures_manifest, db=db, device=dev)
    assert db.signatures == [] and db.measurements == {} and db.model_operations == []


def test_fit_cached_beside_the_db(fixtures_manifest, dev, tmp_path, monkeypatch):
    """fit runs lazily and caches regressors alongside the db —
    reloaded without refitting while the measurements are unchanged, refitted
    when they change."""
    import paper_2605_07985_b200.sim as sim
    from paper_2605_07985_b200 import store
    from paper_2605_07985_b200.profiler import profile_corpus

    db, _ = profile_corpus(fixtures_manifest, device=dev)
    path = tmp_path / "lat.db"
    db.save(path)
    regs = sim.fit_cached(db, path, dev)
    assert (tmp_path / "lat.db.regressors").exists()
    calls = []
    monkeypatch.setattr(sim, "fit", lambda *a, **k: calls.append(1) or None)
    again = sim.fit_cached(LatencyDB_load(path), path, dev)
    assert calls == []                                           # served from the cache
    for d in regs.index:
        assert regs.regressor(d) == again.regressor(d)
    monkeypatch.undo()
    d = db.signatures[0].digest
    x, y = db.measurements[d]
    db.measurements[d] = (x, y * 1.5)                            # stale now
    assert store.load_regressors(path, db, dev) is None
    fresh = sim.fit_cached(db, path, dev)
    assert fresh.regressor(d).coefficients != regs.regressor(d).coefficients


def LatencyDB_load(path):
    from paper_2605_07985_b200.profiler import LatencyDB

    return LatencyDB.load(path)
