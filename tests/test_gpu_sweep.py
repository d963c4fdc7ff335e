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
