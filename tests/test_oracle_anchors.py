"""The reference's own run-level anchors, on the CPU oracle:

* the analytical latency model restated in oracle/profiler.py
  is bit-identical to the package's host sweep for every entry of every
  builtin manifest (C1-C4, fixtures);
* reference_run: brute-force oracle evaluation of every op at
  each iteration's concrete dims, sharing the scheduler with run;
* an exactly-affine oracle gives run == reference_run within 1e-6
  relative on every iteration (oracle fit -> oracle run here; the GPU form is
  tests/test_gpu_anchors.py);
* A6: 10,000 randomized scheduler property cases.
"""

from __future__ import annotations

import math
import time

import numpy as np
import pytest

from helpers import (ATTN, affine_oracle_batch, affine_oracle_coefs, affine_oracle_sweep,
                     oracle_grid, oracle_hw, oracle_ops, oracle_sweep)
from oracle import profiler as oprof
from oracle import sim as osim

MANIFESTS = ["corpus12", "mixtral", "fixtures", "llama70b"]


def _manifest(name):
    from paper_2605_07985_b200 import modelir

    return modelir.load_manifest(modelir.builtin_manifest_path(name))


@pytest.mark.parametrize("name", MANIFESTS)
def test_oracle_sweep_equals_package_sweep(name):
    """Independent restatement of op_cost/oracle_latency/sweep_points vs the
    package's host sweep (which the K5 device sweep is held to): bit-identical."""
    from paper_2605_07985_b200 import profiler
    from paper_2605_07985_b200.records import synthesize_entries

    man = _manifest(name)
    n = 0
    kinds = set()
    for m in man.models:
        for b in man.backends:
            for e in synthesize_entries(m, b, man.tp_degree):
                x, y = oracle_sweep(e, man.grid, m, man.hardware, b)
                px, py = profiler.sweep(e, man.grid, m, man.hardware, b)
                assert np.array_equal(x, px), (m.name, e.name)
                assert np.array_equal(y.view(np.uint64), py.view(np.uint64)), (m.name, e.name)
                n += 1
                kinds.add(e.name)
    assert n >= 10
    if name == "mixtral":
        assert {"fused_moe", "topk_softmax", "attention", "linear"} <= kinds


def test_op_cost_spec_examples(corpus):
    hw = oracle_hw(corpus.hardware)
    # SPEC.md:480 attention prefill: 2*2*T^2*D*H_q flops at one request without cache
    att = {"name": "attention", "feature": "attention",
           "arg_template": [[[7, "NT"], [32, "MC"], [128, "MC"]], [[7, "NT"], [8, "MC"], [128, "MC"]],
                            [[7, "NT"], [8, "MC"], [128, "MC"]]], "kernel_symbols": []}
    T = 1024
    f, _ = oprof.op_cost(att, {"phase": "prefill", "num_toks": T, "num_reqs": 1, "kv_len": 0}, 2)
    assert f == 2 * 2 * T * T * 128 * 32
    # matmul golden through the generic op table
    lin = {"name": "linear", "feature": "num_toks",
           "arg_template": [[[7, "NT"], [4096, "MC"]], [[4096, "MC"], [4096, "MC"]]],
           "kernel_symbols": ["gemm_f16_tn"]}
    lat = oprof.oracle_latency(lin, {"num_toks": 1024}, hw, (), 2)
    assert abs(lat - 1.1512736656410257e-4) <= 1e-9
    # zero-flop op -> overhead only
    rs = {"name": "reshape", "feature": "num_toks", "arg_template": [], "kernel_symbols": []}
    assert oprof.oracle_latency(rs, {"num_toks": 99}, hw, (), 2) == 5e-6
    # modelir.py:134-143 longest-prefix multiplier (fa decode: 1.05 * 1.0 * 0.95)
    fa = corpus.backend("flashattention-like")
    syms = fa.attention_kernels(32, 8, 128, None, "decode")
    assert oprof.multiplier(fa.cost_multiplier, syms) == fa.multiplier(syms)


def test_batch_latency_consistent_with_sweep_points(corpus):
    """The concrete-batch cost of reference_run equals the sweep-point cost at
    uniform batches (integral tokens per request)."""
    from paper_2605_07985_b200.records import synthesize_entries

    m = corpus.model("llama-3-8b-like")
    b = corpus.backend("flashattention-like")
    hw = oracle_hw(corpus.hardware)
    for e in synthesize_entries(m, b, 1):
        ej = e.to_json()
        for t, r, c, phase in ((512, 8, 4096, "prefill"), (64, 64, 512, "decode"),
                               (2048, 1, 0, "prefill")):
            q = t // r if phase == "prefill" else 1
            reqs = [(q, phase == "prefill", c)] * r
            pt = {"phase": phase, "num_toks": t, "num_reqs": r, "kv_len": c}
            got = oprof.batch_latency(ej, reqs, hw, b.cost_multiplier, m.dtype_bytes)
            want = oprof.oracle_latency(ej, pt, hw, b.cost_multiplier, m.dtype_bytes)
            assert math.isclose(got, want, rel_tol=1e-12), (e.name, phase)


def _c1(corpus):
    m = corpus.model("llama-3-8b-like")
    b = corpus.backend("flashattention-like")
    return m, b


def _c1_requests(n, rate, seed=1):
    from paper_2605_07985_b200 import modelir

    spec = modelir.WorkloadSpec(mode="stream", rate=rate, num_requests=n,
                                prompt_len=modelir.LengthDist(950, 1232),
                                output_len=modelir.LengthDist(388, 397), max_len=8192)
    reqs = modelir.sample_workload(spec, seed=seed)
    return ([r.arrival_s for r in reqs], [r.prompt_tokens for r in reqs],
            [r.output_tokens for r in reqs], [r.cached_tokens for r in reqs])


def test_reference_run_kats(corpus):
    """SPEC.md:606-612 examples + SPEC.md:602 single-request TTFT."""
    from paper_2605_07985_b200.records import synthesize_entries

    m, b = _c1(corpus)
    ents = [e.to_json() for e in synthesize_entries(m, b, 1)]
    hw = oracle_hw(corpus.hardware)
    kw = dict(entries=ents, hw=hw, cost_multiplier=b.cost_multiplier, dtype_bytes=m.dtype_bytes,
              chunk=8192, max_batch=256, kv_bytes_per_token=m.kv_bytes_per_token(),
              kv_capacity=10 ** 11, log=True)
    r = osim.reference_run([0.0], [10000], [3], [0], **kw)
    assert [f[0] for f in r["feats"]][:2] == [8192, 1808]
    assert r["ttft"][0] == r["lat"][0] + r["lat"][1]
    # each iteration = sum of repeat x oracle at the concrete batch (brute force)
    lat0 = 0.0
    for e in ents:
        lat0 = lat0 + float(e["repeat_count"]) * oprof.batch_latency(
            e, [(8192, True, 0)], hw, b.cost_multiplier, m.dtype_bytes)
    assert r["lat"][0] == lat0
    # deterministic per seed; empty workload -> zero iterations
    arr, pr, ou, ca = _c1_requests(20, 2.0)
    a1 = osim.reference_run(arr, pr, ou, ca, **kw)
    a2 = osim.reference_run(arr, pr, ou, ca, **kw)
    assert a1["compositions"] == a2["compositions"] and np.array_equal(a1["ttft"], a2["ttft"])
    assert osim.reference_run([], [], [], [], **kw)["n_iter"] == 0


def test_affine_invariant_oracle(corpus):
    """SPEC.md:629 on the oracle side: exactly-affine oracle latencies ->
    oracle fit -> run equals reference_run within 1e-6 relative on every
    iteration, with identical batch compositions."""
    from paper_2605_07985_b200.records import synthesize_entries

    m, b = _c1(corpus)
    ents = synthesize_entries(m, b, 1)
    coefs = affine_oracle_coefs(ents)
    fits = []
    for e, c in zip(ents, coefs):
        x, y = affine_oracle_sweep(e, c, corpus.grid, m.max_context)
        kind = ATTN if e.feature == "attention" else 0
        fits.append((kind, osim.fit(kind, x, y, np.array([0, y.shape[0]], dtype=np.int64))))
    ops = oracle_ops(ents, fits)
    ej, oracle = affine_oracle_batch(ents, coefs)
    arr, pr, ou, ca = _c1_requests(60, 2.0)
    kw = dict(chunk=8192, max_batch=256, kv_bytes_per_token=m.kv_bytes_per_token(),
              kv_capacity=10 ** 11, log=True)
    run = osim.run_shard(arr, pr, ou, ca, ops, **kw)
    ref = osim.reference_run(arr, pr, ou, ca, ej, oracle_hw(corpus.hardware), b.cost_multiplier,
                             m.dtype_bytes, oracle=oracle, **kw)
    assert run["compositions"] == ref["compositions"]
    la, lb = np.array(run["lat"]), np.array(ref["lat"])
    assert np.max(np.abs(la - lb) / lb) <= 1e-6
    ok = ~np.isnan(ref["tpot"])
    assert np.max(np.abs(run["ttft"] - ref["ttft"]) / ref["ttft"]) <= 1e-6
    assert np.max(np.abs(run["tpot"][ok] - ref["tpot"][ok]) / ref["tpot"][ok]) <= 1e-6


def _random_case(rng):
    n = int(rng.integers(1, 12))
    arr = np.cumsum(rng.exponential(0.004, n)).tolist()
    pr = rng.integers(1, 700, n).tolist()
    ou = rng.integers(1, 12, n).tolist()
    ca = [int(p) if rng.random() < 0.15 else (int(rng.integers(0, p)) if rng.random() < 0.1 else 0)
          for p in pr]
    chunk = int(rng.integers(16, 1024))
    mb = int(rng.integers(1, min(chunk, 16) + 1))
    kvb = int(rng.integers(1, 5))
    cap = int(max((p + o) * kvb for p, o in zip(pr, ou)) * rng.uniform(1, 4))
    return arr, pr, ou, ca, chunk, mb, kvb, cap


def _one_op():
    return [{"feat": osim.FEAT_NUM_TOKS, "coef": [1e-3, 1e-6 * 16384], "inv": [1.0 / 16384],
             "repeat": 1, "window_slot": 0}]


def test_a6_scheduler_properties_10k():
    """A6: 10,000 randomized cases — chunk budget, batch cap, KV
    cap, token conservation, clock monotonicity, no finish before arrival,
    determinism."""
    rng = np.random.default_rng(0xA6)
    t0 = time.perf_counter()
    ops = _one_op()
    for case in range(10_000):
        arr, pr, ou, ca, chunk, mb, kvb, cap = _random_case(rng)
        kw = dict(ops=ops, chunk=chunk, max_batch=mb, kv_bytes_per_token=kvb, kv_capacity=cap,
                  log=True)
        r = osim.run_shard(arr, pr, ou, ca, **kw)
        assert r["status"] == "ok", case
        reserved_max = 0
        for comp, (nt, pf, bsz, _, _) in zip(r["compositions"], r["feats"]):
            assert nt <= chunk and pf <= nt and 1 <= bsz <= mb          # budget, batch cap
            reserved_max = max(reserved_max, sum((pr[i] + ou[i]) * kvb for i, _, _ in comp))
        assert reserved_max <= cap                                       # KV-memory cap
        pre = [0] * len(pr)
        dec = [0] * len(pr)
        for comp in r["compositions"]:
            for i, t, is_pf in comp:
                (pre if is_pf else dec)[i] += t
        for i in range(len(pr)):                                         # token conservation
            assert pre[i] == pr[i] - ca[i]
            assert dec[i] == ou[i] - (1 if pr[i] > ca[i] else 0)
        clocks = r["clocks"]
        assert all(b > a for a, b in zip(clocks, clocks[1:]))           # clock monotonicity
        assert all(t > 0 for t in r["ttft"])                            # no finish before arrival
        if case % 10 == 0:                                               # determinism
            r2 = osim.run_shard(arr, pr, ou, ca, **kw)
            assert r2["compositions"] == r["compositions"] and r2["clocks"] == r["clocks"]
    assert time.perf_counter() - t0 < 120
