"""Pin the CPU oracle: every golden vector / KAT the reference holds for this
path, plus fixtures generated from the reference itself
(tests/golden/make_golden.py)."""

from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import GOLDEN
from helpers import AFFINE, ATTN, synth_fit_data
from oracle import profiler as oprof
from oracle import sim as osim


def test_sha256_empty_kat():
    # SPEC.md:452
    assert oprof.signature_hash(b"").hex() == \
        "e3b0c44298fc1c149afbf4c8996fb92427ae41e4649b934ca495991b7852b855"


def test_roofline_golden_values(corpus):
    hw = corpus.hardware
    # SPEC.md:482 matmul 1024x4096x4096 fp16 on A100-like, A9: 1e-9 abs
    flops, nbytes = oprof.matmul_cost(1024, 4096, 4096, 2)
    assert (flops, nbytes) == (34359738368, 50331648)
    lat = oprof.roofline_latency(flops, nbytes, hw.peak_flops, hw.mem_bw)
    assert abs(lat - 1.1512736656410257e-4) <= 1e-9
    # SPEC.md:483 decode GEMV is memory-bound
    f, b = oprof.matmul_cost(1, 4096, 4096, 2)
    assert b / hw.mem_bw > f / hw.peak_flops
    # SPEC.md:484 zero-flop op -> overhead only
    assert oprof.roofline_latency(0, 0, hw.peak_flops, hw.mem_bw) == 5e-6


def test_comm_golden_values():
    # SPEC.md:489-493
    assert abs(oprof.comm_latency(2, 2 ** 20, 5e-6, 5e-12) - 7.62144e-6) <= 1e-9
    assert oprof.comm_latency(4, 0, 5e-6, 5e-12) == 2 * 3 / 4 * 5e-6


def test_product_latency_model_matches_oracle(corpus):
    from paper_2605_07985_b200 import profiler
    from paper_2605_07985_b200.records import RunnableEntry

    e = RunnableEntry("operator", "linear", (((1024, "NT"), (4096, "MC")), ((4096, "MC"), (4096, "MC"))),
                      kernel_symbols=("gemm_f16_tn",))
    lat = profiler.oracle_latency(e, {"num_toks": 1024}, corpus.hardware, corpus.backends[0], 2)
    assert abs(lat - 1.1512736656410257e-4) <= 1e-9
    assert profiler.comm_latency("nvlink8", 2, 2 ** 20, corpus.hardware) == \
        oprof.comm_latency(2, 2 ** 20, 5e-6, 5e-12)


def test_census_table2(corpus):
    """Attention N/R per geometry group; the
    census itself is the reference's test_modelir.py:109-124 (golden file)."""
    from paper_2605_07985_b200 import modelir
    from paper_2605_07985_b200.records import corpus_entries

    gold = json.loads((GOLDEN / "reference_modelir.json").read_text())["corpus12"]["census"]
    cfgs = corpus_entries(corpus)
    ents = [(m, e.to_json()) for m, _, es in cfgs for e in es if e.name == "attention"]
    n_by, r_by = {}, {}
    _, skipped = oprof.dedup([e for _, e in ents])
    for i, (m, e) in enumerate(ents):
        key = modelir.geometry_key(m, m.layer_attention.index(e["window"]))
        n_by[key] = n_by.get(key, 0) + 1
        r_by[key] = r_by.get(key, 0) + (i in skipped)
    assert n_by == gold
    assert r_by == {"q32/kv8/d128/full": 21, "q28/kv4/d128/full": 3, "q32/kv32/d128/full": 3,
                    "q32/kv8/d128/swa4096": 0, "q32/kv8/d128/swa32768": 0}
    assert sum(n_by.values()) - sum(r_by.values()) == 15


def test_census_saturates_within_four_models(corpus):
    from paper_2605_07985_b200.records import corpus_entries

    seen, curve = set(), []
    cur_model = None
    for m, _, es in corpus_entries(corpus):
        for e in es:
            if e.name == "attention":
                seen.add(oprof.signature_hash(oprof.canonicalize(e.to_json())))
        if m.name != cur_model:
            cur_model = m.name
        curve.append((m.name, len(seen)))
    per_model = []
    for name, n in curve:
        if not per_model or per_model[-1][0] != name:
            per_model.append([name, n])
        per_model[-1][1] = n
    counts = [n for _, n in per_model]
    assert counts[:4] == [6, 9, 12, 15] and counts[-1] == 15          # SPEC.md:708 (A3)
    assert counts[3] >= 0.95 * counts[-1]


def test_a3_overall_reuse_and_saturation(corpus):
    """A3 over every record of the 12-model x 3-backend corpus, not
    only attention: unique signatures = N - R, count-reuse ratio >= 50%, and the
    cumulative unique count reaches >= 95% of its final value within the first
    four models (manifest order)."""
    from paper_2605_07985_b200.records import corpus_entries

    seen, n, r, per_model, cur = set(), 0, 0, [], None
    for m, _, es in corpus_entries(corpus):
        for e in es:
            h = oprof.signature_hash(oprof.canonicalize(e.to_json()))
            n += 1
            r += h in seen
            seen.add(h)
        if m.name != cur:
            cur = m.name
            per_model.append(0)
        per_model[-1] = len(seen)
    assert len(seen) == n - r
    assert r / n >= 0.5
    assert per_model[3] >= 0.95 * per_model[-1]
    assert (n, r, len(seen)) == (486, 439, 47)


def test_dedup_rerun_and_empty_db():
    ents = [{"name": "linear", "granularity": "operator", "arg_template": [[[8, "NT"], [64, "MC"]]],
             "kernel_symbols": ["g"], "attrs": {}}] * 3
    to_profile, skipped = oprof.dedup(ents)
    assert to_profile == [0] and skipped == [1, 2]
    keys = {oprof.signature_hash(oprof.canonicalize(ents[0]))}
    assert oprof.dedup(ents, keys)[0] == []


def test_canonical_semantics():
    """A4: equal geometry+backend -> equal; attrs / symbols differ -> differ;
    workload-tainted values never enter the signature."""
    base = {"name": "attention", "granularity": "module",
            "arg_template": [[[538, "NT"], [32, "MC"], [128, "MC"]]],
            "kernel_symbols": ["fa_b", "fa_a"], "attrs": {"causal": True}}
    other_prompt = json.loads(json.dumps(base))
    other_prompt["arg_template"][0][0] = [4111, "NT"]
    assert oprof.canonicalize(base) == oprof.canonicalize(other_prompt)
    swa = json.loads(json.dumps(base))
    swa["attrs"]["sliding_window"] = 4096
    assert oprof.canonicalize(base) != oprof.canonicalize(swa)
    sym = json.loads(json.dumps(base))
    sym["kernel_symbols"] = ["fa_a", "fa_c"]
    assert oprof.canonicalize(base) != oprof.canonicalize(sym)
    mix = json.loads(json.dumps(base))
    mix["arg_template"][0][1] = [32, "MIX{2:NR,16:MC}"]
    assert oprof.canonicalize(base) != oprof.canonicalize(mix)     # Mix dims excluded (A.2)
    c = oprof.canonicalize(base)
    assert c.startswith(b"sigfmt=1") and len(c) == 8 + 4 + 9 + 4 + 2 * 12 + 4 + 2 * 8 + 32


def test_fit_exact_linear_and_insufficient():
    # SPEC.md:562 exactly linear -> fit_error < 1e-6 ; SPEC.md:564 2 records -> insufficient
    x = np.array([[1, 16, 128, 512, 2048, 8192, 3, 9]], dtype=np.uint32)
    y = 5e-6 + 2e-9 * x[0].astype(np.float64)
    r = osim.fit(AFFINE, x, y, np.array([0, 6, 8]))
    assert r["status"].tolist() == [0, 1] and r["fit_err"][0] < 1e-6
    assert r["have"][1] == 2


@pytest.mark.parametrize("kind", [AFFINE, ATTN])
def test_fit_agrees_with_lstsq(kind):
    """The pinned normal-equation/Cholesky formulation agrees with numpy lstsq
    on full-rank designs (<= 1e-9 relative on predictions)."""
    x, y, off = synth_fit_data(kind, 40, 200, seed=kind)
    r = osim.fit(kind, x, y, off)
    for s in range(40):
        a, b = off[s], off[s + 1]
        f = x[:, a:b].astype(np.float64) * r["inv"][s][:, None]
        X = osim.design(kind, f)
        c_ls = np.linalg.lstsq(X, y[a:b], rcond=None)[0]
        p_ls = X @ c_ls
        p = osim.eval_poly(kind, r["coef"][s], r["inv"][s], x[:, a:b].T)
        assert np.max(np.abs(p - p_ls) / np.abs(p_ls)) < 1e-9


def test_predict_clamp_and_flags():
    table = {"coef": np.array([[-1.0, 0.5]]), "inv": np.array([[1.0]]),
             "lo": np.array([[2]], np.uint32), "hi": np.array([[10]], np.uint32)}
    r = osim.predict(AFFINE, table, np.array([0, 0, 1]), np.array([[1, 4, 4]], np.uint32))
    assert r["out"][0] == 1e-7 and r["clamped"][0] and r["extrap"][0]
    assert r["out"][1] == 1.0 and not r["extrap"][1]
    assert np.isnan(r["out"][2]) and r["bad"][2]


def _one_op_table():
    # latency = 1e-3 + 1e-6 * num_toks (affine entry), single op, repeat 1
    return [{"feat": osim.FEAT_NUM_TOKS, "coef": [1e-3, 1e-6 * 16384], "inv": [1.0 / 16384],
             "repeat": 1, "window_slot": 0}]


def test_scheduler_chunk_kats():
    """10000-token prompt at chunk 8192 -> 8192 then 1808;
    SPEC.md:583: 64 decodes leave 8128 of the budget."""
    r = osim.run_shard([0.0], [10000], [1], [0], _one_op_table(), chunk=8192, max_batch=256,
                       kv_bytes_per_token=1, kv_capacity=10 ** 12, log=True)
    assert [f[0] for f in r["feats"]] == [8192, 1808]
    # single request TTFT == sum of its prefill-iteration latencies
    assert r["ttft"][0] == r["lat"][0] + r["lat"][1]
    running = [{"left": 0} for _ in range(64)]
    sched, _ = osim.schedule_step(running, lambda k: None, 8192, 256, lambda w: True)
    assert sum(t for _, t, _, _ in sched) == 64
    waiting = [{"prompt": 9000, "cached": 0, "output": 5, "left": 9000}]
    sched, n_adm = osim.schedule_step(running, lambda k: waiting[k] if k < 1 else None, 8192,
                                      256, lambda w: True)
    assert n_adm == 1 and sched[-1][1] == 8128


def test_scheduler_fcfs_blocking():
    # two identical requests, max_batch 1 -> second TTFT includes the first's prefill
    r = osim.run_shard([0.0, 0.0], [100, 100], [3, 3], [0, 0], _one_op_table(), chunk=256,
                       max_batch=1, kv_bytes_per_token=1, kv_capacity=10 ** 9, log=True)
    assert r["ttft"][1] > r["ttft"][0] + 2 * r["lat"][0] * 0.99
    # empty workload -> zero iterations
    e = osim.run_shard([], [], [], [], _one_op_table(), chunk=256, max_batch=1,
                       kv_bytes_per_token=1, kv_capacity=10)
    assert e["n_iter"] == 0


def test_scheduler_invariants_random():
    """A6-style property run: chunk budget, batch cap, KV cap, token conservation,
    clock monotonicity, determinism."""
    rng = np.random.default_rng(0xD001)
    for case in range(60):
        n = int(rng.integers(1, 40))
        arr = np.cumsum(rng.exponential(0.01, n)).tolist()
        pr = rng.integers(1, 3000, n).tolist()
        ou = rng.integers(1, 30, n).tolist()
        ca = [int(p) if rng.random() < 0.2 else 0 for p in pr]
        chunk = int(rng.integers(64, 4096))
        mb = int(rng.integers(1, min(chunk, 64) + 1))
        kvb = 3
        cap = int(max((p + o) * kvb for p, o in zip(pr, ou)) * rng.uniform(1, 6))
        kw = dict(ops=_one_op_table(), chunk=chunk, max_batch=mb, kv_bytes_per_token=kvb,
                  kv_capacity=cap, log=True)
        r = osim.run_shard(arr, pr, ou, ca, **kw)
        assert r["status"] == "ok"
        for nt, pf, b, _, _ in r["feats"]:
            assert nt <= chunk and pf <= nt and 1 <= b <= mb
        assert sum(f[1] for f in r["feats"]) == sum(p - c for p, c in zip(pr, ca))
        assert sum(f[0] - f[1] for f in r["feats"]) == sum(o - (1 if p > c else 0)
                                                           for p, c, o in zip(pr, ca, ou))
        assert all(t > 0 for t in r["ttft"])
        r2 = osim.run_shard(arr, pr, ou, ca, **kw)
        assert r2["feats"] == r["feats"] and np.array_equal(r2["ttft"], r["ttft"])


def test_mape_kat():
    assert abs(osim.mape([10, 20], [10, 25]) - 0.10) < 1e-15
    assert osim.mape([3.0], [3.0]) == 0.0
    with pytest.raises(ZeroDivisionError):
        osim.mape([1], [0])


@pytest.mark.parametrize("kind", [0, 1])
def test_predict_one_equals_batch_predict(kind):
    """The per-item oracle predict (plain Python floats) is bit-identical to
    the vectorised one, flags included."""
    import numpy as np

    from helpers import synth_fit_data, synth_queries
    from oracle import sim as osim

    x, y, off = synth_fit_data(kind, 64, 32, seed=kind)
    f = osim.fit(kind, x, y, off)
    table = {k: f[k] for k in ("coef", "inv", "lo", "hi")}
    table["coef"][3, 0] = -1.0                                   # a clamped signature
    sig, xq = synth_queries(kind, table, 3000, seed=5, outside=0.1)
    ref = osim.predict(kind, table, sig, xq)
    rows = {i: (list(table["coef"][i]), list(table["inv"][i]), list(table["lo"][i]),
                list(table["hi"][i])) for i in range(64)}
    for q in range(sig.shape[0]):
        p, e, c = osim.predict_one(kind, rows, int(sig[q]), [int(v) for v in xq[:, q]])
        assert np.float64(p).view(np.uint64) == ref["out"][q].view(np.uint64)
        assert e == bool(ref["extrap"][q]) and c == bool(ref["clamped"][q])


def test_packed_serving_form_matches_scaled_evaluation():
    """The folded 96-B serving form (pack_attn / predict_packed, the contract of
    DOOLY_KIND_ATTN_PACKED) differs from the scaled 10-column evaluation by
    rounding only: <= 1e-12 relative, identical flags and unknown rows."""
    from helpers import synth_queries

    x, y, off = synth_fit_data(ATTN, 300, 48, seed=77)
    f = osim.fit(ATTN, x, y, off)
    table = {k: f[k] for k in ("coef", "inv", "lo", "hi")}
    sig, xq = synth_queries(ATTN, table, 200_000, seed=3, outside=0.05)
    a = osim.predict(ATTN, table, sig, xq)
    b = osim.predict_packed(osim.pack_attn(table), sig, xq)
    live = ~a["clamped"] & ~a["bad"]
    assert np.max(np.abs(a["out"][live] - b["out"][live]) / a["out"][live]) <= 1e-12
    for k in ("extrap", "bad"):
        assert np.array_equal(a[k], b[k])
