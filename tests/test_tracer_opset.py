"""Record producer: taint lattice, tainted runner and
operation-set finder, checked against SPEC.md's examples and properties and
against the runnable sets the rest of the pipeline was pinned on."""

from __future__ import annotations

import json
import random

import pytest

from paper_2605_07985_b200 import modelir, opset, taint as T, tracer
from paper_2605_07985_b200.errors import (ContextUnavailable, MalformedTrace, MixValueConflict,
                                          RetraceFailed, ShapeMismatch, UnknownComponent)
from paper_2605_07985_b200.records import canonical_bytes, dump_runnable_set, synthesize_entries


def _man(name):
    return modelir.load_manifest(modelir.builtin_manifest_path(name))


# ------------------------------------------------------------------- taint


def test_combine_table1_rules():
    assert T.combine(T.BOT, T.NT) == T.NT                              # absorption
    assert T.combine(T.MC, T.MC) == T.MC                               # preservation
    assert T.combine(T.NT, T.MC, 269, 40) == "MIX{40:MC,269:NT}"       # conflict (§5.2)
    assert T.combine("MIX{8:NR,128:MC}", T.NT, None, 64) == "MIX{8:NR,64:NT,128:MC}"   # extend
    assert T.combine("MIX{2:NR,40:MC}", "MIX{40:MC,269:NT}") == "MIX{2:NR,40:MC,269:NT}"
    with pytest.raises(MixValueConflict):
        T.combine("MIX{8:MC,40:MC}", T.NR, None, 8)


def test_combine_lattice_properties():
    rng = random.Random(7)
    pool = [T.BOT, T.MC, T.NT, T.NR]
    vals = {T.MC: 40, T.NT: 269, T.NR: 2}

    def rnd():
        t = rng.choice(pool)
        return t, vals.get(t, 1)

    for _ in range(300):
        (a, va), (b, vb), (c, vc) = rnd(), rnd(), rnd()
        assert T.combine(a, b, va, vb) == T.combine(b, a, vb, va)
        assert T.combine(a, a, va, va) == a
        ab = T.combine(a, b, va, vb)
        bc = T.combine(b, c, vb, vc)
        # values of a mix operand are its components; a base keeps its value
        vab = va * vb if T.is_mix(ab) else (va if ab == a else vb)
        vbc = vb * vc if T.is_mix(bc) else (vb if bc == b else vc)
        assert T.combine(ab, c, vab, vc) == T.combine(a, bc, va, vbc)


def test_split_and_reevaluate_examples():
    assert T.split("MIX{40:MC,269:NT}", 40) == (T.MC, T.NT)
    assert T.split("MIX{2:NR,40:MC,269:NT}", 269) == (T.NT, "MIX{2:NR,40:MC}")
    with pytest.raises(UnknownComponent):
        T.split("MIX{40:MC,269:NT}", 7)
    assert T.reevaluate("MIX{40:MC,269:NT}", {T.NT: 1}) == (40, T.MC)
    assert T.reevaluate("MIX{40:MC,269:NT}", {T.NT: 2048})[0] == 81920
    assert T.reevaluate("MIX{8:NR,128:MC}", {T.NR: 64})[0] == 8192
    assert T.reevaluate("MIX{40:MC,269:NT}", {})[0] == 40 * 269          # identity


def test_taint_text_round_trip_and_registry():
    for t in (T.BOT, T.MC, T.NT, T.NR, "MIX{40:MC,269:NT}", "MIX{2:NR,40:MC,269:NT}"):
        assert T.parse(t) == t
    for bad in ("MIX{269:NT,40:MC}", "MIX{40:MC}", "XX", "MIX{40:ZZ,2:NR}"):
        with pytest.raises(ValueError):
            T.parse(bad)
    reg = T.Registry()
    assert not reg.register(4096, T.MC) and reg.lookup(4096) == T.MC
    assert not reg.register(4096, T.MC)                                  # idempotent
    assert not reg.register(8, T.MC) and reg.register(8, T.NR)           # collision (§7.3)
    assert reg.lookup(8) is None and reg.lookup(7) is None and 8 in reg.collisions
    assert T.Registry.from_snapshot(reg.snapshot()).snapshot() == reg.snapshot()


# -------------------------------------------------------------- tracer


def test_seed_sources_and_collisions():
    cfg = _man("corpus12").model("llama-3.1-8b-like")
    reg = tracer.seed_sources(cfg, tracer.DummyBatch(2, 269))
    e = reg.entries
    assert e[4096] == T.MC and e[8] == T.MC and e[2] == T.NR and e[269] == T.NT and e[538] == T.NT
    assert not reg.collisions
    reg = tracer.seed_sources(cfg, tracer.DummyBatch(8, 269))
    assert 8 in reg.collisions                      # collides with the KV head count


def test_retrace_on_collision():
    cfg = _man("corpus12").model("llama-3.1-8b-like")
    tr = tracer.run_trace(cfg, _man("corpus12").backends[0], tracer.DummyBatch(8, 269))
    assert tr.batch != tracer.DummyBatch(8, 269) and not tr.registry.collisions
    moe = _man("mixtral").models[0]                 # top_k = 2 collides with num_reqs 2
    assert tracer.choose_batch(moe).num_reqs != 2
    with pytest.raises(RetraceFailed):
        orig = tracer.choose_batch
        try:
            tracer.choose_batch = lambda cfg, tp=1, skip=(): tracer.DummyBatch(8, 269)
            tracer.run_trace(cfg, _man("corpus12").backends[0], tracer.DummyBatch(8, 269))
        finally:
            tracer.choose_batch = orig


def test_map_and_preserve_dims_examples():
    reg = tracer.seed_sources(_man("corpus12").model("llama-3.1-8b-like"), tracer.DummyBatch(2, 269))
    assert tracer.map_dims("reshape", [(269, T.NT), (40, T.MC)], [10760], reg) == [
        (10760, "MIX{40:MC,269:NT}")]
    assert tracer.map_dims("reshape", [(10760, "MIX{40:MC,269:NT}")], [-1, 40], reg) == [
        (269, T.NT), (40, T.MC)]
    assert tracer.map_dims("create", [], [tracer.TInt(2, T.NR), tracer.TInt(4096, T.MC)], reg) == [
        (2, T.NR), (4096, T.MC)]
    assert tracer.map_dims("create", [], [4096, 7], reg) == [(4096, T.MC), (7, T.BOT)]
    with pytest.raises(ShapeMismatch):
        tracer.map_dims("reshape", [(269, T.NT), (40, T.MC)], [100, 100], reg)
    assert tracer.preserve_dims("matmul", [[(538, T.NT), (4096, T.MC)], [(14336, T.MC), (4096, T.MC)]],
                                None, reg) == [(538, T.NT), (14336, T.MC)]
    x = [(538, T.NT), (4096, T.MC)]
    assert tracer.preserve_dims("elementwise", [x], [538, 4096], reg) == x
    assert tracer.preserve_dims("elementwise", [x], [538, 8], reg) == [(538, T.NT), (8, T.MC)]


def test_trace_structure_determinism_and_chrome_round_trip():
    man = _man("corpus12")
    cfg = man.model("llama-3.1-8b-like")
    tr = tracer.run_trace(cfg, man.backends[0])
    a = tr.to_chrome()
    assert a == tracer.run_trace(cfg, man.backends[0]).to_chrome()       # byte-identical
    evs = tracer.TaintedTrace.events_from_chrome(a)
    assert evs == tr.events                                              # lossless
    tree = opset.build_tree(evs)
    assert len(tree.roots) == 1
    layers = [c for c in tree.roots[0].children if c.event.name == "decoder_layer"]
    assert len(layers) == 32
    qkv = next(n for n in tree.walk() if n.event.name == "linear")
    assert qkv.event.input_dims[0] == [(538, T.NT), (4096, T.MC)]
    # nesting: every child strictly inside its parent, siblings disjoint
    for n in tree.walk():
        kids = sorted(n.children, key=lambda c: c.event.begin)
        for c in kids:
            assert n.event.begin < c.event.begin and c.event.end < n.event.end
        for p, q in zip(kids, kids[1:]):
            assert p.event.end < q.event.begin
    tp4 = tracer.run_trace(cfg, man.backends[0], tp=4)
    coll = [e for e in tp4.events if e.name == "all_reduce"]
    assert len(coll) == 2 * cfg.num_layers and all(e.begin == e.end for e in coll)


def test_differential_taint_classification():
    """§7.3 protocol: across two batch sizes and two prompt lengths every
    MODEL_CONFIG dim is constant and every workload dim scales with the batch."""
    man = _man("corpus12")
    for cfg in man.models[:4]:
        b = man.backends[0]
        traces = [tracer.run_trace(cfg, b, tracer.DummyBatch(r, t)) for r, t in
                  ((3, 271), (5, 271), (3, 277), (5, 277))]
        for evs in zip(*(tr.events for tr in traces)):
            for dims in zip(*(e.input_dims for e in evs)):
                for col in zip(*dims):
                    taints = {t for _, t in col}
                    assert len(taints) == 1
                    t = taints.pop()
                    sizes = [s for s, _ in col]
                    toks = [tr.batch.num_tokens for tr in traces]
                    if t == T.MC:
                        assert len(set(sizes)) == 1
                    elif t == T.NT:
                        assert sizes == toks
                    else:
                        assert t != T.BOT


# ------------------------------------------------------------- opset


def test_build_tree_examples():
    E = tracer.TraceEvent
    t = opset.build_tree([E(0, None, "module", "r", 0, 10), E(1, 0, "operation", "a", 2, 5),
                          E(2, 0, "operation", "b", 6, 8)])
    assert len(t.roots) == 1 and [c.event.name for c in t.roots[0].children] == ["a", "b"]
    assert opset.build_tree([]).roots == []
    with pytest.raises(MalformedTrace):
        opset.build_tree([E(0, None, "module", "r", 0, 10), E(1, 0, "operation", "a", 2, 5),
                          E(2, 0, "operation", "b", 4, 8)])


def test_prune_repeats_swa_and_conservation():
    man = _man("corpus12")
    cfg = man.model("llama-3.1-8b-like")
    tree = opset.build_tree(tracer.run_trace(cfg, man.backends[0]).events)
    pr = opset.prune(tree)
    layers = [c for c in pr.roots[0].children if c.event.name == "decoder_layer"]
    assert [c.repeat for c in layers] == [32]
    assert pr.kernel_count() == tree.kernel_count()
    again = opset.prune(pr)
    assert [(n.fp, n.repeat) for n in again.walk()] == [(n.fp, n.repeat) for n in pr.walk()]
    cmd = man.model("command-r7b-like")
    ents = opset.runnable_set(cmd, man.backends[0])
    att = [(e.window, e.repeat_count) for e in ents if e.name == "attention"]
    assert sorted(att, key=str) == sorted([(None, 8), (4096, 24)], key=str)
    tree = opset.build_tree(tracer.run_trace(cmd, man.backends[0]).events)
    assert opset.covered_kernel_count(ents) == tree.kernel_count()


def test_resolve_granularity_and_context():
    man = _man("corpus12")
    ents = opset.runnable_set(man.model("llama-3.1-8b-like"), man.backends[0])
    mods = [e for e in ents if e.granularity == "module"]
    assert [e.name for e in mods] == ["attention"] and mods[0].context_required
    assert len(mods[0].kernel_symbols) == 3                  # absorbed its 3 kernel leaves
    assert all(not e.context_required for e in ents if e.granularity == "operator")
    names = [e.name for e in ents]
    assert names[0] == "embedding" and names[-1] == "linear"
    lin = next(e for e in ents if e.name == "linear")
    assert opset.generate_inputs(lin, {"num_toks": 2048, "num_reqs": 8})[0] == (2048, 4096)
    eng = opset.EngineContext()
    ctx = opset.emulate_context(mods[0], eng, {"num_toks": 2048, "num_reqs": 1, "phase": "prefill"})
    assert ctx["seq_lens"] == [2048] and ctx["phase"] == "prefill"
    ctx = opset.emulate_context(mods[0], eng, {"num_toks": 64, "num_reqs": 64, "phase": "decode",
                                               "kv_len": 512})
    assert ctx["batch_size"] == 64 and ctx["context_lens"] == [512] * 64
    with pytest.raises(ContextUnavailable):
        opset.emulate_context(lin, eng, {"num_toks": 4, "num_reqs": 1})
    moe = opset.runnable_set(_man("mixtral").models[0], _man("mixtral").backends[0])
    assert [e.name for e in moe if e.granularity == "module"] == ["attention", "fused_moe"]


@pytest.mark.parametrize("manifest", ["corpus12", "fixtures", "mixtral", "llama70b"])
def test_runnable_sets_match_the_pinned_record_sets(manifest):
    """The tracer -> opset pipeline reproduces, entry for entry, the runnable
    sets the dedup / fit / simulate parity tests were pinned on (Table-2
    census, N/R counts): same canonical bytes (hence digests), repeats,
    kernel symbols, features and windows."""
    man = _man(manifest)
    for m in man.models:
        for b in man.backends:
            tr = tracer.run_trace(m, b, tp=man.tp_degree)
            got = opset.runnable_set(m, b, man.tp_degree, tr)
            want = synthesize_entries(m, b, man.tp_degree)
            assert len(got) == len(want), (m.name, b.name)
            for g, w in zip(got, want):
                assert canonical_bytes(g) == canonical_bytes(w), (m.name, g.name)
                assert (g.repeat_count, g.kernel_symbols, g.feature, g.window, g.attrs,
                        g.granularity) == (w.repeat_count, w.kernel_symbols, w.feature,
                                           w.window, w.attrs, w.granularity)
                toks = {s for a in g.arg_template for s, t in a if t == T.NT}
                assert toks <= {tr.batch.num_tokens}
            json.loads(dump_runnable_set(got))


def test_taint_matches_reference_golden():
    """800 seeded cases generated by the reference's taint.py
    (tests/golden/make_taint_golden.py): same result text or same exception."""
    from conftest import GOLDEN
    from paper_2605_07985_b200 import errors

    cases = json.loads((GOLDEN / "reference_taint.json").read_text())["cases"]
    fns = {"combine": lambda a, b, va, vb: T.combine(a, b, va, vb),
           "split": lambda a, k: T.split(a, k),
           "reevaluate": lambda a, subs: T.reevaluate(a, subs)}
    for c in cases:
        try:
            got = fns[c["op"]](*c["args"])
        except (ValueError, errors.DoolyError) as exc:
            assert type(exc).__name__ == c.get("error"), (c, exc)
            continue
        assert "error" not in c, (c, got)
        want = c["result"]
        assert (list(got) if isinstance(got, tuple) else got) == want, (c, got)


@pytest.mark.parametrize("seed", range(25))
def test_runnable_sets_random_architectures(seed):
    """Random valid architectures (GQA/MHA, interleaved or listed sliding
    windows, MoE, tensor parallelism): the traced and resolved runnable set
    equals the closed-form one, and the kernel multiset is conserved."""
    rng = random.Random(seed)
    tp = rng.choice([1, 1, 2, 4])
    kv = tp * rng.choice([1, 2, 4, 8])
    q = kv * rng.choice([1, 2, 4, 8])
    d = rng.choice([64, 128, 256])
    n_layers = rng.randint(1, 24)
    kinds = [rng.choice([None, None, 1024, 4096]) for _ in range(n_layers)]
    moe = None
    if rng.random() < 0.3:
        e = rng.choice([4, 8, 16])
        moe = modelir.MoESpec(e, rng.randint(1, 3), tp * rng.choice([512, 1792]))
    cfg = modelir.ModelConfig(
        name=f"rand{seed}", hidden_dim=q * d, num_layers=n_layers, num_q_heads=q,
        num_kv_heads=kv, head_dim=d, intermediate_size=tp * rng.choice([1024, 3584, 7168]),
        vocab_size=tp * rng.choice([8000, 32000, 64128]), dtype_bytes=rng.choice([1, 2]),
        max_context=rng.choice([4096, 32768]), layer_attention=tuple(kinds), moe=moe)
    cfg.validate()
    backend = _man("corpus12").backends[seed % 3]
    tr = tracer.run_trace(cfg, backend, tp=tp)
    assert not tr.registry.collisions
    tree = opset.build_tree(tr.events)
    got = opset.resolve(opset.prune(tree))
    want = synthesize_entries(cfg, backend, tp)
    assert [canonical_bytes(e) for e in got] == [canonical_bytes(e) for e in want]
    assert [(e.repeat_count, e.kernel_symbols, e.window) for e in got] == \
        [(e.repeat_count, e.kernel_symbols, e.window) for e in want]
    assert opset.covered_kernel_count(got) == tree.kernel_count()
