"""Host-side logic (no GPU): the C-ABI library, packed record layout, manifest /
workload parity with the reference, LatencyDB, trace sharding."""

from __future__ import annotations

import json
import re
import struct

import numpy as np
import pytest

from conftest import GOLDEN, ROOT
from oracle import profiler as oprof


# ------------------------------------------------------------------ C-ABI


def _header_functions():
    text = (ROOT / "include" / "dooly_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*[\w\s\*]+?\b(dooly_\w+)\s*\(", text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2605_07985_b200 import _lib

    lib = _lib.load_library()
    declared = _header_functions()
    assert len(declared) >= 14
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.EXPORTS)
    assert lib.dooly_version() == 1


def test_library_rejects_bad_arguments_without_gpu():
    from paper_2605_07985_b200 import _lib

    lib = _lib.load_library()
    assert lib.dooly_predict(None, 0, None, 0, None, None, 0, None, None, None, None) == 1
    assert lib.dooly_fit_grid_packed(None, None, 0, None, 0, None, None, None, None, None, 0,
                                     None) == 1
    assert lib.dooly_dedup_workspace_size(1000, 10) >= 2048 * 4
    # attention grid workspace: factor + 3 feature planes + the (f1, f2) group plane
    a = lib.dooly_fit_grid_workspace_size(1, 4096)
    assert a == lib.dooly_fit_grid_workspace_size(1, 0) + 3 * 4096 * 8 + 4096 // 4 * 16
    assert lib.dooly_fit_grid_workspace_size(0, 4096) == lib.dooly_fit_grid_workspace_size(0, 0) + 4096 * 8


def test_struct_layouts_match_header():
    import ctypes

    from paper_2605_07985_b200 import _lib
    from paper_2605_07985_b200.sim import AFFINE_ROW, ATTN_ROW

    assert AFFINE_ROW.itemsize == _lib.AFFINE_ROW_BYTES == 32
    assert ATTN_ROW.itemsize == _lib.ATTN_ROW_BYTES == 128
    assert ctypes.sizeof(_lib.Sched) == 4 * 4 + 3 * 8
    assert _lib.OpList.bytes_per_tok.offset % 8 == 0


# ------------------------------------------------------------ packed records


def _canonical_from_words(p, i: int) -> bytes:
    """Decode one packed record back into the sigfmt=1 message (what the GPU builds)."""
    w = p.words
    o = int(p.rec_off[i])
    op, nd, ns, attr = int(w[o]), int(w[o + 1]) & 0xFFFF, int(w[o + 1]) >> 16, int(w[o + 2])
    name = bytes(p.op_bytes[p.op_off[op]:p.op_off[op + 1]])
    out = b"sigfmt=1" + struct.pack("<I", len(name)) + name + struct.pack("<I", nd)
    for k in range(nd):
        out += struct.pack("<III", int(w[o + 4 + 3 * k]), int(w[o + 5 + 3 * k]),
                           int(w[o + 6 + 3 * k]))
    out += struct.pack("<I", ns)
    ids = [int(w[o + 4 + 3 * nd + k]) for k in range(ns)]
    assert ids == sorted(ids)
    for sid in ids:
        s = bytes(p.sym_bytes[p.sym_off[sid]:p.sym_off[sid + 1]])
        out += struct.pack("<I", len(s)) + s
    if attr != 0xFFFFFFFF:
        out += bytes(p.attr_digests[attr])
    return out


@pytest.mark.parametrize("tp", [1, 2])
def test_packed_records_reproduce_oracle_canonical_bytes(corpus, fixtures_manifest, tp):
    from paper_2605_07985_b200.records import corpus_entries, pack_entries

    man = fixtures_manifest if tp == 2 else corpus
    ents = [e for _, _, es in corpus_entries(man, tp=tp) for e in es]
    p = pack_entries(ents)
    for i, e in enumerate(ents):
        want = oprof.canonicalize(e.to_json())
        assert _canonical_from_words(p, i) == want


def test_pack_uniform_equals_generic_packer():
    import bench
    from paper_2605_07985_b200.records import RunnableEntry, pack_entries

    packed, _ = bench.synth_records(500, seed=3)
    for i in range(0, 500, 37):
        msg = _canonical_from_words(packed, i)
        # rebuild the same record through the generic entry path
        o = int(packed.rec_off[i])
        w = packed.words
        pos_val = [(int(w[o + 4 + 3 * k]), int(w[o + 5 + 3 * k]) | (int(w[o + 6 + 3 * k]) << 32))
                   for k in range(3)]
        args = [[(9, "NT")] * 5]
        for pos, val in pos_val:
            args[0][pos] = (val, "MC")
        name = packed.op_names[int(w[o])]
        syms = [bytes(packed.sym_bytes[packed.sym_off[s]:packed.sym_off[s + 1]]).decode()
                for s in (int(w[o + 13]), int(w[o + 14]))]
        e = RunnableEntry("operator", name, (tuple(args[0]),), kernel_symbols=tuple(syms))
        assert _canonical_from_words(pack_entries([e]), 0) == msg


def test_synth_records_dedup_ratio():
    import bench

    packed, _ = bench.synth_records(20000, seed=0)
    digs = [oprof.signature_hash(_canonical_from_words(packed, i)) for i in range(packed.n)]
    res = oprof.dedup_digests(digs)
    assert 0.15 * packed.n < res["n_unique"] < 0.35 * packed.n


def test_runnable_set_json_roundtrip(corpus):
    from paper_2605_07985_b200.records import (canonical_bytes, dump_runnable_set,
                                               load_runnable_set, synthesize_entries)

    ents = synthesize_entries(corpus.models[0], corpus.backends[0], 1)
    back = load_runnable_set(dump_runnable_set(ents))
    assert [canonical_bytes(e) for e in back] == [canonical_bytes(e) for e in ents]
    assert [e.repeat_count for e in back] == [e.repeat_count for e in ents]


def test_synthesizer_layer_pruning(corpus):
    """Command-R7B-like: 2 attention representatives, counts 8 (full) and 24 (swa4096)
    (SPEC.md:366); coverage: sum of repeats of attention entries == num_layers."""
    from paper_2605_07985_b200.records import synthesize_entries

    cfg = corpus.model("command-r7b-like")
    att = [e for e in synthesize_entries(cfg, corpus.backends[0]) if e.name == "attention"]
    assert sorted((e.window or 0, e.repeat_count) for e in att) == [(0, 8), (4096, 24)]
    for m in corpus.models:
        att = [e for e in synthesize_entries(m, corpus.backends[1]) if e.name == "attention"]
        assert sum(e.repeat_count for e in att) == m.num_layers


# ------------------------------------------------------------------ modelir


def test_modelir_matches_reference_golden(corpus, fixtures_manifest):
    from paper_2605_07985_b200 import modelir

    gold = json.loads((GOLDEN / "reference_modelir.json").read_text())
    for name, man in (("corpus12", corpus), ("fixtures", fixtures_manifest)):
        g = gold[name]
        assert modelir.dumps_canonical(modelir.manifest_to_json(man)) == g["canonical"]
        for cfg in man.models:
            assert [modelir.geometry_key(cfg, i) for i in range(cfg.num_layers)] == \
                g["geometry"][cfg.name]
        for key, want in g["attention"].items():
            mname, bname, w, phase = key.split("|")
            cfg, b = man.model(mname), man.backend(bname)
            win = None if w == "None" else int(w)
            syms = b.attention_kernels(cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, win, phase)
            assert list(syms) == want["symbols"]
            assert b.multiplier(syms) == want["multiplier"]
    d = modelir.DEFAULT_GRID
    assert gold["default_grid"]["token_counts"] == list(d.token_counts)
    for f, want in gold["shrink"].items():
        s = d.shrink(int(f))
        assert list(s.token_counts) == want["token_counts"]
        assert list(s.kv_lens) == want["kv_lens"]


@pytest.mark.parametrize("name", ["c1", "dur", "prefill_heavy", "decode_heavy"])
def test_sample_workload_matches_reference(name):
    from paper_2605_07985_b200 import modelir

    g = json.loads((GOLDEN / f"workload_{name}.json").read_text())
    reqs = modelir.sample_workload(modelir.workload_from_json(g["spec"]), g["seed"])
    assert [[r.arrival_s, r.prompt_tokens, r.output_tokens, r.cached_tokens] for r in reqs] == \
        g["requests"]


def test_manifest_validation_errors():
    from paper_2605_07985_b200 import modelir
    from paper_2605_07985_b200.errors import ParseError, ValidationError

    raw = {"name": "bad", "hidden_dim": 4000, "num_layers": 2, "num_q_heads": 32,
           "num_kv_heads": 8, "head_dim": 128, "intermediate_size": 8192, "vocab_size": 1000,
           "max_context": 2048}
    with pytest.raises(ValidationError, match="hidden_dim"):
        modelir.model_from_json(raw).validate()
    with pytest.raises(ParseError):
        modelir.load_manifest(ROOT / "README.md")


# ------------------------------------------------------------------ LatencyDB


def test_latency_db_roundtrip_and_duplicate_key(tmp_path):
    from paper_2605_07985_b200.errors import DuplicateKey, StoreUnavailable
    from paper_2605_07985_b200.profiler import LatencyDB
    from paper_2605_07985_b200.records import RunnableEntry

    db = LatencyDB()
    e = RunnableEntry("operator", "linear", (((8, "NT"), (64, "MC")),), kernel_symbols=("g",))
    d = b"\x01" * 32
    with pytest.raises(StoreUnavailable):
        db.insert_measurements(d, [[1, 2]], [1e-5, 2e-5])
    cid = db.add_configuration("a100-like", "m", "b", 1)
    db.add_signature(d, e)
    db.model_operations.append((cid, d, 3))
    db.insert_measurements(d, [[1, 2, 4]], [1e-5, 2e-5, 4e-5])
    db.insert_measurements(d, [[4, 8]], [4e-5, 8e-5])          # same key, same value: ok
    with pytest.raises(DuplicateKey):
        db.insert_measurements(d, [[8]], [9e-5])
    db.save(tmp_path / "db.npz")
    back = LatencyDB.load(tmp_path / "db.npz")
    assert back.has(d) and back.configurations == db.configurations
    assert np.array_equal(back.measurements[d][0], db.measurements[d][0])
    assert back.model_operations == db.model_operations
    assert "CREATE TABLE signatures(\n  hash BLOB PRIMARY KEY" in back.schema_dump()


def test_sweep_points_cardinality(corpus):
    from paper_2605_07985_b200 import profiler
    from paper_2605_07985_b200.records import synthesize_entries

    cfg = corpus.model("llama-3-8b-like")
    ents = synthesize_entries(cfg, corpus.backends[1])
    lin = [e for e in ents if e.name == "linear"][0]
    att = [e for e in ents if e.name == "attention"][0]
    assert len(profiler.sweep_points(lin, corpus.grid, cfg.max_context)) == 6
    pts = profiler.sweep_points(att, corpus.grid, cfg.max_context)
    assert len(pts) >= 11 and {p["phase"] for p in pts} == {"prefill", "decode"}
    x, y = profiler.sweep(att, corpus.grid, cfg, corpus.hardware, corpus.backends[1])
    assert x.shape == (3, len(pts)) and np.all(y > 0)


# ------------------------------------------------------------------ sharding


def test_sharded_trace_layout():
    import torch

    from paper_2605_07985_b200.sim import ShardedTrace

    n, S = 23, 4
    arr = np.arange(n, dtype=np.float64)
    t = ShardedTrace.from_arrays(arr, np.full(n, 5, np.uint32), np.full(n, 2, np.uint32),
                                 np.zeros(n, np.uint32), S, torch.device("cpu"))
    off = t.shard_off.numpy()
    assert off[-1] == n and list(np.diff(off)) == [6, 6, 6, 5]
    assert list(t.order[:6]) == [0, 4, 8, 12, 16, 20]
    assert np.array_equal(t.arrival.numpy(), arr[t.order])


def test_shard_range_partitions():
    from paper_2605_07985_b200.dist import shard_range

    for n in (0, 1, 7, 100):
        for size in (1, 2, 3, 8):
            parts = [shard_range(n, r, size) for r in range(size)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(size - 1))
