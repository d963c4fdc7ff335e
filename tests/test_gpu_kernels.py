"""GPU parity of every libdooly_b200 kernel against the CPU oracle (C-ABI path).

Bars (BASELINE.json north_star): dedup bit-exact; predictions bit-exact given
the same regressor row (the evaluation order is the pinned contract) and
within 1e-9 relative of the oracle's own fit; coefficients within 1e-9
normwise in the scaled basis; TTFT/TPOT within 1e-6 relative (we assert
bit-equality, which is stronger).
"""

from __future__ import annotations

import hashlib
import os

import numpy as np
import pytest
import torch

from helpers import ATTN, AFFINE, rows_to_table, synth_fit_data, synth_queries, table_to_rows
from oracle import profiler as oprof
from oracle import sim as osim

pytestmark = pytest.mark.gpu

COEF_TOL = 1e-9      # normwise, scaled basis
PRED_TOL = 1e-9      # relative
ERR_TOL = 1e-9


def _i32(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32))


# ------------------------------------------------------------------ fit (K2)


def _fit_gpu(kind, x, y, off, dev):
    from paper_2605_07985_b200.sim import fit_tables

    fr = fit_tables(kind, _i32(x).to(dev), torch.from_numpy(y).to(dev),
                    torch.from_numpy(off).to(dev))
    torch.cuda.synchronize()
    return fr


@pytest.mark.parametrize("kind", [AFFINE, ATTN])
@pytest.mark.parametrize("ragged", [False, True])
def test_fit_matches_oracle(kind, ragged, dev):
    x, y, off = synth_fit_data(kind, 300, 512, seed=3 + kind, ragged=ragged)
    fr = _fit_gpu(kind, x, y, off, dev)
    ref = osim.fit(kind, x, y, off)
    rows = fr.rows()
    got = rows_to_table(kind, rows)
    assert np.array_equal(fr.status.cpu().numpy(), ref["status"])
    assert np.array_equal(got["lo"], ref["lo"]) and np.array_equal(got["hi"], ref["hi"])
    assert np.array_equal(got["inv"], ref["inv"])          # IEEE 1/max on both sides
    dc = np.abs(got["coef"] - ref["coef"]).max(axis=1) / np.abs(ref["coef"]).max(axis=1)
    assert dc.max() <= COEF_TOL, dc.max()
    fe = fr.fit_err.cpu().numpy()
    assert np.allclose(fe, ref["fit_err"], rtol=ERR_TOL, atol=0)
    # predictions of the two fits on the training points agree to 1e-9 relative
    pg = osim.eval_poly(kind, got["coef"][np.repeat(np.arange(300), np.diff(off))],
                        got["inv"][np.repeat(np.arange(300), np.diff(off))], x.T)
    pr = osim.eval_poly(kind, ref["coef"][np.repeat(np.arange(300), np.diff(off))],
                        ref["inv"][np.repeat(np.arange(300), np.diff(off))], x.T)
    assert np.max(np.abs(pg - pr) / np.abs(pr)) <= PRED_TOL


def test_fit_exact_linear_and_insufficient(dev):
    # SPEC.md:562 exact linear data -> fit_error < 1e-6; SPEC.md:564 2 points -> insufficient
    xs = np.array([[1, 16, 128, 512, 2048, 8192, 5, 7]], dtype=np.uint32)
    y = 5e-6 + 1.25e-9 * xs[0].astype(np.float64)
    off = np.array([0, 6, 8], dtype=np.int64)
    fr = _fit_gpu(AFFINE, xs, y, off, dev)
    st = fr.status.cpu().numpy()
    assert st.tolist() == [0, 1]
    assert fr.fit_err.cpu().numpy()[0] < 1e-6
    rows = fr.rows()
    assert rows["lo"][1] > rows["hi"][1]      # unfitted row marker


def test_fit_rank_deficient_drops_columns(dev):
    # chunk-constant style collinearity: batch fixed at 8 -> f2 == 1 == intercept
    rng = np.random.default_rng(5)
    n = 64
    x = np.stack([rng.integers(0, 4096, n), np.full(n, 8), rng.integers(0, 1 << 16, n)]).astype(np.uint32)
    y = 1e-5 + 1e-9 * x[0] + 3e-11 * x[2]
    off = np.array([0, n], dtype=np.int64)
    fr = _fit_gpu(ATTN, x, y, off, dev)
    ref = osim.fit(ATTN, x, y, off)
    got = rows_to_table(ATTN, fr.rows())
    assert fr.status.cpu().numpy()[0] == 0
    # same dropped set (exact zeros) and the same predictions
    assert np.array_equal(got["coef"][0] == 0, ref["coef"][0] == 0)
    pg = osim.eval_poly(ATTN, got["coef"][0], got["inv"][0], x.T)
    pr = osim.eval_poly(ATTN, ref["coef"][0], ref["inv"][0], x.T)
    assert np.max(np.abs(pg - pr) / pr) <= PRED_TOL


# -------------------------------------------------------------- predict (K3)


PACKED = 2   # KIND_ATTN_PACKED: attention rows repacked to 96 B by dooly_attn_pack


def _predict_gpu(kind, rows, sig, x, dev, offset=0, packed=False):
    from paper_2605_07985_b200.sim import pack_attn, predict_batch

    table = torch.from_numpy(rows.view(np.uint8).reshape(len(rows), -1).copy()).to(dev)
    if packed:
        table, kind = pack_attn(table), PACKED
    n = sig.shape[0]
    # `offset` elements of misalignment (offset % 4 != 0 exercises the scalar path)
    sbuf = torch.zeros(n + offset, dtype=torch.int32, device=dev)
    sbuf[offset:] = _i32(sig).to(dev)
    xflat = torch.zeros(x.shape[0] * n + offset, dtype=torch.int32, device=dev)
    xflat[offset:] = _i32(x).to(dev).reshape(-1)
    out, flags, err = predict_batch(kind, table, sbuf[offset:], xflat[offset:])
    torch.cuda.synchronize()
    return out.cpu().numpy(), flags.cpu().numpy().view(np.uint32), int(err.item())


def _unpack_bits(words: np.ndarray, n: int) -> np.ndarray:
    b = np.unpackbits(words.view(np.uint8), bitorder="little")
    return b[:n].astype(bool)


@pytest.mark.parametrize("kind", [AFFINE, ATTN, PACKED])
@pytest.mark.parametrize("n_q,offset", [(1, 0), (127, 0), (4096 * 3 + 5, 0), (1000, 1), (99999, 3)])
def test_predict_bit_exact(kind, n_q, offset, dev):
    packed = kind == PACKED
    kind = ATTN if packed else kind
    x, y, off = synth_fit_data(kind, 257, 64, seed=11 + kind)
    ref_fit = osim.fit(kind, x, y, off)
    table = {k: ref_fit[k] for k in ("coef", "inv", "lo", "hi")}
    # force some clamping: shift one signature's intercept far negative
    table["coef"][7, 0] = -1.0
    rows = table_to_rows(kind, table)
    sig, xq = synth_queries(kind, table, n_q, seed=n_q, outside=0.05)
    out, flags, err = _predict_gpu(kind, rows, sig, xq, dev, offset, packed)
    ref = (osim.predict_packed(osim.pack_attn(table), sig, xq) if packed
           else osim.predict(kind, table, sig, xq))
    if packed:
        # the folded serving form vs the scaled evaluation: rounding only
        # (well inside the north_star's 1e-9 relative on latencies)
        sc = osim.predict(kind, table, sig, xq)
        live = ~sc["clamped"]
        assert np.max(np.abs(ref["out"][live] - sc["out"][live]) / sc["out"][live]) <= 1e-12
        assert np.array_equal(ref["extrap"], sc["extrap"])
    assert err == np.iinfo(np.int64).max
    assert np.array_equal(out.view(np.uint64), ref["out"].view(np.uint64))   # bit-exact
    nw = (n_q + 31) // 32
    assert np.array_equal(_unpack_bits(flags[0, :nw], n_q), ref["extrap"])
    assert np.array_equal(_unpack_bits(flags[1, :nw], n_q), ref["clamped"])


@pytest.mark.parametrize("mode", ["coop", "coop8", "coop1", "staged", "pair", "pair4", "pair4b", "pair3",
                                  "vec", "hybrid", "hybrid:0.9", "hybrid:0"])
@pytest.mark.parametrize("n_q", [8, 160 * 7, 160 * 1000 + 88])
def test_predict_packed_cooperative_kernel(mode, n_q, dev, monkeypatch):
    """Every packed-attention kernel (paired default, one lane per row, the
    cp.async-staged, the 3-lanes-per-row and the TMA gather4 + paired hybrid
    variants, the latter at several TMA shares) is bit-identical to the
    oracle, flags and unknown/unfitted rows included."""
    mode, _, frac = mode.partition(":")
    monkeypatch.setenv("DOOLY_PREDICT_ATTN", mode)
    if frac:
        monkeypatch.setenv("DOOLY_PREDICT_TMA_FRAC", frac)
    x, y, off = synth_fit_data(ATTN, 257, 64, seed=21)
    ref_fit = osim.fit(ATTN, x, y, np.array([0, 3, *off[2:]], dtype=np.int64))  # row 0 unfitted
    table = {k: ref_fit[k] for k in ("coef", "inv", "lo", "hi")}
    table["coef"][7, 0] = -1.0
    table["lo"][0], table["hi"][0] = table["lo"][1], table["hi"][1]             # box, but unfitted
    rows = table_to_rows(ATTN, table)
    rows["lo"][0] = 0xFFFFFFFF
    rows["hi"][0] = 0
    sig, xq = synth_queries(ATTN, table, n_q, seed=n_q, outside=0.05)
    sig[::97] = 300                                                             # unknown
    out, flags, err = _predict_gpu(ATTN, rows, sig, xq, dev, 0, True)
    tab = dict(table)
    tab["lo"], tab["hi"] = rows["lo"].copy(), rows["hi"].copy()
    ref = osim.predict_packed(osim.pack_attn(tab), sig, xq)
    assert np.array_equal(out.view(np.uint64), ref["out"].view(np.uint64))
    nw = (n_q + 31) // 32
    assert np.array_equal(_unpack_bits(flags[0, :nw], n_q), ref["extrap"])
    assert np.array_equal(_unpack_bits(flags[1, :nw], n_q), ref["clamped"])
    assert err == int(np.argmax(ref["bad"]))


@pytest.mark.parametrize("kind", [AFFINE, ATTN, PACKED])
def test_predict_unknown_signature(kind, dev):
    packed = kind == PACKED
    kind = ATTN if packed else kind
    x, y, off = synth_fit_data(kind, 8, 32, seed=2)
    x[:, : off[3]] = x[:, : off[3]]
    ref_fit = osim.fit(kind, x, y, np.array([0, 2, *off[2:]], dtype=np.int64))  # sig 0: 2 pts
    table = {k: ref_fit[k] for k in ("coef", "inv", "lo", "hi")}
    rows = table_to_rows(kind, table)
    sig = np.array([3, 0, 5, 100, 2], dtype=np.uint32)
    xq = np.tile(table["lo"][3][:, None], (1, 5)).astype(np.uint32)
    out, _, err = _predict_gpu(kind, rows, sig, xq, dev, packed=packed)
    assert err == 1                               # first bad query: unfitted sig 0
    assert np.isnan(out[1]) and np.isnan(out[3]) and np.isfinite(out[0])


def test_predict_host_pipeline_matches_device(dev):
    """Pinned-host entry points (chunked multi-stream pipeline, mixed kinds and a
    ragged last chunk) return exactly what the device call returns."""
    from paper_2605_07985_b200.sim import pack_attn, predict_batch, predict_host, predict_host_many

    outs = []
    batches = []
    for kind in (AFFINE, ATTN):
        x, y, off = synth_fit_data(kind, 97, 40, seed=31 + kind)
        ref_fit = osim.fit(kind, x, y, off)
        table = {k: ref_fit[k] for k in ("coef", "inv", "lo", "hi")}
        rows = table_to_rows(kind, table)
        t = torch.from_numpy(rows.view(np.uint8).reshape(len(rows), -1).copy()).to(dev)
        k = kind
        if kind == ATTN:
            t, k = pack_attn(t), PACKED
        n = 100_003 + 8 * kind
        sig, xq = synth_queries(kind, table, n, seed=5 + kind, outside=0.02)
        dev_out, dev_flags, _ = predict_batch(k, t, _i32(sig).to(dev), _i32(xq).to(dev))
        hs, hx = _i32(sig).pin_memory(), _i32(xq).pin_memory()
        ho = torch.empty(n, dtype=torch.float64).pin_memory()
        hf = torch.zeros((2, (n + 31) // 32), dtype=torch.int32).pin_memory()
        predict_host(k, t, hs, hx, ho, hf, chunk=4096 * 3, n_streams=2)
        assert torch.equal(ho, dev_out.cpu())
        assert torch.equal(hf, dev_flags.cpu())            # SPEC.md:569 flags reach the host
        assert int(hf[0].count_nonzero()) > 0              # some extrapolated queries
        outs.append((dev_out.cpu(), dev_flags.cpu()))
        batches.append((k, t, hs, hx, torch.empty(n, dtype=torch.float64).pin_memory(),
                        torch.zeros((2, (n + 31) // 32), dtype=torch.int32).pin_memory()))
    predict_host_many(batches, chunk=8192, n_streams=3)
    for (_, _, _, _, o, f), (want, want_f) in zip(batches, outs):
        assert torch.equal(o, want) and torch.equal(f, want_f)


def test_attn_pack_header_and_refusals(dev):
    """Pack header fields; tables the 96-B form cannot represent exactly are refused,
    and an unchecked refused table makes predict flag every query (never mispredict)."""
    from paper_2605_07985_b200.sim import PACK_HEADER, pack_attn, predict_batch

    x, y, off = synth_fit_data(ATTN, 64, 32, seed=5)
    ref_fit = osim.fit(ATTN, x, y, off)
    table = {k: ref_fit[k].copy() for k in ("coef", "inv", "lo", "hi")}
    t = lambda tb: torch.from_numpy(table_to_rows(ATTN, tb).view(np.uint8).reshape(64, -1).copy()).to(dev)
    pk = pack_attn(t(table))
    h = pk[0].cpu().numpy().view(PACK_HEADER)[0]
    assert int(h["ok"]) == 1 and int(h["n_sig"]) == 64 and int(h["magic"]) == 0x66504144
    assert list(h["max_hi"]) == list(table["hi"].max(axis=0))
    assert list(h["width"]) == [int(v).bit_length() for v in table["hi"].max(axis=0)]
    bad = {k: v.copy() for k, v in table.items()}
    bad["inv"][3, 1] = np.nextafter(bad["inv"][3, 1], 1.0)       # not 1/hi
    with pytest.raises(ValueError):
        pack_attn(t(bad))
    wide = {k: v.copy() for k, v in table.items()}
    wide["hi"][5] = [0xFFFFFFF0, 0xFFFFFFF0, 0xFFFFFFF0]            # 96 box bits > 64
    wide["inv"][5] = 1.0 / wide["hi"][5].astype(np.float64)
    with pytest.raises(ValueError):
        pack_attn(t(wide))
    pk = pack_attn(t(wide), check=False)
    sig = torch.zeros(40, dtype=torch.int32, device=dev)
    xq = torch.zeros((3, 40), dtype=torch.int32, device=dev)
    out, _, err = predict_batch(PACKED, pk, sig, xq)
    assert int(err.item()) == 0 and torch.isnan(out).all()


def test_predict_scalar_api_raises(dev):
    from paper_2605_07985_b200.errors import UnknownSignature
    from paper_2605_07985_b200.sim import FitResult, Regressors, predict

    x, y, off = synth_fit_data(AFFINE, 4, 16, seed=9)
    fr = _fit_gpu(AFFINE, x, y, off, dev)
    regs = Regressors({AFFINE: fr}, {b"a" * 32: (AFFINE, 1)}, dev)
    p = predict(regs, b"a" * 32, [int(x[0, off[1]])])
    ref = osim.predict(AFFINE, rows_to_table(AFFINE, fr.rows()), np.array([1]), x[:, off[1]:off[1] + 1])
    assert float(p) == ref["out"][0] and not p.extrapolated
    with pytest.raises(UnknownSignature):
        predict(regs, b"b" * 32, [1])


# ------------------------------------------------------------- SHA-256 / dedup


def test_sha256_messages_kat_and_random(dev):
    from paper_2605_07985_b200.profiler import signature_hash, signature_hash_batch

    assert signature_hash(b"").hex() == \
        "e3b0c44298fc1c149afbf4c8996fb92427ae41e4649b934ca495991b7852b855"
    rng = np.random.default_rng(0)
    msgs = [rng.bytes(int(n)) for n in rng.integers(0, 700, size=3000)]
    msgs += [b"a" * n for n in range(0, 130)]          # every padding boundary
    got = signature_hash_batch(msgs)
    assert got == [hashlib.sha256(m).digest() for m in msgs]


def test_record_hash_matches_oracle_canonical(corpus, dev):
    from paper_2605_07985_b200.profiler import DeviceRecords, hash_records
    from paper_2605_07985_b200.records import corpus_entries, pack_entries

    for tp in (1, 4):
        ents = [e for _, _, es in corpus_entries(corpus, tp=tp) for e in es]
        recs = DeviceRecords.from_packed(pack_entries(ents), dev)
        got = hash_records(recs).cpu().numpy()
        want = [oprof.signature_hash(oprof.canonicalize(e.to_json())) for e in ents]
        assert [bytes(r) for r in got] == want


def _dedup_gpu(digs: np.ndarray, db: np.ndarray, dev):
    from paper_2605_07985_b200.profiler import dedup_digests

    r = dedup_digests(torch.from_numpy(digs).to(dev),
                      torch.from_numpy(db).to(dev) if db is not None else None)
    return {"first": r.first.cpu().numpy().tolist(), "uid": r.uid.cpu().numpy().tolist(),
            "is_new": r.is_new.cpu().numpy().astype(bool).tolist(),
            "in_db": r.in_db.cpu().numpy().astype(bool).tolist(), "n_unique": r.n_unique}


@pytest.mark.parametrize("insert", ["thread", "group"])
@pytest.mark.parametrize("n,n_distinct,n_db", [(1, 1, 0), (1000, 100, 0), (50000, 20000, 5000),
                                               (200000, 150000, 0)])
def test_dedup_bit_exact(n, n_distinct, n_db, insert, dev, monkeypatch):
    """Both insert kernels (one thread per key; 8-lane groups per 256-bit key,
    DOOLY_DEDUP_INSERT=group) against the oracle."""
    if insert == "group":
        monkeypatch.setenv("DOOLY_DEDUP_INSERT", "group")
    rng = np.random.default_rng(n)
    pool = rng.integers(0, 256, size=(n_distinct, 32), dtype=np.uint8)
    # collisions on the probe word (first 4 bytes) but different digests
    pool[1::7, :4] = pool[0, :4]
    digs = pool[rng.integers(0, n_distinct, size=n)]
    db = pool[rng.choice(n_distinct, size=n_db, replace=False)] if n_db else np.zeros((0, 32), np.uint8)
    got = _dedup_gpu(digs, db, dev)
    ref = oprof.dedup_digests([bytes(d) for d in digs], [bytes(d) for d in db])
    assert got == ref


def test_dedup_empty(dev):
    got = _dedup_gpu(np.zeros((0, 32), np.uint8), None, dev)
    assert got["n_unique"] == 0 and got["first"] == []


def test_corpus_census_and_rerun(corpus, dev):
    """Table 2: attention 42 occurrences, 27
    reuses, groups 24/21, 6/3, 6/3, 3/0, 3/0; re-run profiles nothing."""
    from paper_2605_07985_b200 import modelir
    from paper_2605_07985_b200.profiler import LatencyDB, dedup
    from paper_2605_07985_b200.records import corpus_entries

    db = LatencyDB()
    groups: dict = {}
    for m, b, ents in corpus_entries(corpus):
        att = [e for e in ents if e.name == "attention"]
        to_profile, skipped = dedup(att, db, device=dev)
        for e in att:
            key = modelir.geometry_key(m, m.layer_attention.index(e.window))
            g = groups.setdefault(key, [0, 0])
            g[0] += 1
        for e in skipped:
            key = modelir.geometry_key(m, m.layer_attention.index(e.window))
            groups[key][1] += 1
    assert groups == {"q32/kv8/d128/full": [24, 21], "q28/kv4/d128/full": [6, 3],
                      "q32/kv32/d128/full": [6, 3], "q32/kv8/d128/swa4096": [3, 0],
                      "q32/kv8/d128/swa32768": [3, 0]}
    assert len(db.signatures) == 42 - 27
    again = [e for _, _, es in corpus_entries(corpus) for e in es if e.name == "attention"]
    to_profile, skipped = dedup(again, db, device=dev)
    assert to_profile == [] and len(skipped) == 42


def test_a3_overall_reuse_on_gpu(corpus, dev):
    """A3 through the GPU dedup, config by config into one DB over
    the whole corpus (every record kind): N = 486, R = 439, 47 unique = N - R,
    reuse >= 50%, >= 95% of the uniques seen within the first four models."""
    from paper_2605_07985_b200.profiler import LatencyDB, dedup
    from paper_2605_07985_b200.records import corpus_entries

    db = LatencyDB()
    n = r = 0
    per_model, cur = [], None
    for m, _, ents in corpus_entries(corpus):
        to_profile, skipped = dedup(ents, db, device=dev)
        n += len(ents)
        r += len(skipped)
        if m.name != cur:
            cur = m.name
            per_model.append(0)
        per_model[-1] = len(db.signatures)
    assert (n, r, len(db.signatures)) == (486, 439, 47)
    assert r / n >= 0.5 and per_model[3] >= 0.95 * per_model[-1]


def test_dedup_packed_large_uniform(dev):
    """C5-style bulk records (vectorised packer) vs oracle digests + dedup."""
    from paper_2605_07985_b200.profiler import DeviceRecords, dedup_packed
    from paper_2605_07985_b200.records import pack_uniform
    from bench import synth_records

    packed, n_dims = synth_records(200_000, seed=4)
    recs = DeviceRecords.from_packed(packed, dev)
    res = dedup_packed(recs)
    digs = res.digests.cpu().numpy()
    # spot-check digests against the oracle's canonical hash on a sample
    rng = np.random.default_rng(0)
    w = packed.words
    for i in rng.choice(packed.n, size=300, replace=False):
        o = int(packed.rec_off[i])
        ent = _entry_from_words(packed, o)
        assert bytes(digs[i]) == oprof.signature_hash(oprof.canonicalize(ent))
    ref = oprof.dedup_digests([bytes(d) for d in digs])
    assert res.n_unique == ref["n_unique"]
    assert res.first.cpu().numpy().tolist() == ref["first"]
    assert res.uid.cpu().numpy().tolist() == ref["uid"]


def _entry_from_words(p, o):
    w = p.words
    op, nd, ns, attr = int(w[o]), int(w[o + 1]) & 0xFFFF, int(w[o + 1]) >> 16, int(w[o + 2])
    flat = []
    scal = []
    pos_val = [(int(w[o + 4 + 3 * k]), int(w[o + 5 + 3 * k]) | (int(w[o + 6 + 3 * k]) << 32))
               for k in range(nd)]
    # rebuild an arg template whose MC positions are exactly pos_val (others NT)
    maxpos = max([pv[0] for pv in pos_val if pv[0] < 65536], default=-1)
    pm = dict(pos_val)
    flat = [[pm.get(i, 7), "MC" if i in pm else "NT"] for i in range(maxpos + 1)]
    for k in range(max([pv[0] - 65536 for pv in pos_val if pv[0] >= 65536], default=-1) + 1):
        scal.append([pm.get(65536 + k, 3), "MC" if 65536 + k in pm else "NR"])
    syms = []
    for k in range(ns):
        sid = int(w[o + 4 + 3 * nd + k])
        syms.append(bytes(p.sym_bytes[p.sym_off[sid]:p.sym_off[sid + 1]]).decode())
    name = bytes(p.op_bytes[p.op_off[op]:p.op_off[op + 1]]).decode()
    ent = {"name": name, "granularity": "operator", "arg_template": [flat], "scalars": scal,
           "kernel_symbols": syms, "attrs": {}}
    assert attr == 0xFFFFFFFF
    return ent


# --------------------------------------------------------------- sim (K4)


def _random_oplist(rng, n_aff, n_attn, window, tp):
    from paper_2605_07985_b200 import _lib

    ops = []
    for e in range(12):
        r = rng.random()
        if r < 0.25:
            ops.append({"feat": osim.FEAT_ATTN, "row": int(rng.integers(n_attn)),
                        "window_slot": int(window > 0 and rng.random() < 0.5),
                        "repeat": int(rng.integers(1, 40))})
        elif r < 0.35:
            ops.append({"feat": osim.FEAT_NUM_SEQS, "row": int(rng.integers(n_aff)),
                        "window_slot": 0, "repeat": 1})
        else:
            ops.append({"feat": osim.FEAT_NUM_TOKS, "row": int(rng.integers(n_aff)),
                        "window_slot": 0, "repeat": int(rng.integers(1, 80))})
    if tp > 1:
        ops.append({"feat": osim.FEAT_COMM, "row": 0, "window_slot": 0, "repeat": 160,
                    "bytes_per_tok": 8192 * 2})
    ol = _lib.OpList()
    ol.n_ops = len(ops)
    ol.tp = tp
    ol.comm_alpha, ol.comm_beta = 5e-6, 5e-12
    for i, o in enumerate(ops):
        ol.feat[i], ol.row[i], ol.repeat[i] = o["feat"], o["row"], o["repeat"]
        ol.window_slot[i] = o["window_slot"]
        ol.bytes_per_tok[i] = o.get("bytes_per_tok", 0)
    return ops, ol


def _sim_setup(seed, window=0, tp=1):
    from paper_2605_07985_b200.sim import CallTree, Regressors, FitResult

    rng = np.random.default_rng(seed)
    xa, ya, oa = synth_fit_data(AFFINE, 20, 24, seed=seed)
    xt, yt, ot = synth_fit_data(ATTN, 6, 64, seed=seed + 1)
    fa, ft = osim.fit(AFFINE, xa, ya, oa), osim.fit(ATTN, xt, yt, ot)
    ta = {k: fa[k] for k in ("coef", "inv", "lo", "hi")}
    tt = {k: ft[k] for k in ("coef", "inv", "lo", "hi")}
    ops, ol = _random_oplist(rng, 20, 6, window, tp)
    for o in ops:
        if o["feat"] == osim.FEAT_ATTN:
            o["coef"], o["inv"] = list(tt["coef"][o["row"]]), list(tt["inv"][o["row"]])
        elif o["feat"] != osim.FEAT_COMM:
            o["coef"], o["inv"] = list(ta["coef"][o["row"]]), list(ta["inv"][o["row"]])
    return ta, tt, ops, ol


def _regs(ta, tt, dev):
    from paper_2605_07985_b200.sim import FitResult, Regressors

    def fr(kind, t):
        rows = table_to_rows(kind, t)
        tab = torch.from_numpy(rows.view(np.uint8).reshape(len(rows), -1).copy()).to(dev)
        n = len(rows)
        return FitResult(kind, tab, torch.zeros(n, dtype=torch.float64, device=dev),
                         torch.zeros(n, dtype=torch.uint8, device=dev))

    return Regressors({AFFINE: fr(AFFINE, ta), ATTN: fr(ATTN, tt)}, {}, dev)


@pytest.mark.parametrize("tp", [1, 4])
def test_iter_eval_bit_exact(tp, dev):
    from paper_2605_07985_b200.sim import CallTree, iter_latency_batch

    ta, tt, ops, ol = _sim_setup(21 + tp, window=4096, tp=tp)
    regs = _regs(ta, tt, dev)
    rng = np.random.default_rng(tp)
    n = 20000
    feats = np.stack([rng.integers(1, 8192, n), rng.integers(0, 8192, n), rng.integers(1, 256, n),
                      rng.integers(0, 1 << 21, n), rng.integers(0, 1 << 20, n)]).astype(np.uint32)
    ct = CallTree([], ol, 4096)
    got = iter_latency_batch(_i32(feats).to(dev), ct, regs).cpu().numpy()
    want = np.array([osim.iter_latency(tuple(int(v) for v in feats[:, i]), ops, tp, 5e-6, 5e-12)
                     for i in range(n)])
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def _workload(n, seed, rate=4.0, cached_frac=0.0):
    rng = np.random.default_rng(seed)
    arr = np.cumsum(rng.exponential(1.0 / rate, size=n))
    pr = rng.integers(1, 9000, size=n).astype(np.uint32)
    ou = rng.integers(1, 300, size=n).astype(np.uint32)
    ca = np.where(rng.random(n) < cached_frac, pr, 0).astype(np.uint32)
    return arr, pr, ou, ca


@pytest.mark.parametrize("seed,n,shards,window,tp,cap", [
    (1, 400, 1, 0, 1, 10**15), (2, 3000, 8, 4096, 1, 10**15), (3, 2000, 4, 0, 4, 3 * 10**10),
    (4, 1500, 3, 1024, 1, 4 * 10**9)])
def test_sim_run_bit_exact(seed, n, shards, window, tp, cap, dev):
    from paper_2605_07985_b200 import _lib
    from paper_2605_07985_b200.sim import CallTree, ShardedTrace, collect, run_sharded

    ta, tt, ops, ol = _sim_setup(seed, window=window, tp=tp)
    regs = _regs(ta, tt, dev)
    arr, pr, ou, ca = _workload(n, seed, cached_frac=0.1 if seed % 2 else 0.0)
    sc = _lib.Sched()
    sc.chunk, sc.max_batch, sc.window = 2048, 64, window
    sc.kv_bytes_per_token, sc.kv_capacity_bytes, sc.max_iterations = 131072, cap, 10**7
    trace = ShardedTrace.from_arrays(arr, pr, ou, ca, shards, dev)
    res = run_sharded(trace, CallTree([], ol, window), sc, regs, log_cap=4000)
    met = collect(trace, res)
    ref = osim.run_shards(arr.tolist(), pr.tolist(), ou.tolist(), ca.tolist(), shards, ops=ops,
                          chunk=2048, max_batch=64, kv_bytes_per_token=131072, kv_capacity=cap,
                          window=window, tp=tp, alpha=5e-6, beta=5e-12)
    assert res.n_iter.cpu().numpy().tolist() == ref["n_iter"]
    assert np.array_equal(res.clock.cpu().numpy(), np.array(ref["clock"]))
    assert np.array_equal(met.ttft.view(np.uint64), ref["ttft"].view(np.uint64))
    assert np.array_equal(np.isnan(met.tpot), np.isnan(ref["tpot"]))
    m = ~np.isnan(ref["tpot"])
    assert np.array_equal(met.tpot[m], ref["tpot"][m])
    # per-iteration features + latency of shard 0 (schedule compositions identical)
    r0 = osim.run_shard(arr[0::shards].tolist(), pr[0::shards].tolist(), ou[0::shards].tolist(),
                        ca[0::shards].tolist(), ops, 2048, 64, 131072, cap, window, tp, 5e-6,
                        5e-12, log=True)
    k = min(len(r0["lat"]), 4000)
    lf = res.log_feat.cpu().numpy().view(np.uint32)[0, :k]
    assert [tuple(int(v) for v in row) for row in lf] == [tuple(f) for f in r0["feats"][:k]]
    assert np.array_equal(res.log_lat.cpu().numpy()[0, :k], np.array(r0["lat"][:k]))


@pytest.mark.parametrize("seed,n,shards,window,tp", [(5, 600, 1, 0, 1), (6, 2500, 5, 4096, 4)])
def test_sim_eval_host_schedule_bit_exact(seed, n, shards, window, tp, dev):
    """dooly_sim_eval on the oracle event loop's own schedule: identical iteration
    latencies, clocks (idle jumps included) and TTFT/TPOT, bit for bit."""
    from paper_2605_07985_b200.sim import CallTree, sim_eval

    ta, tt, ops, ol = _sim_setup(seed, window=window, tp=tp)
    regs = _regs(ta, tt, dev)
    arr, pr, ou, ca = _workload(n, seed, rate=2.0, cached_frac=0.1)
    feats, start, clocks, lat, off = [], [], [], [], [0]
    first = np.full(n, -1, dtype=np.int64)
    last = np.full(n, -1, dtype=np.int64)
    ttft_ref = np.full(n, np.nan)
    tpot_ref = np.full(n, np.nan)
    for s in range(shards):
        idx = np.arange(s, n, shards)
        r = osim.run_shard(arr[idx].tolist(), pr[idx].tolist(), ou[idx].tolist(),
                           ca[idx].tolist(), ops, 2048, 64, 131072, 10**15, window, tp, 5e-6,
                           5e-12, log=True)
        base = off[-1]
        feats += r["feats"]
        start += r["start"]
        clocks += r["clocks"]
        lat += r["lat"]
        off.append(base + len(r["lat"]))
        f, l = np.array(r["first_it"]), np.array(r["last_it"])
        first[idx] = np.where(f >= 0, f + base, -1)
        last[idx] = np.where(l >= 0, l + base, -1)
        ttft_ref[idx], tpot_ref[idx] = r["ttft"], r["tpot"]
    assert any(v > 0 for v in start)                       # idle jumps are exercised
    it_feat = _i32(np.array(feats, dtype=np.uint32).T.copy()).to(dev)
    t = lambda a, dt: torch.from_numpy(np.asarray(a, dtype=dt)).to(dev)
    it_lat, clock, ttft, tpot = sim_eval(
        CallTree([], ol, window), regs, it_feat, t(arr, np.float64),
        t(first.astype(np.int32), np.int32), t(last.astype(np.int32), np.int32),
        _i32(ou.astype(np.uint32)).to(dev), it_start=t(start, np.float64),
        it_off=t(off, np.int64))
    assert np.array_equal(it_lat.cpu().numpy(), np.array(lat))
    assert np.array_equal(clock.cpu().numpy(), np.array(clocks))
    g1, g2 = ttft.cpu().numpy(), tpot.cpu().numpy()
    assert np.array_equal(g1.view(np.uint64), ttft_ref.view(np.uint64))
    assert np.array_equal(np.isnan(g2), np.isnan(tpot_ref))
    m = ~np.isnan(tpot_ref)
    assert np.array_equal(g2[m], tpot_ref[m])
    with pytest.raises(ValueError):                        # out-of-range iteration index
        bad = first.copy()
        bad[0] = len(lat) + 5
        sim_eval(CallTree([], ol, window), regs, it_feat, t(arr, np.float64),
                 t(bad.astype(np.int32), np.int32), t(last.astype(np.int32), np.int32),
                 _i32(ou.astype(np.uint32)).to(dev), it_start=t(start, np.float64),
                 it_off=t(off, np.int64))


def test_dedup_single_call_matches_two_calls(corpus, dev):
    from paper_2605_07985_b200.profiler import (DeviceRecords, dedup_digests, dedup_packed,
                                                hash_records)
    from paper_2605_07985_b200.records import pack_entries, synthesize_entries

    ents = [e for m in corpus.models for b in corpus.backends for e in synthesize_entries(m, b)]
    recs = DeviceRecords.from_packed(pack_entries(ents), dev)
    one = dedup_packed(recs)
    dig = hash_records(recs)
    two = dedup_digests(dig, one.digests[:7].clone())
    one_db = dedup_packed(recs, one.digests[:7].clone())
    assert torch.equal(one.digests, dig)
    for a, b in ((one_db.first, two.first), (one_db.uid, two.uid), (one_db.is_new, two.is_new),
                 (one_db.in_db, two.in_db)):
        assert torch.equal(a, b)
    assert one_db.n_unique == two.n_unique == one.n_unique


@pytest.mark.parametrize("source", ["corpus", "synth"])
@pytest.mark.parametrize("with_db", [False, True])
@pytest.mark.parametrize("insert", ["thread", "group"])
def test_dedup_record_grouping_matches_ungrouped(source, with_db, insert, corpus, dev,
                                                 monkeypatch):
    """dooly_dedup hashes each distinct packed content once (records that
    differ only in the repeat count share a digest), copies the digest to the
    rest, and inserts only each group's smallest index into the digest table
    (the others resolve through it): every output equals the path that hashes
    and inserts every record (DOOLY_DEDUP_GROUP=0), with either insert kernel,
    and the digests equal the standalone dooly_sha256_records of every record."""
    if insert == "group":
        monkeypatch.setenv("DOOLY_DEDUP_INSERT", "group")
    from paper_2605_07985_b200.profiler import DeviceRecords, dedup_packed, hash_records
    from paper_2605_07985_b200.records import pack_entries, synthesize_entries
    from bench import synth_records

    rng = np.random.default_rng(5)
    if source == "corpus":
        ents = [e for m in corpus.models for b in corpus.backends for e in synthesize_entries(m, b)]
        ents = [ents[i] for i in rng.permutation(len(ents))] * 3
        packed = pack_entries(ents)
        # vary the repeat count (w3, not hashed) of every record
        packed.words[packed.rec_off[:packed.n] + 3] = rng.integers(1, 1 << 20, packed.n)
    else:
        packed, _ = synth_records(300_000, seed=9)
    recs = DeviceRecords.from_packed(packed, dev)
    db = hash_records(recs)[rng.choice(recs.n, 5, replace=False)].clone() if with_db else None
    monkeypatch.delenv("DOOLY_DEDUP_GROUP", raising=False)
    g = dedup_packed(recs, db)
    monkeypatch.setenv("DOOLY_DEDUP_GROUP", "0")
    u = dedup_packed(recs, db)
    assert torch.equal(g.digests, u.digests)
    assert torch.equal(g.digests, hash_records(recs))
    for a, b in ((g.first, u.first), (g.uid, u.uid), (g.is_new, u.is_new), (g.in_db, u.in_db)):
        assert torch.equal(a, b)
    assert g.n_unique == u.n_unique
    if source == "corpus":
        assert g.n_unique < recs.n // 3


def test_sim_non_termination(dev):
    from paper_2605_07985_b200 import _lib
    from paper_2605_07985_b200.errors import NonTermination
    from paper_2605_07985_b200.sim import CallTree, ShardedTrace, collect, run_sharded

    ta, tt, ops, ol = _sim_setup(7)
    regs = _regs(ta, tt, dev)
    arr, pr, ou, ca = _workload(50, 7)
    sc = _lib.Sched()
    sc.chunk, sc.max_batch, sc.window = 2048, 64, 0
    sc.kv_bytes_per_token, sc.kv_capacity_bytes, sc.max_iterations = 1, 10**12, 10
    trace = ShardedTrace.from_arrays(arr, pr, ou, ca, 1, dev)
    with pytest.raises(NonTermination):
        collect(trace, run_sharded(trace, CallTree([], ol, 0), sc, regs))


def test_library_launch_counter(dev):
    from paper_2605_07985_b200 import _lib

    before = _lib.launch_count(dev)
    x, y, off = synth_fit_data(AFFINE, 4, 16, seed=1)
    _fit_gpu(AFFINE, x, y, off, dev)
    assert _lib.launch_count(dev) == before + 1


def test_sim_run_max_batch_1024(dev):
    """The largest running batch the C-ABI accepts (1024 slots x 40 B of
    per-warp shared memory) against the oracle event loop, bit for bit."""
    from paper_2605_07985_b200 import _lib
    from paper_2605_07985_b200.sim import CallTree, ShardedTrace, collect, run_sharded

    ta, tt, ops, ol = _sim_setup(9, window=0, tp=1)
    regs = _regs(ta, tt, dev)
    arr, pr, ou, ca = _workload(4000, 9, rate=400.0)
    sc = _lib.Sched()
    sc.chunk, sc.max_batch, sc.window = 8192, 1024, 0
    sc.kv_bytes_per_token, sc.kv_capacity_bytes, sc.max_iterations = 131072, 10**15, 10**7
    trace = ShardedTrace.from_arrays(arr, pr, ou, ca, 2, dev)
    res = run_sharded(trace, CallTree([], ol, 0), sc, regs)
    met = collect(trace, res)
    ref = osim.run_shards(arr.tolist(), pr.tolist(), ou.tolist(), ca.tolist(), 2, ops=ops,
                          chunk=8192, max_batch=1024, kv_bytes_per_token=131072,
                          kv_capacity=10**15, window=0, tp=1, alpha=5e-6, beta=5e-12)
    assert res.n_iter.cpu().numpy().tolist() == ref["n_iter"]
    assert np.array_equal(met.ttft.view(np.uint64), ref["ttft"].view(np.uint64))
    m = ~np.isnan(ref["tpot"])
    assert np.array_equal(met.tpot[m], ref["tpot"][m])
