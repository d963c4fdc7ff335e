"""Seeded randomized parity sweeps on the GPU: many small configurations per
kernel family, each against the CPU oracle at the same bar as the targeted
tests (bit-exact for the serving loop and predictions, the fit contract for
coefficients).  The serving-loop sweep varies exactly what its exact decode
windows depend on (arrival rate, batch cap, chunk, KV cap, windows, cached
prompts, tensor parallelism)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from helpers import AFFINE, ATTN, rows_to_table, synth_fit_data, synth_queries, table_to_rows
from oracle import sim as osim
from test_gpu_kernels import PACKED, _predict_gpu, _regs, _sim_setup, _unpack_bits

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", range(40))
def test_sim_run_random_configs(case, dev):
    from paper_2605_07985_b200 import _lib
    from paper_2605_07985_b200.sim import CallTree, ShardedTrace, collect, run_sharded

    rng = np.random.default_rng(1000 + case)
    window = int(rng.choice([0, 0, 512, 4096]))
    tp = int(rng.choice([1, 1, 2, 4]))
    shards = int(rng.integers(1, 7))
    n = int(rng.integers(50, 900))
    rate = float(rng.choice([0.5, 4.0, 40.0, 400.0]))
    chunk = int(rng.choice([256, 2048, 8192]))
    max_batch = int(rng.choice([1, 4, 32, 256]))
    cap = int(rng.choice([10**15, 6 * 10**9, 2 * 10**9]))
    ta, tt, ops, ol = _sim_setup(2000 + case, window=window, tp=tp)
    regs = _regs(ta, tt, dev)
    arr = np.cumsum(rng.exponential(1.0 / rate, size=n))
    pr = rng.integers(1, 6000, size=n).astype(np.uint32)
    ou = rng.integers(1, 400, size=n).astype(np.uint32)
    ca = np.where(rng.random(n) < 0.15, pr, 0).astype(np.uint32)
    sc = _lib.Sched()
    sc.chunk, sc.max_batch, sc.window = chunk, max_batch, window
    sc.kv_bytes_per_token, sc.kv_capacity_bytes, sc.max_iterations = 131072, cap, 10**7
    trace = ShardedTrace.from_arrays(arr, pr, ou, ca, shards, dev)
    res = run_sharded(trace, CallTree([], ol, window), sc, regs)
    met = collect(trace, res)
    ref = osim.run_shards(arr.tolist(), pr.tolist(), ou.tolist(), ca.tolist(), shards, ops=ops,
                          chunk=chunk, max_batch=max_batch, kv_bytes_per_token=131072,
                          kv_capacity=cap, window=window, tp=tp, alpha=5e-6, beta=5e-12)
    assert res.n_iter.cpu().numpy().tolist() == ref["n_iter"]
    assert np.array_equal(res.clock.cpu().numpy(), np.array(ref["clock"]))
    assert np.array_equal(met.ttft.view(np.uint64), ref["ttft"].view(np.uint64))
    m = ~np.isnan(ref["tpot"])
    assert np.array_equal(np.isnan(met.tpot), ~m)
    assert np.array_equal(met.tpot[m].view(np.uint64), ref["tpot"][m].view(np.uint64))


@pytest.mark.parametrize("case", range(120))
def test_sim_run_window_edges(case, dev):
    """The serving loop's windows at their edges, every shard's per-iteration
    features and latencies against the oracle event loop: short outputs (many
    finishes inside a window, requests finishing in their admitting iteration),
    fully cached prompts (first decode step at admission), prompts longer than
    the chunk (partial prefills end the window at iteration 0), batch and KV
    caps that block the FCFS head (windows run across arrivals until the first
    finish), bursts and idle gaps."""
    from paper_2605_07985_b200 import _lib
    from paper_2605_07985_b200.sim import CallTree, ShardedTrace, collect, run_sharded

    rng = np.random.default_rng(5000 + case)
    window = int(rng.choice([0, 0, 0, 64]))
    tp = int(rng.choice([1, 2]))
    shards = int(rng.integers(8, 33))
    n = int(rng.integers(200, 1200))
    chunk = int(rng.choice([64, 512, 8192]))
    max_batch = int(rng.choice([2, 8, 48, 64]))
    max_batch = min(max_batch, chunk)
    cap = int(rng.choice([10**15, 3 * 10**8, 8 * 10**8]))
    ta, tt, ops, ol = _sim_setup(6000 + case, window=window, tp=tp)
    regs = _regs(ta, tt, dev)
    gaps = rng.exponential(1.0 / float(rng.choice([2.0, 50.0, 2000.0])), size=n)
    gaps[rng.random(n) < 0.05] *= 200.0        # idle gaps
    gaps[rng.random(n) < 0.2] = 0.0            # bursts (equal arrival times)
    arr = np.cumsum(gaps)
    pr = rng.integers(1, 3 * chunk if rng.random() < 0.5 else 600, size=n).astype(np.uint32)
    pr = np.minimum(pr, 2000).astype(np.uint32)
    ou = np.where(rng.random(n) < 0.3, rng.integers(1, 4, size=n),
                  rng.integers(1, 60, size=n)).astype(np.uint32)
    ca = np.where(rng.random(n) < 0.2, pr, np.where(rng.random(n) < 0.2, pr // 2, 0)).astype(np.uint32)
    kvb = 131072
    cap = max(cap, int((int(pr.max()) + int(ou.max())) * kvb))   # every request fits alone
    sc = _lib.Sched()
    sc.chunk, sc.max_batch, sc.window = chunk, max_batch, window
    sc.kv_bytes_per_token, sc.kv_capacity_bytes, sc.max_iterations = kvb, cap, 10**7
    trace = ShardedTrace.from_arrays(arr, pr, ou, ca, shards, dev)
    log_cap = 6000
    res = run_sharded(trace, CallTree([], ol, window), sc, regs, log_cap=log_cap)
    met = collect(trace, res)
    n_iter = res.n_iter.cpu().numpy().tolist()
    lf = res.log_feat.cpu().numpy().view(np.uint32)
    ll = res.log_lat.cpu().numpy()
    for s in range(shards):
        r = osim.run_shard(arr[s::shards].tolist(), pr[s::shards].tolist(), ou[s::shards].tolist(),
                           ca[s::shards].tolist(), ops, chunk, max_batch, kvb, cap, window, tp,
                           5e-6, 5e-12, log=True)
        assert n_iter[s] == r["n_iter"], s
        k = min(r["n_iter"], log_cap)
        assert [tuple(int(v) for v in row) for row in lf[s, :k]] == \
            [tuple(f) for f in r["feats"][:k]], s
        assert np.array_equal(ll[s, :k], np.array(r["lat"][:k])), s
        idx = np.arange(s, n, shards)
        assert np.array_equal(met.ttft[idx].view(np.uint64), np.asarray(r["ttft"]).view(np.uint64)), s
        rt = np.asarray(r["tpot"])
        assert np.array_equal(np.isnan(met.tpot[idx]), np.isnan(rt)), s
        m = ~np.isnan(rt)
        assert np.array_equal(met.tpot[idx][m].view(np.uint64), rt[m].view(np.uint64)), s


@pytest.mark.parametrize("mode", ["0", "1"])
@pytest.mark.parametrize("case", range(6))
def test_sim_run_window_eval_modes(mode, case, dev, monkeypatch):
    """The window's evaluation fallbacks (DOOLY_SIM_PV=1: per-lane product
    columns, 0: the plain per-lane loop — used when the decode-product table
    does not fit in shared memory) give the same bit-exact runs."""
    monkeypatch.setenv("DOOLY_SIM_PV", mode)
    test_sim_run_window_edges(case, dev)


@pytest.mark.parametrize("case", range(24))
def test_predict_random_tables(case, dev):
    """Random table sizes, query counts and misalignments; fitted, unfitted
    (lo > hi) and clamped rows; out-of-box and out-of-range queries."""
    rng = np.random.default_rng(3000 + case)
    kind = [AFFINE, ATTN, PACKED][case % 3]
    packed = kind == PACKED
    k = ATTN if packed else kind
    n_sig = int(rng.integers(1, 3000))
    x, y, off = synth_fit_data(k, n_sig, 48, seed=case)
    f = osim.fit(k, x, y, off)
    table = {key: f[key].copy() for key in ("coef", "inv", "lo", "hi")}
    neg = rng.random(n_sig) < 0.05
    table["coef"][neg, 0] = -abs(table["coef"][neg, 0]) - 1.0      # clamped predictions
    n_q = int(rng.integers(1, 200_000))
    offset = int(rng.choice([0, 0, 1, 3]))
    sig, xq = synth_queries(k, table, n_q, seed=case + 7, outside=0.1)
    sig[rng.random(n_q) < 0.002] = n_sig + 5                       # unknown signatures
    if packed:
        unfit = np.zeros(n_sig, bool)
    else:
        unfit = rng.random(n_sig) < 0.03                            # unfitted rows: lo > hi
        table["lo"][unfit] = 0xFFFFFFFF
        table["hi"][unfit] = 0
        table["coef"][unfit] = np.nan
        table["inv"][unfit] = np.nan
    rows = table_to_rows(k, table)
    out, flags, err = _predict_gpu(k, rows, sig, xq, dev, offset, packed)
    # packed tables serve the folded 96-B rows (oracle predict_packed is their contract)
    ref = (osim.predict_packed(osim.pack_attn(table), sig, xq) if packed
           else osim.predict(k, table, sig, xq))
    bad = np.flatnonzero(ref["bad"])
    assert err == (int(bad[0]) if bad.size else np.iinfo(np.int64).max)
    ok = ~ref["bad"]
    assert np.array_equal(out[ok].view(np.uint64), ref["out"][ok].view(np.uint64))
    assert np.isnan(out[~ok]).all()
    nw = (n_q + 31) // 32
    assert np.array_equal(_unpack_bits(flags[0, :nw], n_q), ref["extrap"])
    assert np.array_equal(_unpack_bits(flags[1, :nw], n_q), ref["clamped"])


@pytest.mark.parametrize("case", range(20))
def test_fit_random_csr(case, dev):
    """Random signature counts and point counts per signature, including
    signatures below the minimum (InsufficientData status), against the oracle."""
    from paper_2605_07985_b200.sim import fit_tables

    rng = np.random.default_rng(4000 + case)
    kind = AFFINE if case % 2 == 0 else ATTN
    n_sig = int(rng.integers(1, 400))
    x, y, off = synth_fit_data(kind, n_sig, int(rng.integers(12, 300)), seed=case, ragged=True)
    counts = np.diff(off)
    need = 4 if kind == AFFINE else 11
    short = rng.random(n_sig) < 0.1                                 # cut to 1..need-1 points
    new_counts = np.where(short, np.minimum(counts, rng.integers(1, need, n_sig)), counts)
    keep = np.concatenate([np.arange(off[s], off[s] + new_counts[s]) for s in range(n_sig)])
    x, y = np.ascontiguousarray(x[:, keep]), y[keep]
    off = np.concatenate([[0], np.cumsum(new_counts)]).astype(np.int64)
    ref = osim.fit(kind, x, y, off)
    fr = fit_tables(kind, torch.from_numpy(np.ascontiguousarray(x).view(np.int32)).to(dev),
                    torch.from_numpy(y).to(dev), torch.from_numpy(off).to(dev))
    torch.cuda.synchronize()
    got = rows_to_table(kind, fr.rows())
    st = fr.status.cpu().numpy()
    assert np.array_equal(st, ref["status"])
    ok = st == 0
    assert np.array_equal(got["lo"][ok], ref["lo"][ok]) and np.array_equal(got["hi"][ok], ref["hi"][ok])
    assert np.array_equal(got["inv"][ok], ref["inv"][ok])
    if ok.any():
        c, r = got["coef"][ok], ref["coef"][ok]
        d = np.abs(c - r).max(axis=1) / np.abs(r).max(axis=1)
        assert d.max() <= 1e-9, d.max()
        fe, fr_ = fr.fit_err.cpu().numpy()[ok], ref["fit_err"][ok]
        assert np.all(np.abs(fe - fr_) <= 1e-9 * fr_ + 1e-12)


@pytest.mark.parametrize("shift", [0, 1, 3])
def test_fit_csr_affine_warp_large_ragged(shift, dev, monkeypatch):
    """The warp-per-signature affine CSR kernel on ragged signatures of 1k-6k
    points at every head misalignment (offsets shifted by `shift` points, so
    the 4-point vector body starts after a 1-3 point head), against the oracle
    and against the staged CTA kernel (DOOLY_FIT_CSR_AFFINE=stage)."""
    from paper_2605_07985_b200.sim import fit_tables

    x, y, off = synth_fit_data(AFFINE, 60, 6000, seed=90 + shift, ragged=True)
    pad = np.full((1, shift), 7, np.uint32)
    x = np.ascontiguousarray(np.concatenate([pad, x], axis=1))
    y = np.concatenate([np.full(shift, 1e-5), y])
    off = np.concatenate([[0], off + shift]).astype(np.int64)     # signature 0: the padding
    xt = torch.from_numpy(x.view(np.int32)).to(dev)
    yt, ot = torch.from_numpy(y).to(dev), torch.from_numpy(off).to(dev)
    ref = osim.fit(AFFINE, x, y, off)
    fr = fit_tables(AFFINE, xt, yt, ot)
    monkeypatch.setenv("DOOLY_FIT_CSR_AFFINE", "stage")
    fs = fit_tables(AFFINE, xt, yt, ot)
    torch.cuda.synchronize()
    for res in (fr, fs):
        got = rows_to_table(AFFINE, res.rows())
        st = res.status.cpu().numpy()
        assert np.array_equal(st, ref["status"])
        ok = st == 0
        assert np.array_equal(got["lo"][ok], ref["lo"][ok]) and np.array_equal(got["hi"][ok], ref["hi"][ok])
        d = np.abs(got["coef"][ok] - ref["coef"][ok]).max(axis=1) / np.abs(ref["coef"][ok]).max(axis=1)
        assert d.max() <= 1e-9, d.max()
        fe, fr_ = res.fit_err.cpu().numpy()[ok], ref["fit_err"][ok]
        assert np.all(np.abs(fe - fr_) <= 1e-9 * fr_ + 1e-12)


@pytest.mark.parametrize("shift", [0, 2])
def test_fit_csr_attn_fused_matches_split(shift, dev, monkeypatch):
    """The fused attention CSR kernel (the default: pass 1, solve and pass 2 in
    one warp per signature) against the moments / solve / MAPE kernels and the oracle, on
    ragged signatures of 100-5000 points at two head alignments (the vector
    path and the point-by-point path)."""
    from paper_2605_07985_b200.sim import fit_tables

    x, y, off = synth_fit_data(ATTN, 80, 5000, seed=70 + shift, ragged=True)
    pad = np.full((3, shift), 5, np.uint32)
    x = np.ascontiguousarray(np.concatenate([pad, x], axis=1))
    y = np.concatenate([np.full(shift, 1e-5), y])
    off = np.concatenate([[0], off + shift]).astype(np.int64)
    xt = torch.from_numpy(x.view(np.int32)).to(dev)
    yt, ot = torch.from_numpy(y).to(dev), torch.from_numpy(off).to(dev)
    fused = fit_tables(ATTN, xt, yt, ot)
    monkeypatch.setenv("DOOLY_FIT_CSR_ATTN", "split")
    split = fit_tables(ATTN, xt, yt, ot)
    torch.cuda.synchronize()
    assert torch.equal(fused.status, split.status)
    ok = (split.status == 0).cpu().numpy()
    a = fused.table.view(torch.float64).cpu().numpy()[ok, :10]
    b = split.table.view(torch.float64).cpu().numpy()[ok, :10]
    assert np.max(np.abs(a - b).max(axis=1) / np.abs(b).max(axis=1)) <= 1e-14
    assert torch.equal(fused.table[:, 80:], split.table[:, 80:])        # scaling + box
    fe, fs = fused.fit_err.cpu().numpy()[ok], split.fit_err.cpu().numpy()[ok]
    assert np.all(np.abs(fe - fs) <= 1e-12 * fs)
    ref = osim.fit(ATTN, x, y, off)
    assert np.array_equal(fused.status.cpu().numpy(), ref["status"])
    got = rows_to_table(ATTN, fused.rows())
    d = np.abs(got["coef"][ok] - ref["coef"][ok]).max(axis=1) / np.abs(ref["coef"][ok]).max(axis=1)
    assert d.max() <= 1e-9, d.max()
