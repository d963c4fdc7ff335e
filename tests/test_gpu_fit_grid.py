"""Shared-grid fit (dooly_fit_grid) vs the CPU oracle and vs the CSR fit.

Contract: the same rows, statuses and fit_err as ``fit`` over the same points
repeated per signature — coefficients within 1e-9 normwise
in the scaled basis, fit_err within 1e-9 relative, box and inv_scale exact."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from helpers import ATTN, AFFINE, rows_to_table
from oracle import sim as osim

pytestmark = pytest.mark.gpu

COEF_TOL = 1e-9
ERR_TOL = 1e-9


def _grid(kind, n_pts, rng):
    if kind == AFFINE:
        return np.sort(rng.integers(1, 32769, n_pts)).astype(np.uint32)[None, :]
    side = round(n_pts ** (1 / 3))
    t = np.unique(np.geomspace(1, 32768, side).astype(np.int64))
    b = np.unique(np.geomspace(1, 256, side).astype(np.int64))
    k = np.unique(np.linspace(0, 1 << 22, side).astype(np.int64))
    g = np.stack(np.meshgrid(t, b, k, indexing="ij")).reshape(3, -1)
    return g.astype(np.uint32)


def _ys(kind, x, n_sig, rng, noise=1e-3):
    xf = x.astype(np.float64)
    if kind == AFFINE:
        a = rng.uniform(5e-6, 2e-5, (n_sig, 1))
        b = rng.uniform(1e-9, 1e-7, (n_sig, 1))
        y = a + b * xf[0]
    else:
        c = rng.uniform(1e-12, 1e-9, (n_sig, 3))
        y = (1e-5 + c[:, :1] * xf[0] + c[:, 1:2] * xf[1] * 100 + c[:, 2:3] * xf[2]
             + 1e-15 * xf[0] * xf[0])
    return np.abs(y * (1 + noise * rng.standard_normal(y.shape))) + 1e-9


def _fit_grid_gpu(kind, x, y, dev):
    from paper_2605_07985_b200.sim import fit_grid

    fr = fit_grid(kind, torch.from_numpy(np.ascontiguousarray(x).view(np.int32)).to(dev),
                  torch.from_numpy(y).to(dev))
    torch.cuda.synchronize()
    return fr


def _oracle(kind, x, y):
    n_sig, n = y.shape
    xr = np.tile(x, (1, n_sig))
    off = np.arange(n_sig + 1, dtype=np.int64) * n
    return osim.fit(kind, xr, y.reshape(-1), off), xr, off


@pytest.mark.parametrize("kind", [AFFINE, ATTN])
@pytest.mark.parametrize("n_sig,n_pts", [(1, 512), (37, 512), (301, 512), (37, 510), (9, 4096), (7, 64), (5, 136), (13, 768)])
@pytest.mark.parametrize("kernel", ["warp", "stage", "db", "ws", "ring", "ring6", "ring2"])
def test_fit_grid_matches_oracle_and_csr(kind, n_sig, n_pts, kernel, dev, monkeypatch):
    """n_pts % 4 == 0 takes the warp-per-signature kernel, its register
    double-buffered form (db: n_pts % 256 == 0, the affine default) or the
    shared-memory staged one (DOOLY_FIT_GRID_KERNEL=stage); 510 the direct one."""
    from paper_2605_07985_b200.sim import fit_tables

    monkeypatch.setenv("DOOLY_FIT_GRID_KERNEL", kernel)

    rng = np.random.default_rng(17 + kind + n_sig)
    x = _grid(kind, n_pts, rng)[:, :n_pts]
    y = _ys(kind, x, n_sig, rng)
    fr = _fit_grid_gpu(kind, x, y, dev)
    ref, xr, off = _oracle(kind, x, y)
    got = rows_to_table(kind, fr.rows())
    assert np.array_equal(fr.status.cpu().numpy(), ref["status"])
    assert np.array_equal(got["lo"], ref["lo"]) and np.array_equal(got["hi"], ref["hi"])
    assert np.array_equal(got["inv"], ref["inv"])
    dc = np.abs(got["coef"] - ref["coef"]).max(axis=1) / np.abs(ref["coef"]).max(axis=1)
    assert dc.max() <= COEF_TOL, dc.max()
    # fit_err is a MAPE, so | |a-y| - |b-y| | <= |a-b| bounds its difference by the
    # mean relative difference of the two fits' training predictions (each
    # within the 1e-9 prediction contract); near-noise-level residuals amplify
    # ~1e-12 coefficient differences, so a flat 1e-9 relative bar on fit_err
    # would test summation order, not correctness.
    fe = fr.fit_err.cpu().numpy()
    for s in range(n_sig):
        pg = np.maximum(osim.eval_poly(kind, got["coef"][s], got["inv"][s], x.T), 1e-7)
        pr = np.maximum(osim.eval_poly(kind, ref["coef"][s], ref["inv"][s], x.T), 1e-7)
        assert np.max(np.abs(pg - pr) / np.abs(pr)) <= 1e-9
        bound = np.mean(np.abs(pg - pr) / y[s])
        assert abs(fe[s] - ref["fit_err"][s]) <= bound * (1 + 1e-6) + 1e-12 * ref["fit_err"][s], (
            s, fe[s], ref["fit_err"][s], bound)
    # the CSR kernel over the repeated points gives the same regressors
    csr = fit_tables(kind, torch.from_numpy(xr.view(np.int32)).to(dev), torch.from_numpy(
        y.reshape(-1)).to(dev), torch.from_numpy(off).to(dev))
    c2 = rows_to_table(kind, csr.rows())
    d2 = np.abs(got["coef"] - c2["coef"]).max(axis=1) / np.abs(c2["coef"]).max(axis=1)
    assert d2.max() <= 2 * COEF_TOL


def test_fit_grid_insufficient_and_empty(dev):
    rng = np.random.default_rng(3)
    x = np.array([[1, 16, 128]], dtype=np.uint32)        # 3 points < need 4
    y = _ys(AFFINE, x, 5, rng)
    fr = _fit_grid_gpu(AFFINE, x, y, dev)
    assert fr.status.cpu().numpy().tolist() == [1] * 5
    assert np.isnan(fr.fit_err.cpu().numpy()).all()
    rows = fr.rows()
    assert (rows["lo"] > rows["hi"]).all()
    x3 = _grid(ATTN, 8, rng)[:, :10]                      # 10 points < need 11
    fr = _fit_grid_gpu(ATTN, x3, _ys(ATTN, x3, 2, rng), dev)
    assert fr.status.cpu().numpy().tolist() == [1, 1]
    fr = _fit_grid_gpu(ATTN, _grid(ATTN, 64, rng), np.zeros((0, 64)), dev)
    assert fr.table.shape[0] == 0


def test_fit_grid_rank_deficient_drops_columns(dev):
    rng = np.random.default_rng(5)
    x = _grid(ATTN, 512, rng)
    x[1] = 8                                              # batch constant: f2 == 1 == intercept
    y = _ys(ATTN, x, 9, rng, noise=0.0)
    fr = _fit_grid_gpu(ATTN, x, y, dev)
    ref, xr, off = _oracle(ATTN, x, y)
    got = rows_to_table(ATTN, fr.rows())
    assert np.array_equal(got["coef"] == 0, ref["coef"] == 0)
    pg = osim.eval_poly(ATTN, got["coef"][0], got["inv"][0], x.T)
    pr = osim.eval_poly(ATTN, ref["coef"][0], ref["inv"][0], x.T)
    assert np.max(np.abs(pg - pr) / pr) <= 1e-9


@pytest.mark.parametrize("kind", [AFFINE, ATTN])
@pytest.mark.parametrize("factor", ["0", "1"])
def test_fit_grid_db_and_warp_bit_identical(kind, factor, dev, monkeypatch):
    """The double-buffered kernel runs the warp kernel's per-lane arithmetic in
    the same order (per-point or grouped attention passes alike), so tables,
    fit_err and statuses are bit-identical."""
    monkeypatch.setenv("DOOLY_FIT_GRID_FACTOR", factor)
    rng = np.random.default_rng(29 + kind)
    x = _grid(kind, 4096, rng)[:, :4096]
    y = _ys(kind, x, 2000, rng)
    out = {}
    for k in ("warp", "db"):
        monkeypatch.setenv("DOOLY_FIT_GRID_KERNEL", k)
        out[k] = _fit_grid_gpu(kind, x, y, dev)
    a, b = out["warp"], out["db"]
    assert torch.equal(a.table, b.table) and torch.equal(a.status, b.status)
    assert torch.equal(a.fit_err.view(torch.int64), b.fit_err.view(torch.int64))


def test_fit_grid_grouped_attention_passes(dev, monkeypatch):
    """Sweep grids with the kv axis innermost take the grouped attention passes
    (prefill_toks and batch factored out of each aligned 4-point group); a
    shuffled grid falls back to the per-point passes.  Both meet the oracle
    contract and agree with each other."""
    rng = np.random.default_rng(41)
    x = _grid(ATTN, 4096, rng)[:, :4096]
    y = _ys(ATTN, x, 300, rng)
    ref, _, _ = _oracle(ATTN, x, y)
    grouped = _fit_grid_gpu(ATTN, x, y, dev)
    monkeypatch.setenv("DOOLY_FIT_GRID_FACTOR", "0")
    plain = _fit_grid_gpu(ATTN, x, y, dev)
    monkeypatch.delenv("DOOLY_FIT_GRID_FACTOR")
    perm = rng.permutation(x.shape[1])
    shuffled = _fit_grid_gpu(ATTN, np.ascontiguousarray(x[:, perm]), np.ascontiguousarray(y[:, perm]),
                             dev)
    for fr in (grouped, plain, shuffled):
        got = rows_to_table(ATTN, fr.rows())
        dc = np.abs(got["coef"] - ref["coef"]).max(axis=1) / np.abs(ref["coef"]).max(axis=1)
        assert dc.max() <= COEF_TOL, dc.max()
        fe = fr.fit_err.cpu().numpy()
        assert np.max(np.abs(fe - ref["fit_err"]) / ref["fit_err"]) <= 1e-8
    a, b = (rows_to_table(ATTN, f.rows())["coef"] for f in (grouped, plain))
    assert np.max(np.abs(a - b).max(axis=1) / np.abs(b).max(axis=1)) <= 1e-12


@pytest.mark.parametrize("n_sig,n_pts,kernel", [(300, 4096, "warp"), (37, 512, "db"), (5, 64, "stage"),
                                                (9, 125, "warp"), (4, 8, "warp"), (300, 4096, "ws"),
                                                (1000, 2048, "ws"), (3, 512, "ws")])
def test_fit_grid_packed_equals_attn_pack(n_sig, n_pts, kernel, dev, monkeypatch):
    """dooly_fit_grid_packed's epilogue writes the 96-B serving table
    byte-identical to dooly_attn_pack of the fitted table (header included),
    for every grid kernel and for unfitted tables (too few points)."""
    from paper_2605_07985_b200.sim import fit_grid, pack_attn

    monkeypatch.setenv("DOOLY_FIT_GRID_KERNEL", kernel)
    rng = np.random.default_rng(n_sig + n_pts)
    x = _grid(ATTN, n_pts, rng)[:, :n_pts]
    y = _ys(ATTN, x, n_sig, rng)
    xt = torch.from_numpy(np.ascontiguousarray(x).view(np.int32)).to(dev)
    yt = torch.from_numpy(y).to(dev)
    packed = torch.full((n_sig + 1, 96), 0xAB, dtype=torch.uint8, device=dev)
    fr = fit_grid(ATTN, xt, yt, packed=packed)
    ref = pack_attn(fr.table)
    torch.cuda.synchronize()
    assert torch.equal(packed, ref)
    plain = fit_grid(ATTN, xt, yt)
    assert torch.equal(plain.table, fr.table) and torch.equal(plain.status, fr.status)


@pytest.mark.parametrize("factor", ["0", "1"])
@pytest.mark.parametrize("n_sig", [1, 149, 3001])
def test_fit_grid_ws_matches_warp(factor, n_sig, dev, monkeypatch):
    """The warp-specialised TMA-ring attention kernel (default) against the
    warp kernel: same statuses and boxes, coefficients within 1e-12 normwise
    (only the summation order differs), fit_err within 1e-12 relative; more
    signatures than CTAs x stages so the ring wraps."""
    monkeypatch.setenv("DOOLY_FIT_GRID_FACTOR", factor)
    rng = np.random.default_rng(7 + n_sig)
    x = _grid(ATTN, 4096, rng)[:, :4096]
    y = _ys(ATTN, x, n_sig, rng)
    out = {}
    for k in ("warp", "ws"):
        monkeypatch.setenv("DOOLY_FIT_GRID_KERNEL", k)
        out[k] = _fit_grid_gpu(ATTN, x, y, dev)
    a = rows_to_table(ATTN, out["warp"].rows())
    b = rows_to_table(ATTN, out["ws"].rows())
    assert torch.equal(out["warp"].status, out["ws"].status)
    for k in ("lo", "hi", "inv"):
        assert np.array_equal(a[k], b[k])
    dc = np.abs(a["coef"] - b["coef"]).max(axis=1) / np.abs(a["coef"]).max(axis=1)
    assert dc.max() <= 1e-12, dc.max()
    fa, fb = out["warp"].fit_err.cpu().numpy(), out["ws"].fit_err.cpu().numpy()
    assert np.max(np.abs(fa - fb) / fa) <= 1e-12


@pytest.mark.parametrize("variant", ["ring", "ring6", "ring2"])
@pytest.mark.parametrize("n_sig", [1, 149, 3001])
def test_fit_grid_ring_matches_warp(variant, n_sig, dev, monkeypatch):
    """The per-warp bulk-copy ring kernel (f3-periodic grouped grids) against
    the warp kernel: same statuses, boxes and inv; coefficients within 1e-12
    normwise and fit_err within 1e-10 relative (the order of the per-lane MAPE
    sums differs; the contract is 1e-9); more signatures than warps x stages so every ring wraps across
    signature boundaries, and the packed serving rows written by its epilogue
    byte-identical to dooly_attn_pack of its own table."""
    from paper_2605_07985_b200.sim import fit_grid, pack_attn

    rng = np.random.default_rng(11 + n_sig)
    # the C5 shape: 16 x 16 x 16 (prefill_toks, batch, kv_tokens), kv innermost
    t = 2 ** np.arange(16)
    bt = np.arange(1, 17) * 8
    kv = np.linspace(0, 1 << 22, 16).astype(np.int64)
    x = np.stack(np.meshgrid(t, bt, kv, indexing="ij")).reshape(3, -1).astype(np.uint32)
    y = _ys(ATTN, x, n_sig, rng)
    out = {}
    for k in ("warp", variant):
        monkeypatch.setenv("DOOLY_FIT_GRID_KERNEL", k)
        out[k] = _fit_grid_gpu(ATTN, x, y, dev)
    a = rows_to_table(ATTN, out["warp"].rows())
    b = rows_to_table(ATTN, out[variant].rows())
    assert torch.equal(out["warp"].status, out[variant].status)
    assert int((out[variant].status != 0).sum().item()) == 0
    for k in ("lo", "hi", "inv"):
        assert np.array_equal(a[k], b[k])
    dc = np.abs(a["coef"] - b["coef"]).max(axis=1) / np.abs(a["coef"]).max(axis=1)
    assert dc.max() <= 1e-12, dc.max()
    fa, fb = out["warp"].fit_err.cpu().numpy(), out[variant].fit_err.cpu().numpy()
    assert np.max(np.abs(fa - fb) / fa) <= 1e-10
    xt = torch.from_numpy(np.ascontiguousarray(x).view(np.int32)).to(dev)
    yt = torch.from_numpy(y).to(dev)
    packed = torch.full((n_sig + 1, 96), 0xAB, dtype=torch.uint8, device=dev)
    fr = fit_grid(ATTN, xt, yt, packed=packed)
    torch.cuda.synchronize()
    assert torch.equal(packed, pack_attn(fr.table))
