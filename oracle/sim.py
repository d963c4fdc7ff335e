"""Oracle: regression fit, prediction, iteration latency and the serving event
loop (TTFT/TPOT).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Restates SPEC.md:533-649
with the SURVEY App. A pins:
  A.7  design columns [1, f1, f2, f3, f1^2, f2^2, f3^2, f1f2, f1f3, f2f3] (attention)
       or [1, f] (affine) on features scaled by 1/max; FP64 normal equations
       solved by Cholesky, dropping columns whose pivot <= 1e-9 x diagonal;
  A.8  need = max(4, p + 1) points;  A.9 axis-aligned training box;
  A.10 clamp each entry at 1e-7 s before the repeat multiply;
  A.11 fixed evaluation order, separate multiply and add (numpy / Python floats
       never contract), sequential f64 clock;
  A.12-A.14 cached tokens, KV reservation cap, replica sharding i mod S;
  A.15 fit_error = training MAPE of the clamped predictor.
"""

from __future__ import annotations

import math

import numpy as np

AFFINE, ATTN = 0, 1
PLANES = {AFFINE: 1, ATTN: 3}
NCOL = {AFFINE: 2, ATTN: 10}
NEED = {AFFINE: 4, ATTN: 11}
FLOOR = 1e-7
DROP_TOL = 1e-9
FEAT_NUM_TOKS, FEAT_NUM_SEQS, FEAT_ATTN, FEAT_COMM = 0, 1, 2, 3


# ------------------------------------------------------------------------ fit


def inv_scale(hi: np.ndarray) -> np.ndarray:
    hi = np.asarray(hi, dtype=np.float64)
    return np.where(hi > 0, 1.0 / np.where(hi > 0, hi, 1.0), 1.0)


def design(kind: int, f: np.ndarray) -> np.ndarray:
    """f: (..., P, n) scaled features -> (..., n, p) design matrix (App. A.7)."""
    one = np.ones_like(f[..., 0, :])
    if kind == AFFINE:
        cols = [one, f[..., 0, :]]
    else:
        a, b, c = f[..., 0, :], f[..., 1, :], f[..., 2, :]
        cols = [one, a, b, c, a * a, b * b, c * c, a * b, a * c, b * c]
    return np.stack(cols, axis=-1)


def cholesky_drop_solve(G: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Batched (..., p, p) SPD-or-semidefinite solve; columns whose Cholesky
    pivot falls to <= DROP_TOL x their original diagonal get coefficient 0."""
    G = np.asarray(G, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    p = G.shape[-1]
    L = np.zeros_like(G)
    keep = np.zeros(G.shape[:-1], dtype=bool)
    for j in range(p):
        s = G[..., j, j].copy()
        for k in range(j):
            s = s - L[..., j, k] * L[..., j, k]
        kj = s > DROP_TOL * G[..., j, j]
        keep[..., j] = kj
        d = np.where(kj, np.sqrt(np.where(kj, s, 1.0)), 0.0)
        L[..., j, j] = d
        for i in range(j + 1, p):
            t = G[..., i, j].copy()
            for k in range(j):
                t = t - L[..., i, k] * L[..., j, k]
            L[..., i, j] = np.where(kj, t / np.where(kj, d, 1.0), 0.0)
    z = np.zeros_like(b)
    for j in range(p):
        t = b[..., j].copy()
        for k in range(j):
            t = t - L[..., j, k] * z[..., k]
        z[..., j] = np.where(keep[..., j], t / np.where(keep[..., j], L[..., j, j], 1.0), 0.0)
    c = np.zeros_like(b)
    for j in range(p - 1, -1, -1):
        t = z[..., j].copy()
        for k in range(j + 1, p):
            t = t - L[..., k, j] * c[..., k]
        c[..., j] = np.where(keep[..., j], t / np.where(keep[..., j], L[..., j, j], 1.0), 0.0)
    return c


def eval_poly(kind: int, c: np.ndarray, inv: np.ndarray, x: np.ndarray) -> np.ndarray:
    """Unclamped polynomial; c (..., p), inv (..., P), x (..., P) or broadcastable.

    Operation order is the parity contract shared with the GPU (common.cuh)."""
    xf = np.asarray(x, dtype=np.float64)
    if kind == AFFINE:
        f = xf[..., 0] * inv[..., 0]
        return c[..., 0] + c[..., 1] * f
    f1 = xf[..., 0] * inv[..., 0]
    f2 = xf[..., 1] * inv[..., 1]
    f3 = xf[..., 2] * inv[..., 2]
    p = c[..., 0]
    p = p + c[..., 1] * f1
    p = p + c[..., 2] * f2
    p = p + c[..., 3] * f3
    p = p + c[..., 4] * (f1 * f1)
    p = p + c[..., 5] * (f2 * f2)
    p = p + c[..., 6] * (f3 * f3)
    p = p + c[..., 7] * (f1 * f2)
    p = p + c[..., 8] * (f1 * f3)
    p = p + c[..., 9] * (f2 * f3)
    return p


def clamp(p: np.ndarray):
    p = np.asarray(p, dtype=np.float64)
    cl = p < FLOOR
    return np.where(cl, FLOOR, p), cl


def fit(kind: int, x: np.ndarray, y: np.ndarray, off: np.ndarray) -> dict:
    """SPEC.md:556-564 per signature over CSR ranges.  x (P, N) u32, y (N,) f64."""
    n_sig = len(off) - 1
    P, p = PLANES[kind], NCOL[kind]
    out = {"coef": np.full((n_sig, p), np.nan), "inv": np.full((n_sig, P), np.nan),
           "lo": np.full((n_sig, P), 0xFFFFFFFF, dtype=np.uint32),
           "hi": np.zeros((n_sig, P), dtype=np.uint32), "fit_err": np.full(n_sig, np.nan),
           "status": np.ones(n_sig, dtype=np.uint8), "have": np.diff(off)}
    for s in range(n_sig):
        a, b = int(off[s]), int(off[s + 1])
        if b - a < NEED[kind]:
            continue                     # InsufficientData(sig, have, need)
        r = fit_uniform(kind, x[None, :, a:b], y[None, a:b])
        for k in ("coef", "inv", "lo", "hi", "fit_err"):
            out[k][s] = r[k][0]
        out["status"][s] = 0
    return out


def fit_uniform(kind: int, x: np.ndarray, y: np.ndarray) -> dict:
    """Vectorised fit of S signatures with the same point count: x (S, P, n), y (S, n)."""
    x = np.asarray(x)
    lo = x.min(axis=2).astype(np.uint32)
    hi = x.max(axis=2).astype(np.uint32)
    inv = inv_scale(hi)
    f = x.astype(np.float64) * inv[:, :, None]
    X = design(kind, f)                               # (S, n, p)
    G = np.einsum("sni,snj->sij", X, X)
    rhs = np.einsum("sni,sn->si", X, y)
    c = cholesky_drop_solve(G, rhs)
    pred = eval_poly(kind, c[:, None, :], inv[:, None, :], np.moveaxis(x, 1, 2))
    pred, _ = clamp(pred)
    err = np.mean(np.abs(pred - y) / y, axis=1)
    return {"coef": c, "inv": inv, "lo": lo, "hi": hi, "fit_err": err}


def fit_error(kind: int, coef: np.ndarray, inv: np.ndarray, x: np.ndarray,
              y: np.ndarray) -> np.ndarray:
    """A.15 training MAPE of GIVEN coefficients: c (S, p), inv (S, P), x (S, P, n)
    or (P, n) shared, y (S, n).  Checks a device fit_err against the
    device's own coefficients (fit_err parity then follows coefficient parity)."""
    x = np.asarray(x)
    xq = np.moveaxis(x, -2, -1)
    if xq.ndim == 2:
        xq = xq[None]
    pred = eval_poly(kind, coef[:, None, :], inv[:, None, :], xq)
    pred, _ = clamp(pred)
    return np.mean(np.abs(pred - y) / y, axis=1)


def predict(kind: int, table: dict, sig: np.ndarray, x: np.ndarray) -> dict:
    """SPEC.md:566-574 for a batch: x (P, Q).  Unknown/unfitted rows -> NaN, bad."""
    sig = np.asarray(sig, dtype=np.int64)
    n_sig = table["coef"].shape[0]
    known = (sig >= 0) & (sig < n_sig)
    s = np.where(known, sig, 0)
    lo, hi = table["lo"][s], table["hi"][s]
    known &= lo[:, 0] <= hi[:, 0]
    xq = np.asarray(x).T                                      # (Q, P)
    raw = eval_poly(kind, table["coef"][s], table["inv"][s], xq)
    out, cl = clamp(raw)
    out = np.where(known, out, np.nan)
    extrap = np.any((xq < lo) | (xq > hi), axis=1) & known
    return {"out": out, "extrap": extrap, "clamped": cl & known, "bad": ~known}


def pack_attn(table: dict) -> dict:
    """The folded 96-B serving table of an attention table (include/dooly_b200.h
    dooly_attn_row96; csrc/common.cuh fold_row96): coefficients carried into
    raw-feature space with the row's inv_scale, grouped by feature — sector k
    = (e_k, a_k, b_k, d_k): a_k = c_{1+k} i_k, b_k = (c_{4+k} i_k) i_k,
    d_0 = (c7 i_0) i_1, d_1 = (c9 i_1) i_2, d_2 = (c8 i_0) i_2, e_0 = c0 —
    in this exact rounding order.  Returns {"w": (S, 3, 4) with e_1 = e_2 = 0,
    "lo", "hi"}."""
    c = np.asarray(table["coef"], dtype=np.float64)
    inv = np.asarray(table["inv"], dtype=np.float64)
    i0, i1, i2 = inv[:, 0], inv[:, 1], inv[:, 2]
    w = np.zeros((c.shape[0], 3, 4))
    w[:, 0] = np.stack([c[:, 0], c[:, 1] * i0, (c[:, 4] * i0) * i0, (c[:, 7] * i0) * i1], axis=1)
    w[:, 1] = np.stack([np.zeros_like(i1), c[:, 2] * i1, (c[:, 5] * i1) * i1, (c[:, 9] * i1) * i2],
                       axis=1)
    w[:, 2] = np.stack([np.zeros_like(i2), c[:, 3] * i2, (c[:, 6] * i2) * i2, (c[:, 8] * i0) * i2],
                       axis=1)
    return {"w": w, "lo": table["lo"], "hi": table["hi"]}


def eval_folded(w: np.ndarray, x: np.ndarray) -> np.ndarray:
    """The serving row's per-feature 3-way tree over raw features
    (common.cuh eval_row96): s_k = ((e_k + a_k x_k) + b_k (x_k x_k)) +
    d_k (x_k x_{k+1 mod 3}); p = (s_0 + s_1) + s_2.  w (..., 3, 4), x (..., 3)."""
    xf = np.asarray(x, dtype=np.float64)
    s = []
    for k in range(3):
        xk, xn = xf[..., k], xf[..., (k + 1) % 3]
        e, a, b, d = w[..., k, 0], w[..., k, 1], w[..., k, 2], w[..., k, 3]
        s.append(((e + a * xk) + b * (xk * xk)) + d * (xk * xn))
    return (s[0] + s[1]) + s[2]


def predict_packed(packed: dict, sig: np.ndarray, x: np.ndarray) -> dict:
    """SPEC.md:566-574 served from the folded table (DOOLY_KIND_ATTN_PACKED)."""
    sig = np.asarray(sig, dtype=np.int64)
    n_sig = packed["w"].shape[0]
    known = (sig >= 0) & (sig < n_sig)
    s = np.where(known, sig, 0)
    lo, hi = packed["lo"][s], packed["hi"][s]
    known &= lo[:, 0] <= hi[:, 0]
    xq = np.asarray(x).T
    out, cl = clamp(eval_folded(packed["w"][s], xq))
    out = np.where(known, out, np.nan)
    extrap = np.any((xq < lo) | (xq > hi), axis=1) & known
    return {"out": out, "extrap": extrap, "clamped": cl & known, "bad": ~known}


def predict_one(kind: int, rows: dict, s: int, xs) -> tuple:
    """SPEC.md:566-574 for ONE query in plain Python floats (the per-item form
    of ``predict``; same operation order, so bit-identical):
    ``rows`` maps a signature index to (coef list, inv list, lo list, hi list).
    Returns (latency, extrapolated, clamped); an unknown or unfitted signature
    gives (nan, False, False)."""
    row = rows.get(s)
    if row is None or row[2][0] > row[3][0]:
        return math.nan, False, False
    c, inv, lo, hi = row
    if kind == AFFINE:
        p = c[0] + c[1] * (float(xs[0]) * inv[0])
    else:
        f1, f2, f3 = float(xs[0]) * inv[0], float(xs[1]) * inv[1], float(xs[2]) * inv[2]
        p = c[0]
        p = p + c[1] * f1
        p = p + c[2] * f2
        p = p + c[3] * f3
        p = p + c[4] * (f1 * f1)
        p = p + c[5] * (f2 * f2)
        p = p + c[6] * (f3 * f3)
        p = p + c[7] * (f1 * f2)
        p = p + c[8] * (f1 * f3)
        p = p + c[9] * (f2 * f3)
    ext = any(v < a or v > b for v, a, b in zip(xs, lo, hi))
    return (FLOOR, ext, True) if p < FLOOR else (p, ext, False)


# -------------------------------------------------------------- iter_latency


def entry_value(op: dict, feats: tuple, tp: int, alpha: float, beta: float) -> float:
    """One op's clamped prediction for iteration features
    (num_toks, prefill_toks, batch, kv_tokens, kv_tokens_window)."""
    num_toks, prefill, batch, kv, kvw = feats
    if op["feat"] == FEAT_COMM:
        nbytes = num_toks * op["bytes_per_tok"]
        return 2 * (tp - 1) / tp * (alpha + nbytes / tp * beta)
    c, inv = op["coef"], op["inv"]
    if op["feat"] == FEAT_ATTN:
        f1 = float(prefill) * inv[0]
        f2 = float(batch) * inv[1]
        f3 = float(kvw if op["window_slot"] else kv) * inv[2]
        p = c[0]
        for coef, m in zip(c[1:], (f1, f2, f3, f1 * f1, f2 * f2, f3 * f3, f1 * f2, f1 * f3,
                                   f2 * f3)):
            p = p + coef * m
    else:
        f = float(batch if op["feat"] == FEAT_NUM_SEQS else num_toks) * inv[0]
        p = c[0] + c[1] * f
    return FLOOR if p < FLOOR else p


def iter_latency(feats: tuple, ops: list, tp: int = 1, alpha: float = 0.0,
                 beta: float = 0.0) -> float:
    """sum in list order of repeat x clamped prediction (+ comm)."""
    lat = 0.0
    for op in ops:
        lat = lat + float(op["repeat"]) * entry_value(op, feats, tp, alpha, beta)
    return lat


# ------------------------------------------------------------ schedule / run


def schedule_step(running: list, waiting_head, chunk: int, max_batch: int, kv_ok) -> tuple:
    """SPEC.md:576-584 + D1 (:632): decode requests take 1 token each from the
    chunk budget, then running partial prefills in running order, then FCFS
    admission while max_batch, KV memory (kv_ok) and budget permit.

    running: list of dicts {left, ...}; waiting_head(k) -> k-th waiting request
    dict or None.  Returns ([(req, tokens, is_prefill, admitted)], n_admitted)."""
    budget = chunk
    sched = []
    for r in running:
        if r["left"] == 0:
            sched.append((r, 1, False, False))
            budget -= 1
    for r in running:
        if r["left"] > 0:
            take = min(r["left"], budget)
            budget -= take
            sched.append((r, take, True, False))
    n_adm = 0
    while len(running) + n_adm < max_batch and budget > 0:
        w = waiting_head(n_adm)
        if w is None or not kv_ok(w):
            break
        work = w["prompt"] - w["cached"]
        take = min(work, budget) if work > 0 else 1
        budget -= take
        sched.append((w, take, work > 0, True))
        n_adm += 1
    return sched, n_adm


def run_shard(arrival, prompt, output, cached, ops: list, chunk: int, max_batch: int,
              kv_bytes_per_token: int, kv_capacity: int, window: int = 0, tp: int = 1,
              alpha: float = 0.0, beta: float = 0.0, max_iterations: int = 50_000_000,
              log: bool = False, latency=None) -> dict:
    """SPEC.md:596-604 event loop for one replica (requests sorted by arrival).

    ``latency(reqs, feats) -> seconds`` replaces the regression iteration
    latency (``iter_latency`` over ``ops``): reference_run
    passes the brute-force oracle here, so both runs share this scheduler code.
    reqs = [(tokens, is_prefill, kv_before)] per scheduled request."""
    n = len(arrival)
    ttft = [math.nan] * n
    tpot = [math.nan] * n
    clock = 0.0
    arrive = admit = it = 0
    running: list = []
    reserved = 0
    feats_log, lat_log = [], []
    start_log, clock_log = [], []          # idle jump target (0.0 if busy), clock after it
    comp_log = []                          # batch composition: ((request, tokens, prefill), ...)
    first_it, last_it = [-1] * n, [-1] * n
    jump = 0.0
    status = "ok"

    def make(i):
        return {"i": i, "prompt": int(prompt[i]), "output": int(output[i]),
                "cached": int(cached[i]), "left": int(prompt[i]) - int(cached[i]),
                "dec": 0, "kv": int(cached[i]), "t_first": 0.0}

    while True:
        while arrive < n and arrival[arrive] <= clock:
            arrive += 1
        if not running and admit == arrive:
            if arrive == n:
                break
            clock = float(arrival[arrive])          # idle: jump to the next arrival
            jump = clock
            continue
        if it >= max_iterations:
            status = "non_termination"
            break

        def head(k):
            return make(admit + k) if admit + k < arrive else None

        def kv_ok(w, _res=[reserved]):
            need = (w["prompt"] + w["output"]) * kv_bytes_per_token
            if _res[0] + need > kv_capacity:
                return False
            _res[0] += need
            return True

        sched, n_adm = schedule_step(running, head, chunk, max_batch, kv_ok)
        if not running and n_adm == 0:
            status = "kv_capacity"
            break
        for (r, _, _, adm) in sched:
            if adm:
                running.append(r)
                reserved += (r["prompt"] + r["output"]) * kv_bytes_per_token
        admit += n_adm
        active = [(r, t, pf) for (r, t, pf, _) in sched if t > 0]
        num_toks = sum(t for _, t, _ in active)
        prefill = sum(t for _, t, pf in active if pf)
        batch = len(active)
        kv = sum(r["kv"] for r, _, _ in active)
        kvw = sum(min(r["kv"], window) for r, _, _ in active) if window else 0
        feats = (num_toks, prefill, batch, kv, kvw)
        if latency is None:
            lat = iter_latency(feats, ops, tp, alpha, beta)
        else:
            lat = latency([(t, pf, r["kv"]) for r, t, pf in active], feats)
        clock = clock + lat
        it += 1
        if log:
            comp_log.append(tuple((r["i"], t, pf) for r, t, pf in active))
            feats_log.append(feats)
            lat_log.append(lat)
            start_log.append(jump)
            clock_log.append(clock)
        jump = 0.0
        done = []
        for r, t, pf in active:
            r["kv"] += t
            if pf:
                r["left"] -= t
                if r["left"] > 0:
                    continue
            r["dec"] += 1
            if r["dec"] == 1:
                r["t_first"] = clock
                ttft[r["i"]] = clock - arrival[r["i"]]
                first_it[r["i"]] = it - 1
            if r["dec"] >= r["output"]:
                last_it[r["i"]] = it - 1
                if r["output"] >= 2:
                    tpot[r["i"]] = (clock - r["t_first"]) / (r["output"] - 1)
                done.append(r)
        if done:
            ids = {id(r) for r in done}
            for r in done:
                reserved -= (r["prompt"] + r["output"]) * kv_bytes_per_token
            running = [r for r in running if id(r) not in ids]
    return {"ttft": np.array(ttft), "tpot": np.array(tpot), "n_iter": it, "clock": clock,
            "status": status, "feats": feats_log, "lat": lat_log, "start": start_log,
            "clocks": clock_log, "first_it": first_it, "last_it": last_it,
            "compositions": comp_log}


def reference_run(arrival, prompt, output, cached, entries: list, hw: dict, cost_multiplier,
                  dtype_bytes: int, chunk: int, max_batch: int, kv_bytes_per_token: int,
                  kv_capacity: int, tp: int = 1, hidden: int = 0, num_layers: int = 0,
                  oracle=None, max_iterations: int = 50_000_000, log: bool = False) -> dict:
    """SPEC.md:606-612 reference_run: the same event loop, but every iteration's
    latency is the direct oracle evaluation of every runnable entry at the
    batch's concrete dims (no regression): sum in list order of
    repeat x oracle(entry, reqs), then the TP all-reduces (2 per layer of
    num_toks x hidden x dtype bytes, App. A.16).

    ``oracle(entry, reqs) -> seconds`` defaults to the roofline model at the
    concrete batch (oracle.profiler.batch_latency); SPEC.md:629's invariant is
    tested with an exactly-affine oracle here.  entries are runnable-set JSON
    dicts; hw: {peak_flops, mem_bw, comm_alpha, comm_beta}."""
    from . import profiler as oprof

    if oracle is None:
        def oracle(entry, reqs):
            return oprof.batch_latency(entry, reqs, hw, cost_multiplier, dtype_bytes)

    def latency(reqs, feats):
        lat = 0.0
        for e in entries:
            lat = lat + float(e["repeat_count"]) * oracle(e, reqs)
        if tp > 1:
            nbytes = feats[0] * hidden * dtype_bytes
            comm = 2 * (tp - 1) / tp * (hw["comm_alpha"] + nbytes / tp * hw["comm_beta"])
            lat = lat + float(2 * num_layers) * comm
        return lat

    return run_shard(arrival, prompt, output, cached, [], chunk, max_batch, kv_bytes_per_token,
                     kv_capacity, 0, tp, 0.0, 0.0, max_iterations, log, latency)


def percentile_mape(pred, truth, percentiles=(25, 50, 75, 90, 95, 99)) -> dict:
    """A5: relative error of each reported percentile of a metric
    (NaNs — e.g. TPOT of 1-token requests — dropped on both sides)."""
    p = np.asarray(pred, dtype=np.float64)
    t = np.asarray(truth, dtype=np.float64)
    p, t = p[~np.isnan(p)], t[~np.isnan(t)]
    out = {}
    for q in percentiles:
        a, b = float(np.percentile(p, q)), float(np.percentile(t, q))
        out[f"p{q}"] = abs(a - b) / b
    return out


def run_shards(arrival, prompt, output, cached, n_shards: int, **kw) -> dict:
    """App. A.14: request i -> shard i mod S; results back in request order."""
    n = len(arrival)
    ttft = np.full(n, np.nan)
    tpot = np.full(n, np.nan)
    n_iter, clocks, status = [], [], []
    for s in range(n_shards):
        idx = np.arange(s, n, n_shards)
        r = run_shard([arrival[i] for i in idx], [prompt[i] for i in idx],
                      [output[i] for i in idx], [cached[i] for i in idx], **kw)
        ttft[idx] = r["ttft"]
        tpot[idx] = r["tpot"]
        n_iter.append(r["n_iter"])
        clocks.append(r["clock"])
        status.append(r["status"])
    return {"ttft": ttft, "tpot": tpot, "n_iter": n_iter, "clock": clocks, "status": status}


def mape(pred, truth) -> float:
    """SPEC.md:614-622."""
    if len(pred) != len(truth):
        raise ValueError("LengthMismatch")
    if any(t == 0 for t in truth):
        raise ZeroDivisionError("ZeroTruth")
    return sum(abs(p - t) / t for p, t in zip(pred, truth)) / len(truth) if truth else 0.0
