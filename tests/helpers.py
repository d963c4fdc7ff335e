"""Seeded synthetic inputs shared by the CPU and GPU tests (and bench.py)."""

from __future__ import annotations

import numpy as np

AFFINE, ATTN = 0, 1


def synth_fit_data(kind: int, n_sig: int, n_pts, seed: int = 0, noise: float = 1e-3,
                   ragged: bool = False):
    """Per-signature points inside a random training box; y = positive
    ground-truth polynomial x (1 + noise).  Returns x (P, N) u32, y (N,), off."""
    rng = np.random.default_rng(seed)
    counts = (rng.integers(max(1, n_pts // 2), n_pts + 1, size=n_sig) if ragged
              else np.full(n_sig, n_pts))
    off = np.zeros(n_sig + 1, dtype=np.int64)
    off[1:] = np.cumsum(counts)
    N = int(off[-1])
    P = 1 if kind == AFFINE else 3
    sig_of = np.repeat(np.arange(n_sig), counts)
    if kind == AFFINE:
        lo = rng.integers(1, 64, size=n_sig)
        hi = lo + rng.integers(64, 32768, size=n_sig)
        x = rng.integers(lo[sig_of], hi[sig_of] + 1).astype(np.uint32)[None, :]
        a = rng.uniform(5e-6, 2e-5, size=n_sig)
        b = rng.uniform(1e-9, 1e-7, size=n_sig)
        y = a[sig_of] + b[sig_of] * x[0]
    else:
        hi = np.stack([rng.integers(256, 32768, size=n_sig),
                       rng.integers(8, 256, size=n_sig),
                       rng.integers(4096, 1 << 22, size=n_sig)], axis=1)
        x = np.stack([rng.integers(0, hi[sig_of, k] + 1) for k in range(3)]).astype(np.uint32)
        c = rng.uniform(1e-12, 1e-9, size=(n_sig, 3))
        y = (1e-5 + c[sig_of, 0] * x[0] + c[sig_of, 1] * x[1] * 100 + c[sig_of, 2] * x[2]
             + 1e-15 * x[0].astype(np.float64) ** 2 + 1e-16 * x[0].astype(np.float64) * x[2])
    y = y * (1.0 + noise * rng.standard_normal(N))
    return np.ascontiguousarray(x, dtype=np.uint32), np.abs(y) + 1e-9, off


def rows_to_table(kind: int, rows: np.ndarray) -> dict:
    """Product table rows (structured numpy) -> oracle table dict."""
    P = 1 if kind == AFFINE else 3
    return {"coef": np.asarray(rows["c"], dtype=np.float64).reshape(len(rows), -1),
            "inv": np.asarray(rows["inv"], dtype=np.float64).reshape(len(rows), P),
            "lo": np.asarray(rows["lo"], dtype=np.uint32).reshape(len(rows), P),
            "hi": np.asarray(rows["hi"], dtype=np.uint32).reshape(len(rows), P)}


def table_to_rows(kind: int, table: dict) -> np.ndarray:
    """Oracle table dict -> product row bytes (structured numpy)."""
    from paper_2605_07985_b200.sim import ROW_DTYPE

    n = table["coef"].shape[0]
    rows = np.zeros(n, dtype=ROW_DTYPE[kind])
    for field, key in (("c", "coef"), ("inv", "inv"), ("lo", "lo"), ("hi", "hi")):
        rows[field] = np.asarray(table[key]).reshape(rows[field].shape)
    return rows


def synth_queries(kind: int, table: dict, n_q: int, seed: int = 1, outside: float = 0.0):
    """Uniform signature, features uniform inside that signature's box
    (a fraction ``outside`` pushed beyond the box to exercise the flag)."""
    rng = np.random.default_rng(seed)
    n_sig = table["coef"].shape[0]
    sig = rng.integers(0, n_sig, size=n_q).astype(np.int64)
    lo = table["lo"][sig].astype(np.int64)
    hi = table["hi"][sig].astype(np.int64)
    x = (lo + (rng.random(lo.shape) * (hi - lo + 1)).astype(np.int64)).clip(lo, hi)
    if outside:
        m = rng.random(n_q) < outside
        x[m] = hi[m] + 1 + rng.integers(0, 1000, size=(m.sum(), x.shape[1]))
    return sig.astype(np.uint32), np.ascontiguousarray(x.T.astype(np.uint32))


def oracle_grid(grid) -> dict:
    """modelir.SweepGrid -> the oracle's plain grid dict."""
    return {"token_counts": tuple(grid.token_counts), "request_counts": tuple(grid.request_counts),
            "kv_lens": tuple(grid.kv_lens), "prefill_chunk": grid.prefill_chunk,
            "max_batch": grid.max_batch}


def oracle_hw(hw) -> dict:
    return {"peak_flops": hw.peak_flops, "mem_bw": hw.mem_bw, "comm_alpha": hw.comm_alpha,
            "comm_beta": hw.comm_beta}


def oracle_sweep(entry, grid, model, hw, backend):
    """oracle/profiler.py sweep of one RunnableEntry (JSON form) — the checker."""
    from oracle import profiler as oprof

    return oprof.sweep(entry.to_json(), oracle_grid(grid), model.max_context, oracle_hw(hw),
                       backend.cost_multiplier, model.dtype_bytes)


# ---------------------------------------------- SPEC.md:629 exactly-affine oracle


def affine_oracle_coefs(entries) -> list:
    """Per-entry coefficients of an oracle whose latency is EXACTLY affine in
    the entry's regression features: non-attention
    a + b * num_toks; attention a + b1 * prefill_toks + b2 * batch + b3 * kv_tokens.
    Deterministic in the entry's signature (entries sharing a signature share
    the oracle, as they share the regressor)."""
    import hashlib

    from paper_2605_07985_b200.records import canonical_bytes

    out = []
    for e in entries:
        i = hashlib.sha256(canonical_bytes(e)).digest()[0]
        a = 5e-6 * (1.0 + 0.25 * (i % 7))
        if e.feature == "attention":
            out.append((a, 2e-9 * (1 + i % 3), 3e-7 * (1 + i % 5), 1e-10 * (1 + i % 4)))
        else:
            out.append((a, 1.5e-8 * (1 + i % 11)))
    return out


def affine_oracle_value(entry, coef, feats) -> float:
    if entry.feature == "attention":
        a, b1, b2, b3 = coef
        return a + b1 * feats[0] + b2 * feats[1] + b3 * feats[2]
    return coef[0] + coef[1] * feats[0]


def affine_oracle_batch(entries, coefs):
    """oracle(entry_json, reqs) for oracle.sim.reference_run: the affine
    latency at the iteration's concrete dims (features summed over requests,
    kv capped at the entry's window — App. A.6)."""
    by_key = {}
    for e, c in zip(entries, coefs):
        by_key[id(e)] = c
    table = [(e.to_json(), e, c) for e, c in zip(entries, coefs)]

    def oracle(entry_json, reqs):
        for ej, e, c in table:
            if ej is entry_json:
                break
        else:
            raise KeyError("unknown entry")
        if e.feature == "attention":
            w = e.window
            pre = sum(t for t, pf, _ in reqs if pf)
            kv = sum(min(k, w) if w else k for _, _, k in reqs)
            return affine_oracle_value(e, c, (pre, len(reqs), kv))
        return affine_oracle_value(e, c, (sum(t for t, _, _ in reqs),))

    return [ej for ej, _, _ in table], oracle


def affine_oracle_sweep(entry, coef, grid, max_context):
    """Measurements of one entry under the affine oracle at its sweep points."""
    from oracle import profiler as oprof

    ej = entry.to_json()
    pts = oprof.sweep_points(ej, oracle_grid(grid), max_context)
    x = np.array([oprof.point_features(ej, p) for p in pts], dtype=np.uint32).T
    y = np.array([affine_oracle_value(entry, coef, x[:, j].tolist()) for j in range(x.shape[1])])
    return np.ascontiguousarray(x), y


def oracle_ops(entries, fits) -> list:
    """Oracle regression op list (oracle.sim.iter_latency format) from per-entry
    oracle fits [(kind, fit dict)] in entry order."""
    from oracle import sim as osim

    ops = []
    for e, (kind, r) in zip(entries, fits):
        ops.append({"feat": osim.FEAT_ATTN if kind == ATTN else
                    (osim.FEAT_NUM_SEQS if e.feature == "num_seqs" else osim.FEAT_NUM_TOKS),
                    "coef": list(r["coef"][0]), "inv": list(r["inv"][0]),
                    "repeat": e.repeat_count, "window_slot": 1 if e.window else 0})
    return ops
