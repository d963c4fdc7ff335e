"""Oracle: signature canonicalisation, SHA-256, dedup, analytical latency model.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Input entries are dicts in
the runnable-set export format: name, granularity, arg_template
(list of args, each a list of [size, taint_string]), scalars, attrs,
kernel_symbols, repeat_count.
"""

from __future__ import annotations

import hashlib
import struct


# ---------------------------------------------------------------- canonicalize


def model_dims(entry: dict) -> list:
    """only MODEL_CONFIG dims and scalars.  App. A.2: a dim
    counts iff its taint string is exactly "MC" (Base(MC); BOT and MIX excluded);
    positions number the flattened argument template from 0; scalars sit at
    65536 + scalar index (D2)."""
    flat = [d for arg in entry["arg_template"] for d in arg]
    dims = [(i, int(size)) for i, (size, taint) in enumerate(flat) if taint == "MC"]
    dims += [(65536 + k, int(v)) for k, (v, taint) in enumerate(entry.get("scalars", []))
             if taint == "MC"]
    return sorted(dims)


def _encode_attr(value) -> bytes:
    # App. A.3 type tags: b(bool) i(int64) f(float64) s(utf-8 str) n(None)
    if value is True or value is False:
        return b"b" + bytes([1 if value else 0])
    if isinstance(value, int):
        return b"i" + value.to_bytes(8, "little", signed=True)
    if isinstance(value, float):
        return b"f" + struct.pack("<d", value)
    if isinstance(value, str):
        return b"s" + len(value.encode()).to_bytes(4, "little") + value.encode()
    if value is None:
        return b"n"
    raise TypeError(value)


def attr_digest(attrs: dict) -> bytes:
    """SPEC.md:419 'attr_digest: 32-byte hash of sorted (key, primitive value) pairs'."""
    body = b""
    for key in sorted(attrs, key=lambda k: k.encode()):
        kb = key.encode()
        body += len(kb).to_bytes(4, "little") + kb + _encode_attr(attrs[key])
    return hashlib.sha256(body).digest()


def canonicalize(entry: dict) -> bytes:
    """SPEC.md:438-446 with layout D1 and widths of App. A.1:
    'sigfmt=1' | u32 len(name) | name | u32 n | (u32 pos, u64 val)* ascending pos |
    u32 n_sym | (u32 len | bytes)* bytewise-sorted | attr_digest (modules only)."""
    out = bytearray(b"sigfmt=1")
    name = entry["name"].encode()
    out += len(name).to_bytes(4, "little") + name
    dims = model_dims(entry)
    out += len(dims).to_bytes(4, "little")
    for pos, val in dims:
        out += pos.to_bytes(4, "little") + val.to_bytes(8, "little")
    syms = sorted({s.encode() for s in entry["kernel_symbols"]})
    out += len(syms).to_bytes(4, "little")
    for s in syms:
        out += len(s).to_bytes(4, "little") + s
    if entry["granularity"] == "module":
        out += attr_digest(entry.get("attrs", {}))
    return bytes(out)


def signature_hash(canonical: bytes) -> bytes:
    """standard SHA-256 (hashlib, FIPS 180-4)."""
    return hashlib.sha256(canonical).digest()


def dedup_digests(digests: list, db_keys=()) -> dict:
    """SPEC.md:456-464 + App. A.4 (global order, first occurrence wins).

    Returns per-record first index, uid (rank among first occurrences in index
    order), is_new (first occurrence and not in the DB) and in_db, plus the
    number of distinct digests."""
    db = set(db_keys)
    first_of: dict = {}
    uid_of: dict = {}
    first, uid, is_new, in_db = [], [], [], []
    for i, d in enumerate(digests):
        if d not in first_of:
            first_of[d] = i
            uid_of[d] = len(uid_of)
        f = first_of[d]
        first.append(f)
        uid.append(uid_of[d])
        in_db.append(d in db)
        is_new.append(f == i and d not in db)
    return {"first": first, "uid": uid, "is_new": is_new, "in_db": in_db,
            "n_unique": len(first_of)}


def dedup(entries: list, db_keys=()) -> tuple:
    """(to_profile, skipped) index lists; skipped <=> hash already present."""
    res = dedup_digests([signature_hash(canonicalize(e)) for e in entries], db_keys)
    to_profile = [i for i, n in enumerate(res["is_new"]) if n]
    skipped = [i for i, n in enumerate(res["is_new"]) if not n]
    return to_profile, skipped


# ---------------------------------------------------------- analytical model
#
# oracle_latency = overhead + multiplier * max(flops/peak_flops,
# bytes/mem_bw); multiplier = product over kernel symbols of the longest-prefix
# cost_multiplier (modelir.py:134-143); overhead 5 us.
# The SPEC names only the matmul and attention-prefill flop counts ("2·M·K·N",
# "2·2·T²·D·H_q etc."); the remaining per-op formulas are the
# builder's pin (App. A.18), restated here from that table and
# NOT imported from the package.  Arithmetic follows Python left-to-right
# operator order exactly as written (the K5 device sweep is held bit-identical
# to it).

OVERHEAD_S = 5e-6


def roofline_latency(flops: float, nbytes: float, peak_flops: float, mem_bw: float,
                     multiplier: float = 1.0, overhead: float = OVERHEAD_S) -> float:
    """overhead + multiplier * max(flops/peak, bytes/bw)."""
    return overhead + multiplier * max(flops / peak_flops, nbytes / mem_bw)


def matmul_cost(m: int, k: int, n: int, dtype_bytes: int) -> tuple:
    """SPEC.md:480 'matmul: 2·M·K·N flops'; bytes = (MK + KN + MN) * dtype."""
    return 2 * m * k * n, (m * k + k * n + m * n) * dtype_bytes


def comm_latency(tp: int, nbytes: int, alpha: float, beta: float) -> float:
    """SPEC.md:486-494 ring all-reduce: 2(tp-1)/tp * (alpha + bytes/tp * beta)."""
    return 2 * (tp - 1) / tp * (alpha + nbytes / tp * beta)


def multiplier(cost_multiplier, symbols) -> float:
    """modelir.py:134-143: product over symbols of the value of the longest key
    that prefixes the symbol (first key wins a tie; unlisted symbols cost 1)."""
    product = 1.0
    for sym in symbols:
        best, best_len = 1.0, -1
        for key, value in cost_multiplier:
            if sym.startswith(key) and len(key) > best_len:
                best, best_len = value, len(key)
        product *= best
    return product


def _sizes(entry: dict) -> list:
    return [[int(size) for size, _ in arg] for arg in entry["arg_template"]]


def _attention_cost(hq: int, hkv: int, d: int, reqs, dtype_bytes: int) -> tuple:
    """Attention over requests (q_i new tokens, c_i cached tokens): each query
    token attends to its request's c_i + q_i keys (QK^T and PV, 2 flops per
    MAC: 4·hq·d per (query, key) pair — SPEC.md:480's 2·2·T²·D·H_q at one
    request without cache); bytes = K and V of every visible key plus Q in and
    O out.  At a uniform sweep point this is exactly ``op_cost``'s formula."""
    flops = 0.0
    kv_keys = 0.0
    q_tok = 0.0
    for q, c in reqs:
        flops = flops + 4.0 * hq * d * q * (c + q)
        kv_keys = kv_keys + (c + q)
        q_tok = q_tok + q
    return flops, float(dtype_bytes * (kv_keys * 2 * hkv * d + 2 * q_tok * hq * d))


# op kind -> (flops, bytes) at token count t (and request count r); the table
# of App. A.18.  a = per-argument dim sizes, s = scalar values.
def _linear(a, s, t, r, dt, feature):
    k, n = a[1][1], a[1][0]
    m = r if feature == "num_seqs" else t
    return 2.0 * m * k * n, float((m * k + k * n + m * n) * dt)


def _embedding(a, s, t, r, dt, feature):
    return 0.0, float(2 * t * a[1][1] * dt + 4 * t)          # ids in, rows gathered + written


def _rms_norm(a, s, t, r, dt, feature):
    h = a[0][1]
    return 4.0 * t * h, float((2 * t * h + h) * dt)


def _rotary(a, s, t, r, dt, feature):
    w = a[0][1] * a[0][2] + a[1][1] * a[1][2]                  # q and k head widths
    return 3.0 * t * w, float(2 * t * w * dt)


def _silu_and_mul(a, s, t, r, dt, feature):
    width = a[0][1]                                            # 2 x intermediate
    return 2.0 * t * width, float((t * width + t * width // 2) * dt)


def _topk_softmax(a, s, t, r, dt, feature):
    e = a[0][1]
    return 5.0 * t * e, float(t * e * (dt + 8))               # logits in; f32 weight + i32 id out


def _fused_moe(a, s, t, r, dt, feature):
    n_exp, width, h = a[1]                                     # w13: (E, 2I, h)
    top_k = s[0]
    gemm_cols = width + width // 2                             # gate+up (2I) and down (I)
    experts_read = min(n_exp, t * top_k)
    return (2.0 * t * top_k * gemm_cols * h,
            float((experts_read * gemm_cols * h + 2 * t * h) * dt))


def _reshape(a, s, t, r, dt, feature):
    return 0.0, 0.0


OP_COST = {"linear": _linear, "embedding": _embedding, "rms_norm": _rms_norm,
           "rotary_embedding": _rotary, "silu_and_mul": _silu_and_mul,
           "topk_softmax": _topk_softmax, "fused_moe": _fused_moe, "reshape": _reshape}


def op_cost(entry: dict, point: dict, dtype_bytes: int) -> tuple:
    """(flops, bytes) of one op instance at a sweep point."""
    a = _sizes(entry)
    t = point.get("num_toks", 1)
    if entry["name"] == "attention":
        hq, d, hkv = a[0][1], a[0][2], a[1][1]
        r, c = point["num_reqs"], point["kv_len"]
        if entry.get("window"):
            c = min(c, entry["window"])
        q = t / r if point["phase"] == "prefill" else 1.0
        ctx = c + q
        return (4.0 * hq * d * r * q * ctx,
                float(dtype_bytes * (r * ctx * 2 * hkv * d + 2 * r * q * hq * d)))
    fn = OP_COST.get(entry["name"])
    if fn is None:
        raise KeyError(f"no cost formula for op kind {entry['name']!r}")   # OraclePanic
    scalars = [int(v) for v, _ in entry.get("scalars", [])]
    return fn(a, scalars, t, point.get("num_reqs", 1), dtype_bytes, entry.get("feature"))


def phase_symbols(entry: dict, phase: str) -> list:
    """Attention entries carry decode-phase symbols (tracer D3);
    a prefill-phase instance runs the prefill kernel (modelir.py:122-132)."""
    if entry.get("feature") != "attention":
        return list(entry["kernel_symbols"])
    return [s.replace("_decode_attn_", f"_{phase}_attn_") for s in entry["kernel_symbols"]]


def oracle_latency(entry: dict, point: dict, hw: dict, cost_multiplier,
                   dtype_bytes: int = 2) -> float:
    """SPEC.md:476-484 at one sweep point.  hw: {peak_flops, mem_bw}."""
    flops, nbytes = op_cost(entry, point, dtype_bytes)
    mult = multiplier(cost_multiplier, phase_symbols(entry, point.get("phase", "decode")))
    return OVERHEAD_S + mult * max(flops / hw["peak_flops"], nbytes / hw["mem_bw"])


def sweep_points(entry: dict, grid: dict, max_context: int) -> list:
    """SPEC.md:466-474, D3 (:515), App. A.5: affine entries sweep their one
    feature; attention sweeps toks x reqs x kv x {prefill, decode}, skipping
    prefill points with t < r and points past the model's max_context.
    grid: {token_counts, request_counts, kv_lens, prefill_chunk, max_batch}."""
    toks = [t for t in grid["token_counts"] if t <= min(grid["prefill_chunk"], max_context)]
    reqs = [r for r in grid["request_counts"] if r <= grid["max_batch"]]
    feature = entry.get("feature", "num_toks")
    if feature == "num_toks":
        return [{"num_toks": t} for t in toks]
    if feature == "num_seqs":
        return [{"num_reqs": r} for r in reqs]
    out = [{"phase": "prefill", "num_toks": t, "num_reqs": r, "kv_len": c}
           for t in toks for r in reqs if t >= r
           for c in grid["kv_lens"] if c + -(-t // r) <= max_context]
    out += [{"phase": "decode", "num_toks": r, "num_reqs": r, "kv_len": c}
            for r in reqs for c in grid["kv_lens"] if c + 1 <= max_context]
    return out


def point_features(entry: dict, point: dict) -> tuple:
    """App. A.6 regression features: (num_toks,) / (num_reqs,) or, for
    attention, (prefill_toks, batch, kv_tokens) with kv capped at the window."""
    feature = entry.get("feature", "num_toks")
    if feature == "num_toks":
        return (point["num_toks"],)
    if feature == "num_seqs":
        return (point["num_reqs"],)
    c = point["kv_len"]
    if entry.get("window"):
        c = min(c, entry["window"])
    return (point["num_toks"] if point["phase"] == "prefill" else 0, point["num_reqs"],
            point["num_reqs"] * c)


def sweep(entry: dict, grid: dict, max_context: int, hw: dict, cost_multiplier,
          dtype_bytes: int = 2) -> tuple:
    """The measurements of one signature: x (P, n) u32 features, y (n,) f64."""
    import numpy as np

    pts = sweep_points(entry, grid, max_context)
    x = np.array([point_features(entry, p) for p in pts], dtype=np.uint32).T
    y = np.array([oracle_latency(entry, p, hw, cost_multiplier, dtype_bytes) for p in pts])
    return np.ascontiguousarray(x), y


def batch_latency(entry: dict, reqs, hw: dict, cost_multiplier, dtype_bytes: int = 2) -> float:
    """SPEC.md:606-612 reference_run's per-op cost: the oracle evaluated at one
    scheduled iteration's CONCRETE dims.  reqs: [(tokens, is_prefill, kv_before)]
    per scheduled request.  Non-attention ops see M = the iteration's token
    count (or request count); attention sums over requests with each
    request's own cached length (capped at the window) and runs the prefill
    kernel when any request is prefilling (App. A.17)."""
    a = _sizes(entry)
    t = sum(q for q, _, _ in reqs)
    phase = "prefill" if any(pf for _, pf, _ in reqs) else "decode"
    if entry["name"] == "attention":
        w = entry.get("window")
        flops, nbytes = _attention_cost(a[0][1], a[1][1], a[0][2],
                                        [(q, min(c, w) if w else c) for q, _, c in reqs],
                                        dtype_bytes)
    else:
        scalars = [int(v) for v, _ in entry.get("scalars", [])]
        flops, nbytes = OP_COST[entry["name"]](a, scalars, t, len(reqs), dtype_bytes,
                                               entry.get("feature"))
    mult = multiplier(cost_multiplier, phase_symbols(entry, phase))
    return OVERHEAD_S + mult * max(flops / hw["peak_flops"], nbytes / hw["mem_bw"])
