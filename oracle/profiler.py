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


def roofline_latency(flops: float, nbytes: float, peak_flops: float, mem_bw: float,
                     multiplier: float = 1.0, overhead: float = 5e-6) -> float:
    """overhead + multiplier * max(flops/peak, bytes/bw)."""
    return overhead + multiplier * max(flops / peak_flops, nbytes / mem_bw)


def matmul_cost(m: int, k: int, n: int, dtype_bytes: int) -> tuple:
    """SPEC.md:480 'matmul: 2·M·K·N flops'; bytes = (MK + KN + MN) * dtype."""
    return 2 * m * k * n, (m * k + k * n + m * n) * dtype_bytes


def comm_latency(tp: int, nbytes: int, alpha: float, beta: float) -> float:
    """SPEC.md:486-494 ring all-reduce: 2(tp-1)/tp * (alpha + bytes/tp * beta)."""
    return 2 * (tp - 1) / tp * (alpha + nbytes / tp * beta)
