"""Taint-labelled operation records, their canonical form, and the packed
columnar layout the GPU dedup kernel consumes.

* ``RunnableEntry`` mirrors the reference's runnable-set entry (SPEC.md:318-321,
  export format SPEC.md:404): granularity, op name, argument template of
  tainted dims (taint strings use the grammar of taint.py:215-239), tainted
  scalars, attrs, kernel symbols, repeat count.  Two hot-path fields ride
  along: ``feature`` (which iteration quantity the simulator regresses the
  entry on) and ``window`` (sliding window of an attention module).
* ``canonical_bytes`` is signature canonicalisation (layout
  D1/D2 SPEC.md:513-514 with the byte widths pinned in SURVEY App. A.1-A.3).
* ``RecordPacker`` turns entries into the u32 record stream + string tables of
  include/dooly_b200.h (the canonical message is rebuilt on the GPU).
* ``runnable_entries`` is the record producer: tracer.run_trace ->
  opset.build_tree / prune / resolve.
  ``synthesize_entries`` is the closed-form runnable set of one
  (model, backend, tp) in `run_trace` op order with layer
  pruning; tests hold the traced sets equal to it entry for
  entry, and ``producer="synth"`` selects it.
"""

from __future__ import annotations

import hashlib
import json
import struct
from dataclasses import dataclass, field
from typing import Iterable, Optional, Sequence

import numpy as np

from .modelir import BackendSpec, ModelConfig

SIGFMT = b"sigfmt=1"
SCALAR_POS_BASE = 1 << 16           # SPEC.md:514 (D2)
NO_ATTR = 0xFFFFFFFF
FEATURES = ("num_toks", "num_seqs", "attention")


@dataclass(frozen=True)
class RunnableEntry:
    granularity: str                       # "operator" | "module"
    name: str
    arg_template: tuple                    # ((size, taint_str), ...) per tensor argument
    scalars: tuple = ()                    # ((value, taint_str), ...)
    context_required: bool = False
    attrs: tuple = ()                      # sorted ((key, primitive), ...)
    kernel_symbols: tuple = ()
    repeat_count: int = 1
    feature: str = "num_toks"
    window: Optional[int] = None

    def model_dims(self) -> list:
        """(position, value) of every Base(MODEL_CONFIG) dim and scalar (App. A.2)."""
        out = []
        pos = 0
        for arg in self.arg_template:
            for size, taint in arg:
                if taint == "MC":
                    out.append((pos, int(size)))
                pos += 1
        for k, (value, taint) in enumerate(self.scalars):
            if taint == "MC":
                out.append((SCALAR_POS_BASE + k, int(value)))
        return out

    def to_json(self) -> dict:
        return {"granularity": self.granularity, "name": self.name,
                "arg_template": [[list(d) for d in a] for a in self.arg_template],
                "scalars": [list(s) for s in self.scalars],
                "context_required": self.context_required, "attrs": dict(self.attrs),
                "kernel_symbols": list(self.kernel_symbols), "repeat_count": self.repeat_count,
                "feature": self.feature, "window": self.window}

    @staticmethod
    def from_json(d: dict) -> "RunnableEntry":
        return RunnableEntry(
            granularity=d["granularity"], name=d["name"],
            arg_template=tuple(tuple((int(s), str(t)) for s, t in a) for a in d["arg_template"]),
            scalars=tuple((int(v), str(t)) for v, t in d.get("scalars", [])),
            context_required=bool(d.get("context_required", False)),
            attrs=tuple(sorted(d.get("attrs", {}).items())),
            kernel_symbols=tuple(d.get("kernel_symbols", ())),
            repeat_count=int(d.get("repeat_count", 1)),
            feature=d.get("feature", "num_toks"), window=d.get("window"))


def dump_runnable_set(entries: Sequence[RunnableEntry]) -> str:
    return json.dumps([e.to_json() for e in entries], sort_keys=True)


def load_runnable_set(text: str) -> list:
    return [RunnableEntry.from_json(d) for d in json.loads(text)]


# ----------------------------------------------------------------- canonical form


def _attr_value_bytes(v) -> bytes:
    if isinstance(v, bool):
        return b"b" + (b"\x01" if v else b"\x00")
    if isinstance(v, int):
        return b"i" + struct.pack("<q", v)
    if isinstance(v, float):
        return b"f" + struct.pack("<d", v)
    if isinstance(v, str):
        raw = v.encode()
        return b"s" + struct.pack("<I", len(raw)) + raw
    if v is None:
        return b"n"
    raise TypeError(f"attr values must be primitives, got {type(v).__name__}")


def attr_digest(attrs) -> bytes:
    """SHA-256 of the attrs sorted by UTF-8 key (App. A.3); 32 bytes."""
    items = sorted(dict(attrs).items(), key=lambda kv: kv[0].encode())
    body = b"".join(struct.pack("<I", len(k.encode())) + k.encode() + _attr_value_bytes(v)
                    for k, v in items)
    return hashlib.sha256(body).digest()


def canonical_bytes(entry: RunnableEntry) -> bytes:
    """The sigfmt=1 canonical serialisation (App. A.1)."""
    name = entry.name.encode()
    dims = sorted(entry.model_dims())
    syms = sorted(s.encode() for s in set(entry.kernel_symbols))
    parts = [SIGFMT, struct.pack("<I", len(name)), name, struct.pack("<I", len(dims))]
    parts += [struct.pack("<IQ", p, v) for p, v in dims]
    parts.append(struct.pack("<I", len(syms)))
    parts += [struct.pack("<I", len(s)) + s for s in syms]
    if entry.granularity == "module":
        parts.append(attr_digest(entry.attrs))
    return b"".join(parts)


# -------------------------------------------------------------------- packing


@dataclass
class PackedRecords:
    """Columnar record batch; numpy on the host, ``.to(device)`` for the GPU."""

    words: np.ndarray          # u32
    rec_off: np.ndarray        # i64, n
    op_bytes: np.ndarray       # u8
    op_off: np.ndarray         # i64, n_ops + 1
    sym_bytes: np.ndarray      # u8
    sym_off: np.ndarray        # i64, n_sym + 1
    attr_digests: np.ndarray   # u8, (n_attr, 32)
    repeat: np.ndarray         # u32, n
    op_names: list = field(default_factory=list)

    @property
    def n(self) -> int:
        return int(self.rec_off.shape[0])

    def nbytes(self) -> int:
        return int(self.words.nbytes + self.rec_off.nbytes)


class RecordPacker:
    """Interns op names / symbols / attr digests and emits packed records.

    Symbol ids are assigned in bytewise-sorted order at ``finish`` so that a
    record's ascending id list IS the sorted-symbol order of the canonical form.
    """

    def __init__(self) -> None:
        self._ops: dict = {}
        self._attrs: dict = {}
        self._recs: list = []

    def add(self, e: RunnableEntry) -> None:
        op = self._ops.setdefault(e.name, len(self._ops))
        if e.granularity == "module":
            dig = attr_digest(e.attrs)
            attr = self._attrs.setdefault(dig, len(self._attrs))
        else:
            attr = NO_ATTR
        dims = sorted(e.model_dims())
        self._recs.append((op, dims, sorted(set(e.kernel_symbols)), attr, e.repeat_count))

    def extend(self, entries: Iterable[RunnableEntry]) -> "RecordPacker":
        for e in entries:
            self.add(e)
        return self

    def finish(self) -> PackedRecords:
        sym_list = sorted({s.encode() for r in self._recs for s in r[2]})
        sym_id = {s: i for i, s in enumerate(sym_list)}
        words: list = []
        off = np.empty(len(self._recs), dtype=np.int64)
        for i, (op, dims, syms, attr, rep) in enumerate(self._recs):
            off[i] = len(words)
            ids = sorted(sym_id[s.encode()] for s in syms)
            words += [op, len(dims) | (len(ids) << 16), attr, rep]
            for p, v in dims:
                words += [p, v & 0xFFFFFFFF, v >> 32]
            words += ids
        op_names = sorted(self._ops, key=self._ops.get)
        ob, oo = _string_table([n.encode() for n in op_names])
        sb, so = _string_table(sym_list)
        ad = np.zeros((len(self._attrs), 32), dtype=np.uint8)
        for dig, i in self._attrs.items():
            ad[i] = np.frombuffer(dig, dtype=np.uint8)
        return PackedRecords(np.asarray(words, dtype=np.uint32), off, ob, oo, sb, so, ad,
                             np.asarray([r[4] for r in self._recs], dtype=np.uint32), op_names)


def _string_table(items: Sequence[bytes]):
    off = np.zeros(len(items) + 1, dtype=np.int64)
    if items:
        off[1:] = np.cumsum([len(s) for s in items])
    data = np.frombuffer(b"".join(items), dtype=np.uint8).copy() if items else np.zeros(0, np.uint8)
    return data, off


def pack_entries(entries: Sequence[RunnableEntry]) -> PackedRecords:
    return RecordPacker().extend(entries).finish()


def pack_uniform(op_names: Sequence[str], op_ids: np.ndarray, dim_pos: np.ndarray,
                 dim_val: np.ndarray, symbols: Sequence[str], sym_ids: np.ndarray,
                 attr_digests: np.ndarray, attr_ids: np.ndarray,
                 repeat: np.ndarray) -> PackedRecords:
    """Vectorised packing of n records that share (n_dims, n_sym) — the bulk
    path for synthetic corpora (config C5).  ``symbols`` must be sorted
    bytewise and each row of ``sym_ids`` ascending; ``dim_pos`` ascending."""
    n, nd = dim_pos.shape
    ns = sym_ids.shape[1]
    enc = [s.encode() for s in symbols]
    if enc != sorted(enc):
        raise ValueError("symbols must be sorted bytewise")
    stride = 4 + 3 * nd + ns
    w = np.empty((n, stride), dtype=np.uint32)
    w[:, 0] = op_ids
    w[:, 1] = nd | (ns << 16)
    w[:, 2] = attr_ids
    w[:, 3] = repeat
    v = dim_val.astype(np.uint64)
    w[:, 4:4 + 3 * nd:3] = dim_pos
    w[:, 5:5 + 3 * nd:3] = (v & 0xFFFFFFFF).astype(np.uint32)
    w[:, 6:6 + 3 * nd:3] = (v >> 32).astype(np.uint32)
    w[:, 4 + 3 * nd:] = sym_ids
    ob, oo = _string_table([s.encode() for s in op_names])
    sb, so = _string_table(enc)
    return PackedRecords(w.reshape(-1), np.arange(n, dtype=np.int64) * stride, ob, oo, sb, so,
                         np.ascontiguousarray(attr_digests, dtype=np.uint8),
                         repeat.astype(np.uint32), list(op_names))


# ---------------------------------------------------------------- synthesizer

_DUMMY_REQS, _DUMMY_TOKS = 2, 269     # tracer D1: collision-free primes


def _gemm_symbol(dtype_bytes: int) -> str:
    return f"gemm_f{8 * dtype_bytes}_tn"


def synthesize_entries(cfg: ModelConfig, backend: BackendSpec, tp: int = 1) -> list:
    """Runnable set of one (model, backend, tp) configuration.

    Per layer representative (layers collapse unless their attention window
    differs, opset D1 SPEC.md:407): input norm, qkv linear, rope, attention
    module (decode-phase kernel symbols, tracer D3 SPEC.md:304), o linear,
    post norm, then dense MLP (gate_up linear, act, down linear) or MoE (router
    linear, top-k softmax, expert module).  Embedding first, final norm and
    lm_head last.  Model-config dims are sharded by ``tp``.
    """
    tok = (_DUMMY_REQS * _DUMMY_TOKS, "NT")
    h, d = cfg.hidden_dim, cfg.head_dim
    hq, hkv = cfg.num_q_heads // tp, cfg.num_kv_heads // tp
    inter = cfg.intermediate_size // tp
    vocab = cfg.vocab_size // tp
    gemm = (_gemm_symbol(cfg.dtype_bytes),)

    def mc(v):
        return (v, "MC")

    def op(name, args, syms, rep, feature="num_toks", scalars=()):
        return RunnableEntry("operator", name, tuple(tuple(a) for a in args), tuple(scalars),
                             False, (), tuple(syms), rep, feature)

    def linear(k, n, rep, x=tok, feature="num_toks"):
        return op("linear", [(x, mc(k)), (mc(n), mc(k))], gemm, rep, feature)

    def norm(rep):
        return op("rms_norm", [(tok, mc(h)), (mc(h),)], ("rms_norm_kernel",), rep)

    out = [op("embedding", [(tok,), (mc(vocab), mc(h))], ("embedding_lookup_kernel",), 1)]
    for window in cfg.windows():
        rep = cfg.layers_with(window)
        attrs = (("causal", True),) + ((("sliding_window", window),) if window else ())
        out.append(norm(rep))
        out.append(linear(h, (hq + 2 * hkv) * d, rep))
        out.append(op("rotary_embedding", [(tok, mc(hq), mc(d)), (tok, mc(hkv), mc(d))],
                      ("rotary_embedding_kernel",), rep))
        out.append(RunnableEntry(
            "module", "attention",
            ((tok, mc(hq), mc(d)), (tok, mc(hkv), mc(d)), (tok, mc(hkv), mc(d))),
            (), True, attrs,
            backend.attention_kernels(hq, hkv, d, window, "decode"), rep, "attention", window))
        out.append(linear(hq * d, h, rep))
        out.append(norm(rep))
        if cfg.moe is None:
            out.append(linear(h, 2 * inter, rep))
            out.append(op("silu_and_mul", [(tok, mc(2 * inter))], ("act_and_mul_kernel",), rep))
            out.append(linear(inter, h, rep))
        else:
            m = cfg.moe
            e_inter = m.expert_intermediate // tp
            out.append(linear(h, m.num_experts, rep))
            out.append(op("topk_softmax", [(tok, mc(m.num_experts))], ("topk_gating_softmax",),
                          rep, scalars=[mc(m.top_k)]))
            out.append(RunnableEntry(
                "module", "fused_moe",
                ((tok, mc(h)), (mc(m.num_experts), mc(2 * e_inter), mc(h)),
                 (mc(m.num_experts), mc(h), mc(e_inter))),
                (mc(m.top_k),), True,
                (("num_experts", m.num_experts), ("top_k", m.top_k)),
                ("moe_align_block_size", "fused_moe_kernel", "moe_sum"), rep, "num_toks"))
    out.append(norm(1))
    # Appendix F: every non-attention op regresses on the token count
    out.append(linear(h, vocab, 1))
    return out


def runnable_entries(cfg: ModelConfig, backend: BackendSpec, tp: int = 1,
                     producer: str = "trace") -> list:
    """The runnable set of one configuration: traced and resolved (default) or
    the closed-form synthesizer."""
    if producer == "synth":
        return synthesize_entries(cfg, backend, tp)
    if producer != "trace":
        raise ValueError(f"unknown record producer {producer!r}")
    from .opset import runnable_set

    return runnable_set(cfg, backend, tp)


def corpus_entries(manifest, tp: Optional[int] = None, producer: str = "trace") -> list:
    """All (model, backend) runnable sets in manifest order — models outer,
    backends inner (dedup order, App. A.4).  Returns [(model, backend, entries)]."""
    tp = manifest.tp_degree if tp is None else tp
    return [(m, b, runnable_entries(m, b, tp, producer)) for m in manifest.models
            for b in manifest.backends]
