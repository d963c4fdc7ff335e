"""Tainted runner: one symbolic forward pass of a model under
an attention backend, with every tensor dimension and scalar labelled by its
provenance taint, recorded as a module / operation / kernel event forest.

This is the upstream producer of the hot path's records:
``opset.resolve`` turns the trace into the runnable set that ``profiler.dedup``
canonicalises and hashes.  It is host-side, control-heavy and low-volume (a few
hundred events per model), so it stays in Python.

* Scalars are ``TInt`` (value, taint); arithmetic on them applies the taint
  combination rules, so weight shapes such as (q + 2 kv) x head_dim carry
  MODEL_CONFIG without a registry lookup (paper §4.1, "recursively taints
  member values").  Tensor-parallel sharding divides by an untainted degree.
* ``map_dims`` (create / reshape / permute / concat) and ``preserve_dims``
  (dimension-preserving ops) are the two dim-propagation rules of SPEC.md:263-287.
* Events get synthetic ticks from a depth-first counter (D2: parents span their
  children; collectives have zero duration).  The dummy batch is collision-free
  by construction (D1: primes not among the model's values); a caller-supplied
  colliding batch is retraced once (Appendix B).
* The trace exports to Chrome Trace Event JSON with an ``args.dooly`` extension
  and imports back losslessly.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import Optional, Sequence

from . import taint as T
from .errors import RetraceFailed, ShapeMismatch
from .modelir import BackendSpec, ModelConfig

TOKS_PRIMES = (269, 271, 277, 281, 283, 293, 307, 311, 313, 317, 331, 337)
REQS_PRIMES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


@dataclass(frozen=True)
class DummyBatch:
    num_reqs: int
    tokens_per_req: int

    @property
    def num_tokens(self) -> int:
        return self.num_reqs * self.tokens_per_req


@dataclass(frozen=True)
class TInt:
    """A tainted integer scalar."""

    value: int
    taint: str = T.BOT

    def _other(self, o):
        return o if isinstance(o, TInt) else TInt(int(o))

    def __mul__(self, o):
        o = self._other(o)
        return TInt(self.value * o.value, T.combine(self.taint, o.taint, self.value, o.value))

    __rmul__ = __mul__

    def __add__(self, o):
        o = self._other(o)
        return TInt(self.value + o.value, T.combine(self.taint, o.taint, self.value, o.value))

    __radd__ = __add__

    def __floordiv__(self, o):
        """Division by an untainted degree (tensor parallelism) keeps the taint."""
        o = self._other(o)
        if self.value % o.value:
            raise ShapeMismatch(f"{self.value} not divisible by {o.value}")
        return TInt(self.value // o.value, T.combine(self.taint, o.taint, self.value, o.value)
                    if o.taint != T.BOT else self.taint)

    def dim(self) -> tuple:
        return (self.value, self.taint)


@dataclass
class TraceEvent:
    id: int
    parent_id: Optional[int]
    category: str                      # module | operation | kernel
    name: str
    begin: int
    end: int
    input_dims: list = field(default_factory=list)     # [[(size, taint), ...] per tensor]
    scalars: list = field(default_factory=list)        # [(value, taint), ...]
    attrs: dict = field(default_factory=dict)
    kernel_symbols: list = field(default_factory=list)


@dataclass
class TaintedTrace:
    events: list
    registry: T.Registry
    model: ModelConfig
    backend: BackendSpec
    batch: DummyBatch
    tp: int
    ambiguities: list = field(default_factory=list)

    # ---- Chrome Trace Event JSON (array form, complete events), lossless
    def to_chrome(self) -> str:
        out = []
        for e in self.events:
            out.append({"name": e.name, "cat": e.category, "ph": "X", "ts": e.begin,
                        "dur": e.end - e.begin, "pid": 0, "tid": 0,
                        "args": {"dooly": {
                            "id": e.id, "parent": e.parent_id,
                            "dims": [[[s, t] for s, t in a] for a in e.input_dims],
                            "scalars": [[v, t] for v, t in e.scalars],
                            "attrs": e.attrs, "kernel_symbols": list(e.kernel_symbols)}}})
        return json.dumps(out, sort_keys=True, separators=(",", ":"))

    @staticmethod
    def events_from_chrome(text: str) -> list:
        evs = []
        for d in json.loads(text):
            x = d["args"]["dooly"]
            evs.append(TraceEvent(
                x["id"], x["parent"], d["cat"], d["name"], d["ts"], d["ts"] + d["dur"],
                [[(int(s), T.parse(t)) for s, t in a] for a in x["dims"]],
                [(int(v), T.parse(t)) for v, t in x["scalars"]], dict(x["attrs"]),
                list(x["kernel_symbols"])))
        return evs


# ------------------------------------------------------------------ sources


def model_values(cfg: ModelConfig, tp: int = 1) -> dict:
    """Every shape value of the model (fields and the derived / sharded values
    the forward pass uses) -> MODEL_CONFIG.  dtype_bytes is a byte width, not a
    dimension, and is not registered (SPEC.md:238 example registers 2 as NR)."""
    vals = {cfg.hidden_dim, cfg.num_layers, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim,
            cfg.intermediate_size, cfg.vocab_size, cfg.max_context,
            cfg.num_q_heads * cfg.head_dim, cfg.num_kv_heads * cfg.head_dim}
    vals |= {w for w in cfg.layer_attention if w}
    if cfg.moe is not None:
        vals |= {cfg.moe.num_experts, cfg.moe.top_k, cfg.moe.expert_intermediate}
    if tp > 1:
        vals |= {cfg.num_q_heads // tp, cfg.num_kv_heads // tp, cfg.intermediate_size // tp,
                 cfg.vocab_size // tp}
        if cfg.moe is not None:
            vals.add(cfg.moe.expert_intermediate // tp)
    return {v: T.MC for v in vals if v >= 1}


def seed_sources(cfg: ModelConfig, batch: DummyBatch, tp: int = 1) -> T.Registry:
    """model values as MODEL_CONFIG, num_reqs as NUM_REQS, the
    total token count and tokens_per_req as NUM_TOKS; collisions recorded."""
    reg = T.Registry()
    for v, t in sorted(model_values(cfg, tp).items()):
        reg.register(v, t)
    reg.register(batch.num_reqs, T.NR)
    reg.register(batch.num_tokens, T.NT)
    reg.register(batch.tokens_per_req, T.NT)
    return reg


def choose_batch(cfg: ModelConfig, tp: int = 1, skip: Sequence[DummyBatch] = ()) -> DummyBatch:
    """D1: tokens_per_req from primes >= 269, num_reqs from small primes, skipping
    any value (or product) the model uses; the first admissible pair wins."""
    used = set(model_values(cfg, tp))
    for r in REQS_PRIMES:
        for t in TOKS_PRIMES:
            b = DummyBatch(r, t)
            if b in skip or {r, t, r * t} & used or r == t:
                continue
            return b
    raise RetraceFailed(f"no collision-free dummy batch for {cfg.name}")


# ------------------------------------------------------------ dim propagation


def map_dims(op_kind: str, inputs: Sequence, params, reg: T.Registry) -> list:
    """SPEC.md:263-271.

    create:  params = scalars [TInt | int]: each dim takes its scalar's taint
             (an untainted int is resolved through the registry, else BOT).
    reshape: params = output sizes, at most one -1 (inferred).  Merged dims
             combine their taints; a split of a MIX recovers components with
             taint.split; a split of a base taint inherits it; anything else
             is resolved through the registry.
    permute: params = permutation of the input dims.
    concat:  inputs = list of dim lists, params = axis; the axis dim combines.
    """
    def resolve(v):
        return reg.lookup(v) or T.BOT

    if op_kind == "create":
        return [(p.value, p.taint) if isinstance(p, TInt) else (int(p), resolve(int(p)))
                for p in params]
    if op_kind == "permute":
        return [tuple(inputs[i]) for i in params]
    if op_kind == "concat":
        axis = params
        out = [tuple(d) for d in inputs[0]]
        size, taint = out[axis]
        for other in inputs[1:]:
            s2, t2 = other[axis]
            taint = T.combine(taint, t2, size, s2)
            size += s2
        out[axis] = (size, taint)
        return out
    if op_kind != "reshape":
        raise ValueError(f"unknown map_dims op {op_kind!r}")
    total = 1
    for s, _ in inputs:
        total *= s
    sizes = list(params)
    if sizes.count(-1) > 1:
        raise ShapeMismatch("at most one inferred dimension")
    known = 1
    for s in sizes:
        if s != -1:
            known *= s
    if -1 in sizes:
        if known == 0 or total % known:
            raise ShapeMismatch(f"cannot infer a dim: {total} elements into {sizes}")
        sizes[sizes.index(-1)] = total // known
        known = total
    if known != total:
        raise ShapeMismatch(f"{total} elements reshaped to {sizes}")
    # group input and output dims by equal running products
    out, i, j = [], 0, 0
    inputs = [tuple(d) for d in inputs]
    while i < len(inputs) or j < len(sizes):
        gi, go = [inputs[i]] if i < len(inputs) else [], [sizes[j]] if j < len(sizes) else []
        i, j = i + len(gi), j + len(go)
        pi = gi[0][0] if gi else 1
        po = go[0] if go else 1
        while pi != po:
            if pi < po:
                gi.append(inputs[i])
                pi *= inputs[i][0]
                i += 1
            else:
                go.append(sizes[j])
                po *= sizes[j]
                j += 1
        if len(gi) == 1 and len(go) == 1:
            out.append(gi[0])
        elif len(go) == 1:                                  # merge
            taint, size = gi[0][1], gi[0][0]
            for s, t in gi[1:]:
                taint = T.combine(taint, t, size, s)
                size *= s
            out.append((go[0], taint))
        elif len(gi) == 1:                                  # split
            s_in, t_in = gi[0]
            if T.is_mix(t_in):
                rest, got = t_in, []
                for s in go:
                    if s in T.components(rest):
                        lab, rest = T.split(rest, s)
                        got.append((s, lab))
                    else:
                        got.append((s, None))
                missing = [k for k, (_, t) in enumerate(got) if t is None]
                for k in missing:      # the one unmatched dim takes the residual
                    got[k] = (got[k][0], rest if len(missing) == 1 else resolve(got[k][0]))
                out.extend(got)
            elif t_in != T.BOT:
                out.extend((s, t_in) for s in go)
            else:
                out.extend((s, resolve(s)) for s in go)
        else:
            out.extend((s, resolve(s)) for s in go)
    return out


def preserve_dims(op_kind: str, inputs: Sequence, out_shape: Sequence[int],
                  reg: T.Registry) -> list:
    """each output dim inherits the taint of the first
    size-matching input dim (argument order, heuristic H1), else the registry,
    else BOT; ``matmul`` (x [.., k] times weight [n, k]) inherits positionally."""
    if op_kind == "matmul":
        x, w = inputs[0], inputs[1]
        return [tuple(d) for d in x[:-1]] + [tuple(w[0])]
    out = []
    for s in out_shape:
        hit = next((d for a in inputs for d in a if d[0] == s), None)
        out.append(tuple(hit) if hit is not None else (s, reg.lookup(s) or T.BOT))
    return out


# ------------------------------------------------------------------ the pass


class _Recorder:
    def __init__(self):
        self.events: list = []
        self.stack: list = []
        self.tick = 0

    def open(self, category, name, dims=(), scalars=(), attrs=None, kernels=()):
        ev = TraceEvent(len(self.events), self.stack[-1].id if self.stack else None, category,
                        name, self.tick, -1, [list(a) for a in dims], list(scalars),
                        dict(attrs or {}), list(kernels))
        self.tick += 1
        self.events.append(ev)
        self.stack.append(ev)
        return ev

    def close(self):
        ev = self.stack.pop()
        ev.end = self.tick
        self.tick += 1

    def op(self, name, dims=(), scalars=(), kernels=(), attrs=None):
        """An operation event with one kernel child per symbol."""
        self.open("operation", name, dims, scalars, attrs, kernels)
        for k in kernels:
            self.open("kernel", k)
            self.close()
        self.close()

    def collective(self, name, dims):
        """Collectives are hooked as no-ops: zero duration (paper §4)."""
        ev = TraceEvent(len(self.events), self.stack[-1].id, "operation", name, self.tick,
                        self.tick, [list(a) for a in dims])
        self.events.append(ev)
        self.tick += 1


def _trace_once(cfg: ModelConfig, backend: BackendSpec, batch: DummyBatch, tp: int,
                reg: T.Registry) -> list:
    rec = _Recorder()
    mc = lambda v: TInt(v, T.MC)                                        # noqa: E731
    toks = TInt(batch.num_tokens, reg.lookup(batch.num_tokens) or T.BOT)
    h, d = mc(cfg.hidden_dim), mc(cfg.head_dim)
    hq, hkv = mc(cfg.num_q_heads) // tp, mc(cfg.num_kv_heads) // tp
    inter, vocab = mc(cfg.intermediate_size) // tp, mc(cfg.vocab_size) // tp
    gemm = f"gemm_f{8 * cfg.dtype_bytes}_tn"

    def weight(*dims):
        return map_dims("create", [], dims, reg)

    def linear(name, x, n):
        """nn.Linear module: x [.., k] @ weight [n, k] -> [.., n]."""
        w = weight(n, TInt(x[-1][0], x[-1][1]))
        rec.open("module", name)
        rec.op("linear", [x, w], kernels=(gemm,))
        rec.close()
        return preserve_dims("matmul", [x, w], None, reg)

    def rms_norm(name, x):
        rec.open("module", name)
        rec.op("rms_norm", [x, weight(h)], kernels=("rms_norm_kernel",))
        rec.close()
        return preserve_dims("elementwise", [x], [s for s, _ in x], reg)

    rec.open("module", cfg.name)
    ids = map_dims("create", [], [toks], reg)
    rec.open("module", "embed_tokens")
    rec.op("embedding", [ids, weight(vocab, h)], kernels=("embedding_lookup_kernel",))
    rec.close()
    x = map_dims("create", [], [toks, h], reg)
    for layer in range(cfg.num_layers):
        window = cfg.layer_attention[layer]
        rec.open("module", "decoder_layer")
        a = rms_norm("input_layernorm", x)
        rec.open("module", "self_attn")
        qkv = linear("qkv_proj", a, (hq + 2 * hkv) * d)
        # q / k / v views: split the fused projection, then heads x head_dim
        q = map_dims("reshape", [(toks.value, toks.taint), ((hq * d).value, T.MC)],
                     [toks.value, hq.value, d.value], reg)
        k = map_dims("reshape", [(toks.value, toks.taint), ((hkv * d).value, T.MC)],
                     [toks.value, hkv.value, d.value], reg)
        v = [tuple(t) for t in k]
        rec.op("view", [qkv])
        rec.open("module", "rotary_emb")
        rec.op("rotary_embedding", [q, k], kernels=("rotary_embedding_kernel",))
        rec.close()
        attrs = {"causal": True}
        if window:
            attrs["sliding_window"] = window
        # decode phase traced by default (tracer D3)
        syms = backend.attention_kernels(hq.value, hkv.value, d.value, window, "decode")
        rec.open("module", "attention", [q, k, v], attrs=attrs)
        rec.op("attention", [q, k, v], kernels=syms)
        rec.close()
        o_in = map_dims("reshape", q, [toks.value, -1], reg)
        rec.op("view", [q])
        x_attn = linear("o_proj", o_in, h)
        rec.close()                                                      # self_attn
        if tp > 1:
            rec.collective("all_reduce", [x_attn])
        m = rms_norm("post_attention_layernorm", x_attn)
        if cfg.moe is None:
            rec.open("module", "mlp")
            gu = linear("gate_up_proj", m, 2 * inter)
            rec.open("module", "act_fn")
            rec.op("silu_and_mul", [gu], kernels=("act_and_mul_kernel",))
            rec.close()
            down_in = [gu[0], (inter.value, inter.taint)]
            linear("down_proj", down_in, h)
            rec.close()
        else:
            moe = cfg.moe
            n_exp, top_k = mc(moe.num_experts), mc(moe.top_k)
            e_inter = mc(moe.expert_intermediate) // tp
            rec.open("module", "block_sparse_moe")
            logits = linear("gate", m, n_exp)
            rec.op("topk_softmax", [logits], [top_k.dim()], kernels=("topk_gating_softmax",))
            w13 = weight(n_exp, 2 * e_inter, h)
            w2 = weight(n_exp, h, e_inter)
            rec.open("module", "fused_moe", [m, w13, w2], [top_k.dim()],
                     attrs={"num_experts": moe.num_experts, "top_k": moe.top_k})
            # routing is uniform-random under the trace seed (D4); the expert
            # kernels see the aligned block layout, not per-expert shapes
            rec.op("fused_moe", [m, w13, w2], [top_k.dim()],
                   kernels=("moe_align_block_size", "fused_moe_kernel", "moe_sum"))
            rec.close()
            rec.close()
        if tp > 1:
            rec.collective("all_reduce", [m])
        rec.close()                                                      # decoder_layer
        x = m
    f = rms_norm("norm", x)
    linear("lm_head", f, vocab)
    rec.close()                                                          # model
    return rec.events


def run_trace(cfg: ModelConfig, backend: BackendSpec, batch: Optional[DummyBatch] = None,
              tp: int = 1) -> TaintedTrace:
    """the symbolic forward pass.  A supplied batch that
    collides with a model value is retraced once with a fresh collision-free
    batch (Appendix B); a second collision raises RetraceFailed."""
    b = batch or choose_batch(cfg, tp)
    tried: list = []
    for _ in range(2):
        reg = seed_sources(cfg, b, tp)
        amb = sorted(reg.collisions)
        if not amb:
            return TaintedTrace(_trace_once(cfg, backend, b, tp, reg), reg, cfg, backend, b, tp)
        tried.append(b)
        b = choose_batch(cfg, tp, skip=tried)
    raise RetraceFailed(f"{cfg.name}: dummy batches {tried} both collided")
