"""Operation Set Finder: trace -> call tree -> pruned tree ->
minimal runnable set, the record stream the hot path dedups.

* ``build_tree`` nests events by interval containment (not by the recorded
  parent ids), so an imported Chrome trace is rebuilt from its ticks alone.
* ``fingerprint`` hashes (category, name, attrs, kernel symbols, the taints of
  every dim with MODEL_CONFIG values kept and workload values dropped, child
  fingerprints) — D1: layers with a different window must not collapse, a
  different token count must not split them.
* ``prune`` collapses structurally identical siblings (not only adjacent ones:
  interleaved sliding-window layers collapse per kind) into the first instance
  with a repeat count; the kernel multiset weighted by repeats is conserved.
* ``resolve`` walks kernels bottom-up: an operation whose kind runs standalone
  becomes an operator entry; a context-dependent one (attention, MoE dispatch)
  is absorbed by its nearest stateful ancestor module, run with emulated
  context, as one module entry.  Views and collectives launch no kernel and
  are skipped.
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass, field
from typing import Optional, Sequence

from . import taint as T
from .errors import ContextUnavailable, MalformedTrace, Unresolvable
from .records import RunnableEntry
from .tracer import TaintedTrace, TraceEvent, run_trace

STANDALONE = frozenset({"embedding", "linear", "rms_norm", "rotary_embedding", "silu_and_mul",
                        "topk_softmax"})
CONTEXT_DEPENDENT = frozenset({"attention", "fused_moe"})
STATEFUL_MODULES = frozenset({"attention", "fused_moe"})       # D3: the engine's registry
VERIFY_POINT = {"num_toks": 4, "num_reqs": 1, "phase": "decode", "kv_len": 1}   # D2


@dataclass
class CallNode:
    event: TraceEvent
    children: list = field(default_factory=list)
    repeat: int = 1
    fp: str = ""

    def kernels(self) -> list:
        """Kernel leaves of this subtree in trace order (one instance)."""
        if self.event.category == "kernel":
            return [self.event.name]
        return [k for c in self.children for k in c.kernels()]

    def kernel_count(self) -> int:
        """Kernel launches this subtree stands for, repeats included."""
        if self.event.category == "kernel":
            return self.repeat
        return self.repeat * sum(c.kernel_count() for c in self.children)


@dataclass
class CallTree:
    roots: list

    def walk(self):
        stack = list(reversed(self.roots))
        while stack:
            n = stack.pop()
            yield n
            stack.extend(reversed(n.children))

    def kernel_count(self) -> int:
        return sum(r.kernel_count() for r in self.roots)


def build_tree(events: Sequence[TraceEvent]) -> CallTree:
    """parentage by interval containment.  Overlapping
    siblings raise MalformedTrace."""
    roots: list = []
    stack: list = []
    for ev in sorted(events, key=lambda e: (e.begin, -e.end, e.id)):
        if ev.end < ev.begin:
            raise MalformedTrace(f"event {ev.id} ends before it begins")
        while stack and stack[-1].event.end <= ev.begin and not (
                stack[-1].event.begin == ev.begin and ev.end <= stack[-1].event.end):
            stack.pop()
        node = CallNode(ev)
        if stack:
            top = stack[-1].event
            if ev.end > top.end:
                raise MalformedTrace(f"event {ev.id} [{ev.begin},{ev.end}] overlaps "
                                     f"{top.id} [{top.begin},{top.end}]")
            stack[-1].children.append(node)
        else:
            roots.append(node)
        stack.append(node)
    tree = CallTree(roots)
    for r in roots:
        _fingerprint(r)
    return tree


def _dim_key(size: int, taint: str):
    if taint == T.MC:
        return [size, taint]
    if T.is_mix(taint):
        return [None, [[v if lab == T.MC else None, lab]
                       for v, lab in sorted(T.components(taint).items())]]
    return [None, taint]


def _fingerprint(node: CallNode) -> str:
    for c in node.children:
        _fingerprint(c)
    e = node.event
    doc = [e.category, e.name, sorted(e.attrs.items()), list(e.kernel_symbols),
           [[_dim_key(s, t) for s, t in a] for a in e.input_dims],
           [_dim_key(v, t) for v, t in e.scalars], [c.fp for c in node.children]]
    node.fp = hashlib.sha256(json.dumps(doc, separators=(",", ":")).encode()).hexdigest()
    return node.fp


def prune(tree: CallTree) -> CallTree:
    """identical sibling subtrees -> first instance x count.
    Returns a new tree; idempotent."""
    def go(n: CallNode) -> CallNode:
        kids: dict = {}
        for c in n.children:
            p = go(c)
            if p.fp in kids:
                kids[p.fp].repeat += p.repeat
            else:
                kids[p.fp] = p
        return CallNode(n.event, list(kids.values()), n.repeat, n.fp)

    roots: dict = {}
    for r in tree.roots:
        p = go(r)
        if p.fp in roots:
            roots[p.fp].repeat += p.repeat
        else:
            roots[p.fp] = p
    return CallTree(list(roots.values()))


# ---------------------------------------------------------- runnability


@dataclass
class EngineContext:
    """Two-stage context: stage 1 per stateful module kind
    (KV-cache layout, metadata builder), stage 2 regenerated per point."""

    stage1: dict = field(default_factory=lambda: {
        "attention": {"kv_cache_layout": "paged[block=16]", "metadata_builder": "attn_metadata"},
        "fused_moe": {"kv_cache_layout": None, "metadata_builder": "moe_routing"}})


def generate_inputs(entry: RunnableEntry, point: dict) -> list:
    """MODEL_CONFIG dims fixed, NUM_TOKS / NUM_REQS dims set to
    the point, MIX dims recomputed by taint.reevaluate, BOT dims unchanged."""
    subs = {T.NT: int(point["num_toks"]), T.NR: int(point["num_reqs"])}
    out = []
    for arg in entry.arg_template:
        shape = []
        for size, t in arg:
            if t in T.WORKLOAD:
                shape.append(subs[t])
            elif T.is_mix(t):
                shape.append(T.reevaluate(t, subs)[0])
            else:
                shape.append(int(size))
        out.append(tuple(shape))
    return out


def emulate_context(entry: RunnableEntry, engine: EngineContext, point: dict) -> dict:
    """stage-2 metadata for a stateful entry at one point."""
    if not entry.context_required or entry.name not in engine.stage1:
        raise ContextUnavailable(f"{entry.name}: not a stateful module")
    phase = point.get("phase", "decode")
    n_req = int(point["num_reqs"])
    if phase == "prefill":
        toks = int(point["num_toks"])
        base, extra = divmod(toks, n_req)
        seq = [base + (1 if i < extra else 0) for i in range(n_req)]
        ctx = {"phase": "prefill", "seq_lens": seq, "batch_size": n_req}
    else:
        kv = int(point.get("kv_len", 0))
        ctx = {"phase": "decode", "seq_lens": [kv + 1] * n_req, "batch_size": n_req,
               "context_lens": [kv] * n_req}
    ctx["slot_mapping"] = list(range(sum(ctx["seq_lens"])))[:n_req]
    return dict(engine.stage1[entry.name], **ctx)


def is_runnable(node: CallNode, ctx: Optional[EngineContext] = None) -> bool:
    """an operation of a standalone kind whose shape function
    runs at the small verification point; a stateful module with context."""
    e = node.event
    if e.category == "operation":
        if e.name not in STANDALONE:
            return False
        return all(s >= 1 for shape in generate_inputs(_entry_of(node, 1), VERIFY_POINT)
                   for s in shape)
    if e.category == "module" and e.name in STATEFUL_MODULES:
        return ctx is not None
    return False


def _entry_of(node: CallNode, repeat: int, kernels: Optional[list] = None) -> RunnableEntry:
    e = node.event
    module = e.category == "module"
    attrs = tuple(sorted(e.attrs.items())) if module else ()
    return RunnableEntry(
        "module" if module else "operator", e.name,
        tuple(tuple((int(s), t) for s, t in a) for a in e.input_dims),
        tuple((int(v), t) for v, t in e.scalars), module, attrs,
        tuple(kernels if kernels is not None else e.kernel_symbols), repeat,
        "attention" if e.name == "attention" else "num_toks",
        e.attrs.get("sliding_window") if module else None)


def resolve(tree: CallTree, engine: Optional[EngineContext] = None) -> list:
    """the runnable set, one entry per operator-level op or
    absorbing module, in trace order, repeat = product of repeats on the path.
    Every kernel is covered exactly once (coverage conservation)."""
    engine = engine or EngineContext()
    out: list = []

    def go(n: CallNode, path: list, rep: int):
        e = n.event
        rep *= n.repeat
        if e.category == "operation":
            kern = [c for c in n.children if c.event.category == "kernel"]
            if not kern:
                return                              # view / collective: no launch
            if is_runnable(n):
                out.append(_entry_of(n, rep))
                return
            for depth in range(len(path) - 1, -1, -1):
                anc, anc_rep = path[depth]
                if is_runnable(anc, engine):
                    if not any(x[0] is anc for x in covered):
                        covered.append((anc, anc_rep))
                        out.append(_entry_of(anc, anc_rep, anc.kernels()))
                    return
            raise Unresolvable(f"operation {e.name} (event {e.id}) has no runnable ancestor")
        for c in n.children:
            go(c, path + [(n, rep)], rep)

    covered: list = []
    for r in tree.roots:
        go(r, [], 1)
    return out


def runnable_set(cfg, backend, tp: int = 1, trace: Optional[TaintedTrace] = None) -> list:
    """tracer -> build_tree -> prune -> resolve for one (model, backend, tp)."""
    tr = trace or run_trace(cfg, backend, tp=tp)
    return resolve(prune(build_tree(tr.events)))


def covered_kernel_count(entries: Sequence[RunnableEntry]) -> int:
    return sum(len(e.kernel_symbols) * e.repeat_count for e in entries)
