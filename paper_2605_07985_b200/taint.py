"""Provenance taints of integer shape values (reference
``taint.py``), restated for the record producer (tracer.py / opset.py).

A taint is held in its canonical TEXT form, the same grammar the trace file and
the runnable-set JSON carry (taint.py:215-239):

    "BOT" | "MC" | "NT" | "NR" | "MIX{v1:L1,v2:L2,...}"   (values ascending, >= 2)

so a taint is an immutable, hashable, directly serialisable value and the
records' ``arg_template`` needs no conversion.  The lattice operations
(Table 1 of the paper) work on the component map {value: label} of a MIX.
"""

from __future__ import annotations

from typing import Iterable, Mapping, Optional

from .errors import MixValueConflict, UnknownComponent

BOT = "BOT"
MC, NT, NR = "MC", "NT", "NR"          # MODEL_CONFIG, NUM_TOKS, NUM_REQS
LABELS = (MC, NT, NR)
WORKLOAD = frozenset((NT, NR))


def is_mix(t: str) -> bool:
    return t.startswith("MIX{")


def components(t: str) -> dict:
    """{value: label} of a MIX (a base label has none)."""
    if not is_mix(t):
        return {}
    out = {}
    for part in t[4:-1].split(","):
        v, _, lab = part.partition(":")
        out[int(v)] = lab
    return out


def mix(pairs: Iterable) -> str:
    """Normalised taint of (value, label) pairs: one distinct entry collapses to
    its base label (D2 ascending order); a value with two labels
    raises MixValueConflict (D1)."""
    merged: dict = {}
    for v, lab in pairs:
        v = int(v)
        if v < 1:
            raise ValueError(f"mix component values must be positive, got {v}")
        if lab not in LABELS:
            raise ValueError(f"bad taint label {lab!r}")
        if merged.setdefault(v, lab) != lab:
            raise MixValueConflict(f"value {v} assigned both {merged[v]} and {lab}")
    if not merged:
        raise ValueError("a mix needs at least one component")
    if len(merged) == 1:
        return next(iter(merged.values()))
    return "MIX{" + ",".join(f"{v}:{merged[v]}" for v in sorted(merged)) + "}"


def combine(t1: str, t2: str, v1: Optional[int] = None, v2: Optional[int] = None) -> str:
    """t1 (x) t2 (Table 1): absorption, preservation, conflict,
    extend, merge.  v1/v2 are the operands' concrete values, needed whenever a
    new component is recorded."""
    if t1 == BOT:
        return t2
    if t2 == BOT or t1 == t2:
        return t1
    m1, m2 = is_mix(t1), is_mix(t2)
    if not m1 and not m2:                       # two different base labels: conflict
        if v1 is None or v2 is None:
            raise ValueError("the conflict rule needs both concrete values")
        return mix([(v1, t1), (v2, t2)])
    if m1 and m2:                               # merge
        return mix(list(components(t1).items()) + list(components(t2).items()))
    if not m1:                                  # extend is symmetric
        t1, t2, v1, v2 = t2, t1, v2, v1
    if v2 is None:
        raise ValueError("the extend rule needs the base operand's value")
    return mix(list(components(t1).items()) + [(v2, t2)])


def split(t: str, known_value: int) -> tuple:
    """(component, residual) of a MIX by one factor value."""
    comps = components(t)
    if known_value not in comps:
        raise UnknownComponent(f"value {known_value} not in {t}")
    rest = [(v, lab) for v, lab in comps.items() if v != known_value]
    return comps[known_value], mix(rest)


def reevaluate(t: str, subs: Mapping) -> tuple:
    """(new size, taint) of a MIX with workload components substituted
    (D3): MODEL_CONFIG values are kept, the size is the product,
    size-1 workload components are dropped only when one component remains."""
    if not is_mix(t):
        raise ValueError("reevaluate needs a MIX taint")
    if any(lab not in WORKLOAD for lab in subs):
        raise ValueError("substitutions may only cover NT / NR")
    new, size = {}, 1
    for v, lab in components(t).items():
        nv = int(subs.get(lab, v)) if lab in WORKLOAD else v
        size *= nv
        if new.setdefault(nv, lab) != lab:
            raise MixValueConflict(f"reevaluate collided value {nv} between {new[nv]} and {lab}")
    keep = [(v, lab) for v, lab in new.items() if not (v == 1 and lab in WORKLOAD)]
    return size, mix(keep if len(keep) == 1 else new.items())


def parse(text: str) -> str:
    """Validate a serialised taint; returns it unchanged if canonical."""
    if text == BOT or text in LABELS:
        return text
    if is_mix(text) and text.endswith("}"):
        pairs = []
        for part in text[4:-1].split(","):
            v, sep, lab = part.partition(":")
            if not sep or not v.isdigit():
                raise ValueError(f"unparseable taint {text!r}")
            pairs.append((int(v), lab))
        vals = [v for v, _ in pairs]
        if len(pairs) < 2 or vals != sorted(set(vals)) or mix(pairs) != text:
            raise ValueError(f"non-canonical mix serialisation {text!r}")
        return text
    raise ValueError(f"unparseable taint {text!r}")


class Registry:
    """Global value -> taint map with collision tracking.
    A value registered with two different taints moves to ``collisions`` and
    looks up as unknown (None) from then on."""

    def __init__(self) -> None:
        self._entries: dict = {}
        self._collisions: set = set()

    def register(self, value: int, taint: str) -> bool:
        """True when this registration detects (or re-hits) a collision."""
        if value < 1:
            raise ValueError(f"registry values must be positive, got {value}")
        if taint == BOT:
            raise ValueError("BOT is never registered (D4)")
        if value in self._collisions:
            return True
        prior = self._entries.setdefault(value, taint)
        if prior == taint:
            return False
        del self._entries[value]
        self._collisions.add(value)
        return True

    def lookup(self, value: int) -> Optional[str]:
        return self._entries.get(value)

    @property
    def entries(self) -> dict:
        return dict(self._entries)

    @property
    def collisions(self) -> frozenset:
        return frozenset(self._collisions)

    def snapshot(self) -> dict:
        return {"entries": {str(v): self._entries[v] for v in sorted(self._entries)},
                "collisions": sorted(self._collisions)}

    @classmethod
    def from_snapshot(cls, data: Mapping) -> "Registry":
        reg = cls()
        reg._entries = {int(v): parse(t) for v, t in data.get("entries", {}).items()}
        reg._collisions = {int(v) for v in data.get("collisions", [])}
        return reg
