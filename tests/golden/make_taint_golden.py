"""Golden vectors for the taint lattice from the reference's own taint.py
(run in the build container only; /root/reference does not exist on the GPU box).

    python tests/golden/make_taint_golden.py

Writes tests/golden/reference_taint.json: seeded random combine / split /
reevaluate cases with the reference's result (text form) or exception name,
checked against paper_2605_07985_b200/taint.py by tests/test_tracer_opset.py.
"""

from __future__ import annotations

import importlib
import json
import random
import sys
from pathlib import Path

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "reference_taint.json"


def main() -> None:
    sys.path.insert(0, str(REF_SRC))
    try:
        t = importlib.import_module("dooly.taint")
    finally:
        sys.path.pop(0)
    rng = random.Random(2605)
    labels = [t.MODEL_CONFIG, t.NUM_TOKS, t.NUM_REQS]
    values = [1, 2, 4, 8, 40, 64, 128, 269, 538, 4096]

    def rand_taint():
        r = rng.random()
        if r < 0.15:
            return t.BOT
        if r < 0.55:
            return t.Base(rng.choice(labels))
        n = rng.randint(2, 4)
        try:
            return t.mix_from([(rng.choice(values), rng.choice(labels)) for _ in range(n)])
        except Exception:
            return t.Base(rng.choice(labels))

    def run(fn):
        try:
            res = fn()
        except Exception as exc:      # noqa: BLE001 — the class name is the golden
            return {"error": type(exc).__name__}
        if isinstance(res, tuple):
            return {"result": [x if isinstance(x, int) else t.taint_to_str(x) for x in res]}
        return {"result": t.taint_to_str(res)}

    cases = []
    for _ in range(400):
        a, b = rand_taint(), rand_taint()
        va, vb = rng.choice(values), rng.choice(values)
        cases.append({"op": "combine", "args": [t.taint_to_str(a), t.taint_to_str(b), va, vb],
                      **run(lambda: t.combine(a, b, va, vb))})
    for _ in range(200):
        a = rand_taint()
        k = rng.choice(values)
        cases.append({"op": "split", "args": [t.taint_to_str(a), k], **run(lambda: t.split(a, k))})
    for _ in range(200):
        a = rand_taint()
        subs = {lab.code: rng.choice(values) for lab in (t.NUM_TOKS, t.NUM_REQS)
                if rng.random() < 0.7}
        cases.append({"op": "reevaluate", "args": [t.taint_to_str(a), subs],
                      **run(lambda: t.reevaluate(a, {t.TaintLabel(c): v for c, v in subs.items()}))})
    OUT.write_text(json.dumps({"source": "reference pkg/src/dooly/taint.py", "cases": cases},
                              indent=0) + "\n")
    print(f"wrote {len(cases)} cases to {OUT}")


if __name__ == "__main__":
    main()
