"""Affine and packed-attention predict batches back to back on one stream vs
concurrently on two streams (C5 shapes: 0.5M rows per kind, 0.5e9 queries per
kind by default).  Prints one JSON line."""

from __future__ import annotations

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from paper_2605_07985_b200 import _lib  # noqa: E402
from paper_2605_07985_b200.sim import pack_attn, predict_batch  # noqa: E402
from predict_sweep import gen_queries, synth_table  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--sigs", type=int, default=500_000)
    ap.add_argument("--queries", type=int, default=500_000_000)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    jobs = []
    for kind in (_lib.KIND_AFFINE, _lib.KIND_ATTN):
        t = synth_table(kind, a.sigs, dev)
        sig, x = gen_queries(kind, t, a.queries, dev, 1 + kind)
        if kind == _lib.KIND_ATTN:
            t, kind = pack_attn(t), _lib.KIND_ATTN_PACKED
        out = torch.empty(a.queries, dtype=torch.float64, device=dev)
        flags = torch.empty((2, (a.queries + 31) // 32), dtype=torch.int32, device=dev)
        err = torch.full((1,), torch.iinfo(torch.int64).max, dtype=torch.int64, device=dev)
        jobs.append((kind, t, sig, x, out, flags, err))
    side = torch.cuda.Stream(dev)
    main_s = torch.cuda.current_stream(dev)

    def serial():
        for j in jobs:
            predict_batch(*j)

    def concurrent():
        side.wait_stream(main_s)
        predict_batch(*jobs[0])
        with torch.cuda.stream(side):
            predict_batch(*jobs[1])
        main_s.wait_stream(side)

    res = {}
    for name, fn in (("serial", serial), ("concurrent", concurrent)):
        fn()
        ms = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        ms.sort()
        res[name + "_ms"] = ms[len(ms) // 2]
    res["queries"] = 2 * a.queries
    print(json.dumps(res))


if __name__ == "__main__":
    main()
