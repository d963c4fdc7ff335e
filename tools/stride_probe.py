"""Packed attention rows in 96-B vs 128-B slots under the paired predict kernel
(experiment: a 128-B slot keeps a row's three sectors in one line, so the
paired loads' two same-row sectors always coalesce).  Run once with the
default library (96-B slots) and once with a PAIR_STRIDE_D=16 build
(DOOLY_LIB_PATH=tools/_build/libdooly_stride128.so --slot 128; a PAIR_SPLIT build
with --slot split); the
checksums must agree.

    python tools/stride_probe.py --slot 96|128|split [--sigs 500000] [--queries 500000000]
"""

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
from paper_2605_07985_b200.sim import pack_attn  # noqa: E402
from predict_sweep import gen_queries, synth_table  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--slot", default="96", choices=["96", "128", "split"])
    ap.add_argument("--sigs", type=int, default=500_000)
    ap.add_argument("--queries", type=int, default=500_000_000)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    table = synth_table(_lib.KIND_ATTN, a.sigs, dev)
    sig, x = gen_queries(_lib.KIND_ATTN, table, a.queries, dev, 1)
    t96 = pack_attn(table)
    del table
    if a.slot == "128":
        t = torch.zeros((a.sigs + 1, 128), dtype=torch.uint8, device=dev)
        t[:, :96] = t96
    elif a.slot == "split":
        # header padded to 128 B, then sectors 0-1 of every row (64-B slots), then sector 2
        n = a.sigs
        t = torch.zeros(128 + 96 * n, dtype=torch.uint8, device=dev)
        t[:96] = t96[0]
        t[128:128 + 64 * n] = t96[1:, :64].reshape(-1)
        t[128 + 64 * n:] = t96[1:, 64:].reshape(-1)
    else:
        t = t96
    lib = _lib.load_library()
    ctx = _lib.ctx_for(dev)
    out = torch.empty(a.queries, dtype=torch.float64, device=dev)
    flags = torch.empty((2, (a.queries + 31) // 32), dtype=torch.int32, device=dev)
    err = torch.full((1,), torch.iinfo(torch.int64).max, dtype=torch.int64, device=dev)
    st = _lib.stream_ptr(dev)

    def run():
        _lib.check(lib.dooly_predict(ctx, _lib.KIND_ATTN_PACKED, t.data_ptr(), a.sigs,
                                     sig.data_ptr(), x.data_ptr(), a.queries, out.data_ptr(),
                                     flags.data_ptr(), err.data_ptr(), st), ctx)

    run()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ms = []
    for _ in range(a.reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    ms.sort()
    med = ms[len(ms) // 2]
    print(json.dumps({"slot": a.slot, "ms": med, "gq_per_s": a.queries / med / 1e6,
                      "checksum_out": float(out.sum().item()),
                      "checksum_flags": int(flags.to(torch.int64).sum().item()),
                      "err": int(err.item())}))


if __name__ == "__main__":
    main()
