"""Time K3 predict per table layout at C5 scale (synthetic rows, random gathers).

    python tools/predict_sweep.py --sigs 1000000 --queries 200000000 --reps 5

Rows are synthesised directly on the device (random coefficients, random
training boxes, inv = 1/hi) — only the gather/evaluate/stream cost is measured.
Prints one JSON line per layout with ms per launch and queries/s."""

from __future__ import annotations

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_07985_b200 import _lib  # noqa: E402
from paper_2605_07985_b200.sim import pack_attn, predict_batch  # noqa: E402


def synth_table(kind: int, n_sig: int, dev, seed: int = 0) -> torch.Tensor:
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    P = _lib.PLANES[kind]
    n_c = 2 if kind == _lib.KIND_AFFINE else 10
    hi = torch.randint(64, 32768, (n_sig, P), generator=g, device=dev, dtype=torch.int64)
    lo = (hi.double() * torch.rand((n_sig, P), generator=g, device=dev, dtype=torch.float64) * 0.1).long()
    c = torch.rand((n_sig, n_c), generator=g, device=dev, dtype=torch.float64) * 1e-5 + 1e-6
    inv = 1.0 / hi.double()
    box = torch.cat([lo, hi], dim=1).to(torch.int32).contiguous().view(torch.float64)  # (n, P)
    rows = torch.cat([c, inv, box], dim=1)
    return rows.contiguous().view(torch.uint8).reshape(n_sig, -1)


def gen_queries(kind: int, table: torch.Tensor, n_q: int, dev, seed: int):
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    n_sig = table.shape[0]
    words = table.view(torch.int32).reshape(n_sig, -1)
    lo_hi = ([(words[:, 6], words[:, 7])] if kind == _lib.KIND_AFFINE
             else [(words[:, 26 + k], words[:, 29 + k]) for k in range(3)])
    sig = torch.randint(0, n_sig, (n_q,), generator=g, device=dev, dtype=torch.int64)
    x = torch.empty((len(lo_hi), n_q), dtype=torch.int32, device=dev)
    for k, (lo, hi) in enumerate(lo_hi):
        l, h = lo[sig].long(), hi[sig].long()
        u = torch.rand(n_q, generator=g, device=dev, dtype=torch.float64)
        x[k] = torch.minimum(l + (u * (h - l + 1)).long(), h).int()
    return sig.int(), x


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--sigs", type=int, default=1_000_000)
    ap.add_argument("--queries", type=int, default=200_000_000)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--layouts", default="affine,attn,attn96")
    ap.add_argument("--vs-ldg", action="store_true",
                    help="attn96: compare out/flags bit for bit with DOOLY_PREDICT_ATTN unset (the default kernel)")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    base = {"affine": _lib.KIND_AFFINE, "attn": _lib.KIND_ATTN, "attn96": _lib.KIND_ATTN}
    for name in a.layouts.split(","):
        kind = base[name]
        table = synth_table(kind, a.sigs, dev)
        sig, x = gen_queries(kind, table, a.queries, dev, 1)
        if name == "attn96":
            table, kind = pack_attn(table), _lib.KIND_ATTN_PACKED
        out = torch.empty(a.queries, dtype=torch.float64, device=dev)
        flags = torch.empty((2, (a.queries + 31) // 32), dtype=torch.int32, device=dev)
        err = torch.full((1,), torch.iinfo(torch.int64).max, dtype=torch.int64, device=dev)
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        for _ in range(2):
            predict_batch(kind, table, sig, x, out, flags, err)
        ms = []
        for _ in range(a.reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            predict_batch(kind, table, sig, x, out, flags, err)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        ms.sort()
        med = ms[len(ms) // 2]
        ok = int(err.item()) == torch.iinfo(torch.int64).max
        line = {"layout": name, "sigs": a.sigs, "queries": a.queries, "ms": med,
                "mode": os.environ.get("DOOLY_PREDICT_ATTN", "default"),
                "tma_frac": os.environ.get("DOOLY_PREDICT_TMA_FRAC"),
                "gq_per_s": a.queries / med / 1e6, "all_known": ok,
                "checksum": float(out.sum().item())}
        if a.vs_ldg and name == "attn96":
            env = os.environ.pop("DOOLY_PREDICT_ATTN", None)
            out2, flags2 = torch.empty_like(out), torch.empty_like(flags)
            err2 = torch.full_like(err, torch.iinfo(torch.int64).max)
            predict_batch(kind, table, sig, x, out2, flags2, err2)
            torch.cuda.synchronize()
            if env is not None:
                os.environ["DOOLY_PREDICT_ATTN"] = env
            line["bit_identical_vs_ldg"] = bool(torch.equal(out.view(torch.int64),
                                                            out2.view(torch.int64))
                                                and torch.equal(flags, flags2)
                                                and torch.equal(err, err2))
            del out2, flags2, err2
        print(json.dumps(line), flush=True)
        del table, sig, x, out, flags, err, flush
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
