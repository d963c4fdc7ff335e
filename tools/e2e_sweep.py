"""Sweep predict_host pipelining (streams x chunk) and measure raw pinned copy
bandwidth, to see how close the e2e path is to the host link.

    python tools/e2e_sweep.py
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_07985_b200 import _lib  # noqa: E402
from paper_2605_07985_b200.sim import pack_attn, predict_host  # noqa: E402
from tools.predict_sweep import gen_queries, synth_table  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    nb = 1 << 30
    h = torch.empty(nb, dtype=torch.uint8).pin_memory()
    d = torch.empty(nb, dtype=torch.uint8, device=dev)
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                     ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        print(json.dumps({"copy": name, "gb_per_s": 5 * nb / (time.perf_counter() - t) / 1e9}))
    s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        with torch.cuda.stream(s_h2d):
            d[: nb // 2].copy_(h[: nb // 2], non_blocking=True)
        with torch.cuda.stream(s_d2h):
            h[nb // 2:].copy_(d[nb // 2:], non_blocking=True)
    torch.cuda.synchronize()
    print(json.dumps({"copy": "duplex (half each way)", "gb_per_s": 5 * nb / (time.perf_counter() - t) / 1e9}))
    del h, d
    n = 100_000_000
    for kind, name in ((0, "affine"), (1, "attn96")):
        table = synth_table(kind, 500_000, dev)
        sig, x = gen_queries(kind, table, n, dev, 1)
        pk = kind
        if kind == 1:
            table, pk = pack_attn(table), _lib.KIND_ATTN_PACKED
        hs, hx = sig.cpu().pin_memory(), x.cpu().pin_memory()
        ho = torch.empty(n, dtype=torch.float64).pin_memory()
        for ns in (2, 3, 4):
            for ch in (1 << 22, 1 << 23, 1 << 24):
                predict_host(pk, table, hs, hx, ho, chunk=ch, n_streams=ns)
                t = time.perf_counter()
                for _ in range(3):
                    predict_host(pk, table, hs, hx, ho, chunk=ch, n_streams=ns)
                dt = (time.perf_counter() - t) / 3
                print(json.dumps({"kind": name, "streams": ns, "chunk": ch,
                                  "g_per_s": n / dt / 1e9,
                                  "link_gb_per_s": n * (4 + 4 * x.shape[0] + 8) / dt / 1e9}),
                      flush=True)


if __name__ == "__main__":
    main()
