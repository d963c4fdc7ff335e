"""The C5 grid fits of both kinds back to back on one stream vs on two
concurrent streams (affine is HBM-bound, attention y-latency-bound).
Prints one JSON line."""

from __future__ import annotations

import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2605_07985_b200.sim import fit_grid  # noqa: E402


def main() -> None:
    dev = torch.device("cuda", 0)
    n = 500_000
    data = {k: bench.gen_grid_fit_data(k, n, 4096, dev, seed=k) for k in (0, 1)}
    packed = torch.empty((n + 1, 96), dtype=torch.uint8, device=dev)
    outs = {k: fit_grid(k, *data[k], packed=packed if k == 1 else None) for k in (0, 1)}
    side = torch.cuda.Stream(dev)
    main_s = torch.cuda.current_stream(dev)

    def serial():
        for k in (0, 1):
            fit_grid(k, *data[k], outs[k], packed=packed if k == 1 else None)

    def concurrent():
        side.wait_stream(main_s)
        with torch.cuda.stream(side):
            fit_grid(1, *data[1], outs[1], packed=packed)
        fit_grid(0, *data[0], outs[0])
        main_s.wait_stream(side)

    res = {}
    for name, fn in (("serial", serial), ("concurrent", concurrent)):
        fn()
        ms = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        ms.sort()
        res[name + "_ms"] = ms[2]
    res["all_ok"] = all(int((outs[k].status != 0).sum().item()) == 0 for k in (0, 1))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
