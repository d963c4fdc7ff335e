"""Time the shared-grid fit (dooly_fit_grid) at C5 scale against the CSR fit.

    python tools/fit_grid_bench.py --sigs 500000 --points 4096 [--csr]

C5 (BASELINE.json configs[4]): affine signatures over 4096 token counts in
[1, 32768]; attention signatures over a 16x16x16 (prefill_toks, batch,
kv_tokens) grid.  y is generated on the device per signature."""

from __future__ import annotations

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2605_07985_b200.sim import fit_grid, fit_tables  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--sigs", type=int, default=500_000)
    ap.add_argument("--points", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--csr", action="store_true")
    ap.add_argument("--kinds", default="0,1")
    ap.add_argument("--vs-warp", action="store_true",
                    help="check the table bit-identical to DOOLY_FIT_GRID_KERNEL=warp")
    ap.add_argument("--vs-unfactored", action="store_true",
                    help="max coefficient difference against DOOLY_FIT_GRID_FACTOR=0")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    for kind in [int(k) for k in a.kinds.split(",")]:
        x, y = bench.gen_grid_fit_data(kind, a.sigs, a.points, dev, seed=kind)
        fr = fit_grid(kind, x, y)
        ms = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fr = fit_grid(kind, x, y, fr)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        line = {"kind": kind, "sigs": a.sigs, "points": a.points, "grid_ms": min(ms),
                "grid_fits_per_s": a.sigs / min(ms) * 1e3,
                "y_gb_per_s": a.sigs * a.points * 8 / min(ms) / 1e6,
                "all_ok": int((fr.status != 0).sum().item()) == 0}
        if a.vs_warp:
            env = os.environ.get("DOOLY_FIT_GRID_KERNEL")
            os.environ["DOOLY_FIT_GRID_KERNEL"] = "warp"
            fw = fit_grid(kind, x, y)
            torch.cuda.synchronize()
            if env is None:
                del os.environ["DOOLY_FIT_GRID_KERNEL"]
            else:
                os.environ["DOOLY_FIT_GRID_KERNEL"] = env
            line["bit_identical_vs_warp"] = bool(torch.equal(fw.table, fr.table) and torch.equal(
                fw.fit_err.view(torch.int64), fr.fit_err.view(torch.int64)) and torch.equal(
                fw.status, fr.status))
            del fw
        if a.vs_unfactored:
            os.environ["DOOLY_FIT_GRID_FACTOR"] = "0"
            fu = fit_grid(kind, x, y)
            torch.cuda.synchronize()
            del os.environ["DOOLY_FIT_GRID_FACTOR"]
            nc = 2 if kind == 0 else 10
            ga, gu = fr.table.view(torch.float64), fu.table.view(torch.float64)
            d = (ga[:, :nc] - gu[:, :nc]).abs().amax(1) / gu[:, :nc].abs().amax(1)
            line["max_coef_rel_diff_vs_unfactored"] = float(d.max().item())
            line["fit_err_max_rel_diff"] = float(((fr.fit_err - fu.fit_err).abs() /
                                                  fu.fit_err.abs()).max().item())
            del fu
        if a.csr:
            xr = x.repeat(1, a.sigs)
            off = torch.arange(a.sigs + 1, dtype=torch.int64, device=dev) * a.points
            fc = fit_tables(kind, xr, y.reshape(-1), off)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fc = fit_tables(kind, xr, y.reshape(-1), off, fc)
            e1.record()
            torch.cuda.synchronize()
            line["csr_ms"] = e0.elapsed_time(e1)
            ga = fr.table.view(torch.float64)
            gc = fc.table.view(torch.float64)
            nc = 2 if kind == 0 else 10
            d = (ga[:, :nc] - gc[:, :nc]).abs().amax(1) / gc[:, :nc].abs().amax(1)
            line["max_coef_rel_diff_vs_csr"] = float(d.max().item())
            del xr, fc
        print(json.dumps(line), flush=True)
        del x, y, fr
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
