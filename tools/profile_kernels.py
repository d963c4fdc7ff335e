"""Launch every libdooly_b200 hot kernel on C5-shaped inputs, for ncu.

    ncu --set full --import-source on -k regex:'fit_grid_stage|fit_stage|fit_moments_attn|fit_mape_attn|predict_vec|sha256_rec|dedup_insert|sim_run' \
        -c 16 -o gpurun_out/prof python tools/profile_kernels.py

Sizes are scaled down from bench.py (same shapes per unit) so a full ncu
replay finishes in minutes; per-unit numbers (bytes/query, bytes/point) are
what profiles/ compares against the roofline.
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--sigs", type=int, default=40_000)
    ap.add_argument("--points", type=int, default=4096)
    ap.add_argument("--queries", type=int, default=100_000_000)
    ap.add_argument("--records", type=int, default=1_000_000)
    ap.add_argument("--repeat", type=int, default=2)
    ap.add_argument("--only", default="fit,fitgrid,predict,dedup,sim")
    args = ap.parse_args()

    import torch

    import bench
    from paper_2605_07985_b200.profiler import DedupWorkspace, DeviceRecords, dedup_packed
    from paper_2605_07985_b200.sim import fit_grid, fit_tables, pack_attn, predict_batch

    dev = torch.device("cuda", 0)
    only = set(args.only.split(","))
    tables = {}
    for kind in (0, 1):
        x, y, off = bench.gen_fit_data(kind, args.sigs, args.points, dev, seed=kind)
        off_d = torch.from_numpy(off).to(dev)
        fr = None
        for _ in range(args.repeat if "fit" in only else 1):
            fr = fit_tables(kind, x, y, off_d, fr)
        tables[kind] = fr.table
        del x, y
    torch.cuda.synchronize()
    if "fitgrid" in only:
        for kind in (0, 1):
            xg, yg = bench.gen_grid_fit_data(kind, args.sigs, args.points, dev, seed=kind)
            fg = None
            for _ in range(args.repeat):
                fg = fit_grid(kind, xg, yg, fg)
            del xg, yg
    if "predict" in only:
        for kind in (0, 1):
            # table sized like C5 (0.5M rows) by tiling the fitted rows
            reps = max(1, 500_000 // tables[kind].shape[0])
            table = tables[kind].repeat(reps, 1)
            sig, xq = bench.gen_queries(kind, table, args.queries // 2, dev, seed=7)
            pk = kind
            if kind == 1:   # the serving form bench.py times (96-B packed rows)
                table, pk = pack_attn(table), 2
            out = torch.empty(sig.numel(), dtype=torch.float64, device=dev)
            for _ in range(args.repeat):
                predict_batch(pk, table, sig, xq, out)
            del sig, xq, out
    if "dedup" in only:
        packed, _ = bench.synth_records(args.records, seed=1)
        recs = DeviceRecords.from_packed(packed, dev)
        ws = DedupWorkspace(dev)
        for _ in range(args.repeat):
            dedup_packed(recs, workspace=ws)
    torch.cuda.synchronize()
    print("profile driver done")


if __name__ == "__main__":
    main()
