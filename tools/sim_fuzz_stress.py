"""Extended seeded sweeps of the GPU fuzz tests beyond the cases the suite runs:
the serving loop's window-edge fuzz (every shard bit-exact against the oracle
event loop), and with --kernels also the random predict tables (values and
flag planes bit-exact) and random CSR fits (coefficients within 1e-9):

    python tools/sim_fuzz_stress.py [--start 120] [--count 2000] [--kernels 500]
"""

from __future__ import annotations

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main() -> None:
    import torch

    import test_gpu_fuzz as F

    ap = argparse.ArgumentParser()
    ap.add_argument("--start", type=int, default=120)
    ap.add_argument("--count", type=int, default=2000)
    ap.add_argument("--kernels", type=int, default=0,
                    help="also this many extra random predict-table and CSR-fit cases")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    t0 = time.time()
    for case in range(a.start, a.start + a.count):
        F.test_sim_run_window_edges(case, dev)
    print(f"{a.count} window-edge configurations bit-exact ({time.time() - t0:.0f} s)", flush=True)
    if a.kernels:
        t0 = time.time()
        for case in range(1000, 1000 + a.kernels):
            F.test_predict_random_tables(case, dev)
        print(f"{a.kernels} random predict tables bit-exact ({time.time() - t0:.0f} s)", flush=True)
        t0 = time.time()
        for case in range(1000, 1000 + a.kernels):
            F.test_fit_random_csr(case, dev)
        print(f"{a.kernels} random CSR fits within the contract ({time.time() - t0:.0f} s)")


if __name__ == "__main__":
    main()
