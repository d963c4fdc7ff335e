"""Extended seeded sweep of the serving loop's window-edge fuzz (the cases of
tests/test_gpu_fuzz.py::test_sim_run_window_edges beyond the 120 the suite
runs), every shard bit-exact against the oracle event loop:

    python tools/sim_fuzz_stress.py [--start 120] [--count 2000]
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
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    t0 = time.time()
    for case in range(a.start, a.start + a.count):
        F.test_sim_run_window_edges(case, dev)
    print(f"{a.count} window-edge configurations bit-exact ({time.time() - t0:.0f} s)")


if __name__ == "__main__":
    main()
