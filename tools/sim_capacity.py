"""Find the near-capacity request rate of one C4 replica (Llama-3-70B-like,
tp=4, flashattention-like, a100-like HW) with the device event loop: sweep the
per-replica Poisson rate and report TTFT percentiles and iterations.

    python tools/sim_capacity.py [--requests 20000] [--shards 148]
"""

from __future__ import annotations

import argparse
import json
import math
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=20000)
    ap.add_argument("--shards", type=int, default=148)
    ap.add_argument("--rates", default="0.5,1,2,3,4,5,6,8,10")
    args = ap.parse_args()

    import torch

    from paper_2605_07985_b200 import modelir
    from paper_2605_07985_b200.profiler import profile_corpus
    from paper_2605_07985_b200.sim import (SchedConfig, ShardedTrace, build_calltree, collect,
                                           fit, make_sched, run_sharded)

    dev = torch.device("cuda", 0)
    man = modelir.load_manifest(modelir.builtin_manifest_path("llama70b"))
    model, backend, hw = man.models[0], man.backends[1], man.hardware
    db, _ = profile_corpus(modelir.CorpusManifest((model,), (backend,), hw, man.tp_degree,
                                                  man.grid), device=dev)
    regs = fit(db, dev)
    ct = build_calltree(model, backend, regs, hw, man.tp_degree)
    cfg = make_sched(model, hw, man.tp_degree, SchedConfig(chunk=8192, max_batch=256), ct)
    n = args.requests
    rng = np.random.default_rng(1)
    sig_p = math.sqrt(2 * math.log(1232 / 950))
    sig_o = math.sqrt(2 * math.log(397 / 388))
    pr = np.clip(np.rint(rng.lognormal(math.log(950), sig_p, n)), 1, 8192 - 512).astype(np.uint32)
    ou = np.clip(np.rint(rng.lognormal(math.log(388), sig_o, n)), 1, 512).astype(np.uint32)
    gaps = rng.exponential(1.0, size=n)
    for rate in [float(r) for r in args.rates.split(",")]:
        arr = np.cumsum(gaps / (rate * args.shards))
        trace = ShardedTrace.from_arrays(arr, pr, ou, np.zeros(n, np.uint32), args.shards, dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = run_sharded(trace, ct, cfg, regs)
        e1.record()
        torch.cuda.synchronize()
        m = collect(trace, res)
        print(json.dumps({"rate_per_replica": rate, "ms": e0.elapsed_time(e1),
                          "iterations": int(res.n_iter.sum().item()),
                          "ttft": m.percentiles["ttft"], "tpot": m.percentiles["tpot"],
                          "makespan_s": float(res.clock.max().item())}))


if __name__ == "__main__":
    main()
