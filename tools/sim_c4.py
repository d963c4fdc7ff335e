"""Run the C4 serving simulation once (Llama-3-70B-like tp=4,
1M-request Poisson trace, S fixed replicas) — for ncu captures of
sim_run_kernel and for layout / build-knob experiments (SIM_WARPS_N, SIM_UNROLL,
DOOLY_SIM_PV).

    python tools/sim_c4.py [--shards 64] [--requests 1000000] [--reps 3]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--shards", type=int, default=64)
    ap.add_argument("--requests", type=int, default=1_000_000)
    ap.add_argument("--rate", type=float, default=4.0)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    from paper_2605_07985_b200 import modelir
    from paper_2605_07985_b200.profiler import profile_corpus
    from paper_2605_07985_b200.sim import (SchedConfig, ShardedTrace, build_calltree, fit,
                                           make_sched, run_sharded)

    dev = torch.device("cuda", 0)
    man = modelir.load_manifest(modelir.builtin_manifest_path("llama70b"))
    model, backend, hw = man.models[0], man.backends[1], man.hardware
    db, _ = profile_corpus(modelir.CorpusManifest((model,), (backend,), hw, man.tp_degree,
                                                  man.grid), device=dev)
    regs = fit(db, dev)
    ct = build_calltree(model, backend, regs, hw, man.tp_degree)
    cfg = make_sched(model, hw, man.tp_degree, SchedConfig(chunk=8192, max_batch=256), ct)
    arr, pr, ou, ca = bench.c4_trace(a.requests, a.shards, a.rate)
    trace = ShardedTrace.from_arrays(arr, pr, ou, ca, a.shards, dev)
    res = run_sharded(trace, ct, cfg, regs)
    ms = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = run_sharded(trace, ct, cfg, regs, out=res)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    n_it = res.n_iter.cpu()
    print(json.dumps({"shards": a.shards, "requests": a.requests, "ms": min(ms), "n_ops": ct.n_ops,
                      "iterations": int(n_it.sum()), "max_iterations": int(n_it.max()),
                      "us_per_iteration_longest": min(ms) * 1e3 / int(n_it.max()),
                      "ttft_checksum": float(torch.nan_to_num(res.ttft).sum())}))


if __name__ == "__main__":
    main()
