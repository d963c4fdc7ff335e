"""C1 (BASELINE.json configs[0], the reference's CPU-runnable case) end to end:
Llama-3-8B-like / flashattention-like on a100-like, tp 1; dedup + sweep + fit,
then TTFT/TPOT for the reference's own 1k-request trace
(tests/golden/workload_c1.json).  Times the GPU path (profile_and_fit + the
device serving loop) and the CPU oracle (oracle.profiler dedup, host sweep,
oracle.sim fit and event loop) on the same inputs; prints one JSON line.

    python tools/c1_pipeline.py [--reps 3]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_07985_b200 import modelir  # noqa: E402
from paper_2605_07985_b200.profiler import profile_and_fit  # noqa: E402
from paper_2605_07985_b200.sim import (SchedConfig, ShardedTrace, build_calltree, collect,  # noqa: E402
                                       make_sched, run_sharded)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    corpus = modelir.load_manifest(modelir.builtin_manifest_path("corpus12"))
    model = corpus.model("llama-3-8b-like")
    backend = corpus.backend("flashattention-like")
    man = modelir.CorpusManifest((model,), (backend,), corpus.hardware, 1, corpus.grid)
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "workload_c1.json")))
    reqs = [modelir.Request(*r) for r in g["requests"]]
    arr = np.array([r.arrival_s for r in reqs])
    pr = np.array([r.prompt_tokens for r in reqs], dtype=np.uint32)
    ou = np.array([r.output_tokens for r in reqs], dtype=np.uint32)
    ca = np.array([r.cached_tokens for r in reqs], dtype=np.uint32)
    sched = SchedConfig(chunk=8192, max_batch=256)

    def gpu_once():
        t0 = time.perf_counter()
        _, regs, _ = profile_and_fit(man, device=dev)
        t1 = time.perf_counter()
        ct = build_calltree(model, backend, regs, corpus.hardware, 1)
        cfg = make_sched(model, corpus.hardware, 1, sched, ct)
        trace = ShardedTrace.from_arrays(arr, pr, ou, ca, 1, dev)
        res = run_sharded(trace, ct, cfg, regs)
        met = collect(trace, res)
        t2 = time.perf_counter()
        return t1 - t0, t2 - t1, met, int(res.n_iter.sum().item())

    gpu_once()
    runs = [gpu_once() for _ in range(a.reps)]
    fit_s = min(r[0] for r in runs)
    sim_s = min(r[1] for r in runs)
    met, n_it = runs[-1][2], runs[-1][3]
    # device-only time of the serving loop (CUDA events)
    _, regs, _ = profile_and_fit(man, device=dev)
    ct = build_calltree(model, backend, regs, corpus.hardware, 1)
    cfg = make_sched(model, corpus.hardware, 1, sched, ct)
    trace = ShardedTrace.from_arrays(arr, pr, ou, ca, 1, dev)
    res = run_sharded(trace, ct, cfg, regs)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = run_sharded(trace, ct, cfg, regs, out=res)
    e1.record()
    torch.cuda.synchronize()
    dev_ms = e0.elapsed_time(e1)
    # CPU oracle on the same inputs: dedup + host sweep + oracle fit + event loop
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from helpers import rows_to_table
    from oracle import profiler as oprof
    from oracle import sim as osim
    from paper_2605_07985_b200.profiler import _kind_of, sweep
    from paper_2605_07985_b200.records import synthesize_entries

    t0 = time.perf_counter()
    ents = synthesize_entries(model, backend, 1)
    seen = set()
    for e in ents:                                   # first occurrences (dedup)
        d = oprof.signature_hash(oprof.canonicalize(e.to_json()))
        if d in seen:
            continue
        seen.add(d)
        x, y = sweep(e, corpus.grid, model, corpus.hardware, backend)
        kind = _kind_of(e)
        osim.fit(kind, np.asarray(x, dtype=np.uint32).reshape(osim.PLANES[kind], -1),
                 np.asarray(y, dtype=np.float64), np.array([0, len(y)], dtype=np.int64))
    cpu_fit_s = time.perf_counter() - t0
    tabs = {k: rows_to_table(k, regs.tables[k].rows()) for k in regs.tables}
    ops = []
    for i in range(ct.n_ops):
        feat, row = ct.oplist.feat[i], ct.oplist.row[i]
        op = {"feat": feat, "repeat": ct.oplist.repeat[i], "window_slot": ct.oplist.window_slot[i],
              "bytes_per_tok": ct.oplist.bytes_per_tok[i]}
        if feat != osim.FEAT_COMM:
            t = tabs[1 if feat == osim.FEAT_ATTN else 0]
            op.update(coef=list(t["coef"][row]), inv=list(t["inv"][row]))
        ops.append(op)
    t0 = time.perf_counter()
    ref = osim.run_shard(arr.tolist(), pr.tolist(), ou.tolist(), ca.tolist(), ops, 8192, 256,
                         cfg.kv_bytes_per_token, cfg.kv_capacity_bytes, ct.window, 1)
    cpu_sim_s = time.perf_counter() - t0
    same = bool(np.array_equal(met.ttft.view(np.uint64), np.array(ref["ttft"]).view(np.uint64)))
    line = {"workload": "C1: llama-3-8b-like / flashattention-like, 1k-request reference trace",
            "cpu_oracle_fit_s": cpu_fit_s, "cpu_oracle_sim_s": cpu_sim_s,
            "ttft_bit_identical_to_oracle": same,
            "iterations": n_it, "gpu_fit_s": fit_s, "gpu_sim_wall_s": sim_s,
            "gpu_sim_device_ms": dev_ms, "gpu_us_per_iteration": dev_ms * 1e3 / n_it,
            "ttft_p50_s": float(np.nanpercentile(met.ttft, 50)),
            "tpot_p50_s": float(np.nanpercentile(met.tpot, 50))}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
