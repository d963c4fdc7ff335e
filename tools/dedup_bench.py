"""Time the SHA-256 record hash (K1a) and the full dedup (K1) at C5 size.

    python tools/dedup_bench.py [--records 4000000] [--reps 10]
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
from paper_2605_07985_b200.profiler import (DedupWorkspace, DeviceRecords, dedup_packed,  # noqa: E402
                                            hash_records)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--records", type=int, default=4_000_000)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    packed, _ = bench.synth_records(a.records, seed=11)
    recs = DeviceRecords.from_packed(packed, dev)
    ws = DedupWorkspace(dev)
    ref = hash_records(recs).clone()
    res = dedup_packed(recs, workspace=ws)
    torch.cuda.synchronize()

    def timed(fn):
        fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.reps

    sha_ms = timed(lambda: hash_records(recs))
    dd_ms = timed(lambda: dedup_packed(recs, workspace=ws))
    from paper_2605_07985_b200.profiler import dedup_digests
    dig = res.digests
    ins = {}
    for mode in ("thread", "group"):
        if mode == "group":
            os.environ["DOOLY_DEDUP_INSERT"] = "group"
        else:
            os.environ.pop("DOOLY_DEDUP_INSERT", None)
        r = dedup_digests(dig, workspace=ws)
        ins[mode] = {"ms": timed(lambda: dedup_digests(dig, workspace=ws)),
                     "same": bool(torch.equal(r.first, res.first) and torch.equal(r.uid, res.uid))}
    os.environ.pop("DOOLY_DEDUP_INSERT", None)
    # the same digests from the default kernel variant (DOOLY_SHA_VARIANT unset)
    var = os.environ.pop("DOOLY_SHA_VARIANT", None)
    base = hash_records(recs).clone()
    if var is not None:
        os.environ["DOOLY_SHA_VARIANT"] = var
    same = bool(torch.equal(ref, base))
    print(json.dumps({"records": a.records, "sha_ms": sha_ms, "dedup_ms": dd_ms,
                      "records_per_s": a.records / dd_ms * 1e3, "unique": int(res.n_unique),
                      "digests_unchanged": same, "dedup_digests_by_insert": ins}))


if __name__ == "__main__":
    main()
