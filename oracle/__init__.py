"""CPU oracle — TEST INFRASTRUCTURE ONLY.

A plain restatement (Python + hashlib + numpy, one thread unless stated) of the
reference's hot-path algorithm.  The reference ships this path only as a
specification (`/root/reference/SPEC.md:413-649`; `profiler`/`sim` modules are
absent from `pkg/src`), so every function here cites the SPEC line it follows
and the SURVEY App. A pin that resolves a spec gap.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import this package, and only as the checker or
the timed CPU baseline — never as part of the product path.

Pinning status:
  * signature canonicalisation / SHA-256 / dedup — pinned by the SHA-256 KAT
     and the Table-2 attention census N/R 42/27 (SPEC.md:708,
    test_modelir.py:109-124) via tests/golden/reference_modelir.json;
  * analytical latency + comm model — pinned by the SPEC golden values
    (A9 SPEC.md:714);
  * workload trace — pinned by request lists generated with the reference's
    own sample_workload (tests/golden/workload_*.json);
  * fit / predict / iter_latency / run — PARITY UNPINNED by reference tests
    (none exist); only the SPEC examples (exact-linear fit_error, clamp floor,
    InsufficientData, scheduler chunk KATs, single-request TTFT, mape) pin them.
"""
