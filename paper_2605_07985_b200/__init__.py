"""B200-native Dooly latency-database hot path.

Drop-in for the reference's (specified but unshipped) `dooly.profiler` /
`dooly.sim` hot path: signature canonicalisation + dedup, per-signature
latency-regression fitting, batched latency prediction and the simulator's
per-iteration gather-evaluate-reduce into TTFT/TPOT — all on hand-written
sm_100a kernels behind the C-ABI in include/dooly_b200.h.
"""

from . import errors, modelir, records  # noqa: F401  (host-only, importable without a GPU)

__all__ = ["errors", "modelir", "records", "profiler", "sim", "dist"]


def __getattr__(name):  # lazy: profiler/sim import torch
    if name in ("profiler", "sim", "dist"):
        import importlib

        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
