"""Generate golden fixtures by importing the reference package (run in the build
container only; /root/reference does not exist on the GPU box).

    python tests/golden/make_golden.py

Writes:
  paper_2605_07985_b200/data/{corpus12,fixtures}.json  — the reference's shipped
      manifests re-serialised (model-config data consumed by configs C1/C2)
  tests/golden/reference_modelir.json — outputs of the reference's modelir on
      those manifests: attention census (test_modelir.py:109-124), geometry
      keys, attention kernel symbols and multipliers, DEFAULT_GRID, shrink()
  tests/golden/workload_*.json — reference sample_workload() request lists
"""

from __future__ import annotations

import importlib
import json
import sys
from pathlib import Path

REF_SRC = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent


def _load_reference():
    # The reference is an implicit namespace package named `dooly`.
    sys.path.insert(0, str(REF_SRC))
    try:
        return importlib.import_module("dooly.modelir")
    finally:
        sys.path.pop(0)


WORKLOADS = {
    # C1 trace: Poisson 0.5 req/s, 1000 requests, Table-3 lengths, seed 1
    "c1": ({"mode": "stream", "rate": 0.5, "num_requests": 1000,
            "prompt_len": {"median": 950, "mean": 1232},
            "output_len": {"median": 388, "mean": 397}, "max_len": 8192}, 1),
    "dur": ({"mode": "stream", "rate": 2.0, "duration_s": 120.0,
             "prompt_len": {"median": 300, "mean": 420},
             "output_len": {"median": 50, "mean": 50}, "max_len": 4096}, 7),
    "prefill_heavy": ({"mode": "single_batch", "kind": "prefill_heavy",
                       "total_tokens": 16384, "batch_size": 4}, 0),
    "decode_heavy": ({"mode": "single_batch", "kind": "decode_heavy",
                      "cached_context": 2048, "batch_size": 8}, 0),
}


def main() -> None:
    mir = _load_reference()
    data_dir = REPO / "paper_2605_07985_b200" / "data"
    data_dir.mkdir(parents=True, exist_ok=True)
    out: dict = {}
    for name in ("corpus12", "fixtures"):
        man = mir.load_manifest(mir.builtin_manifest_path(name))
        (data_dir / f"{name}.json").write_text(
            json.dumps(mir.manifest_to_json(man), indent=1, sort_keys=True) + "\n")
        census: dict = {}
        geoms = {}
        syms = {}
        for cfg in man.models:
            keys = sorted({mir.geometry_key(cfg, i) for i in range(cfg.num_layers)})
            geoms[cfg.name] = [mir.geometry_key(cfg, i) for i in range(cfg.num_layers)]
            for k in keys:
                census[k] = census.get(k, 0) + len(man.backends)
            for b in man.backends:
                for w in sorted({w for w in cfg.layer_attention}, key=lambda v: (v is not None, v)):
                    for phase in ("prefill", "decode"):
                        s = b.attention_kernels(cfg.num_q_heads, cfg.num_kv_heads,
                                                cfg.head_dim, w, phase)
                        syms[f"{cfg.name}|{b.name}|{w}|{phase}"] = {
                            "symbols": list(s), "multiplier": b.multiplier(s)}
        out[name] = {"census": census, "geometry": geoms, "attention": syms,
                     "canonical": mir.dumps_canonical(mir.manifest_to_json(man))}
    g = mir.DEFAULT_GRID
    out["default_grid"] = {"token_counts": list(g.token_counts),
                           "request_counts": list(g.request_counts),
                           "kv_lens": list(g.kv_lens), "prefill_chunk": g.prefill_chunk,
                           "max_batch": g.max_batch}
    out["shrink"] = {str(f): {"token_counts": list(g.shrink(f).token_counts),
                              "request_counts": list(g.shrink(f).request_counts),
                              "kv_lens": list(g.shrink(f).kv_lens)} for f in (2, 3, 4)}
    (HERE / "reference_modelir.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")

    for name, (raw, seed) in WORKLOADS.items():
        spec = mir.workload_from_json(raw)
        reqs = mir.sample_workload(spec, seed)
        rows = [[r.arrival_s, r.prompt_tokens, r.output_tokens, r.cached_tokens] for r in reqs]
        (HERE / f"workload_{name}.json").write_text(
            json.dumps({"spec": raw, "seed": seed, "requests": rows}) + "\n")
    print("golden fixtures written")


if __name__ == "__main__":
    main()
