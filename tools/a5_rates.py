"""A5 errors of the product pipeline vs reference_run on C1 at
rates around C1's capacity:  python tools/a5_rates.py  (needs a GPU)."""
import sys, torch
sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import test_gpu_anchors as A
from paper_2605_07985_b200 import modelir
man = modelir.load_manifest(modelir.builtin_manifest_path("corpus12"))
dev = torch.device("cuda", 0)
for rate in [3.0, 5.0, 6.0, 7.0, 8.0]:
    err = A._a5(man, "llama-3-8b-like", rate, dev)
    print("RATE", rate, "ttft max %.4f tpot max %.4f same %s" % (max(err["ttft"].values()), max(err["tpot"].values()), err["same_compositions"]), err["ttft"], err["tpot"], flush=True)
