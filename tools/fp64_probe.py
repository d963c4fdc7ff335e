"""FP64 vector (DFMA) vs FP64 tensor (mma.sync .f64) throughput on this B200.

    python tools/fp64_probe.py
"""

from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_build", "fp64_probe.so")


def build() -> None:
    os.makedirs(os.path.dirname(SO), exist_ok=True)
    src = os.path.join(HERE, "fp64_probe.cu")
    if os.path.exists(SO) and os.path.getmtime(SO) >= os.path.getmtime(src):
        return
    subprocess.check_call(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                           "-Xcompiler", "-fPIC", "--cudart", "static", "-o", SO, src])


def main() -> None:
    build()
    lib = C.CDLL(SO)
    lib.probe_fp64.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
    lib.probe_fp64.restype = C.c_double
    dev = torch.device("cuda", 0)
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    names = {0: "dfma", 1: "dmma_m8n8k4", 2: "dmma_m16n8k4", 3: "dmma_m16n8k16",
             4: "dmma+dfma (half each)"}
    for which in (0, 1, 4):
        for per_sm, threads in ((4, 256), (8, 256)):
            iters = 20000
            lib.probe_fp64(which, n_sm * per_sm, threads, 100, out.data_ptr(), st)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fmas = lib.probe_fp64(which, n_sm * per_sm, threads, iters, out.data_ptr(), st)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b)
            print(json.dumps({"op": names[which], "ctas_per_sm": per_sm, "threads": threads,
                              "ms": ms, "tflops": 2 * fmas / ms / 1e9}), flush=True)


if __name__ == "__main__":
    main()
