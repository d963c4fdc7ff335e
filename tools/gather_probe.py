"""Measure the random-row gather ceiling that bounds K3 predict (and the L2
read cap) on this B200.

    python tools/gather_probe.py            # builds tools/_build/gather_probe.so first if needed

For each row size used by the predict tables (32 B affine, 96 B packed
attention, 128 B attention) and table sizes matching the C5 bench, prints
rows/s and gathered bytes/s.  Compare with bench.py's per-kind kernel_ms."""

from __future__ import annotations

import ctypes as C
import json
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_build", "gather_probe.so")


def build() -> None:
    os.makedirs(os.path.dirname(SO), exist_ok=True)
    src = os.path.join(HERE, "gather_probe.cu")
    if os.path.exists(SO) and os.path.getmtime(SO) >= os.path.getmtime(src):
        return
    subprocess.check_call(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a",
                           "-shared", "-Xcompiler", "-fPIC", "--cudart", "static", "-o", SO, src])


def main() -> None:
    build()
    lib = C.CDLL(SO)
    lib.probe_gather.argtypes = [C.c_void_p, C.c_uint32, C.c_int, C.c_int64, C.c_void_p, C.c_int,
                                 C.c_void_p]
    lib.probe_tma_gather.argtypes = [C.c_void_p, C.c_uint32, C.c_int, C.c_int, C.c_int64,
                                     C.c_void_p, C.c_int, C.c_void_p]
    lib.probe_tma_gather4.argtypes = lib.probe_tma_gather.argtypes
    lib.probe_l2_stream.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_int, C.c_void_p]
    dev = torch.device("cuda", 0)
    only = set(sys.argv[1:])
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    sink = torch.zeros(2, dtype=torch.int64, device=dev)   # [checksum hits, timeouts]
    st = torch.cuda.current_stream().cuda_stream

    def timed(fn, reps=5):
        fn()
        ms = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        return sorted(ms)[len(ms) // 2]

    if "gather4" in only:
        gather4(lib, dev, n_sm, sink, st, timed)
        return
    if "coop" in only:
        lib.probe_coop_gather.argtypes = lib.probe_gather.argtypes
        n_q, rows = 500_000_000, 500_000
        for stride in (96, 128):
            table = torch.rand((rows * stride) // 8, dtype=torch.float64, device=dev)
            for per_sm in (4, 8):
                ms = timed(lambda: lib.probe_coop_gather(table.data_ptr(), rows, stride, n_q,
                                                         sink.data_ptr(), n_sm * per_sm, st))
                print(json.dumps({"probe": "coop_gather", "row_bytes": 96, "stride": stride,
                                  "rows": rows, "ctas_per_sm": per_sm, "ms": ms,
                                  "g_rows_per_s": n_q / ms / 1e6}), flush=True)
            if stride == 96:
                lib.probe_coop_smem.argtypes = [C.c_void_p, C.c_uint32, C.c_int64, C.c_void_p,
                                                C.c_int, C.c_void_p]
                for per_sm in (4, 6, 8):
                    ms = timed(lambda: lib.probe_coop_smem(table.data_ptr(), rows, n_q,
                                                           sink.data_ptr(), n_sm * per_sm, st))
                    print(json.dumps({"probe": "coop_smem", "row_bytes": 96, "rows": rows,
                                      "ctas_per_sm": per_sm, "ms": ms,
                                      "g_rows_per_s": n_q / ms / 1e6}), flush=True)
            if stride == 96:
                lib.probe_coop_shfl.argtypes = lib.probe_coop_smem.argtypes
                for per_sm in (4, 6, 8):
                    ms = timed(lambda: lib.probe_coop_shfl(table.data_ptr(), rows, n_q,
                                                           sink.data_ptr(), n_sm * per_sm, st))
                    print(json.dumps({"probe": "coop_shfl", "row_bytes": 96, "rows": rows,
                                      "ctas_per_sm": per_sm, "ms": ms,
                                      "g_rows_per_s": n_q / ms / 1e6}), flush=True)
            for sectors in (3,):
                if stride != 96:
                    continue
                ms = timed(lambda: lib.probe_gather(table.data_ptr(), rows, sectors, n_q,
                                                    sink.data_ptr(), n_sm * 8, st))
                print(json.dumps({"probe": "gather", "row_bytes": 96, "rows": rows, "ms": ms,
                                  "g_rows_per_s": n_q / ms / 1e6}), flush=True)
            del table
        return
    if "hybrid" in only:
        hybrid(lib, dev, n_sm, sink, st, timed)
        return
    if "predmem" in only:
        predict_mem(lib, dev, n_sm, timed)
        return
    for mb in (16, 48):
        buf = torch.rand((mb << 20) // 8, dtype=torch.float64, device=dev)
        reps = 20
        for blocks in (n_sm * 4, n_sm * 8):
            ms = timed(lambda: lib.probe_l2_stream(buf.data_ptr(), buf.numel() * 8, reps,
                                                   sink.data_ptr(), blocks, st))
            print(json.dumps({"probe": "l2_stream", "buffer_mb": mb, "blocks": blocks,
                              "gb_per_s": buf.numel() * 8 * reps / ms / 1e6}), flush=True)
        del buf
    n_q = 500_000_000
    for sectors, rows in ((1, 500_000), (3, 500_000), (4, 500_000), (3, 1_000_000),
                          (4, 1_000_000), (3, 250_000)):
        table = torch.rand((rows * sectors * 32) // 8, dtype=torch.float64, device=dev)
        for blocks in (n_sm * 8,):
            ms = timed(lambda: lib.probe_gather(table.data_ptr(), rows, sectors, n_q,
                                                sink.data_ptr(), blocks, st))
            print(json.dumps({"probe": "gather", "row_bytes": 32 * sectors, "rows": rows,
                              "table_mb": rows * sectors * 32 / 2**20, "ms": ms,
                              "g_rows_per_s": n_q / ms / 1e6,
                              "gb_per_s": n_q * 32 * sectors / ms / 1e6}), flush=True)
        del table
    for rb, rows in ((96, 500_000), (32, 500_000), (128, 500_000)):
        table = torch.rand((rows * rb) // 8, dtype=torch.float64, device=dev)
        for depth in (2, 4, 8):
            for per_sm in (2, 4, 8):
                smem = 4 * depth * (8 + 32 * rb)
                if smem * per_sm > 220 * 1024:
                    continue
                rc = lib.probe_tma_gather(table.data_ptr(), rows, rb, depth, n_q, sink.data_ptr(),
                                          n_sm * per_sm, st)
                if rc != 0:
                    continue
                ms = timed(lambda: lib.probe_tma_gather(table.data_ptr(), rows, rb, depth, n_q,
                                                        sink.data_ptr(), n_sm * per_sm, st))
                print(json.dumps({"probe": "tma_gather", "row_bytes": rb, "rows": rows,
                                  "depth": depth, "ctas_per_sm": per_sm, "ms": ms,
                                  "g_rows_per_s": n_q / ms / 1e6,
                                  "gb_per_s": n_q * rb / ms / 1e6}), flush=True)
        del table


def predict_mem(lib, dev, n_sm, timed):
    """predict_vec_kernel's access pattern with the evaluation removed, on the C5
    bench shapes (0.5M rows, uniform random signatures), next to the product
    kernel timed by tools/predict_sweep.py on the same sizes."""
    lib.probe_predict_mem.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int64,
                                      C.c_void_p, C.c_int, C.c_void_p]
    st = torch.cuda.current_stream().cuda_stream
    n_q, rows = 200_000_000, 500_000
    for sectors, planes, occ in ((1, 1, 3), (3, 3, 2)):
        table = torch.rand((rows * sectors * 32) // 8, dtype=torch.float64, device=dev)
        sig = torch.randint(0, rows, (n_q,), dtype=torch.int32, device=dev)
        x = torch.randint(0, 1 << 15, (planes, n_q), dtype=torch.int32, device=dev)
        out = torch.empty(n_q, dtype=torch.float64, device=dev)
        for per_sm in (occ, occ + 1, occ * 2):
            ms = timed(lambda: lib.probe_predict_mem(table.data_ptr(), sig.data_ptr(), x.data_ptr(),
                                                     sectors, n_q, out.data_ptr(), n_sm * per_sm,
                                                     st))
            print(json.dumps({"probe": "predict_mem", "row_bytes": 32 * sectors, "planes": planes,
                              "rows": rows, "ctas_per_sm": per_sm, "ms": ms,
                              "g_q_per_s": n_q / ms / 1e6}), flush=True)
        del table, sig, x, out


def gather4(lib, dev, n_sm, sink, st, timed):
    n_q = 500_000_000
    for rb, rows in ((96, 500_000), (32, 500_000), (128, 500_000)):
        table = torch.rand((rows * rb) // 8, dtype=torch.float64, device=dev)
        for depth in (2, 4):
            for per_sm in (2, 4, 8):
                smem = 4 * depth * 32 * rb + 128
                if smem * per_sm > 220 * 1024:
                    continue
                rc = lib.probe_tma_gather4(table.data_ptr(), rows, rb, depth, 1 << 20,
                                           sink.data_ptr(), n_sm * per_sm, st)
                torch.cuda.synchronize()
                if rc != 0 or int(sink[1].item()):
                    print(json.dumps({"probe": "tma_gather4", "row_bytes": rb, "depth": depth,
                                      "rc": rc, "timeouts": int(sink[1].item())}), flush=True)
                    sink.zero_()
                    continue
                ms = timed(lambda: lib.probe_tma_gather4(table.data_ptr(), rows, rb, depth, n_q,
                                                         sink.data_ptr(), n_sm * per_sm, st))
                print(json.dumps({"probe": "tma_gather4", "row_bytes": rb, "rows": rows,
                                  "depth": depth, "ctas_per_sm": per_sm, "ms": ms,
                                  "g_rows_per_s": n_q / ms / 1e6, "timeouts": int(sink[1].item()),
                                  "gb_per_s": n_q * rb / ms / 1e6}), flush=True)
        del table


def hybrid(lib, dev, n_sm, sink, st, timed):
    """TMA gather4 warps and LDG.256 warps in the same CTAs on disjoint query
    ranges: if the two paths used separate request interfaces, the total would
    exceed either alone (96-B rows, 0.5M-row table)."""
    lib.probe_hybrid_gather.argtypes = [C.c_void_p, C.c_uint32, C.c_int, C.c_int64, C.c_int64,
                                        C.c_void_p, C.c_int, C.c_void_p]
    n_q, rows = 500_000_000, 500_000
    table = torch.rand((rows * 96) // 8, dtype=torch.float64, device=dev)
    for cfg, per_sm in ((0, 2), (0, 3), (1, 2), (2, 2), (2, 3), (3, 2)):
        for frac in (0.0, 0.3, 0.45, 0.6, 1.0):
            n_tma = int(n_q * frac) // 32 * 32
            rc = lib.probe_hybrid_gather(table.data_ptr(), rows, cfg, min(n_tma, 1 << 20),
                                         min(n_q, 1 << 21), sink.data_ptr(), n_sm * per_sm, st)
            torch.cuda.synchronize()
            if rc != 0 or int(sink[1].item()):
                print(json.dumps({"probe": "hybrid", "cfg": cfg, "rc": rc,
                                  "timeouts": int(sink[1].item())}), flush=True)
                sink.zero_()
                continue
            ms = timed(lambda: lib.probe_hybrid_gather(table.data_ptr(), rows, cfg, n_tma, n_q,
                                                       sink.data_ptr(), n_sm * per_sm, st))
            print(json.dumps({"probe": "hybrid", "cfg": cfg, "ctas_per_sm": per_sm,
                              "tma_frac": frac, "ms": ms, "g_rows_per_s": n_q / ms / 1e6,
                              "timeouts": int(sink[1].item())}), flush=True)
    del table


if __name__ == "__main__":
    sys.exit(main())
