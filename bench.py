"""Benchmark of the Dooly latency-database hot path on B200 (bench contract of
the task README; metric from BASELINE.json: latency predictions/s and
signature fits/s at 1/2/4/8 B200, % of HBM roofline).

Headline step (config C5 of BASELINE.json, per GPU — weak scaling):
    one batch of 1e9 latency queries against the 1M-signature regressor tables
    (0.5e9 affine-kind queries on 0.5M affine rows + 0.5e9 attention-kind
    queries on 0.5M 10-column rows), uniform signature, features uniform inside
    the signature's training box; inputs resident in HBM (~20 GB per step,
    >> 126 MB L2, so no L2 flush is needed).
Also measured in the same run and reported as extra keys:
    fits     — the C5 fit of those 1M signatures x 4096 points on the shared
               sweep grid, the attention serving table (96-B rows) written by
               the fit epilogue; at N > 1 the regressor rows reach every rank
               through the fused peer-memory all-gather (NCCL otherwise);
               roofline per kind (affine HBM, attention FP64 + HBM);
    fits_csr — the same points through the per-signature (CSR) fit;
    dedup    — SHA-256 + first-occurrence dedup of 4M packed records (~1M
               unique); at N > 1 fused digest all-gather (2 ranks) or
               owner-routed all-to-all (4+ ranks);
    sim      — config C4 as BASELINE.md defines it: Llama-3-70B-like (tp=4),
               1M-request Poisson trace over S = 64 fixed replicas, device event
               loop; sim.sim_eval (dooly_sim_eval over the run's own logged
               iterations: 28 B/iteration HBM and FP64 fractions); s1184 the
               same trace over 1184 replicas;
    e2e      — the predict batch through the public host API (pinned host
               buffers, latencies and flag bit-planes back, copies inside the
               timed region);
    cpu_baseline — the CPU oracle on the box's host cores for EVERY metric
               (predictions here; fits / dedup / sim inside their keys): the
               per-item oracle on one thread and the numpy oracle over all
               cores, 1 warm-up + median of 5 on bounded samples, with the
               host's core count, affinity and BLAS threads.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
torchrun launches one rank per GPU (RANK/LOCAL_RANK/WORLD_SIZE from env).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

AFFINE, ATTN = 0, 1
BYTES_PER_QUERY = {AFFINE: 4 + 4 + 8 + 0.25, ATTN: 4 + 12 + 8 + 0.25}   # sig + x + out + 2 flag bits
BYTES_PER_POINT = {AFFINE: 4 + 8, ATTN: 12 + 8}                          # x u32 planes + y f64
BYTES_PER_GRID_POINT = 8                     # shared grid: y f64 per point (x counted once per kind)
FP64_PER_ATTN_POINT = 27          # per-point passes (13 pass 1 + 14 pass 2)
FP64_PER_ATTN_POINT_GROUPED = 16  # grouped passes: 7.25 + 8.75 (4-point groups share f1, f2)
FP64_PER_ATTN_POINT_PERIODIC = 14  # + kv period dividing 128 points: per-position pass 1, 5.25 + 8.75
SHA_ALU_PER_BLOCK = 48 * 18 + 16 * 10          # SASS count, sha256_compress
ALU_PEAK_TINSTR = 64 * 148 * 1.965e9 / 1e12       # ALU pipe lanes/clk/SM x SMs x clock
FP64_PEAK_TINSTR = 64 * 148 * 1.965e9 / 1e12   # 18.6 T DFMA-class instr/s
FALLBACK_HBM_GBS = 6650.0


# ----------------------------------------------------------------- inputs


def synth_records(n: int, seed: int = 0):
    """C5 record stream: n operator records, ~n/4 distinct signatures."""
    from paper_2605_07985_b200.records import pack_uniform

    rng = np.random.default_rng(seed)
    op_names = ["bmm", "conv1d", "linear", "matmul"]
    symbols = sorted(["cutlass_gemm_bf16_128x128", "cutlass_gemm_bf16_256x128",
                      "gemv_f16_split_k", "im2col_f16", "reduce_rows_f32", "splitk_reduce",
                      "xmma_gemm_f16_tn", "xmma_gemm_f16_nt"], key=str.encode)
    side = max(1, int(round(math.sqrt(n / 16))))        # op x K x N ~ n/4 combos
    op = rng.integers(0, 4, size=n)
    k = 64 * rng.integers(1, side + 1, size=n)
    nn = 64 * rng.integers(1, side + 1, size=n)
    pos = np.tile(np.array([1, 3, 4], dtype=np.uint32), (n, 1))
    val = np.stack([k, k, nn], axis=1).astype(np.uint64)
    sym = np.stack([2 * op, 2 * op + 1], axis=1).astype(np.uint32)
    packed = pack_uniform(op_names, op.astype(np.uint32), pos, val, symbols, sym,
                          np.zeros((0, 32), np.uint8), np.full(n, 0xFFFFFFFF, np.uint32),
                          rng.integers(1, 80, size=n).astype(np.uint32))
    return packed, 3


def gen_fit_data(kind: int, n_sig: int, n_pts: int, dev, seed: int):
    """Per-signature training points inside a random box; y = positive
    polynomial x (1 + N(0, 1e-3)).  Built on the device in chunks."""
    import torch

    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    P = 1 if kind == AFFINE else 3
    x = torch.empty((P, n_sig * n_pts), dtype=torch.int32, device=dev)
    y = torch.empty(n_sig * n_pts, dtype=torch.float64, device=dev)
    chunk = max(1, (1 << 26) // n_pts)
    for s0 in range(0, n_sig, chunk):
        s1 = min(n_sig, s0 + chunk)
        m = s1 - s0
        sl = slice(s0 * n_pts, s1 * n_pts)
        if kind == AFFINE:
            lo = torch.randint(1, 64, (m, 1), generator=g, device=dev)
            hi = lo + torch.randint(64, 32768, (m, 1), generator=g, device=dev)
            u = torch.rand((m, n_pts), generator=g, device=dev, dtype=torch.float64)
            xv = torch.minimum(lo + (u * (hi - lo + 1)).long(), hi)
            a = torch.empty((m, 1), dtype=torch.float64, device=dev).uniform_(5e-6, 2e-5, generator=g)
            b = torch.empty((m, 1), dtype=torch.float64, device=dev).uniform_(1e-9, 1e-7, generator=g)
            yv = a + b * xv.double()
            x[0, sl] = xv.reshape(-1).int()
        else:
            hi = torch.stack([torch.randint(256, 32768, (m,), generator=g, device=dev),
                              torch.randint(8, 256, (m,), generator=g, device=dev),
                              torch.randint(4096, 1 << 22, (m,), generator=g, device=dev)], 1)
            cols = []
            for kk in range(3):
                u = torch.rand((m, n_pts), generator=g, device=dev, dtype=torch.float64)
                cols.append(torch.minimum((u * (hi[:, kk:kk + 1] + 1)).long(), hi[:, kk:kk + 1]))
            c = torch.empty((m, 3), dtype=torch.float64, device=dev).uniform_(1e-12, 1e-9, generator=g)
            f0, f1, f2 = (cc.double() for cc in cols)
            yv = (1e-5 + c[:, 0:1] * f0 + c[:, 1:2] * f1 * 100 + c[:, 2:3] * f2
                  + 1e-15 * f0 * f0 + 1e-16 * f0 * f2)
            for kk in range(3):
                x[kk, sl] = cols[kk].reshape(-1).int()
        eps = torch.randn((m, n_pts), generator=g, device=dev, dtype=torch.float64)
        y[sl] = (yv * (1.0 + 1e-3 * eps)).abs().reshape(-1) + 1e-9
    off = np.arange(n_sig + 1, dtype=np.int64) * n_pts
    return x, y, off


def grid_points(kind: int, n_pts: int):
    """C5 sweep grid shared by every signature of a kind (BASELINE.json configs[4]):
    affine — n_pts token counts evenly spanning [1, 32768]; attention — a
    side^3 (prefill_toks, batch, kv_tokens) grid, side = n_pts^(1/3) (16 for 4096)."""
    if kind == AFFINE:
        return np.rint(np.linspace(1, 32768, n_pts)).astype(np.uint32)[None, :]
    side = max(2, round(n_pts ** (1.0 / 3.0)))
    t = np.rint(np.geomspace(1, 32768, side)).astype(np.int64)
    b = np.rint(np.geomspace(1, 256, side)).astype(np.int64)
    k = np.rint(np.linspace(0, 1 << 22, side)).astype(np.int64)
    g = np.stack(np.meshgrid(t, b, k, indexing="ij")).reshape(3, -1)
    return g.astype(np.uint32)


def gen_grid_fit_data(kind: int, n_sig: int, n_pts: int, dev, seed: int):
    """Shared-grid C5 fit input: x (P, n) int32 on device, y (n_sig, n) f64 with
    y = positive per-signature polynomial x (1 + N(0, 1e-3))."""
    import torch

    xg = grid_points(kind, n_pts)
    n = xg.shape[1]
    x = torch.from_numpy(xg.view(np.int32)).to(dev)
    xf = x.view(torch.int32).double()
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    y = torch.empty((n_sig, n), dtype=torch.float64, device=dev)
    chunk = max(1, (1 << 26) // n)
    for s0 in range(0, n_sig, chunk):
        m = min(n_sig, s0 + chunk) - s0
        if kind == AFFINE:
            a = torch.empty((m, 1), dtype=torch.float64, device=dev).uniform_(5e-6, 2e-5, generator=g)
            b = torch.empty((m, 1), dtype=torch.float64, device=dev).uniform_(1e-9, 1e-7, generator=g)
            yv = a + b * xf[0]
        else:
            c = torch.empty((m, 3), dtype=torch.float64, device=dev).uniform_(1e-12, 1e-9, generator=g)
            yv = (1e-5 + c[:, 0:1] * xf[0] + c[:, 1:2] * xf[1] * 100 + c[:, 2:3] * xf[2]
                  + 1e-15 * xf[0] * xf[0] + 1e-16 * xf[0] * xf[2])
        eps = torch.randn((m, n), generator=g, device=dev, dtype=torch.float64)
        y[s0:s0 + m] = (yv * (1.0 + 1e-3 * eps)).abs() + 1e-9
    return x, y


def gen_queries(kind: int, table, n_q: int, dev, seed: int):
    """Uniform signature; features uniform inside that signature's box."""
    import torch

    from paper_2605_07985_b200.sim import ROW_DTYPE

    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    n_sig = table.shape[0]
    words = table.view(torch.int32).reshape(n_sig, -1)
    if kind == AFFINE:
        lo_hi = [(words[:, 6], words[:, 7])]
    else:
        lo_hi = [(words[:, 26 + k], words[:, 29 + k]) for k in range(3)]
    P = len(lo_hi)
    sig = torch.empty(n_q, dtype=torch.int32, device=dev)
    x = torch.empty((P, n_q), dtype=torch.int32, device=dev)
    chunk = 1 << 26
    for q0 in range(0, n_q, chunk):
        q1 = min(n_q, q0 + chunk)
        s = torch.randint(0, n_sig, (q1 - q0,), generator=g, device=dev)
        sig[q0:q1] = s.int()
        for k, (lo, hi) in enumerate(lo_hi):
            l, h = lo[s].long(), hi[s].long()
            u = torch.rand(q1 - q0, generator=g, device=dev, dtype=torch.float64)
            x[k, q0:q1] = torch.minimum(l + (u * (h - l + 1)).long(), h).int()
    return sig, x


# ----------------------------------------------------------------- helpers


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return float(d["hbm_gbs"]), "measured"
        except (ValueError, KeyError):
            pass
    return FALLBACK_HBM_GBS, "fallback"


def link_ceiling(pinned, dev, h2d: int, d2h: int, step_s: float) -> dict:
    """Measured pinned-copy bandwidth of this GPU's host link, each direction alone
    and both at once (full duplex shares the link: ~50 GB/s each way on the
    gpurun B200s, tools/link_probe.py), and the e2e step time those allow: the
    smaller direction's bytes move at the duplex rate alongside the same amount
    of the larger direction, the rest of the larger at its solo rate."""
    import torch

    buf = pinned.view(torch.uint8)
    n = buf.numel() // 2
    a, b = buf[:n], buf[n:2 * n]
    da = torch.empty_like(a, device=dev)
    db = torch.empty_like(b, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def up():
        with torch.cuda.stream(s1):
            da.copy_(a, non_blocking=True)

    def down():
        with torch.cuda.stream(s2):
            b.copy_(db, non_blocking=True)

    def timed(fns, reps=3):
        for f in fns:
            f()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(reps):
            for f in fns:
                f()
        torch.cuda.synchronize()
        return (time.perf_counter() - t) / reps

    bw_up, bw_down = n / timed([up]), n / timed([down])
    bw_dup = n / timed([up, down])            # per direction, both active
    del da, db
    both = min(h2d, d2h)
    ideal = both / bw_dup + (h2d - both) / bw_up + (d2h - both) / bw_down
    return {"h2d_gb_s": bw_up / 1e9, "d2h_gb_s": bw_down / 1e9,
            "duplex_gb_s_each_way": bw_dup / 1e9, "ideal_step_s": ideal, "frac": ideal / step_s}


def gather_ceiling(nq: dict, k_ms: dict):
    """The binding limit of random-row predict on this hardware: the measured
    LDG.256 gather rate of bare 32-B / 96-B rows (tools/gather_probe.py,
    profiles/r1_gather_probe.jsonl).  frac = time at that rate / measured time."""
    p = ROOT / "profiles" / "r1_gather_probe.jsonl"
    if not p.exists():
        return None
    rate = {}
    for ln in p.read_text().splitlines():
        r = json.loads(ln)
        if r.get("probe") == "gather" and r.get("rows") == 500_000:
            rate[r["row_bytes"]] = r["g_rows_per_s"] * 1e9
    if 32 not in rate or 96 not in rate:
        return None
    ideal_ms = (nq[AFFINE] / rate[32] + nq[ATTN] / rate[96]) * 1e3
    out = {"rows_per_s": {"affine_32B": rate[32], "attention_96B": rate[96]},
           "ideal_ms": ideal_ms, "frac": ideal_ms / (k_ms[AFFINE] + k_ms[ATTN]),
           "source": "profiles/r1_gather_probe.jsonl (bare LDG.256 row gathers, 500k rows)"}
    # the predict kernel's own access pattern (streams + gathers + stores) with
    # the evaluation replaced by a sum: the memory-system ceiling it runs against
    mem = {}
    for ln in p.read_text().splitlines():
        r = json.loads(ln)
        if r.get("probe") == "predict_mem" and r.get("rows") == 500_000:
            mem[r["row_bytes"]] = max(mem.get(r["row_bytes"], 0.0), r["g_q_per_s"] * 1e9)
    if 32 in mem and 96 in mem:
        mem_ms = (nq[AFFINE] / mem[32] + nq[ATTN] / mem[96]) * 1e3
        out["access_pattern_ceiling"] = {
            "queries_per_s": {"affine": mem[32], "attention_96B": mem[96]},
            "ideal_ms": mem_ms, "frac": mem_ms / (k_ms[AFFINE] + k_ms[ATTN]),
            "source": "profiles/r1_gather_probe.jsonl predict_mem (tools/gather_probe.py predmem)"}
    return out


def ncu_traffic(kernel_key: str, units: dict):
    """DRAM bytes per step from the committed ncu per-unit measurement
    (profiles/ncu_summary.json x this step's units), or None."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        per = json.loads(p.read_text())[kernel_key]["dram_bytes_per_unit"]
        return sum(float(per[str(k)]) * n for k, n in units.items())
    except (ValueError, KeyError):
        return None


def l1tex_roofline(nq: dict, k_ms: dict, sm_mhz):
    """The binding resource of random-row predict: L1TEX data-pipe wavefronts
    (one per distinct line per warp-wide access, shuffles and shared accesses
    included; peak 1 per clock per SM — ncu l1tex__data_pipe_lsu_wavefronts
    against sm__cycles_elapsed).  Wavefronts per query come from the committed
    ncu measurement (profiles/ncu_summary.json "predict"), the time and clock
    from this run."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists() or not sm_mhz:
        return None
    try:
        per = json.loads(p.read_text())["predict"]["l1tex_wavefronts_per_unit"]
    except (ValueError, KeyError):
        return None
    wf = sum(float(per[str(k)]) * nq[k] for k in (AFFINE, ATTN))
    t = (k_ms[AFFINE] + k_ms[ATTN]) / 1e3
    peak = 148 * sm_mhz * 1e6
    return {"bound": "l1tex data-pipe wavefronts", "achieved": wf / t / 1e9, "peak": peak / 1e9,
            "unit": "G wavefronts/s", "frac": wf / t / peak,
            "wavefronts_per_query": {str(k): float(per[str(k)]) for k in (AFFINE, ATTN)},
            "source": "profiles/ncu_summary.json predict.l1tex_wavefronts_per_unit (ncu), "
                      "peak 1/clk/SM x 148 SMs x this run's median SM clock"}


def xbar_roofline(nq: dict, k_ms: dict, sm_mhz):
    """The unit that binds random-row predict on B200: the L1TEX -> crossbar
    request interface (one L2 request per distinct row sector per warp
    access; ncu l1tex__m_l1tex2xbar_req_cycles_active, peak 1 cycle per clock
    per SM).  Busy cycles per query from the committed ncu measurement
    (profiles/ncu_summary.json "predict"), time and clock from this run."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists() or not sm_mhz:
        return None
    try:
        per = json.loads(p.read_text())["predict"]["xbar_req_cycles_per_unit"]
    except (ValueError, KeyError):
        return None
    cyc = sum(float(per[str(k)]) * nq[k] for k in (AFFINE, ATTN))
    t = (k_ms[AFFINE] + k_ms[ATTN]) / 1e3
    peak = 148 * sm_mhz * 1e6
    return {"bound": "L1TEX->XBAR request interface (L2 requests of the row gathers)",
            "achieved": cyc / t / 1e9, "peak": peak / 1e9, "unit": "G busy-cycles/s",
            "frac": cyc / t / peak,
            "busy_cycles_per_query": {str(k): float(per[str(k)]) for k in (AFFINE, ATTN)},
            "source": "profiles/ncu_summary.json predict.xbar_req_cycles_per_unit (ncu), "
                      "peak 1/clk/SM x 148 SMs x this run's median SM clock"}


class ClockSampler:
    """SM clocks + throttle reasons sampled every ~5 ms through NVML in a
    background thread, restricted to the timed region (mark_start/mark_end)."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self.window = [None, None]
        self.max_mhz = None
        self._stop = False
        self._thread = None

    def __enter__(self):
        import threading

        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons

            def loop():
                while not self._stop:
                    try:
                        self.samples.append((time.perf_counter(),
                                             float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)),
                                             int(get_reasons(h))))
                    except pynvml.NVMLError:
                        pass
                    time.sleep(0.002)

            self._thread = threading.Thread(target=loop, daemon=True)
            self._thread.start()
        except Exception:  # NVML unavailable: report it, never fake clocks
            self._thread = None
        return self

    def mark_start(self):
        self.window[0] = time.perf_counter()

    def mark_end(self):
        self.window[1] = time.perf_counter()

    def __exit__(self, *exc):
        self._stop = True
        if self._thread is not None:
            self._thread.join(timeout=2)

    def summary(self):
        if self._thread is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        t0, t1 = self.window
        t1 = t1 or t0
        inside = [s for s in self.samples if t0 is not None and t0 <= s[0] <= t1]
        pad = 0.0
        # a short timed region can fall between two NVML reads (a read takes
        # ms on some drivers): widen the window until 3 samples, and say so
        while len(inside) < 3 and pad < 0.05 and t0 is not None:
            pad += 0.005
            inside = [s for s in self.samples if t0 - pad <= s[0] <= t1 + pad]
        src = inside if inside else self.samples[-3:]
        reasons = sorted({name for _, _, r in src for bit, name in self.REASONS.items() if r & bit})
        out = {"sm_mhz": float(np.median([s[1] for s in src])) if src else None,
               "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(inside),
               "source": "nvml, 2 ms sampling inside the timed region"}
        if pad:
            out["window_pad_ms"] = round(pad * 1e3, 1)
        return out


def barrier_sync(dist_on: bool):
    import torch
    import torch.distributed as dist

    torch.cuda.synchronize()
    if dist_on:
        dist.barrier()
        torch.cuda.synchronize()


def max_over_ranks(v: float, dist_on: bool) -> float:
    import torch
    import torch.distributed as dist

    if not dist_on:
        return v
    t = torch.tensor([v], dtype=torch.float64,
                     device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# --------------------------------------------------------------- CPU baselines
#
# SURVEY §8(d) "CPU path timing": the CPU oracle (oracle/, the restatement of
# the reference's specified algorithm) on the GPU box's host cores, for every
# metric the bench reports — predictions, fits, dedup records, sim requests —
# as two lines each: the per-item oracle (one Python thread, the "reference CPU
# path") and the vectorised numpy oracle over all host cores (fork pool).
# Method: 1 warm-up run, then the median of 5 timed runs (time.perf_counter),
# each run a bounded sample of the same workload (stated per line).


_CPU_JOBS: list = []     # set before the fork: workers inherit the job inputs


def host_info() -> dict:
    """Core count, affinity and BLAS threading of this host."""
    info = {"os_cpu_count": os.cpu_count(),
            "affinity_cores": len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity")
            else os.cpu_count(),
            "OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS"),
            "method": "1 warm-up run, median of 5 timed runs (time.perf_counter)"}
    try:
        from threadpoolctl import threadpool_info

        info["blas"] = [{"api": i.get("internal_api"), "threads": i.get("num_threads")}
                        for i in threadpool_info()]
    except Exception as exc:  # noqa: BLE001 — report, never guess
        info["blas"] = f"unavailable ({exc})"
    return info


def one_thread():
    """BLAS pinned to one thread (per-item lines, and each fork-pool worker so
    the all-core lines do not oversubscribe the host)."""
    try:
        from threadpoolctl import threadpool_limits

        return threadpool_limits(1)
    except Exception:  # noqa: BLE001
        import contextlib

        return contextlib.nullcontext()


def median_rate(fn, units: float, reps: int = 5) -> tuple:
    """1 warm-up call, then the median of ``reps`` timed calls -> (units/s, median s)."""
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    med = float(np.median(ts))
    return units / med, med


def _cpu_all_cores(worker, jobs: list, threads: int, units: float, post=None) -> tuple:
    """Median-of-5 rate of ``worker`` over ``jobs`` on a fork pool of ``threads``
    processes (inputs inherited through fork; only job indices cross the pipe
    inside the timing)."""
    import multiprocessing as mp

    _CPU_JOBS[:] = jobs
    ctx = mp.get_context("fork")
    with ctx.Pool(threads) as pool:
        def run():
            out = pool.map(worker, range(len(jobs)), chunksize=1)
            if post is not None:
                post(out)
        return median_rate(run, units)


def _w_predict(i):
    from oracle import sim as osim

    with one_thread():
        osim.predict(*_CPU_JOBS[i])
    return 0


def _w_fit(i):
    from oracle import sim as osim

    kind, x, y = _CPU_JOBS[i]
    with one_thread():
        osim.fit_uniform(kind, np.broadcast_to(x, (y.shape[0],) + x.shape), y)
    return 0


def _w_hash(i):
    from oracle import profiler as oprof

    return [oprof.signature_hash(oprof.canonicalize(e)) for e in _CPU_JOBS[i]]


def _w_sim(i):
    from oracle import sim as osim

    args, kw = _CPU_JOBS[i]
    osim.run_shard(*args, **kw)
    return 0


def cpu_predictions(tables_host, queries_host, threads: int, n_item: int, n_numpy: int,
                    n_all: int) -> dict:
    """Predictions/s of the oracle on the C5 batch's own tables
    and queries: per-item predict_one (1 thread), numpy predict (1 thread),
    numpy predict over all cores."""
    from oracle import sim as osim

    out = {}
    # per item (plain Python per query)
    prep = []
    for kind in (AFFINE, ATTN):
        tab = tables_host[kind]
        sig, x = queries_host[kind]
        m = min(n_item // 2, sig.shape[0])
        need = sorted({int(v) for v in sig[:m]})
        rows = {i: (tab["coef"][i].tolist(), tab["inv"][i].tolist(), tab["lo"][i].tolist(),
                    tab["hi"][i].tolist()) for i in need}
        prep.append((kind, rows, [int(v) for v in sig[:m]], x[:, :m].T.tolist()))

    def per_item():
        for kind, rows, sl, xl in prep:
            for q in range(len(sl)):
                osim.predict_one(kind, rows, sl[q], xl[q])

    n1 = sum(len(p[2]) for p in prep)
    with one_thread():
        rate, med = median_rate(per_item, n1)
    out["per_item"] = {"value": rate, "unit": "predictions/s", "cores": 1, "kind": "port",
                       "sample": f"{n1} queries of the C5 batch, oracle/sim.py predict_one "
                                 "(plain Python per query)", "median_s": med}
    # numpy batch, one thread
    jobs1 = [(k, tables_host[k], queries_host[k][0][:n_numpy // 2],
              queries_host[k][1][:, :n_numpy // 2]) for k in (AFFINE, ATTN)]
    n2 = sum(j[2].shape[0] for j in jobs1)
    with one_thread():
        rate, med = median_rate(lambda: [osim.predict(*j) for j in jobs1], n2)
    out["numpy_1thread"] = {"value": rate, "unit": "predictions/s", "cores": 1, "kind": "port",
                            "sample": f"{n2} queries of the C5 batch, oracle/sim.py predict "
                                      "(numpy)", "median_s": med}
    # numpy over all cores
    chunk = max(250_000, -(-n_all // (4 * threads)))
    jobs = []
    for kind in (AFFINE, ATTN):
        sig, x = queries_host[kind]
        m = min(n_all // 2, sig.shape[0])
        for q0 in range(0, m, chunk):
            q1 = min(m, q0 + chunk)
            jobs.append((kind, tables_host[kind], sig[q0:q1], x[:, q0:q1]))
    n3 = sum(j[2].shape[0] for j in jobs)
    rate, med = _cpu_all_cores(_w_predict, jobs, threads, n3)
    out["all_cores"] = {"value": rate, "unit": "predictions/s", "cores": threads, "kind": "port",
                        "sample": f"{n3} queries of the C5 batch, oracle/sim.py predict (numpy) "
                                  f"over {threads} processes", "median_s": med}
    return out


def cpu_fits(grid_x: dict, y_sample: dict, threads: int, n_item: int) -> dict:
    """Fits/s of the oracle (App. A.7) on C5 signatures of the
    shared sweep grids: per-signature oracle.fit (1 thread) and vectorised
    fit_uniform over all cores."""
    from oracle import sim as osim

    out = {}
    per = {k: max(1, n_item // 2) for k in (AFFINE, ATTN)}

    def per_item():
        for k in (AFFINE, ATTN):
            x, y = grid_x[k], y_sample[k][:per[k]]
            n = x.shape[1]
            osim.fit(k, np.tile(x, (1, y.shape[0])), y.reshape(-1),
                     np.arange(y.shape[0] + 1, dtype=np.int64) * n)

    n1 = sum(min(per[k], y_sample[k].shape[0]) for k in (AFFINE, ATTN))
    with one_thread():
        rate, med = median_rate(per_item, n1)
    out["per_item"] = {"value": rate, "unit": "fits/s", "cores": 1, "kind": "port",
                       "sample": f"{n1} C5 signatures (half affine, half attention) x "
                                 f"{grid_x[AFFINE].shape[1]} points, oracle/sim.py fit "
                                 "(one least-squares solve per signature)", "median_s": med}
    jobs = []
    for k in (AFFINE, ATTN):
        y = y_sample[k]
        for s0 in range(0, y.shape[0], 64):
            jobs.append((k, grid_x[k], y[s0:s0 + 64]))
    n2 = sum(y_sample[k].shape[0] for k in (AFFINE, ATTN))
    rate, med = _cpu_all_cores(_w_fit, jobs, threads, n2)
    out["all_cores"] = {"value": rate, "unit": "fits/s", "cores": threads, "kind": "port",
                        "sample": f"{n2} C5 signatures, oracle/sim.py fit_uniform (numpy, 64 "
                                  f"signatures per job) over {threads} processes",
                        "median_s": med}
    return out


def packed_as_entries(packed, n: int) -> list:
    """The first n packed C5 records as runnable-set JSON entries:
    every model-config dim at its packed position, the kernel symbols, operator
    granularity — the oracle canonicalises these to the GPU's exact bytes."""
    w = packed.words
    sym = [bytes(packed.sym_bytes[packed.sym_off[i]:packed.sym_off[i + 1]]).decode()
           for i in range(len(packed.sym_off) - 1)]
    out = []
    for i in range(n):
        o = int(packed.rec_off[i])
        op, nd, ns = int(w[o]), int(w[o + 1]) & 0xFFFF, int(w[o + 1]) >> 16
        dims = {int(w[o + 4 + 3 * k]): int(w[o + 5 + 3 * k]) | (int(w[o + 6 + 3 * k]) << 32)
                for k in range(nd)}
        flat = [[dims[pp], "MC"] if pp in dims else [7, "NT"] for pp in range(max(dims) + 1)]
        out.append({"granularity": "operator", "name": packed.op_names[op],
                    "arg_template": [flat], "scalars": [], "attrs": {},
                    "kernel_symbols": [sym[int(w[o + 4 + 3 * nd + k])] for k in range(ns)],
                    "repeat_count": int(w[o + 3])})
    return out


def cpu_dedup(entries: list, threads: int, n_item: int) -> dict:
    """Records/s of the oracle dedup path: canonicalize ->
    SHA-256 (hashlib) -> first-occurrence dedup (dict), per item on one thread,
    and with the hashing spread over all cores (the dedup merge in the parent)."""
    from oracle import profiler as oprof

    out = {}
    sample = entries[:n_item]
    rate, med = median_rate(lambda: oprof.dedup_digests(
        [oprof.signature_hash(oprof.canonicalize(e)) for e in sample]), len(sample))
    out["per_item"] = {"value": rate, "unit": "records/s", "cores": 1, "kind": "port",
                       "sample": f"{len(sample)} C5 records, oracle/profiler.py canonicalize + "
                                 "signature_hash (hashlib) + dedup_digests (dict)",
                       "median_s": med}
    step = max(1, -(-len(entries) // (4 * threads)))
    jobs = [entries[i:i + step] for i in range(0, len(entries), step)]
    rate, med = _cpu_all_cores(
        _w_hash, jobs, threads, len(entries),
        post=lambda parts: oprof.dedup_digests([d for part in parts for d in part]))
    out["all_cores"] = {"value": rate, "unit": "records/s", "cores": threads, "kind": "port",
                        "sample": f"{len(entries)} C5 records, canonicalize + hashlib over "
                                  f"{threads} processes, dict dedup of all digests in the parent",
                        "median_s": med}
    return out


def cpu_sim(shards: list, kw: dict, threads: int) -> dict:
    """Requests/s of the oracle serving loop (regression
    iteration latency, oracle/sim.py run_shard) on C4 replica samples: one
    shard sample on one thread, and one sample per process over all cores."""
    from oracle import sim as osim

    out = {}
    a0 = shards[0]
    rate, med = median_rate(lambda: osim.run_shard(*a0, **kw), len(a0[0]))
    out["per_item"] = {"value": rate, "unit": "requests/s", "cores": 1, "kind": "port",
                       "sample": f"first {len(a0[0])} requests of one C4 replica, oracle/sim.py "
                                 "run_shard (Python event loop, the GPU's regressor rows)",
                       "median_s": med}
    jobs = [(a, kw) for a in shards[:threads]]
    n = sum(len(a[0]) for a, _ in jobs)
    rate, med = _cpu_all_cores(_w_sim, jobs, threads, n)
    out["all_cores"] = {"value": rate, "unit": "requests/s", "cores": threads, "kind": "port",
                        "sample": f"first {len(a0[0])} requests of each of {len(jobs)} C4 "
                                  f"replicas, one replica per process", "median_s": med}
    return out


def host_regressor_table(kind: int, n_sig: int, seed: int) -> dict:
    """Random fitted-looking regressor table for the reference arm (oracle/sim.py
    layout): training boxes inside the C5 grids (affine num_toks <= 32768;
    attention prefill_toks <= 32768, batch <= 256, kv_tokens <= 2^22),
    inv = 1/hi as the fit computes it, small positive coefficients.  The
    oracle's predict cost does not depend on the coefficient values."""
    rng = np.random.default_rng(seed)
    caps = [32768] if kind == AFFINE else [32768, 256, 1 << 22]
    hi = np.stack([rng.integers(c // 4, c + 1, n_sig) for c in caps], axis=1).astype(np.uint32)
    lo = np.minimum(hi, np.stack([rng.integers(0, 4, n_sig) for _ in caps], axis=1)).astype(np.uint32)
    inv = 1.0 / hi.astype(np.float64)
    p = 2 if kind == AFFINE else 10
    coef = rng.uniform(1e-7, 1e-4, (n_sig, p))
    return {"coef": coef, "inv": inv, "lo": lo, "hi": hi}


# ------------------------------------------------------------------- main arm


def arm_config(args) -> dict:
    """The workload both arms report (the reference arm times a bounded sample of it)."""
    return {"workload": f"C5 scale sweep: {args.sigs:.3g} signatures x {args.points} points "
                        f"fitted on the shared sweep grid (split across the GPUs, one all-gather "
                        f"of the rows), then {args.queries:.3g} queries per GPU per step over the "
                        "full table (half affine, half attention)",
            "queries_per_gpu": args.queries, "signatures": args.sigs,
            "points_per_signature": args.points,
            "l2": "inputs >> L2 (126 MB); no flush"}


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2605_07985_b200 import _lib, dist as ddist
    from paper_2605_07985_b200.profiler import DedupWorkspace, DeviceRecords
    from paper_2605_07985_b200.sim import ROW_DTYPE, predict_batch, predict_host_many

    rank, world = ddist.init_from_env()
    dist_on = world > 1
    dev = ddist.local_device()
    local = dev.index
    torch.cuda.set_device(dev)
    if world != args.gpus and rank == 0:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    _lib.ctx_for(dev)
    hbm_peak, peak_kind = load_peaks()
    seed = 1000 * rank

    # ---------------- fit inputs (C5: one shared sweep grid per kind) and the fit sub-benchmark
    # C5: args.sigs signatures in total; each rank fits a contiguous 1/world of
    # each kind (strong scaling of the fit), one all-gather gives every rank the
    # full table, and every rank serves its own queries over that full table
    n_sig_total = {AFFINE: args.sigs // 2, ATTN: args.sigs - args.sigs // 2}
    n_sig = {k: -(-n_sig_total[k] // world) for k in (AFFINE, ATTN)}
    fit_in = {k: gen_grid_fit_data(k, n_sig[k], args.points, dev, seed + k) for k in (AFFINE, ATTN)}
    n_pts = {k: fit_in[k][0].shape[1] for k in (AFFINE, ATTN)}
    torch.cuda.synchronize()
    from paper_2605_07985_b200._lib import KIND_ATTN_PACKED
    from paper_2605_07985_b200.sim import fit_grid, fit_tables, pack_attn

    from paper_2605_07985_b200.sim import FitResult

    # N > 1: the regressor all-gather fused into the fit (peer stores from the
    # fit epilogue + a device arrival counter) when every GPU pair has peer
    # access; otherwise one NCCL all-gather of the rows after the fit
    peer = None
    if dist_on and os.environ.get("DOOLY_FIT_ALLGATHER", "fused") == "fused" and \
            ddist.PeerFitTable.available(world):
        try:   # raises on every rank together if any rank cannot map its peers
            peer = {k: ddist.PeerFitTable(k, world * n_sig[k], dev) for k in (AFFINE, ATTN)}
        except RuntimeError as exc:
            peer = None
            if rank == 0:
                print(f"fused all-gather unavailable ({exc}); using NCCL", file=sys.stderr)

    # the serving form of the attention table (96-B rows) is part of the fit
    # output: written by the fit epilogue itself on one rank (fit_grid_packed),
    # by dooly_attn_pack after the fused all-gather otherwise
    packed96 = torch.empty((world * n_sig[ATTN] + 1, 96), dtype=torch.uint8, device=dev)

    def do_fit(k):
        if peer is None:
            return fit_grid(k, fit_in[k][0], fit_in[k][1], fit_out.get(k),
                            packed=packed96 if k == ATTN and not dist_on else None)
        r0 = rank * n_sig[k]
        pt = peer[k].fit_grid(fit_in[k][0], fit_in[k][1], r0)
        sl = slice(r0, r0 + n_sig[k])
        return FitResult(k, pt.table[sl], pt.fit_err[sl], pt.status[sl])

    fit_out = {}
    for _ in range(max(1, args.warmup)):
        for k in (AFFINE, ATTN):
            fit_out[k] = do_fit(k)
    fused_note = None
    if peer is not None:
        # the fused path's first use on this box: every rank's rows must have
        # landed in every rank's table (no handshake timed out, no all-zero
        # row); all ranks agree, and fall back to the NCCL all-gather together
        ok = 1
        for k in (AFFINE, ATTN):
            ok &= int(peer[k].timed_out.item()) == 0
            ok &= bool(peer[k].table.view(peer[k].n_total, -1).any(dim=1).all().item())
        flag = torch.tensor([ok], dtype=torch.int32,
                            device=dev if torch.distributed.get_backend() == "nccl" else "cpu")
        torch.distributed.all_reduce(flag, op=torch.distributed.ReduceOp.MIN)
        if int(flag.item()) == 0:
            fused_note = "fused all-gather failed its first-use check on this box; NCCL used"
            if rank == 0:
                print(fused_note, file=sys.stderr)
            peer = None
            fit_out.clear()
            for k in (AFFINE, ATTN):
                fit_out[k] = do_fit(k)
    barrier_sync(dist_on)
    stream = torch.cuda.current_stream()
    ev = {k: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for k in (AFFINE, ATTN)}
    ag0, ag1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fit_ms = {AFFINE: 0.0, ATTN: 0.0}
    ag_ms = 0.0
    fit_steps = max(1, min(args.steps, 3))
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    fit_launches0 = _lib.launch_count(dev)
    t_start.record(stream)
    full = {k: fit_out[k].table for k in (AFFINE, ATTN)}   # one rank: the local rows are the table
    for _ in range(fit_steps):
        for k in (AFFINE, ATTN):
            ev[k][0].record(stream)
            fit_out[k] = do_fit(k)
            ev[k][1].record(stream)
        ag0.record(stream)
        if dist_on:   # the one exchange step: every rank gets every rank's rows
            if peer is None:
                full = {k: ddist.gather_requests(fit_out[k].table).reshape(
                    -1, fit_out[k].table.shape[-1]) for k in (AFFINE, ATTN)}
            else:     # already stored into every rank's full table by the fit epilogues
                full = {k: peer[k].table for k in (AFFINE, ATTN)}
            # serving form (96-B rows) of the full attention table (one rank:
            # written by the fit epilogue itself)
            packed96 = pack_attn(full[ATTN], packed96, check=False)
        else:
            full = {k: fit_out[k].table for k in (AFFINE, ATTN)}
        ag1.record(stream)
        torch.cuda.synchronize()
        for k in (AFFINE, ATTN):
            fit_ms[k] += ev[k][0].elapsed_time(ev[k][1])
        ag_ms += ag0.elapsed_time(ag1)
    t_end.record(stream)
    barrier_sync(dist_on)
    fit_launches = (_lib.launch_count(dev) - fit_launches0) // fit_steps
    fit_total_ms = max_over_ranks(t_start.elapsed_time(t_end) / fit_steps, dist_on)
    status_ok = all(int((fit_out[k].status != 0).sum().item()) == 0 for k in (AFFINE, ATTN))
    if peer is not None:   # every rank's rows landed in this rank's full tables
        for k in (AFFINE, ATTN):
            peer[k].check()
            status_ok &= int((peer[k].status != 0).sum().item()) == 0
    fit_bytes = sum(n_sig[k] * n_pts[k] * BYTES_PER_GRID_POINT for k in (AFFINE, ATTN))
    xa = fit_in[ATTN][0][:2].reshape(2, -1, 4) if n_pts[ATTN] % 4 == 0 else None
    grouped = xa is not None and bool((xa == xa[:, :, :1]).all().item()) and \
        os.environ.get("DOOLY_FIT_GRID_FACTOR", "1") != "0"
    x2 = fit_in[ATTN][0][2]
    periodic = grouped and n_pts[ATTN] % 128 == 0 and \
        bool((x2.reshape(-1, 128) == x2[:128]).all().item()) and \
        os.environ.get("DOOLY_FIT_GRID_FACTOR", "2") not in ("0", "1")
    fp64_attn = FP64_PER_ATTN_POINT_PERIODIC if periodic else \
        FP64_PER_ATTN_POINT_GROUPED if grouped else FP64_PER_ATTN_POINT
    fit_dev_ms = sum(fit_ms.values()) / fit_steps
    fits = {
        "value": world * sum(n_sig.values()) / (fit_total_ms / 1e3), "unit": "fits/s",
        "ms_per_step": fit_total_ms, "signatures": world * sum(n_sig.values()),
        "signatures_per_gpu": sum(n_sig.values()), "points": n_pts,
        "scaling": "strong: C5's signature set is split across the ranks",
        "workload": "C5 shared sweep grid per kind (affine: 4096 token counts in [1, 32768]; "
                    "attention: 16x16x16 (prefill_toks, batch, kv_tokens)); sim.fit_grid",
        "kernel_ms": {"affine": fit_ms[AFFINE] / fit_steps, "attention": fit_ms[ATTN] / fit_steps,
                      "allgather": ag_ms / fit_steps},
        "roofline_by_kind": {
            "affine": {"bound": "hbm", "achieved": n_sig[AFFINE] * n_pts[AFFINE] * BYTES_PER_GRID_POINT
                       / (fit_ms[AFFINE] / fit_steps / 1e3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                       "frac": n_sig[AFFINE] * n_pts[AFFINE] * BYTES_PER_GRID_POINT
                       / (fit_ms[AFFINE] / fit_steps / 1e3) / 1e9 / hbm_peak},
            "attention": {"bound": "fp64 (see fp64_attention); hbm alongside",
                          "hbm_achieved": n_sig[ATTN] * n_pts[ATTN] * BYTES_PER_GRID_POINT
                          / (fit_ms[ATTN] / fit_steps / 1e3) / 1e9, "hbm_peak": hbm_peak,
                          "unit": "GB/s",
                          "hbm_frac": n_sig[ATTN] * n_pts[ATTN] * BYTES_PER_GRID_POINT
                          / (fit_ms[ATTN] / fit_steps / 1e3) / 1e9 / hbm_peak}},
        "launches_per_step": fit_launches,
        "allgather_path": None if not dist_on else (
            "fused: peer-memory row stores in the fit epilogue + device arrival counter"
            if peer is not None else "NCCL all_gather of the regressor rows"
            + (f" ({fused_note})" if fused_note else "")),
        "roofline": {"bound": "hbm", "achieved": fit_bytes / (fit_dev_ms / 1e3) / 1e9,
                     "peak": hbm_peak, "unit": "GB/s",
                     "frac": fit_bytes / (fit_dev_ms / 1e3) / 1e9 / hbm_peak,
                     "traffic": ncu_traffic("fit_grid", {k: n_sig[k] * n_pts[k] for k in (AFFINE, ATTN)}),
                     "alg_bytes_per_point": BYTES_PER_GRID_POINT,
                     "note": "y crosses HBM once (8 B/point); the attention kind is FP64-bound, "
                             "see fp64_attention and DESIGN.md"},
        # FP64 instructions per attention point: per-point passes 27 (pass 1:
        # 3 mul + 4 add + 6 fma; pass 2: 9-fma Horner, clamp, subtract, 1-Newton
        # reciprocal, fma), grouped passes 16, grouped with the per-position
        # pass 1 (grid_r1_step) 14; 64 per clock per SM nominal
        "fp64_attention": {
            "bound": "fp64", "instr_per_point": fp64_attn,
            "passes": "grouped, per-position pass 1 (aligned 4-point groups share "
            "prefill_toks and batch; the kv axis repeats every 128 points)"
            if fp64_attn == FP64_PER_ATTN_POINT_PERIODIC else
            "grouped (aligned 4-point groups share prefill_toks and batch)"
            if fp64_attn == FP64_PER_ATTN_POINT_GROUPED else "per-point",
            "achieved": n_sig[ATTN] * n_pts[ATTN] * fp64_attn
            / (fit_ms[ATTN] / fit_steps / 1e3) / 1e12,
            "peak": FP64_PEAK_TINSTR, "unit": "T FP64 instr/s",
            "frac": n_sig[ATTN] * n_pts[ATTN] * fp64_attn
            / (fit_ms[ATTN] / fit_steps / 1e3) / 1e12 / FP64_PEAK_TINSTR,
            "peak_source": "nominal 64 DFMA/clk/SM x 148 SMs x 1965 MHz (tools/fp64_probe.py "
                           "measures DFMA at 34 TFLOP/s = 17 T instr/s)"},
        "all_fitted": status_ok,
    }
    # the general per-signature (CSR) kernel on the same points, x materialised per signature
    fits_csr = None
    if args.csr_fit:
        csr_ms = {}
        worst = 0.0
        for k in (AFFINE, ATTN):
            xr = fit_in[k][0].repeat(1, n_sig[k])
            off = torch.arange(n_sig[k] + 1, dtype=torch.int64, device=dev) * n_pts[k]
            fc = fit_tables(k, xr, fit_in[k][1].reshape(-1), off)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fc = fit_tables(k, xr, fit_in[k][1].reshape(-1), off, fc)
            e1.record(stream)
            torch.cuda.synchronize()
            csr_ms[k] = e0.elapsed_time(e1)
            nc = 2 if k == AFFINE else 10
            ga, gc = fit_out[k].table.view(torch.float64)[:, :nc], fc.table.view(torch.float64)[:, :nc]
            worst = max(worst, float(((ga - gc).abs().amax(1) / gc.abs().amax(1)).max().item()))
            del xr, fc
        torch.cuda.empty_cache()
        csr_bytes = sum(n_sig[k] * n_pts[k] * BYTES_PER_POINT[k] for k in (AFFINE, ATTN))
        fits_csr = {"value": sum(n_sig.values()) / (sum(csr_ms.values()) / 1e3), "unit": "fits/s",
                    "kernel_ms": {"affine": csr_ms[AFFINE], "attention": csr_ms[ATTN]},
                    "achieved_gbs": csr_bytes / (sum(csr_ms.values()) / 1e3) / 1e9,
                    "alg_bytes_per_point": BYTES_PER_POINT,
                    "max_coef_rel_diff_vs_grid": worst,
                    "path": "sim.fit_tables (dooly_fit): per-signature points, Gram per signature"}
    cpu_on = rank == 0 and world == 1 and args.cpu_sample > 0
    cpu_fit_in = None
    if cpu_on:
        m = max(2, args.cpu_fit_sigs // 2)
        cpu_fit_in = ({k: fit_in[k][0].cpu().numpy().view(np.uint32) for k in (AFFINE, ATTN)},
                      {k: fit_in[k][1][:m].cpu().numpy() for k in (AFFINE, ATTN)})
    del fit_in
    pack_attn(full[ATTN], packed96, check=True)   # raises if not representable
    rows128 = dict(full)   # every rank queries the full table
    tables = {AFFINE: full[AFFINE], ATTN: packed96}
    pkind = {AFFINE: AFFINE, ATTN: KIND_ATTN_PACKED}
    torch.cuda.empty_cache()

    # ---------------- headline: predict
    nq = {AFFINE: args.queries // 2, ATTN: args.queries - args.queries // 2}
    qs = {k: gen_queries(k, rows128[k], nq[k], dev, seed + 7 + k) for k in (AFFINE, ATTN)}
    outs = {k: torch.empty(nq[k], dtype=torch.float64, device=dev) for k in (AFFINE, ATTN)}
    flags = {k: torch.empty((2, (nq[k] + 31) // 32), dtype=torch.int32, device=dev)
             for k in (AFFINE, ATTN)}
    errs = {k: torch.full((1,), torch.iinfo(torch.int64).max, dtype=torch.int64, device=dev)
            for k in (AFFINE, ATTN)}

    def predict_step():
        for k in (AFFINE, ATTN):
            predict_batch(pkind[k], tables[k], qs[k][0], qs[k][1], outs[k], flags[k], errs[k])

    for _ in range(args.warmup):
        predict_step()
    barrier_sync(dist_on)
    launches0 = _lib.launch_count(dev)
    pev = {k: [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)] for k in (AFFINE, ATTN)}
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        time.sleep(0.05)
        clk.mark_start()
        start.record(stream)
        for s in range(args.steps):
            for k in (AFFINE, ATTN):
                pev[k][s][0].record(stream)
                predict_batch(pkind[k], tables[k], qs[k][0], qs[k][1], outs[k], flags[k], errs[k])
                pev[k][s][1].record(stream)
        end.record(stream)
        barrier_sync(dist_on)
        clk.mark_end()
    launches = _lib.launch_count(dev) - launches0
    ms_step = max_over_ranks(start.elapsed_time(end) / args.steps, dist_on)
    k_ms = {k: sum(a.elapsed_time(b) for a, b in pev[k]) / args.steps for k in (AFFINE, ATTN)}
    bad = any(int(errs[k].item()) != torch.iinfo(torch.int64).max for k in (AFFINE, ATTN))
    alg_bytes = sum(nq[k] * BYTES_PER_QUERY[k] for k in (AFFINE, ATTN))
    achieved = alg_bytes / ((k_ms[AFFINE] + k_ms[ATTN]) / 1e3) / 1e9
    value = world * args.queries / (ms_step / 1e3)
    clocks = clk.summary()

    # ---------------- e2e through the public host API (pinned host buffers)
    e2e = None
    if args.e2e_queries > 0:
        n_e = {AFFINE: args.e2e_queries // 2, ATTN: args.e2e_queries - args.e2e_queries // 2}
        host_q = {}
        for k in (AFFINE, ATTN):
            host_q[k] = (qs[k][0][: n_e[k]].cpu().pin_memory(), qs[k][1][:, : n_e[k]].cpu().pin_memory(),
                         torch.empty(n_e[k], dtype=torch.float64).pin_memory(),
                         torch.empty((2, (n_e[k] + 31) // 32), dtype=torch.int32).pin_memory())
        batches = [(pkind[k], tables[k], *host_q[k]) for k in (AFFINE, ATTN)]
        for _ in range(2):
            predict_host_many(batches)
        barrier_sync(dist_on)
        e_steps = max(3, min(args.steps, 5))
        e_times = []
        for _ in range(e_steps):
            t0 = time.perf_counter()
            predict_host_many(batches)          # synchronises (host buffers are the output)
            e_times.append(time.perf_counter() - t0)
        barrier_sync(dist_on)
        # median step: the host link is shared with the rest of the box
        e_s = max_over_ranks(float(np.median(e_times)), dist_on)
        h2d = sum(host_q[k][0].numel() * 4 + host_q[k][1].numel() * 4 for k in (AFFINE, ATTN))
        d2h = sum(host_q[k][2].numel() * 8 + host_q[k][3].numel() * 4 for k in (AFFINE, ATTN))
        e2e = {"value": world * args.e2e_queries / e_s, "unit": "predictions/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "queries_per_step_per_gpu": args.e2e_queries,
               "steps": e_steps, "step_s": e_times, "method": "median of the timed steps",
               "path": "sim.predict_host_many: pinned host -> device -> kernel -> host (latencies "
                       "and the extrapolation/clamp flag bit-planes), both kinds' chunks "
                       "interleaved over 3 streams",
               "link_ceiling": link_ceiling(host_q[AFFINE][2], dev, h2d, d2h, e_s)}
        del host_q

    # ---------------- CPU baselines (rank 0, N=1 only)
    cpu = None
    cpu_threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    if cpu_on:
        tables_host = {}
        qh = {}
        sys.path.insert(0, str(ROOT / "tests"))
        from helpers import rows_to_table

        for k in (AFFINE, ATTN):
            rows = rows128[k].cpu().numpy().view(ROW_DTYPE[k]).reshape(-1)
            tables_host[k] = rows_to_table(k, rows)
            m = args.cpu_sample // 2
            qh[k] = (qs[k][0][:m].cpu().numpy().view(np.uint32),
                     qs[k][1][:, :m].cpu().numpy().view(np.uint32))
        lines = cpu_predictions(tables_host, qh, cpu_threads, args.cpu_sample_items,
                                args.cpu_sample // 5, args.cpu_sample)
        cpu = dict(lines["numpy_1thread"], per_item=lines["per_item"], all_cores=lines["all_cores"],
                   host=host_info())
        fits["cpu_baseline"] = dict(cpu_fits(*cpu_fit_in, cpu_threads, args.cpu_fit_items),
                                    host=host_info())
        del tables_host, qh

    # ---------------- dedup sub-benchmark
    dedup = None
    if args.records > 0:
        packed, _ = synth_records(args.records, seed=rank + 11)
        recs = DeviceRecords.from_packed(packed, dev)
        ws = DedupWorkspace(dev)
        from paper_2605_07985_b200.profiler import dedup_packed, hash_records, dedup_digests

        for _ in range(args.warmup):
            r = dedup_packed(recs, workspace=ws, sync=False)
        barrier_sync(dist_on)
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        d_steps = max(1, min(args.steps, 5))
        sha_ms = 0.0
        tot_ms = 0.0
        dig = torch.empty((recs.n, 32), dtype=torch.uint8, device=dev)
        n_total = world * recs.n   # global record list = the ranks' slices in rank order
        # N > 1: the one exchange step — digests into every rank's gathered array,
        # fused into the hash kernel's epilogue over peer memory when available
        # (else an NCCL all-gather) — then a global first-occurrence resolve on
        # every rank (dist.dedup_sharded)
        # From 4 ranks on, the owner-routed form (all-to-all of digests to their
        # owners and of the results back, dist.dedup_routed) keeps each rank's
        # resolve at ~records_per_gpu keys instead of the whole list.
        xchg = os.environ.get("DOOLY_DEDUP_EXCHANGE", "route" if world >= 4 else "gather")
        routed = dist_on and xchg == "route"
        pdig = ddist.PeerDigests(n_total, dev) if peer is not None and not routed else None
        for _ in range(d_steps):
            e0.record(stream)
            if routed:
                r = ddist.dedup_routed(recs, n_total, None, ws)
                e1.record(stream)
            elif not dist_on:
                # one process: the public batch call (dooly_dedup: record grouping,
                # SHA-256 of the representatives, digest copy, resolve)
                r = dedup_packed(recs, workspace=ws, sync=False)
                full = r.digests
                e1.record(stream)
            else:
                if pdig is not None:
                    full = pdig.hash(recs, rank * recs.n)
                else:
                    hash_records(recs, dig)
                e1.record(stream)
                if pdig is None:
                    full = ddist.all_gather_rows(dig, n_total)
                r = dedup_digests(full, None, ws, sync=False)
            e2.record(stream)
            torch.cuda.synchronize()
            sha_ms += e0.elapsed_time(e1)
            tot_ms += e0.elapsed_time(e2)
        barrier_sync(dist_on)
        tot_ms = max_over_ranks(tot_ms / d_steps, dist_on)
        if pdig is not None:
            pdig.check()
        n_unique = int(r.n_unique) if routed else int(dedup_digests(full, None, ws).n_unique)
        if routed or not dist_on:   # e0 -> e1 spans the whole dedup; time the hash alone once
            e0.record(stream)
            hash_records(recs, dig)
            e1.record(stream)
            torch.cuda.synchronize()
            sha_ms = e0.elapsed_time(e1) * d_steps
        msg_len = 8 + 4 + 6 + 4 + 3 * 12 + 4 + 2 * (4 + 16)  # approx canonical length
        dedup = {"value": world * recs.n / (tot_ms / 1e3), "unit": "records/s",
                 "records_per_gpu": recs.n, "unique": n_unique, "ms_per_step": tot_ms,
                 "exchange": None if not dist_on else (
                     "owner-routed: all-to-all of (digest, index) to the owners, resolve "
                     "there, all-to-all of the results back" if routed else
                     "fused: digests stored into every rank by the hash kernel, global resolve"
                     if pdig is not None else "NCCL all-gather of 32-B digests, global resolve"),
                 "sha_ms": sha_ms / d_steps,
                 "sha_blocks_per_s": recs.n * 2 / (sha_ms / d_steps / 1e3),
                 "bound": "int32 ALU (SHA-256 rounds)",
                 # rotates (SHF) and Ch/Maj/xor (LOP3) are ALU-pipe only: 18 per
                 # scheduled round, 10 per round of the first 16 (the additions run
                 # on the FMA pipe as IMAD); ALU pipe = 64 lanes/clk/SM
                 "alu_roofline": {
                     "instr_per_block": SHA_ALU_PER_BLOCK,
                     "achieved": recs.n * 2 * SHA_ALU_PER_BLOCK / (sha_ms / d_steps / 1e3) / 1e12,
                     "peak": ALU_PEAK_TINSTR, "unit": "T ALU instr/s",
                     "frac": recs.n * 2 * SHA_ALU_PER_BLOCK / (sha_ms / d_steps / 1e3) / 1e12
                     / ALU_PEAK_TINSTR,
                     "note": "compression rounds only; canonical-message construction and "
                             "lock-step padding of shorter messages are the remainder"}}

        if cpu_on:
            ents = packed_as_entries(packed, args.cpu_dedup_records)
            from oracle import profiler as oprof

            for i in range(0, len(ents), max(1, len(ents) // 50)):   # the CPU path hashes the same bytes
                want = bytes(r.digests[i].cpu().numpy())
                assert oprof.signature_hash(oprof.canonicalize(ents[i])) == want
            dedup["cpu_baseline"] = dict(cpu_dedup(ents, cpu_threads, args.cpu_dedup_items),
                                         host=host_info())

    # ---------------- sim sub-benchmark (C4)
    sim = None
    if args.sim_requests > 0:
        sim = bench_sim(args, dev, dist_on, rank, world, cpu_threads if cpu_on else 0)

    if rank == 0:
        line = {
            "metric": "latency predictions/s (C5 predict batch; fits/s, dedup, sim alongside)",
            "value": value, "unit": "predictions/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (C5: seeded device-generated regressor tables and queries)",
            "config": arm_config(args),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": ncu_traffic("predict", nq),
                         "alg_bytes": alg_bytes,
                         "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)"
                         if peak_kind == "measured" else "fallback 6.65 TB/s",
                         "kernel_ms": {"affine": k_ms[AFFINE], "attention": k_ms[ATTN]},
                         "alg_bytes_per_query": BYTES_PER_QUERY,
                         "gather_ceiling": gather_ceiling(nq, k_ms),
                         "l1tex": l1tex_roofline(nq, k_ms, clocks.get("sm_mhz")),
                         "xbar": xbar_roofline(nq, k_ms, clocks.get("sm_mhz"))},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
            "fits": fits, "fits_csr": fits_csr, "dedup": dedup, "sim": sim, "unknown_signature_errors": bad,
        }
        print(json.dumps(line))
    if dist_on:
        dist.barrier()
        dist.destroy_process_group()


def c4_trace(n: int, S: int, rate_per_replica: float):
    """C4 trace: Poisson arrivals at rate_per_replica x S,
    Table-3 length distributions (lognormal with the medians/means of
    PAPER.md:621-623), seed 1."""
    rng = np.random.default_rng(1)
    arr = np.cumsum(rng.exponential(1.0 / (rate_per_replica * S), size=n))
    sig_p = math.sqrt(2 * math.log(1232 / 950))
    sig_o = math.sqrt(2 * math.log(397 / 388))
    pr = np.clip(np.rint(rng.lognormal(math.log(950), sig_p, n)), 1, 8192 - 512).astype(np.uint32)
    ou = np.clip(np.rint(rng.lognormal(math.log(388), sig_o, n)), 1, 512).astype(np.uint32)
    return arr, pr, ou, np.zeros(n, np.uint32)


def bench_sim(args, dev, dist_on, rank, world, cpu_threads: int = 0):
    """C4: Llama-3-70B-like tp=4 serving replicas; regressors from the C4
    manifest's sweep.  The headline sim line is C4 as defined (S = 64 fixed
    replicas, request i -> replica i mod S, replicas round-robin over ranks);
    ``s1184`` reruns the trace over 1184 replicas (8 per SM) as a throughput
    extra; ``sim_eval`` times dooly_sim_eval (K4a iteration evaluation + the
    per-replica clock scan + per-request TTFT/TPOT) over the C4 run's own
    logged iterations."""
    import torch

    from paper_2605_07985_b200 import _lib
    from paper_2605_07985_b200 import dist as ddist
    from paper_2605_07985_b200 import modelir
    from paper_2605_07985_b200.profiler import profile_corpus
    from paper_2605_07985_b200.sim import (SchedConfig, ShardedTrace, build_calltree, fit,
                                           make_sched, run_sharded, sim_eval)

    man = modelir.load_manifest(modelir.builtin_manifest_path("llama70b"))
    model, backend, hw = man.models[0], man.backends[1], man.hardware
    db, _ = profile_corpus(modelir.CorpusManifest((model,), (backend,), hw, man.tp_degree,
                                                  man.grid), device=dev)
    regs = fit(db, dev)
    ct = build_calltree(model, backend, regs, hw, man.tp_degree)
    sched = SchedConfig(chunk=8192, max_batch=256)
    cfg = make_sched(model, hw, man.tp_degree, sched, ct)
    n = args.sim_requests
    conf = (f"llama-3-70b-like tp=4 flashattention-like on a100-like; Poisson "
            f"{args.sim_rate} req/s per replica; chunk 8192, max_batch 256")

    def run_c4(S, log_cap=0):
        arr, pr, ou, ca = c4_trace(n, S, args.sim_rate)
        mine = np.arange(S)[np.arange(S) % world == rank]
        sel = np.concatenate([np.arange(s, n, S) for s in mine])
        sel.sort()
        trace = ShardedTrace.from_arrays(arr[sel], pr[sel], ou[sel], ca[sel], len(mine), dev)
        res = run_sharded(trace, ct, cfg, regs)      # warm-up
        barrier_sync(dist_on)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = run_sharded(trace, ct, cfg, regs, out=res)
        e1.record()
        barrier_sync(dist_on)
        ms = max_over_ranks(e0.elapsed_time(e1), dist_on)
        if log_cap:   # untimed rerun with the per-iteration log (sim_eval's inputs)
            res = run_sharded(trace, ct, cfg, regs, log_cap=log_cap)
        ok = int((res.status != 0).sum().item()) == 0
        ttft = res.ttft.cpu()
        if dist_on:   # global percentiles: every rank's TTFTs, NaN-padded to a common length
            m = int(max_over_ranks(float(ttft.numel()), dist_on))
            pad = torch.full((m,), float("nan"), dtype=torch.float64)
            pad[: ttft.numel()] = ttft
            ttft = ddist.gather_requests(pad.to(dev)).reshape(-1).cpu()
            ok = max_over_ranks(0.0 if ok else 1.0, dist_on) == 0.0
        ttft = ttft.numpy()
        n_it = int(res.n_iter.sum().item())
        line = {"value": n / (ms / 1e3), "unit": "requests/s", "ms": ms, "requests": n,
                "shards": S, "iterations_rank0": n_it, "iterations_per_s": n_it / (ms / 1e3),
                "max_iterations_per_replica": int(res.n_iter.max().item()), "all_ok": ok,
                "ttft_p50_s": float(np.nanpercentile(ttft, 50)),
                "ttft_p99_s": float(np.nanpercentile(ttft, 99)), "config": conf + f" x {S} replicas"}
        return line, trace, res, (arr, pr, ou, ca)

    S = args.sim_shards
    sim, trace, res, c4 = run_c4(S, log_cap=args.sim_log_cap)
    sim["bound"] = ("latency: each replica's event loop is sequential (SPEC.md:638); one warp "
                    "per replica, exact decode windows evaluate up to 32 event-free iterations "
                    "in parallel; S = 64 replicas occupy 64 warps of the GPU")
    # ---- dooly_sim_eval over the C4 run's logged iterations (28 B per iteration
    # + 36 B per request); every logged iteration of every replica
    if args.sim_log_cap > 0:
        n_it = res.n_iter.cpu().numpy()
        if int(n_it.max()) <= args.sim_log_cap:
            S_mine = trace.n_shards
            feats = torch.cat([res.log_feat[s, :int(n_it[s])] for s in range(S_mine)]).t().contiguous()
            off = torch.from_numpy(np.concatenate([[0], np.cumsum(n_it)]).astype(np.int64)).to(dev)
            it_start = torch.zeros(feats.shape[1], dtype=torch.float64, device=dev)
            # request -> a (first, last) iteration pair inside its replica (timing input)
            g = torch.Generator(device=dev)
            g.manual_seed(5)
            req_shard = torch.repeat_interleave(torch.arange(S_mine, device=dev),
                                                trace.shard_off[1:] - trace.shard_off[:-1])
            lo = off[:-1][req_shard]
            span = (off[1:] - off[:-1])[req_shard]
            f_it = (lo + (torch.rand(req_shard.numel(), generator=g, device=dev, dtype=torch.float64)
                          * span).long()).int()
            l_it = torch.minimum(f_it.long() + 380, off[1:][req_shard] - 1).int()
            def once():
                return sim_eval(ct, regs, feats, trace.arrival, f_it, l_it, trace.output,
                                it_start=it_start, it_off=off)
            once()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            l0 = _lib.launch_count(dev)
            e0.record()
            once()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            N_it, N_req = feats.shape[1], trace.arrival.numel()
            nbytes = N_it * 28 + N_req * 36
            feat_of = [ct.oplist.feat[i] for i in range(ct.n_ops)]
            # FP64 instructions per iteration of the call graph's evaluation:
            # affine entry 5 (scale, multiply, add, clamp, repeat product) + 1
            # add; attention entry 27 (3 scalings, 6 monomials, 9 products, 9
            # adds) + repeat product + add; comm entry 6
            fp64_per_it = sum(6 if f in (_lib.FEAT_NUM_TOKS, _lib.FEAT_NUM_SEQS) else
                              29 if f == _lib.FEAT_ATTN else 6 for f in feat_of)
            sim["sim_eval"] = {
                "iterations": N_it, "requests": N_req, "ms": ms,
                "iterations_per_s": N_it / (ms / 1e3), "launches": _lib.launch_count(dev) - l0,
                "roofline": {"hbm_achieved_gbs": nbytes / (ms / 1e3) / 1e9,
                             "hbm_frac": nbytes / (ms / 1e3) / 1e9 / load_peaks()[0],
                             "fp64_achieved_tinstr": N_it * fp64_per_it / (ms / 1e3) / 1e12,
                             "fp64_frac": N_it * fp64_per_it / (ms / 1e3) / 1e12 / FP64_PEAK_TINSTR,
                             "alg_bytes": "28 B/iteration (5 u32 features in, f64 out) + 36 B/request",
                             "fp64_instr_per_iteration": fp64_per_it},
                "inputs": "the S = 64 C4 run's logged per-iteration features (every iteration of "
                          "every replica); it_start zero (no idle jumps), per-request first/last "
                          "iterations drawn inside the request's replica",
                "bound": "the per-replica clock scan is sequential f64 (App. A.11): 64 replicas "
                         "= 64 warps; the iteration evaluation itself is parallel"}
            del feats, it_start
    if args.sim_wide_shards > 0:
        wide, _, _, _ = run_c4(args.sim_wide_shards)
        sim["s1184" if args.sim_wide_shards == 1184 else f"s{args.sim_wide_shards}"] = wide
    # ---- CPU oracle serving loop on replica samples (rank 0, N = 1)
    if cpu_threads and rank == 0 and world == 1:
        sys.path.insert(0, str(ROOT / "tests"))
        from helpers import AFFINE as HA, ATTN as HT, rows_to_table

        tabs = {k: rows_to_table(k, regs.tables[k].rows()) for k in regs.tables}
        ops = []
        for i in range(ct.n_ops):
            feat, row = ct.oplist.feat[i], ct.oplist.row[i]
            op = {"feat": feat, "repeat": ct.oplist.repeat[i],
                  "window_slot": ct.oplist.window_slot[i], "bytes_per_tok": ct.oplist.bytes_per_tok[i]}
            if feat != _lib.FEAT_COMM:
                t = tabs[HT if feat == _lib.FEAT_ATTN else HA]
                op.update(coef=list(t["coef"][row]), inv=list(t["inv"][row]))
            ops.append(op)
        arr, pr, ou, ca = c4
        m = args.cpu_sim_requests
        shards = []
        for s_ in range(min(S, cpu_threads)):
            idx = np.arange(s_, n, S)[:m]
            shards.append((arr[idx].tolist(), pr[idx].tolist(), ou[idx].tolist(), ca[idx].tolist()))
        kw = dict(ops=ops, chunk=8192, max_batch=256, kv_bytes_per_token=cfg.kv_bytes_per_token,
                  kv_capacity=cfg.kv_capacity_bytes, window=ct.window, tp=man.tp_degree,
                  alpha=hw.comm_alpha, beta=hw.comm_beta)
        sim["cpu_baseline"] = dict(cpu_sim(shards, kw, cpu_threads), host=host_info())
    return sim


# ---------------------------------------------------------------- reference arm


def run_reference(args):
    """The reference path has no shipped implementation; the oracle port of its
    specified predict (oracle/sim.py) is timed on all host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sys.path.insert(0, str(ROOT / "tests"))
    from helpers import synth_queries

    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    tables, qh = {}, {}
    for k in (AFFINE, ATTN):
        # regressor tables of the C5 size (sigs / 2 rows per kind, as the GPU arm
        # serves), boxes spanning the C5 sweep grids; queries inside the boxes
        tables[k] = host_regressor_table(k, args.sigs // 2, seed=k)
        qh[k] = synth_queries(k, tables[k], args.ref_sample // 2, seed=k + 1)
    import multiprocessing as mp

    chunk = max(250_000, -(-args.ref_sample // (4 * threads)))
    jobs = []
    for kind in (AFFINE, ATTN):
        sig, x = qh[kind]
        for q0 in range(0, sig.shape[0], chunk):
            jobs.append((kind, tables[kind], sig[q0:q0 + chunk], x[:, q0:q0 + chunk]))
    _CPU_JOBS[:] = jobs
    n_done = sum(j[2].shape[0] for j in jobs)
    times = []
    with mp.get_context("fork").Pool(threads) as pool:
        for _ in range(max(1, args.warmup)):
            pool.map(_w_predict, range(len(jobs)), chunksize=1)
        for _ in range(args.steps):
            t0 = time.perf_counter()
            pool.map(_w_predict, range(len(jobs)), chunksize=1)
            times.append(time.perf_counter() - t0)
    ms = 1e3 * float(np.median(times))
    value = n_done / (ms / 1e3)
    line = {"impl": "reference",
            "metric": "latency predictions/s (C5 predict batch; fits/s, dedup, sim alongside)",
            "value": value, "unit": "predictions/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": arm_config(args),
            "config_sample": {"workload": "C5 predict batch (bounded CPU sample): "
                                          f"{args.sigs // 2} regressor rows per kind",
                              "queries_per_step": args.ref_sample},
            "cpu_baseline": {"value": value, "unit": "predictions/s", "cores": threads,
                             "kind": "port",
                             "sample": f"{n_done} queries per step, oracle/sim.py "
                                       f"predict over {threads} processes (median of "
                                       f"{args.steps} steps after {max(1, args.warmup)} warm-up)",
                             "host": host_info()},
            "e2e": {"value": value, "unit": "predictions/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--queries", type=int, default=1_000_000_000)
    ap.add_argument("--sigs", type=int, default=1_000_000)
    ap.add_argument("--points", type=int, default=4096)
    ap.add_argument("--csr-fit", type=int, default=1, help="also time the per-signature CSR fit")
    ap.add_argument("--records", type=int, default=4_000_000)
    ap.add_argument("--e2e-queries", type=int, default=200_000_000)
    ap.add_argument("--cpu-sample", type=int, default=20_000_000)
    ap.add_argument("--cpu-sample-items", type=int, default=200_000,
                    help="queries of the per-item (plain Python) CPU line")
    ap.add_argument("--ref-sample", type=int, default=40_000_000)
    ap.add_argument("--sim-requests", type=int, default=1_000_000)
    ap.add_argument("--sim-shards", type=int, default=64, help="C4: S fixed replicas")
    ap.add_argument("--sim-wide-shards", type=int, default=1184,
                    help="extra sim line over this many replicas (0: skip)")
    ap.add_argument("--sim-rate", type=float, default=4.0)
    ap.add_argument("--sim-log-cap", type=int, default=400_000,
                    help="per-replica iteration log for the sim_eval timing (0: skip)")
    ap.add_argument("--cpu-fit-sigs", type=int, default=2048)
    ap.add_argument("--cpu-fit-items", type=int, default=64)
    ap.add_argument("--cpu-dedup-records", type=int, default=400_000)
    ap.add_argument("--cpu-dedup-items", type=int, default=50_000)
    ap.add_argument("--cpu-sim-requests", type=int, default=1000)
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "ours":
        print("warning: the bench contract requires --warmup >= 3", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
