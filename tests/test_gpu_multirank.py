"""N > 1 path on the GPU box: two ranks sharing cuda:0 over gloo (gpurun hands out
one GPU, and NCCL refuses two ranks on one device).  The sharded dedup and fit
(paper_2605_07985_b200.dist) run the real sm_100a kernels on each rank's slice,
exchange through the same collective calls the NCCL path makes, and must equal
the single-rank results.  The fused fit + all-gather (PeerFitTable,
dooly_fit_grid_bcast) maps each rank's table into the other through CUDA IPC —
the same mechanism as across NVLink peers, minus the link — and must reproduce
the single-rank table bit for bit.  Then bench.py runs under torchrun at
--gpus 2."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, q) -> None:
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank), DOOLY_DIST_BACKEND="gloo")
    import torch.distributed as dist

    try:
        import bench
        from helpers import AFFINE, ATTN, synth_fit_data
        from paper_2605_07985_b200 import dist as ddist
        from paper_2605_07985_b200.profiler import DeviceRecords, dedup_packed
        from paper_2605_07985_b200.records import pack_uniform  # noqa: F401 (bench uses it)
        from paper_2605_07985_b200.sim import fit_grid, fit_tables

        assert ddist.init_from_env() == (rank, world)
        dev = ddist.local_device()
        assert dev == torch.device("cuda", 0)
        # ---- dedup: global record list split contiguously, digests all-gathered
        n_total = 20_011
        packed, _ = bench.synth_records(n_total, seed=5)
        whole = dedup_packed(DeviceRecords.from_packed(packed, dev))
        a, b = ddist.shard_range(n_total, rank, world)
        mine, _ = bench.synth_records(n_total, seed=5)
        sl = _slice_packed(mine, a, b)
        got = ddist.dedup_sharded(DeviceRecords.from_packed(sl, dev), n_total)
        assert got.n_unique == whole.n_unique
        for name in ("first", "uid", "is_new", "in_db"):
            assert torch.equal(getattr(got, name), getattr(whole, name)[a:b]), name
        assert torch.equal(got.digests, whole.digests[a:b])
        # owner-routed dedup (all-to-all to the digest owners and back)
        got = ddist.dedup_routed(DeviceRecords.from_packed(sl, dev), n_total)
        assert got.n_unique == whole.n_unique
        for name in ("first", "uid", "is_new", "in_db"):
            assert torch.equal(getattr(got, name), getattr(whole, name)[a:b]), name
        assert torch.equal(got.digests, whole.digests[a:b])
        db = whole.digests[::97].clone()                      # some keys already in the DB
        whole_db = dedup_packed(DeviceRecords.from_packed(packed, dev), db)
        got = ddist.dedup_routed(DeviceRecords.from_packed(sl, dev), n_total, db)
        assert got.n_unique == whole_db.n_unique
        for name in ("first", "uid", "is_new", "in_db"):
            assert torch.equal(getattr(got, name), getattr(whole_db, name)[a:b]), name
        # fused hash + all-gather (digests stored into both ranks by the hash kernel)
        pd = ddist.PeerDigests(n_total, dev)
        for _ in range(2):
            got = ddist.dedup_sharded(DeviceRecords.from_packed(sl, dev), n_total, peer_digests=pd)
        torch.cuda.synchronize()
        pd.check()
        assert torch.equal(pd.digests, whole.digests)
        for name in ("first", "uid", "is_new", "in_db"):
            assert torch.equal(getattr(got, name), getattr(whole, name)[a:b]), name
        # ---- fit: contiguous signature ranges, regressor rows all-gathered
        for kind in (AFFINE, ATTN):
            x, y, off = synth_fit_data(kind, 301, 64, seed=kind, ragged=True)
            xt = torch.from_numpy(np.ascontiguousarray(x).view(np.int32)).to(dev)
            yt = torch.from_numpy(y).to(dev)
            ref = fit_tables(kind, xt, yt, torch.from_numpy(off).to(dev))
            shard = ddist.fit_sharded(kind, xt, yt, off)
            # same kernels, but a signature's points sit at a different alignment
            # in the rank's slice (TMA head/tail peeling changes the summation
            # order), so rows agree to the fit contract, not bit for bit
            nc = 2 if kind == AFFINE else 10
            ga, gr = shard.table.view(torch.float64), ref.table.view(torch.float64)
            d = (ga[:, :nc] - gr[:, :nc]).abs().amax(1) / gr[:, :nc].abs().amax(1)
            assert float(d.max()) <= 1e-11, (kind, float(d.max()))
            assert torch.equal(ga[:, nc:], gr[:, nc:]), kind        # scaling + box exact
            assert torch.equal(shard.status, ref.status), kind
            assert torch.allclose(shard.fit_err, ref.fit_err, rtol=1e-11, atol=0), kind
        # ---- fused fit + all-gather: rows stored into every rank's table by the
        # fit epilogue over peer (IPC-mapped) memory, device arrival counter
        assert ddist.PeerFitTable.available(world)
        for kind in (AFFINE, ATTN):
            n_total = 601
            xg, yg = bench.gen_grid_fit_data(kind, n_total, 512, dev, seed=7 + kind)
            ref = fit_grid(kind, xg, yg)
            pt = ddist.PeerFitTable(kind, n_total, dev)
            a, b = ddist.shard_range(n_total, rank, world)
            for _ in range(3):                      # repeated calls: counter targets advance
                pt.fit_grid(xg, yg[a:b], a)
            torch.cuda.synchronize()
            pt.check()
            assert torch.equal(pt.table, ref.table), kind
            assert torch.equal(pt.status, ref.status), kind
            assert torch.equal(pt.fit_err, ref.fit_err), kind
            # the collective form side by side: the same local fit, rows all-gathered
            mine = fit_grid(kind, xg, yg[a:b])
            assert torch.equal(ddist.all_gather_rows(mine.table, n_total), pt.table), kind
            assert torch.equal(ddist.all_gather_rows(mine.fit_err, n_total), pt.fit_err), kind
            dist.barrier()
        dist.barrier()
        q.put((rank, "ok"))
    except Exception as exc:  # surface the failure to the parent
        import traceback

        q.put((rank, repr(exc) + traceback.format_exc()[-1500:]))
        raise
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def _slice_packed(packed, a: int, b: int):
    """Records [a, b) of a packed batch (the string/digest tables are shared)."""
    from dataclasses import replace

    off = packed.rec_off                      # n start offsets into words
    w0 = int(off[a])
    w1 = int(off[b]) if b < packed.n else packed.words.shape[0]
    return replace(packed, words=packed.words[w0:w1].copy(), rec_off=(off[a:b] - w0).copy(),
                   repeat=packed.repeat[a:b].copy())


@pytest.mark.parametrize("world", [2, 8])
def test_ranks_one_gpu_sharded_dedup_and_fit(world):
    """world 8 maps DOOLY_MAX_PEERS = 7 peers per rank (the 8-GPU box case)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    results = dict(q.get(timeout=5) for _ in range(world))
    assert results == {r: "ok" for r in range(world)}, results
    assert all(p.exitcode == 0 for p in procs)


@pytest.mark.parametrize("world,allgather", [(2, "fused"), (8, "fused"), (2, "collective")])
def test_bench_ranks_torchrun(world, allgather):
    """bench.py's N > 1 path end to end (barriers, max-over-ranks timing, the
    fit-table and digest all-gathers, replica-sharded sim) at small sizes: the
    C5 signature set split across the ranks, every rank's queries served from
    the full gathered table."""
    env = dict(os.environ, DOOLY_DIST_BACKEND="gloo", DOOLY_FIT_ALLGATHER=allgather)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(ROOT / "bench.py"),
           "--gpus", str(world), "--steps", "3", "--warmup", "3", "--queries", "4000000",
           "--sigs", "20000", "--points", "512", "--records", "100000",
           "--e2e-queries", "2000000", "--sim-requests", "20000", "--sim-shards", "16",
           "--sim-wide-shards", "0", "--csr-fit", "0"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == world and d["value"] > 0 and d["scaling"] == "weak"
    assert d["fits"]["all_fitted"] and not d["unknown_signature_errors"]
    assert d["fits"]["allgather_path"].startswith("fused" if allgather == "fused" else "NCCL")
    assert d["fits"]["signatures"] == 20_000 and d["fits"]["signatures_per_gpu"] == 20_000 // world
    assert d["dedup"]["exchange"].startswith(
        "owner-routed" if world >= 4 else "fused" if allgather == "fused" else "NCCL")
    assert d["dedup"]["records_per_gpu"] == 100_000 and d["dedup"]["unique"] > 0
    assert d["sim"]["all_ok"] and d["sim"]["requests"] == 20_000
