"""World-size-2 gloo tests of the multi-GPU exchange logic (paper_2605_07985_b200.dist)
on CPU tensors: the same collectives the GPU path runs over NCCL."""

from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, q) -> None:
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    try:
        from helpers import AFFINE, ATTN, synth_fit_data
        from oracle import profiler as oprof
        from oracle import sim as osim
        from paper_2605_07985_b200 import dist as ddist

        dist.init_process_group("gloo", rank=rank, world_size=world)
        assert ddist.world() == (rank, world)
        # 1. uneven contiguous split of rows, gathered back in order
        n = 11
        full = torch.arange(n * 3, dtype=torch.int64).reshape(n, 3)
        a, b = ddist.shard_range(n, rank, world)
        got = ddist.all_gather_rows(full[a:b].clone(), n)
        assert torch.equal(got, full)
        # 2. dedup exchange: hash the local slice, gather digests, resolve globally
        rng = np.random.default_rng(0)
        pool = [bytes(rng.integers(0, 256, 32, dtype=np.uint8)) for _ in range(40)]
        digs = [pool[i] for i in rng.integers(0, 40, size=101)]
        a, b = ddist.shard_range(len(digs), rank, world)
        local = torch.from_numpy(np.frombuffer(b"".join(digs[a:b]), np.uint8).reshape(-1, 32).copy())
        gathered = ddist.all_gather_rows(local, len(digs))
        res = oprof.dedup_digests([bytes(r) for r in gathered.numpy()])
        ref = oprof.dedup_digests(digs)
        assert res["first"][a:b] == ref["first"][a:b] and res["uid"] == ref["uid"]
        # 3. fit exchange: each rank fits its signature range, rows all-gathered
        for kind in (AFFINE, ATTN):
            x, y, off = synth_fit_data(kind, 9, 40, seed=kind)
            a, b = ddist.shard_range(9, rank, world)
            xs, ys, lo = ddist.csr_slice(torch.from_numpy(x), torch.from_numpy(y), off, a, b)
            part = osim.fit(kind, xs.numpy(), ys.numpy(), lo)
            coef = ddist.all_gather_rows(torch.from_numpy(part["coef"]), 9)
            whole = osim.fit(kind, x, y, off)
            assert np.array_equal(coef.numpy(), whole["coef"])
        # 4. per-rank request blocks
        blk = torch.full((5,), float(rank))
        g = ddist.gather_requests(blk)
        assert g.shape == (world, 5) and torch.equal(g[1], torch.ones(5))
        dist.barrier()
        q.put((rank, "ok"))
    except Exception as exc:  # surface the failure to the parent
        q.put((rank, repr(exc)))
        raise
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_two_rank_exchange_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    results = dict(q.get(timeout=5) for _ in range(2))
    assert results == {0: "ok", 1: "ok"}, results
    assert all(p.exitcode == 0 for p in procs)
