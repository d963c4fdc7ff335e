"""In-library communicator and the owner-routed dedup kernels (SURVEY §8(b),
§8(e); include/dooly_b200.h dooly_comm_* and dooly_route_*).

The GPU box hands out one GPU, so NCCL runs here at world size 1 (the
in-place all-gather and the grouped send/recv all-to-all are exercised end to
end through libdooly_b200), and the routed dedup's kernels are checked at
world 3 and 8 by emulating the ranks' exchanges on one device: every rank's
route plan, the owners' resolves, the first-list all-gather, the replies and
the finish run exactly as dist.dedup_routed runs them, with the all-to-alls
replaced by slicing.  The result must equal the single-rank dedup of the
whole list bit for bit (with and without DB keys)."""

from __future__ import annotations

import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_lib_comm_world1_allgather_alltoallv(dev):
    from paper_2605_07985_b200 import _lib
    from paper_2605_07985_b200.errors import CommError

    lib = _lib.load_library()
    idb = (C.c_uint8 * _lib.COMM_ID_BYTES)()
    assert lib.dooly_comm_unique_id(idb) == 0
    h = C.c_void_p()
    assert lib.dooly_comm_init_rank(dev.index, idb, 1, 0, C.byref(h)) == 0
    nr, r0, nl = C.c_int(), C.c_int(), C.c_int()
    assert lib.dooly_comm_size(h, C.byref(nr), C.byref(r0), C.byref(nl)) == 0
    assert (nr.value, r0.value, nl.value) == (1, 0, 1)
    buf = torch.arange(1000, dtype=torch.int64, device=dev)
    want = buf.clone()
    st = (C.c_void_p * 1)(torch.cuda.current_stream(dev).cuda_stream)
    assert lib.dooly_allgather(h, (C.c_void_p * 1)(buf.data_ptr()), 8000, st) == 0
    src = torch.randint(0, 1 << 30, (777, 5), dtype=torch.int64, device=dev)
    dst = torch.empty_like(src)
    cnt = (C.c_int64 * 1)(777)
    assert lib.dooly_alltoallv(h, src.data_ptr(), cnt, dst.data_ptr(), cnt, 40, st[0]) == 0
    torch.cuda.synchronize(dev)
    assert torch.equal(buf, want) and torch.equal(dst, src)
    lib.dooly_comm_destroy(h)
    # single-process form (ncclCommInitAll) over the one device
    h2 = C.c_void_p()
    assert lib.dooly_comm_create(1, (C.c_int * 1)(dev.index), C.byref(h2)) == 0
    lib.dooly_comm_destroy(h2)
    # argument errors are status 1; an NCCL failure maps to CommError (status 7)
    assert lib.dooly_comm_init_rank(dev.index, idb, 2, 5, C.byref(h)) == 1
    with pytest.raises(CommError):
        _lib.check_comm(7, None)


def _owner(d: torch.Tensor, world: int) -> torch.Tensor:
    tail = d[:, 24:32].contiguous().view(torch.int64).reshape(-1)
    return torch.remainder(tail & 0x7FFFFFFFFFFFFFFF, world)


def _plan(lib, ctx, dig, world, gidx0, dev):
    from paper_2605_07985_b200 import _lib

    n = dig.shape[0]
    perm = torch.empty(n, dtype=torch.int64, device=dev)
    counts = torch.empty(world, dtype=torch.int64, device=dev)
    sdig = torch.empty((n, 32), dtype=torch.uint8, device=dev)
    sg = torch.empty(n, dtype=torch.int64, device=dev)
    ws = torch.empty(int(lib.dooly_route_workspace_size(n, world)), dtype=torch.uint8, device=dev)
    _lib.check(lib.dooly_route_plan(ctx, _lib.ptr(dig) if n else 0, n, world, gidx0,
                                    _lib.ptr(perm), counts.data_ptr(), _lib.ptr(sdig),
                                    _lib.ptr(sg), ws.data_ptr(), ws.numel(),
                                    _lib.stream_ptr(dev)), ctx)
    return perm, counts.cpu().tolist(), sdig, sg


def test_route_plan_is_a_stable_owner_bucketing(dev):
    from paper_2605_07985_b200 import _lib

    lib, ctx = _lib.load_library(), _lib.ctx_for(dev)
    g = torch.Generator(device=dev)
    g.manual_seed(3)
    for n, world in ((1, 2), (5000, 3), (70_001, 8), (2048 * 3, 5)):
        dig = torch.randint(0, 256, (n, 32), generator=g, device=dev, dtype=torch.int32).to(torch.uint8)
        perm, counts, sdig, sg = _plan(lib, ctx, dig, world, 1000, dev)
        own = _owner(dig, world)
        want = torch.sort(own, stable=True).indices
        assert torch.equal(perm, want)
        assert counts == torch.bincount(own, minlength=world).cpu().tolist()
        assert torch.equal(sdig, dig[want]) and torch.equal(sg, want + 1000)


@pytest.mark.parametrize("world", [3, 8])
@pytest.mark.parametrize("with_db", [False, True])
def test_routed_dedup_kernels_equal_single_rank(world, with_db, dev):
    """dist.dedup_routed's kernel pipeline with the exchanges emulated on one GPU."""
    import bench
    from paper_2605_07985_b200 import _lib
    from paper_2605_07985_b200 import dist as ddist
    from paper_2605_07985_b200.profiler import DedupWorkspace, DeviceRecords, dedup_packed

    lib, ctx, st = _lib.load_library(), _lib.ctx_for(dev), _lib.stream_ptr(dev)
    n_total = 30_011
    packed, _ = bench.synth_records(n_total, seed=9)
    recs = DeviceRecords.from_packed(packed, dev)
    db = None
    whole = dedup_packed(recs)
    if with_db:
        db = whole.digests[::53].clone()
        whole = dedup_packed(recs, db)
    dig = whole.digests
    ranges = [ddist.shard_range(n_total, r, world) for r in range(world)]
    plans = [_plan(lib, ctx, dig[a:b], world, a, dev) for a, b in ranges]
    dplan = _plan(lib, ctx, db, world, 0, dev) if with_db else None
    # all-to-all 1: owner o receives bucket o of every rank, in rank order
    def bucket(r, o):
        perm, counts, sdig, sg = plans[r]
        s = sum(counts[:o])
        return sdig[s:s + counts[o]], sg[s:s + counts[o]]
    owners = []
    for o in range(world):
        r_dig = torch.cat([bucket(r, o)[0] for r in range(world)])
        r_g = torch.cat([bucket(r, o)[1] for r in range(world)])
        db_own = None
        if with_db:
            dc = dplan[1]
            s = sum(dc[:o])
            db_own = dplan[2][s:s + dc[o]]
        m, n_db = r_dig.shape[0], 0 if db_own is None else db_own.shape[0]
        ws = DedupWorkspace(dev).get(m, n_db)
        first = torch.empty(m, dtype=torch.int64, device=dev)
        uid = torch.empty(m, dtype=torch.int32, device=dev)
        new = torch.empty(m, dtype=torch.uint8, device=dev)
        indb = torch.empty(m, dtype=torch.uint8, device=dev)
        nu = torch.zeros(1, dtype=torch.int64, device=dev)
        _lib.check(lib.dooly_dedup_digests(ctx, _lib.ptr(r_dig), m, _lib.ptr(db_own) if n_db else 0,
                                           n_db, first.data_ptr(), uid.data_ptr(), new.data_ptr(),
                                           indb.data_ptr(), nu.data_ptr(), ws.data_ptr(),
                                           ws.numel(), st), ctx)
        k = int(nu.item())
        firsts = torch.empty(max(k, 1), dtype=torch.int64, device=dev)
        _lib.check(lib.dooly_dedup_firsts(ctx, m, n_db, r_g.data_ptr(), firsts.data_ptr(),
                                          ws.data_ptr(), ws.numel(), st), ctx)
        owners.append((r_g, first, new, indb, firsts[:k]))
    per = max(1, max(o[4].numel() for o in owners))
    all_firsts = torch.full((world, per), torch.iinfo(torch.int64).max, dtype=torch.int64, device=dev)
    for o, ow in enumerate(owners):
        all_firsts[o, :ow[4].numel()] = ow[4]
    assert sum(o[4].numel() for o in owners) == whole.n_unique
    replies = []
    for r_g, first, new, indb, _ in owners:
        m = r_g.shape[0]
        rows = torch.empty((m, 3), dtype=torch.int64, device=dev)
        _lib.check(lib.dooly_route_reply(ctx, r_g.data_ptr(), first.data_ptr(), new.data_ptr(),
                                         indb.data_ptr(), m, all_firsts.data_ptr(), per, world,
                                         rows.data_ptr(), st), ctx)
        replies.append(rows)
    # all-to-all 2: rank r gets, from each owner in order, the rows of its bucket
    for r, (a, b) in enumerate(ranges):
        blocks = []
        for o in range(world):
            off = sum(plans[q][1][o] for q in range(r))
            blocks.append(replies[o][off:off + plans[r][1][o]])
        back = torch.cat(blocks)
        n = b - a
        out = [torch.empty(n, dtype=torch.int64, device=dev), torch.empty(n, dtype=torch.int32, device=dev),
               torch.empty(n, dtype=torch.uint8, device=dev), torch.empty(n, dtype=torch.uint8, device=dev)]
        _lib.check(lib.dooly_route_finish(ctx, back.data_ptr(), plans[r][0].data_ptr(), n,
                                          *[t.data_ptr() for t in out], st), ctx)
        assert torch.equal(out[0], whole.first[a:b])
        assert torch.equal(out[1], whole.uid[a:b])
        assert torch.equal(out[2], whole.is_new[a:b])
        assert torch.equal(out[3], whole.in_db[a:b])
