"""Multi-GPU partitioning of the hot path: one process per GPU,
``torch.distributed`` (NCCL over NVLink on the GPU box, gloo in CPU tests) for
the plumbing.

  dedup   records split contiguously by global index; each rank hashes its own
          slice (the ALU-bound part), ONE all-gather of the 32-B digests, then
          every rank resolves first occurrences over the full digest list (exact
          for any world size) and keeps its slice.
  fit     signatures split into contiguous ranges, no communication during the
          fit, ONE all-gather of the fitted regressor rows (p*8 + box bytes per
          signature) so every rank holds the full table.  On GPUs with peer
          access (NVLink/NVSwitch) the all-gather is fused into the fit:
          ``PeerFitTable`` maps every rank's table into every other rank (CUDA
          IPC) and dooly_fit_grid_bcast's epilogue stores each row into all of
          them, then a device-side arrival counter replaces the collective.
  predict queries split contiguously; no collective (each rank holds the table).
  sim     S fixed replica shards, shard s on rank s mod world ("replicas only",
          no data-path collective); per-request TTFT/TPOT gathered at the end.

Data-path collectives on GPUs go through the NCCL communicator INSIDE
libdooly_b200 (``LibComm``: dooly_comm_init_rank / dooly_allgather /
dooly_alltoallv); torch.distributed is the bootstrap only (it ships the
128-byte NCCL id) and the gloo host path of the CPU tests and of several
ranks sharing one GPU.  DOOLY_COMM=torch switches the GPU path to
torch.distributed's own NCCL collectives (side-by-side checks).
"""

from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np
import torch
import torch.distributed as dist


def world() -> tuple:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def local_device() -> torch.device:
    """This rank's GPU: LOCAL_RANK, folded onto the visible devices (so a
    multi-rank smoke test can share one GPU under the gloo backend)."""
    n = max(1, torch.cuda.device_count())
    return torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")) % n)


def init_from_env(backend: Optional[str] = None) -> tuple:
    """Initialise the default group from torchrun's env (127.0.0.1 rendezvous).

    Backend: NCCL on GPUs unless DOOLY_DIST_BACKEND overrides it (gloo is used
    by the CPU tests and for several ranks sharing one GPU)."""
    if int(os.environ.get("WORLD_SIZE", "1")) > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = backend or os.environ.get("DOOLY_DIST_BACKEND") or (
            "nccl" if torch.cuda.is_available() else "gloo")
        if torch.cuda.is_available():
            torch.cuda.set_device(local_device())
        dist.init_process_group(backend=backend)
    return world()


def shard_range(n: int, rank: int, size: int) -> tuple:
    """Contiguous split of [0, n): the first n % size ranks get one extra."""
    q, r = divmod(n, size)
    a = rank * q + min(rank, r)
    return a, a + q + (1 if rank < r else 0)


def all_gather_rows(local: torch.Tensor, n_total: int, group=None) -> torch.Tensor:
    """Concatenate per-rank row blocks of a contiguous split of n_total rows.

    Blocks differ by at most one row; they are padded to ceil(n/size) rows for
    a single all_gather_into_tensor, then trimmed."""
    rank, size = world()
    if size == 1:
        return local
    per = -(-n_total // size)
    pad = torch.zeros((per,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    out = _gather_cat(pad, size, group)
    keep = [out[r * per: r * per + (shard_range(n_total, r, size)[1] -
                                    shard_range(n_total, r, size)[0])] for r in range(size)]
    return torch.cat(keep, dim=0)


def csr_slice(x: torch.Tensor, y: torch.Tensor, off: np.ndarray, a: int, b: int):
    """Signatures [a, b) of a CSR batch -> (x, y, rebased offsets) views."""
    p0, p1 = int(off[a]), int(off[b])
    return x[:, p0:p1].contiguous(), y[p0:p1].contiguous(), off[a:b + 1] - off[a]


def fit_sharded(kind: int, x: torch.Tensor, y: torch.Tensor, off: np.ndarray, group=None):
    """Fit this rank's contiguous signature range, all-gather the regressor rows."""
    from .sim import FitResult, fit_tables

    rank, size = world()
    n_sig = len(off) - 1
    a, b = shard_range(n_sig, rank, size)
    xs, ys, lo = csr_slice(x, y, off, a, b)
    local = fit_tables(kind, xs, ys, torch.from_numpy(np.ascontiguousarray(lo)).to(y.device))
    if size == 1:
        return local
    return FitResult(kind, all_gather_rows(local.table, n_sig, group),
                     all_gather_rows(local.fit_err, n_sig, group),
                     all_gather_rows(local.status, n_sig, group))


def dedup_sharded(recs_local, n_total: int, db_digests: Optional[torch.Tensor] = None,
                  workspace=None, group=None, peer_digests: Optional["PeerDigests"] = None):
    """Hash the local records, all-gather digests, dedup globally, keep local slice.

    With ``peer_digests`` the hash kernel itself stores every digest into all
    ranks' gathered arrays (fused hash + all-gather) instead of an NCCL call."""
    from .profiler import DedupResult, dedup_digests, hash_records

    rank, size = world()
    if peer_digests is not None:
        full = peer_digests.hash(recs_local, shard_range(n_total, rank, size)[0])
    else:
        local = hash_records(recs_local)
        full = all_gather_rows(local, n_total, group) if size > 1 else local
    res = dedup_digests(full, db_digests, workspace, sync=True)
    a, b = shard_range(n_total, rank, size)
    return DedupResult(res.digests[a:b], res.first[a:b], res.uid[a:b], res.is_new[a:b],
                       res.in_db[a:b], res.n_unique)


def owner_of(digests: torch.Tensor, size: int) -> torch.Tensor:
    """Owning rank of each 32-byte digest: the last 8 bytes modulo the world
    size (the dedup hash table probes the first bytes, so an owner's keys
    still spread over its whole table)."""
    tail = digests[:, 24:32].contiguous().view(torch.int64).reshape(-1)
    return torch.remainder(tail & 0x7FFFFFFFFFFFFFFF, size)


class LibComm:
    """The NCCL communicator inside libdooly_b200 for this process's GPU
    (include/dooly_b200.h dooly_comm_*).  Collective: every rank of the group
    constructs it together (rank 0's NCCL id reaches the others through
    torch.distributed, the bootstrap)."""

    def __init__(self, device: torch.device, group=None):
        from . import _lib

        rank, size = world()
        lib = _lib.load_library()
        idb = (C.c_uint8 * _lib.COMM_ID_BYTES)()
        if rank == 0:
            _lib.check_comm(lib.dooly_comm_unique_id(idb), None)
        box = [bytes(idb)]
        if size > 1:
            dist.broadcast_object_list(box, src=0, group=group)
        idb = (C.c_uint8 * _lib.COMM_ID_BYTES).from_buffer_copy(box[0])
        h = C.c_void_p()
        _lib.check_comm(lib.dooly_comm_init_rank(device.index, idb, size, rank, C.byref(h)), None)
        self.handle, self.rank, self.size, self.device = h, rank, size, device

    def allgather(self, t: torch.Tensor) -> torch.Tensor:
        """Equal-shape per-rank blocks concatenated on dim 0 (dooly_allgather, in place)."""
        from . import _lib

        t = t.contiguous()
        out = torch.empty((t.shape[0] * self.size,) + tuple(t.shape[1:]), dtype=t.dtype,
                          device=t.device)
        nb = t.numel() * t.element_size()
        out.view(-1)[self.rank * t.numel():(self.rank + 1) * t.numel()].copy_(t.view(-1))
        bufs = (C.c_void_p * 1)(out.data_ptr())
        streams = (C.c_void_p * 1)(_lib.stream_ptr(self.device))
        _lib.check_comm(_lib.load_library().dooly_allgather(self.handle, bufs, nb, streams),
                        self.handle)
        return out

    def alltoallv(self, t: torch.Tensor, send: list, recv: list) -> torch.Tensor:
        """Rows of ``t`` split by ``send`` counts to the ranks; ``recv`` rows back."""
        from . import _lib

        t = t.contiguous()
        row = int(np.prod(t.shape[1:], dtype=np.int64)) * t.element_size()
        out = torch.empty((sum(recv),) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        sc = (C.c_int64 * self.size)(*send)
        rc = (C.c_int64 * self.size)(*recv)
        _lib.check_comm(_lib.load_library().dooly_alltoallv(
            self.handle, t.data_ptr() if t.numel() else 0, sc,
            out.data_ptr() if out.numel() else 0, rc, max(row, 1),
            _lib.stream_ptr(self.device)), self.handle)
        return out

    def close(self) -> None:
        from . import _lib

        if self.handle:
            _lib.load_library().dooly_comm_destroy(self.handle)
            self.handle = None


_COMMS: dict = {}


def lib_comm(device: torch.device, group=None):
    """This process's LibComm for ``group`` (created on first use, collectively),
    or None when the data path uses torch.distributed (gloo, or DOOLY_COMM=torch)."""
    if dist.get_backend(group) != "nccl" or os.environ.get("DOOLY_COMM", "lib") == "torch":
        return None
    key = (device.index, id(group))
    if key not in _COMMS:
        _COMMS[key] = LibComm(device, group)
    return _COMMS[key]


def _all_to_all(t: torch.Tensor, send: list, recv: list, group=None) -> torch.Tensor:
    """all-to-all on dim 0 with per-rank split sizes: libdooly's NCCL
    (dooly_alltoallv) on GPUs, torch's NCCL under DOOLY_COMM=torch, gloo
    through host memory."""
    out_shape = (sum(recv),) + tuple(t.shape[1:])
    if dist.get_backend(group) == "nccl":
        comm = lib_comm(t.device, group)
        if comm is not None:
            return comm.alltoallv(t, send, recv)
        out = torch.empty(out_shape, dtype=t.dtype, device=t.device)
        dist.all_to_all_single(out, t.contiguous(), recv, send, group=group)
        return out
    h = t.contiguous().cpu()
    out = torch.empty(out_shape, dtype=t.dtype)
    dist.all_to_all_single(out, h, recv, send, group=group)
    return out.to(t.device)


def dedup_routed(recs_local, n_total: int, db_digests: Optional[torch.Tensor] = None,
                 workspace=None, group=None):
    """Multi-GPU dedup with owner routing: each digest goes to the
    rank that owns it, so every rank resolves ~n_total / world keys instead of
    all of them (the all-gather form resolves the whole list on every rank).
    Every data step is a libdooly kernel (route.cu); the exchanges are the
    communicator's all-to-alls / all-gathers:

      1. hash the local records (K1a);
      2. dooly_route_plan: stable bucket of (digest, global index) by owner;
         all-to-all to the owners — a rank's bucket keeps its records' order
         and ranks send in rank order, so what an owner receives is in
         global order;
      3. the owner resolves its keys (K1b, with its planned share of the DB
         keys) — every copy of a digest is there, so first occurrence, DB
         membership and is_new are exact — and lists its first occurrences'
         global indices (dooly_dedup_firsts);
      4. the owners' sorted first lists are all-gathered; dooly_route_reply
         gives each received record its global first index, its global uid
         (first occurrences over all owners with a smaller global index) and
         flags;
      5. all-to-all of the replies back; dooly_route_finish scatters them
         through the plan's permutation.
    Bit-identical to the single-rank dedup of the whole list."""
    from . import _lib
    from .profiler import DedupResult, DedupWorkspace, hash_records

    rank, size = world()
    dev = recs_local.words.device
    lib = _lib.load_library()
    ctx = _lib.ctx_for(dev)
    st = _lib.stream_ptr(dev)
    a, _ = shard_range(n_total, rank, size)

    def plan(dig, gidx0):
        n = dig.shape[0]
        perm = torch.empty(n, dtype=torch.int64, device=dev)
        counts = torch.empty(size, dtype=torch.int64, device=dev)
        sdig = torch.empty((n, 32), dtype=torch.uint8, device=dev)
        sgidx = torch.empty(n, dtype=torch.int64, device=dev)
        ws = torch.empty(int(lib.dooly_route_workspace_size(n, size)), dtype=torch.uint8,
                         device=dev)
        _lib.check(lib.dooly_route_plan(ctx, _lib.ptr(dig) if n else 0, n, size, gidx0,
                                        _lib.ptr(perm), counts.data_ptr(), _lib.ptr(sdig),
                                        _lib.ptr(sgidx), ws.data_ptr(), ws.numel(), st), ctx)
        return perm, counts, sdig, sgidx

    dig = hash_records(recs_local)
    n = dig.shape[0]
    perm, counts, sdig, sgidx = plan(dig, a)
    send = counts.cpu().tolist()                         # host counts for the exchange
    recv = _all_to_all(counts, [1] * size, [1] * size, group).cpu().tolist()
    r_dig = _all_to_all(sdig, send, recv, group)
    r_gidx = _all_to_all(sgidx, send, recv, group)
    db_own = None
    if db_digests is not None and db_digests.shape[0]:
        _, dcounts, ddig, _ = plan(db_digests.contiguous(), 0)
        dc = dcounts.cpu().tolist()
        o = sum(dc[:rank])
        db_own = ddig[o:o + dc[rank]]
    n_db = 0 if db_own is None else db_own.shape[0]
    m = r_dig.shape[0]
    ws = (workspace or DedupWorkspace(dev)).get(m, n_db)
    first = torch.empty(m, dtype=torch.int64, device=dev)
    uid = torch.empty(m, dtype=torch.int32, device=dev)
    is_new = torch.empty(m, dtype=torch.uint8, device=dev)
    in_db = torch.empty(m, dtype=torch.uint8, device=dev)
    n_unique = torch.zeros(1, dtype=torch.int64, device=dev)
    _lib.check(lib.dooly_dedup_digests(
        ctx, _lib.ptr(r_dig) if m else 0, m, _lib.ptr(db_own) if n_db else 0, n_db,
        _lib.ptr(first), _lib.ptr(uid), _lib.ptr(is_new), _lib.ptr(in_db), n_unique.data_ptr(),
        ws.data_ptr(), ws.numel(), st), ctx)
    n_first = int(n_unique.item())
    firsts = torch.empty(max(n_first, 1), dtype=torch.int64, device=dev)
    _lib.check(lib.dooly_dedup_firsts(ctx, m, n_db, _lib.ptr(r_gidx) if m else 0,
                                      firsts.data_ptr(), ws.data_ptr(), ws.numel(), st), ctx)
    all_counts = _gather_cat(n_unique, size, group)
    per = max(1, int(all_counts.max().item()))
    pad = torch.full((per,), torch.iinfo(torch.int64).max, dtype=torch.int64, device=dev)
    pad[:n_first] = firsts[:n_first]
    all_firsts = _gather_cat(pad, size, group)
    rows = torch.empty((m, 3), dtype=torch.int64, device=dev)
    _lib.check(lib.dooly_route_reply(ctx, _lib.ptr(r_gidx) if m else 0, _lib.ptr(first),
                                     _lib.ptr(is_new), _lib.ptr(in_db), m, all_firsts.data_ptr(),
                                     per, size, _lib.ptr(rows), st), ctx)
    back = _all_to_all(rows, recv, send, group)
    out_first = torch.empty(n, dtype=torch.int64, device=dev)
    out_uid = torch.empty(n, dtype=torch.int32, device=dev)
    out_new = torch.empty(n, dtype=torch.uint8, device=dev)
    out_db = torch.empty(n, dtype=torch.uint8, device=dev)
    _lib.check(lib.dooly_route_finish(ctx, _lib.ptr(back) if n else 0, _lib.ptr(perm), n,
                                      _lib.ptr(out_first), _lib.ptr(out_uid), _lib.ptr(out_new),
                                      _lib.ptr(out_db), st), ctx)
    return DedupResult(dig, out_first, out_uid, out_new, out_db, int(all_counts.sum().item()))


def gather_requests(values: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather equally sized per-rank vectors (e.g. padded TTFT blocks)."""
    rank, size = world()
    if size == 1:
        return values
    return _gather_cat(values.contiguous(), size, group).view((size,) + tuple(values.shape))


def _gather_cat(t: torch.Tensor, size: int, group=None) -> torch.Tensor:
    """all_gather of equal-shape tensors concatenated on dim 0 (one NCCL call:
    libdooly's dooly_allgather, or torch's under DOOLY_COMM=torch)."""
    if dist.get_backend(group) == "nccl":
        comm = lib_comm(t.device, group)
        if comm is not None:
            return comm.allgather(t)
        out = torch.empty((t.shape[0] * size,) + tuple(t.shape[1:]), dtype=t.dtype,
                          device=t.device)
        dist.all_gather_into_tensor(out, t, group=group)
        return out
    # gloo (CPU tests; several ranks sharing one GPU): exchange through host memory
    h = t.cpu()
    parts = [torch.empty_like(h) for _ in range(size)]
    dist.all_gather(parts, h, group=group)
    return torch.cat(parts, dim=0).to(t.device)


class PeerFitTable:
    """Full regressor table replicated on every rank and written in place by every
    rank's fit (dooly_fit_grid_bcast): the fused fit + all-gather.

    Each rank allocates the full (n_total rows) table, fit_err, status and a u32
    arrival counter, shares them with the other ranks through CUDA IPC (torch's
    tensor-sharing reductions, handles exchanged once with all_gather_object),
    and hands the peers' mapped device pointers to the kernel.  ``fit_grid``
    fits this rank's rows [row0, row0 + n) and returns when (on the stream) all
    ranks' rows have landed.  Needs peer access between every pair of GPUs
    (``available``); callers use ``fit_sharded``/NCCL otherwise."""

    def __init__(self, kind: int, n_total: int, device: torch.device, group=None):
        from . import _lib

        self.kind, self.n_total, self.device = kind, n_total, device
        rank, size = world()
        self.rank, self.size = rank, size
        if size - 1 > _lib.MAX_PEERS:
            raise ValueError(f"at most {_lib.MAX_PEERS + 1} ranks per fused fit")
        self.table = torch.zeros((n_total, _lib.ROW_BYTES[kind]), dtype=torch.uint8, device=device)
        self.fit_err = torch.zeros(n_total, dtype=torch.float64, device=device)
        self.status = torch.zeros(n_total, dtype=torch.uint8, device=device)
        self.flag = torch.zeros(4, dtype=torch.int32, device=device)   # [0] arrivals
        self.timed_out = torch.zeros(1, dtype=torch.int32, device=device)
        self._peer_tensors = _share_with_peers(
            [self.table, self.fit_err, self.status, self.flag], group)   # keeps mappings alive
        pe = _lib.GridPeers()
        pe.n_peers = size - 1
        for j, ts in enumerate(self._peer_tensors):
            pe.table[j], pe.fit_err[j], pe.status[j], pe.flag[j] = (t.data_ptr() for t in ts)
        self._peers = pe
        self.calls = 0

    available = staticmethod(lambda size: peer_access_available(size))

    def fit_grid(self, x: torch.Tensor, y: torch.Tensor, row0: int):
        """Fit y's signatures as global rows [row0, row0 + len(y)) into every
        rank's table; returns self once the stream has seen all ranks arrive."""
        from . import _lib
        from .sim import _grid_workspace

        n_sig, n_pts = y.shape
        if row0 < 0 or row0 + n_sig > self.n_total:
            raise ValueError("rows outside the shared table")
        if x.shape != (_lib.PLANES[self.kind], n_pts):
            raise ValueError(f"x must have shape ({_lib.PLANES[self.kind]}, {n_pts})")
        x, y = x.contiguous(), y.contiguous()
        self.calls += 1
        self._peers.row0 = row0
        lib = _lib.load_library()
        ws = _grid_workspace(self.device, self.kind, n_pts)
        ctx = _lib.ctx_for(self.device)
        _lib.check(lib.dooly_fit_grid_bcast(
            ctx, self.kind, x.data_ptr() if x.numel() else 0, n_pts,
            y.data_ptr() if y.numel() else 0, n_sig, self.table.data_ptr(),
            self.fit_err.data_ptr(), self.status.data_ptr(), C.byref(self._peers),
            self.flag.data_ptr(), (self.calls * self.size) & 0xFFFFFFFF,
            self.timed_out.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr(self.device)),
            ctx)
        return self

    def check(self) -> None:
        """Raise if a wait gave up (a peer never arrived); synchronises."""
        if int(self.timed_out.item()):
            raise RuntimeError("fused fit all-gather: a peer rank never signalled (timeout)")


def peer_access_available(size: int) -> bool:
    """Peer access between every pair of the GPUs ``size`` ranks use (a single
    GPU shared by several ranks maps its own memory and qualifies)."""
    n = torch.cuda.device_count()
    if n == 0:
        return False
    devs = sorted({r % n for r in range(size)})
    return all(torch.cuda.can_device_access_peer(a, b) for a in devs for b in devs if a != b)


def _share_with_peers(tensors, group=None) -> list:
    """CUDA-IPC map this rank's ``tensors`` into every other rank (torch's
    tensor-sharing reductions; handles exchanged once with all_gather_object).
    Returns, for each other rank in rank order, its tensors mapped here."""
    from torch.multiprocessing.reductions import reduce_tensor

    from . import _lib

    rank, size = world()
    dev = tensors[0].device
    torch.cuda.synchronize(dev)
    mine = (dev.index, [reduce_tensor(t) for t in tensors])
    handles = [None] * size
    if size > 1:
        dist.all_gather_object(handles, mine, group=group)
    err = None
    try:
        # the fused epilogues run on THIS device and store into the peers'
        # buffers: enable access from here to every peer device (torch opens
        # the IPC handles under the exporting device, which does not)
        ctx = _lib.ctx_for(dev)
        for r in range(size):
            if r != rank and handles[r][0] != dev.index:
                _lib.check(_lib.load_library().dooly_enable_peer_access(ctx, handles[r][0]), ctx)
        peers = [[fn(*args) for fn, args in handles[r][1]] for r in range(size) if r != rank]
    except Exception as exc:  # e.g. IPC not permitted: every rank must learn it together
        peers, err = None, exc
    if size > 1:   # agree on success so no rank is left waiting in a later collective
        ok = torch.tensor([0 if err else 1], dtype=torch.int32,
                          device=tensors[0].device if dist.get_backend(group) == "nccl" else "cpu")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if int(ok.item()) == 0:
            raise RuntimeError(f"peer mapping failed on some rank: {err!r}")
    return peers


class PeerDigests:
    """Gathered digest array replicated on every rank and written in place by
    every rank's hash kernel (dooly_sha256_records_bcast): the fused
    hash + all-gather step of the multi-GPU dedup."""

    def __init__(self, n_total: int, device: torch.device, group=None):
        from . import _lib

        rank, size = world()
        if size - 1 > _lib.MAX_PEERS:
            raise ValueError(f"at most {_lib.MAX_PEERS + 1} ranks per fused hash")
        self.n_total, self.device, self.size = n_total, device, size
        self.digests = torch.zeros((n_total, 32), dtype=torch.uint8, device=device)
        self.flag = torch.zeros(4, dtype=torch.int32, device=device)
        self.timed_out = torch.zeros(1, dtype=torch.int32, device=device)
        self._peer_tensors = _share_with_peers([self.digests, self.flag], group)
        pe = _lib.DigestPeers()
        pe.n_peers = size - 1
        for j, (d, f) in enumerate(self._peer_tensors):
            pe.digest[j], pe.flag[j] = d.data_ptr(), f.data_ptr()
        self._peers = pe
        self.calls = 0

    def hash(self, recs, row0: int) -> torch.Tensor:
        """Hash this rank's records as global rows [row0, row0 + recs.n) into every
        rank's array; returns the full (n_total, 32) digests once (on the stream)
        all ranks have arrived."""
        from . import _lib

        if row0 < 0 or row0 + recs.n > self.n_total:
            raise ValueError("records outside the gathered digest array")
        self.calls += 1
        self._peers.row0 = row0
        ctx = _lib.ctx_for(self.device)
        _lib.check(_lib.load_library().dooly_sha256_records_bcast(
            ctx, recs.words.data_ptr(), recs.rec_off.data_ptr(), recs.n,
            recs.op_bytes.data_ptr(), recs.op_off.data_ptr(), recs.op_off.numel() - 1,
            recs.sym_bytes.data_ptr(), recs.sym_off.data_ptr(), recs.sym_off.numel() - 1,
            recs.attr_digests.data_ptr(), recs.attr_digests.numel() // 32,
            self.digests.data_ptr(), C.byref(self._peers), self.flag.data_ptr(),
            (self.calls * self.size) & 0xFFFFFFFF, self.timed_out.data_ptr(),
            _lib.stream_ptr(self.device)), ctx)
        return self.digests

    def check(self) -> None:
        if int(self.timed_out.item()):
            raise RuntimeError("fused hash all-gather: a peer rank never signalled (timeout)")
