"""Multi-GPU layer: cell-range sharding, diagnostics reduction, particle migration.

SURVEY §8(e).  Cells never interact in this operator ("we only consider
collisions between two particles in the same grid cell"), so the
global grid is split into contiguous cell ranges, one per rank, and every
particle lives on the rank that owns its cell.  ``coulomb_collide`` then runs
locally with ``cell_base`` = the rank's first global cell: the random streams
are keyed by the global cell id, so each shard reproduces the single-GPU
result on the same particles (the hard form of the paper's "nearly identical
regardless of how many MPI processes").  Unlike the paper's
replicated-grid scheme (one O(M) MPI_AllReduce per step) the data
path has no collective; NCCL carries only

  * the 16-double diagnostics vector: all_gather + a rank-ascending sum on the
    device (deterministic for a given world size), and
  * particle migration when a pusher moves particles across shard boundaries:
    a stable partition by owner rank (the binning kernels with key = owner),
    an all_to_all of the counts, and an all_to_all of the packed particles;
    arrivals are appended in source-rank order, so results stay deterministic.

The communication/plan logic here is device-agnostic (it runs on CPU tensors
with the gloo backend in the tests); the per-particle work (partition, pack,
ordered sum) is done by the CUDA kernels behind ``ops`` — the tests inject
CPU stand-ins for those, the product path always uses the CUDA ones.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import torch
import torch.distributed as dist


def shard_cells(global_cells: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced cell range of `rank`: (cell_base, local_cells)."""
    if world < 1 or not (0 <= rank < world) or global_cells < world:
        raise ValueError("need 0 <= rank < world <= global_cells")
    q, r = divmod(global_cells, world)
    base = rank * q + min(rank, r)
    return base, q + (1 if rank < r else 0)


def owner_bounds(global_cells: int, world: int) -> list[int]:
    """bounds[r] = first global cell of rank r; bounds[world] = global_cells."""
    return [shard_cells(global_cells, world, r)[0] for r in range(world)] + [global_cells]


@dataclass
class DistOps:
    """Per-particle kernels the layer needs (CUDA by default)."""
    partition: Callable   # (key int32 [n], nkeys) -> (perm int32 [n], off int32 [nkeys+1]), stable
    gather: Callable      # (v [3][n], cell [n], perm [n], cell_shift) -> (v [3][n], cell [n]) permuted
    sum_ranks: Callable   # (gathered [P][16]) -> [16] rank-ascending sum
    owner: Callable       # (cell_global int32 [n], bounds list) -> owner rank int32 [n]; dead (-1) -> -1
    p2c: Optional[Callable] = None          # (v, cell, cells, sub) -> raw sums [cells][7] (NEXT f4)
    p2c_moments: Optional[Callable] = None  # (raw [cells][7], weight, cell_volume) -> moments [cells][7]
    nccl: Optional["NcclComm"] = None       # the library's own NCCL communicator (C ABI cc_dist_*), or
                                            # None: torch.distributed collectives (gloo tests)


class NcclComm:
    """An NCCL communicator owned by the C library (cc_nccl_comm_init): rank 0 draws the
    unique id, torch.distributed broadcasts it, every rank joins.  Used by reduce_diag /
    migrate through the C ABI entries cc_dist_diag_reduce / cc_dist_alltoall_counts /
    cc_dist_exchange (grouped ncclSend / ncclRecv)."""

    def __init__(self, group=None):
        import ctypes as C
        from . import _lib
        L = _lib.load()
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        uid = (C.c_char * _lib.CC_NCCL_ID_BYTES)()
        if self.rank == 0:
            _lib.check(L.cc_nccl_get_unique_id(uid), "cc_nccl_get_unique_id")
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0, group=group)
        uid = (C.c_char * _lib.CC_NCCL_ID_BYTES).from_buffer_copy(obj[0])
        self.comm = C.c_void_p()
        _lib.check(L.cc_nccl_comm_init(C.byref(self.comm), self.world, self.rank, uid), "cc_nccl_comm_init")

    def close(self):
        from . import _lib
        if self.comm:
            _lib.check(_lib.load().cc_nccl_comm_destroy(self.comm), "cc_nccl_comm_destroy")
            self.comm = None

    @staticmethod
    def _stream(t):
        import ctypes as C
        return C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)

    def diag_reduce(self, diag: torch.Tensor) -> torch.Tensor:
        import ctypes as C
        from . import _lib
        out = diag.contiguous().clone()
        scratch = torch.empty((self.world, out.numel()), dtype=out.dtype, device=out.device)
        _lib.check(_lib.load().cc_dist_diag_reduce(C.c_void_p(out.data_ptr()), C.c_void_p(scratch.data_ptr()),
                                                   self.comm, self._stream(out)), "cc_dist_diag_reduce")
        return out

    def alltoall_counts(self, send: torch.Tensor) -> torch.Tensor:
        import ctypes as C
        from . import _lib
        recv = torch.empty_like(send)
        _lib.check(_lib.load().cc_dist_alltoall_counts(C.c_void_p(send.data_ptr()), C.c_void_p(recv.data_ptr()),
                                                       self.comm, self._stream(send)), "cc_dist_alltoall_counts")
        return recv

    def exchange(self, send: torch.Tensor, recv: torch.Tensor, send_off: list, recv_off: list) -> None:
        """rows of send [r][lds] -> recv [r][ldr] by the per-rank offsets (host lists)."""
        import ctypes as C
        import numpy as np
        from . import _lib
        so = np.asarray(send_off, dtype=np.int64)
        ro = np.asarray(recv_off, dtype=np.int64)
        s2 = send.reshape(-1, send.shape[-1]) if send.dim() > 1 else send.reshape(1, -1)
        r2 = recv.reshape(-1, recv.shape[-1]) if recv.dim() > 1 else recv.reshape(1, -1)
        _lib.check(_lib.load().cc_dist_exchange(
            C.c_void_p(s2.data_ptr()), s2.stride(0) if s2.shape[1] > 0 else 0, C.c_void_p(r2.data_ptr()),
            r2.stride(0) if r2.shape[1] > 0 else 0, s2.shape[0], s2.element_size(), so.ctypes.data_as(C.c_void_p),
            ro.ctypes.data_as(C.c_void_p), self.comm, self._stream(send)), "cc_dist_exchange")


class Migrator:
    """Device-side particle migration between cell-range shards, no host synchronisation
    (C ABI cc_mig_pack -> cc_dist_mig_exchange -> cc_mig_unpack).

    The rank's particles live in ``n`` fixed slots, dead-padded (cell -1): after a
    ``coulomb_collide`` call the live ones are in [0, L) (L = its diag_out[0]) and the
    dead in [L, n).  ``__call__(v, x, cell, diag)`` takes the cell ids as GLOBAL ids
    (a push's output), sends every particle owned by another rank in a fixed-capacity
    slot (``cap`` particles per peer; the message size never depends on a count, so
    nothing is read back to the host), marks it dead here, converts the stayers' ids to
    LOCAL ones and appends the arrivals in (source rank, source order) at [L, L + A).
    ``status`` (device int32 [4], accumulated): leavers dropped for a full slot, ids
    outside every range, arrivals dropped for a full buffer, arrivals received.

    ``exchange``: None -> the library's NCCL communicator ``comm`` (grouped
    ncclSend/ncclRecv of whole slots with ``peers``); a callable(send, recv, slot_bytes)
    replaces it (the tests run several simulated ranks in one process)."""

    def __init__(self, n: int, bounds: list, rank: int, cap: int, device, *, xrows: int = 0,
                 comm: Optional[NcclComm] = None, peers: Optional[list] = None, exchange=None):
        from . import _lib
        L = _lib.load()
        self.n, self.rank, self.cap, self.xrows = n, rank, cap, xrows
        self.P = len(bounds) - 1
        self.bounds = torch.tensor(bounds, dtype=torch.int32, device=device)
        self.slot = int(L.cc_mig_slot_bytes(cap, xrows))
        self.send = torch.empty(self.P * self.slot, dtype=torch.uint8, device=device)
        self.recv = torch.empty(self.P * self.slot, dtype=torch.uint8, device=device)
        self.ws = torch.empty(max(int(L.cc_mig_workspace_bytes(n, self.P)), 256), dtype=torch.uint8, device=device)
        self.status = torch.zeros(4, dtype=torch.int32, device=device)
        self.comm = comm
        self.peers = [p for p in range(self.P) if p != rank] if peers is None else list(peers)
        self.exchange_fn = exchange
        import numpy as np
        self._peers = np.asarray(self.peers, dtype=np.int32)

    @staticmethod
    def _p(t):
        import ctypes as C
        return C.c_void_p(t.data_ptr()) if t is not None else None

    def _stream(self):
        import ctypes as C
        return C.c_void_p(torch.cuda.current_stream(self.send.device).cuda_stream)

    def pack(self, v, x, cell):
        from . import _lib
        ldx = x.stride(0) if (x is not None and self.xrows > 0) else self.n
        _lib.check(_lib.load().cc_mig_pack(self._p(v), v.stride(0), self._p(x) if self.xrows else None, ldx,
                                           self.xrows, self._p(cell), self.n, self._p(self.bounds), self.P, self.rank,
                                           self.cap, self._p(self.send), self._p(self.recv), self._p(self.status),
                                           self._p(self.ws), self.ws.numel(), self._stream()), "cc_mig_pack")

    def exchange(self):
        import ctypes as C
        from . import _lib
        if self.exchange_fn is not None:
            self.exchange_fn(self.send, self.recv, self.slot)
        elif self.peers:
            _lib.check(_lib.load().cc_dist_mig_exchange(self._p(self.send), self._p(self.recv), self.slot,
                                                        self._peers.ctypes.data_as(C.c_void_p), len(self.peers),
                                                        self.comm.comm, self._stream()), "cc_dist_mig_exchange")

    def unpack(self, v, x, cell, diag):
        from . import _lib
        ldx = x.stride(0) if (x is not None and self.xrows > 0) else self.n
        _lib.check(_lib.load().cc_mig_unpack(self._p(v), v.stride(0), self._p(x) if self.xrows else None, ldx,
                                             self.xrows, self._p(cell), self.n, self._p(diag), self._p(self.recv),
                                             self._p(self.bounds), self.P, self.rank, self.cap, self._p(self.status),
                                             self._stream()), "cc_mig_unpack")

    def __call__(self, v, x, cell, diag):
        self.pack(v, x, cell)
        self.exchange()
        self.unpack(v, x, cell, diag)


def torch_exchange(group=None):
    """Migrator exchange through torch.distributed point-to-point ops (batch_isend_irecv of
    whole slots with every other rank); used when the library's own NCCL communicator is not."""
    def fn(send, recv, slot):
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        host = dist.get_backend(group) == "gloo"      # gloo point-to-point: host buffers (smoke runs)
        snd = send.cpu() if host else send
        rcv = recv.cpu() if host else recv
        ops = []
        for p in range(world):
            if p != rank:
                ops.append(dist.P2POp(dist.isend, snd[p * slot:(p + 1) * slot], p, group))
                ops.append(dist.P2POp(dist.irecv, rcv[p * slot:(p + 1) * slot], p, group))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        if host:
            recv.copy_(rcv)
    return fn


def cuda_ops(nccl: Optional[NcclComm] = None) -> DistOps:
    from . import coulomb as cc

    def partition(key, nkeys):
        return cc.cc_bin(key, nkeys)

    def gather(v, cell, perm, cell_shift):
        return cc.cc_gather(v, cell, perm, cell_shift)

    def owner(cell_global, bounds):
        return cc.cc_owner(cell_global, bounds)

    def p2c(v, cell, cells, sub):
        return cc.cc_p2c(v, cell, cells, sub=sub)

    def p2c_moments(raw, weight, cell_volume):
        return cc.cc_p2c_moments(raw, weight=weight, cell_volume=cell_volume)

    return DistOps(partition=partition, gather=gather, sum_ranks=cc.cc_diag_sum_ranks, owner=owner, p2c=p2c,
                   p2c_moments=p2c_moments, nccl=nccl)


def reduce_diag(diag: torch.Tensor, ops: DistOps, group=None) -> torch.Tensor:
    """All-gather every rank's 16-double diagnostics and sum them in rank order."""
    if ops.nccl is not None:
        return ops.nccl.diag_reduce(diag)
    world = dist.get_world_size(group)
    flat = torch.empty(world * diag.numel(), dtype=diag.dtype, device=diag.device)
    dist.all_gather_into_tensor(flat, diag.contiguous().view(-1), group=group)
    return ops.sum_ranks(flat.view(world, diag.numel()))


@dataclass
class Migrated:
    v: torch.Tensor        # [3][n_new] fp64
    cell: torch.Tensor     # [n_new] int32, LOCAL cell ids of the receiving rank (-1 dead)
    sent: list             # particles sent to each rank (incl. self)
    received: list         # particles received from each rank (incl. self)
    payload: Optional[torch.Tensor] = None   # [3][n_new] fp64 rows carried along (e.g. positions)


def migrate(v: torch.Tensor, cell_global: torch.Tensor, global_cells: int, ops: DistOps,
            group=None, keep_dead: bool = False, payload: Optional[torch.Tensor] = None) -> Migrated:
    """Move every particle to the rank owning its (global) cell.

    1. owner rank of every particle (dead particles: dropped unless keep_dead,
       then they stay on this rank);
    2. stable partition by owner (key = owner rank; the binning kernels);
    3. all_to_all of the per-destination counts;
    4. pack (gather in partition order) and all_to_all of velocities and cells;
    5. arrivals concatenated in source-rank order; global -> local cell ids.
    ``payload`` ([3][n] fp64, e.g. the positions of the NEXT f2 push) travels
    with the particles (same pack order, same exchange).
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bounds = owner_bounds(global_cells, world)
    dev = v.device
    own = ops.owner(cell_global, bounds)
    # dead particles: key `world` (dropped) or own rank (kept)
    key = torch.where(own < 0, torch.full_like(own, rank if keep_dead else world), own)
    perm, off = ops.partition(key.to(torch.int32), world + 1)
    off_l = [int(x) for x in off.cpu().tolist()]
    send = [off_l[r + 1] - off_l[r] for r in range(world)]
    n_send = off_l[world]
    send_t = torch.tensor(send, dtype=torch.int64, device=dev)
    if ops.nccl is not None:
        recv_t = ops.nccl.alltoall_counts(send_t)
    else:
        recv_t = torch.empty(world, dtype=torch.int64, device=dev)
        dist.all_to_all_single(recv_t, send_t, group=group)
    recv = [int(x) for x in recv_t.cpu().tolist()]
    pv, pc = ops.gather(v, cell_global, perm[:n_send], 0)
    n_recv = sum(recv)
    rv = torch.empty((3, n_recv), dtype=v.dtype, device=dev)
    rc = torch.empty(n_recv, dtype=torch.int32, device=dev)

    def exchange_rows(src, dst):
        if ops.nccl is not None:
            so = [0]
            for x in send:
                so.append(so[-1] + x)
            ro = [0]
            for x in recv:
                ro.append(ro[-1] + x)
            ops.nccl.exchange(src.contiguous(), dst, so, ro)
        elif src.dim() == 1:
            dist.all_to_all_single(dst, src.contiguous(), output_split_sizes=recv, input_split_sizes=send,
                                   group=group)
        else:
            for c in range(src.shape[0]):
                dist.all_to_all_single(dst[c], src[c].contiguous(), output_split_sizes=recv,
                                       input_split_sizes=send, group=group)

    exchange_rows(pv, rv)
    exchange_rows(pc, rc)
    base = bounds[rank]
    ident = torch.arange(n_recv, dtype=torch.int32, device=dev)
    lv, lc = ops.gather(rv, rc, ident, base)
    lp = None
    if payload is not None:
        px, _ = ops.gather(payload, cell_global, perm[:n_send], 0)
        rx = torch.empty((3, n_recv), dtype=payload.dtype, device=dev)
        exchange_rows(px, rx)
        lp = rx
    return Migrated(lv, lc, send, recv, lp)


# ---------------------------------------------------------------- NEXT f4: the paper's replicated grid
# "each task owns N/P electrons and replicates all M cells.  Steps S1-S2 ... are done in an
# embarrassingly parallel manner at each task.  Steps S3a and S3b are where the communication takes
# place: a local P2C operation, ... followed by an all-reduce with message size O(M)".
# The comparison point for the cell-range shards above: each rank runs coulomb_collide on ALL cells
# (cell_base 0) with its own particles, a rank-distinct random stream (replica_seed) and weight
# P x w (its N/P particles sample the whole plasma: "P simulations of N/P particles");
# pairs never cross ranks (the paper's within-rank pairing).


def replica_seed(seed: int, rank: int) -> int:
    """Rank-distinct Philox key of replica `rank` (independent streams; rank 0 keeps `seed`)."""
    return (seed + rank * 0x9E3779B97F4A7C15) % (1 << 64)


def replicated_moments(v: torch.Tensor, cell: torch.Tensor, cells: int, ops: DistOps, *, weight: float,
                       cell_volume: float, sub: int = 16, group=None) -> torch.Tensor:
    """S3a/S3b of the replicated-grid scheme: local atomic P2C (sub-binned) of this rank's
    particles, one all-reduce (sum) of the [cells][7] raw sums, moments of the union of all ranks'
    particles with the physical weight w."""
    raw = ops.p2c(v, cell, cells, sub)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(raw, op=dist.ReduceOp.SUM, group=group)
    return ops.p2c_moments(raw, weight, cell_volume)


def init_from_env(backend: Optional[str] = None):
    """torchrun environment -> (rank, world, local_rank), process group initialised."""
    import os
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            if torch.cuda.is_available():
                torch.cuda.set_device(local % torch.cuda.device_count())
            dist.init_process_group(backend)
    return rank, world, local
