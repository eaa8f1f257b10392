"""GPU tests of the multi-GPU layer's CUDA kernels (cc_owner, cc_gather, the
rank-ordered diag sum) and of migrate()/reduce_diag() through a 1-rank NCCL
group (a real NCCL communicator on the one GPU a gpurun box gives us)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402

import paper_2508_06771_b200 as cc  # noqa: E402
from paper_2508_06771_b200 import dist as ccd  # noqa: E402

DEV = torch.device("cuda:0")


def test_owner_matches_searchsorted():
    rng = np.random.default_rng(1)
    bounds = [0, 4096, 8192, 12288, 16384]
    cell = rng.integers(-2, 17000, 100_000).astype(np.int32)
    got = cc.cc_owner(torch.from_numpy(cell).to(DEV), bounds).cpu().numpy()
    b = np.asarray(bounds)
    exp = np.searchsorted(b, cell, side="right") - 1
    exp[(cell < 0) | (cell >= b[-1])] = -1
    assert np.array_equal(got, exp)


def test_gather_matches_numpy():
    rng = np.random.default_rng(2)
    n = 50_000
    v = rng.standard_normal((3, n))
    cell = rng.integers(-1, 100, n).astype(np.int32)
    idx = rng.permutation(n)[: n // 2].astype(np.int32)
    gv, gc = cc.cc_gather(torch.from_numpy(v).to(DEV), torch.from_numpy(cell).to(DEV),
                          torch.from_numpy(idx).to(DEV), 10)
    assert np.array_equal(gv.cpu().numpy(), v[:, idx])
    c = cell[idx]
    assert np.array_equal(gc.cpu().numpy(), np.where(c >= 0, c - 10, -1))


@pytest.fixture(scope="module")
def nccl1():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=DEV)
    yield
    dist.destroy_process_group()


def test_reduce_diag_and_migrate_one_rank(nccl1):
    ops = ccd.cuda_ops()
    d = torch.arange(16, dtype=torch.float64, device=DEV)
    assert torch.equal(ccd.reduce_diag(d, ops), d)
    rng = np.random.default_rng(3)
    n = 20_000
    v = rng.standard_normal((3, n))
    cell = rng.integers(-1, 64, n).astype(np.int32)
    m = ccd.migrate(torch.from_numpy(v).to(DEV), torch.from_numpy(cell).to(DEV), 64, ops)
    live = cell >= 0
    assert np.array_equal(m.v.cpu().numpy(), v[:, live])
    assert np.array_equal(m.cell.cpu().numpy(), cell[live])
    assert m.sent == [int(live.sum())] and m.received == [int(live.sum())]


def test_pic_loop_dist_path_one_rank(nccl1):
    """PicLoop's multi-GPU path (device-side Migrator with the positions as payload after every
    push, fixed dead-padded slots) through a real 1-rank NCCL group equals the single-GPU loop
    bitwise: with one rank nothing leaves, ids are already local, the slots stay where they are."""
    import workloads as W
    from paper_2508_06771_b200.pic import PicLoop
    rng = np.random.default_rng(4)
    nx, ny, per = 8, 8, 400
    n = nx * ny * per
    d = 2e-4
    x = np.zeros((3, n))
    x[0], x[1] = rng.uniform(0, nx * d, n), rng.uniform(0, ny * d, n)
    cell = (np.minimum((x[0] / d).astype(int), nx - 1) + nx * np.minimum((x[1] / d).astype(int), ny - 1))
    v = rng.normal(0, W.sigma_v(2.0), (3, n))
    v[0] += 2e5
    g = cc.Grid(2, (nx, ny), (d, d), 2)                 # x absorbing: some electrons leave
    prm = dict(dt=1e-11, weight=W.weight_for(per), cell_volume=W.CELL_VOLUME, subcycles=4)
    args = (torch.from_numpy(x).to(DEV), torch.from_numpy(v).to(DEV), torch.from_numpy(cell.astype(np.int32)).to(DEV), g)
    for comm in (None, ccd.NcclComm()):                 # torch.distributed P2P and the library's NCCL
        a = PicLoop(*args, graph=False, capacity=n + 500, **prm)
        b = PicLoop(*args, dist_ops=ccd.cuda_ops(comm), capacity=n + 500, **prm)
        for _ in range(2):
            a.field_step()
            b.field_step()
        xa, va, ca = a.state
        xb, vb, cb = b.state
        assert int((ca < 0).sum()) > 500                # absorbed electrons (dead slots)
        assert torch.equal(ca, cb) and torch.equal(va, vb) and torch.equal(xa[:2], xb[:2])
        assert b.migrator.status.cpu().tolist() == [0, 0, 0, 0]
        if comm is not None:
            comm.close()


def test_library_nccl_comm_one_rank(nccl1):
    """The C ABI's own NCCL path (cc_nccl_comm_init, cc_dist_diag_reduce,
    cc_dist_alltoall_counts, cc_dist_exchange) through a real 1-rank communicator:
    same results as the torch.distributed path."""
    comm = ccd.NcclComm()
    try:
        ops_c, ops_t = ccd.cuda_ops(comm), ccd.cuda_ops()
        d = torch.arange(16, dtype=torch.float64, device=DEV) * 1.5
        assert torch.equal(ccd.reduce_diag(d, ops_c), ccd.reduce_diag(d, ops_t))
        rng = np.random.default_rng(5)
        n = 30_000
        v = torch.from_numpy(rng.standard_normal((3, n))).to(DEV)
        cell = torch.from_numpy(rng.integers(-1, 64, n).astype(np.int32)).to(DEV)
        x = torch.from_numpy(rng.standard_normal((3, n))).to(DEV)
        a = ccd.migrate(v, cell, 64, ops_c, payload=x)
        b = ccd.migrate(v, cell, 64, ops_t, payload=x)
        assert torch.equal(a.v, b.v) and torch.equal(a.cell, b.cell) and torch.equal(a.payload, b.payload)
        assert a.sent == b.sent and a.received == b.received
    finally:
        comm.close()
