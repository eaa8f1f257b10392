"""World-size-2 gloo tests (CPU) of the multi-GPU layer's host logic:
cell-range sharding, the rank-ordered diagnostics reduction and particle
migration.  The per-particle CUDA kernels behind DistOps (stable partition,
gather, ordered sum, owner lookup) are replaced by plain numpy stand-ins defined
here; their CUDA versions are parity-tested in tests/test_gpu_dist.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_06771_b200.dist import (DistOps, migrate, owner_bounds, reduce_diag, replica_seed,
                                        replicated_moments, shard_cells)


def cpu_ops() -> DistOps:
    def partition(key, nkeys):
        k = key.numpy()
        perm = np.argsort(k, kind="stable").astype(np.int32)
        off = np.concatenate([[0], np.cumsum(np.bincount(k, minlength=nkeys))]).astype(np.int32)
        return torch.from_numpy(perm), torch.from_numpy(off)

    def gather(v, cell, perm, shift):
        p = perm.numpy().astype(np.int64)
        c = cell.numpy()[p]
        return (torch.from_numpy(np.ascontiguousarray(v.numpy()[:, p])),
                torch.from_numpy(np.where(c >= 0, c - shift, -1).astype(np.int32)))

    def sum_ranks(g):
        out = torch.zeros(g.shape[1], dtype=g.dtype)
        for r in range(g.shape[0]):
            out += g[r]
        return out

    def owner(cell, bounds):
        c = cell.numpy()
        b = np.asarray(bounds)
        r = np.searchsorted(b, c, side="right") - 1
        r[(c < b[0]) | (c >= b[-1])] = -1
        return torch.from_numpy(r.astype(np.int32))

    def p2c(v, cell, cells, sub):
        # plain per-cell sums (the CUDA version is the atomic, sub-binned kernel)
        c = cell.numpy()
        vv = v.numpy()
        raw = np.zeros((cells, 7))
        ok = (c >= 0) & (c < cells)
        raw[:, 0] = np.bincount(c[ok], minlength=cells)
        for q in range(3):
            raw[:, 1 + q] = np.bincount(c[ok], weights=vv[q][ok], minlength=cells)
            raw[:, 4 + q] = np.bincount(c[ok], weights=vv[q][ok] ** 2, minlength=cells)
        return torch.from_numpy(raw)

    def p2c_moments(raw, weight, volume):
        return raw.clone()           # the test compares the all-reduced raw sums directly

    return DistOps(partition, gather, sum_ranks, owner, p2c, p2c_moments)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ops = cpu_ops()
        res = {}
        # diagnostics: rank-ordered sum of every rank's vector
        diag = torch.arange(16, dtype=torch.float64) * (rank + 1) + 0.1 * rank
        res["diag"] = reduce_diag(diag, ops).numpy()
        # migration: global grid of 10 cells, every rank starts with random particles
        G = 10
        rng = np.random.default_rng(100 + rank)
        n = 500 + 37 * rank
        cell = rng.integers(-1, G, n).astype(np.int32)
        v = rng.standard_normal((3, n))
        v[0] = np.arange(n) + 1000 * rank             # tag: source rank and index
        x = rng.standard_normal((3, n))
        x[1] = v[0] + 0.5                             # positions (NEXT f2 payload) carry the same tag
        m = migrate(torch.from_numpy(v), torch.from_numpy(cell), G, ops, payload=torch.from_numpy(x))
        res["mig"] = (m.v.numpy(), m.cell.numpy(), m.sent, m.received)
        res["payload"] = m.payload.numpy()
        # NEXT f4: replicated grid — every rank deposits its own particles; one all-reduce
        res["repl"] = replicated_moments(torch.from_numpy(v), torch.from_numpy(cell), G, ops, weight=1.0,
                                         cell_volume=1.0).numpy()
        res["src"] = (v, cell)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_shard_cells_partition():
    for G, P in [(4096 * 8, 8), (10, 3), (7, 7), (100, 1)]:
        ranges = [shard_cells(G, P, r) for r in range(P)]
        assert ranges[0][0] == 0
        for r in range(P - 1):
            assert ranges[r][0] + ranges[r][1] == ranges[r + 1][0]
        assert sum(c for _, c in ranges) == G
        assert max(c for _, c in ranges) - min(c for _, c in ranges) <= 1
    assert owner_bounds(10, 3) == [0, 4, 7, 10]
    with pytest.raises(ValueError):
        shard_cells(2, 3, 0)


def test_world2_diag_and_migration():
    world, port = 2, free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = sum(np.arange(16) * (r + 1) + 0.1 * r for r in range(world))
    for r in range(world):
        assert np.array_equal(out[r]["diag"], expect)
    # migration: every live particle ends on its owner, in (source rank, source order)
    bounds = owner_bounds(10, world)
    for r in range(world):
        v, c, sent, recv = out[r]["mig"]
        assert np.all((c >= 0) & (c < bounds[r + 1] - bounds[r]))
        expect_tags, expect_cells = [], []
        for s in range(world):
            sv, sc = out[s]["src"]
            sel = (sc >= bounds[r]) & (sc < bounds[r + 1])
            expect_tags.append(sv[0][sel])
            expect_cells.append(sc[sel] - bounds[r])
        assert np.array_equal(v[0], np.concatenate(expect_tags))
        assert np.array_equal(out[r]["payload"][1], v[0] + 0.5)      # payload travels with its particle
        assert np.array_equal(c, np.concatenate(expect_cells))
        assert sum(recv) == v.shape[1]
    total_live = sum(int(np.sum(out[s]["src"][1] >= 0)) for s in range(world))
    # replicated-grid P2C: every rank holds the sums over the union of all ranks' particles
    allv = np.concatenate([out[s]["src"][0] for s in range(world)], axis=1)
    allc = np.concatenate([out[s]["src"][1] for s in range(world)])
    ok = allc >= 0
    for r in range(world):
        raw = out[r]["repl"]
        assert np.array_equal(raw[:, 0], np.bincount(allc[ok], minlength=10))
        assert np.allclose(raw[:, 1], np.bincount(allc[ok], weights=allv[0][ok], minlength=10), rtol=1e-12)
        assert np.array_equal(raw, out[0]["repl"])
    assert replica_seed(42, 0) == 42 and len({replica_seed(42, r) for r in range(8)}) == 8
    assert sum(out[r]["mig"][0].shape[1] for r in range(world)) == total_live
