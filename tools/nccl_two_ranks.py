"""Two ranks on ONE GPU through the library's own NCCL communicator (C ABI cc_nccl_comm_init,
cc_dist_diag_reduce, cc_dist_mig_exchange): does NCCL accept two ranks on one device here?
If it does, the rank-ordered diagnostics sum and the device-side migration are checked against
the torch.distributed (gloo) path on the same data.  Launch:
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29533 tools/nccl_two_ranks.py
Prints one line per rank; exit 0 with "nccl-unavailable: <why>" when NCCL refuses."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2508_06771_b200 import dist as ccd  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    try:
        comm = ccd.NcclComm()
        d = torch.full((16,), float(rank + 1), dtype=torch.float64, device=dev) * torch.arange(16, device=dev)
        got = comm.diag_reduce(d)
        torch.cuda.synchronize()
    except Exception as e:   # NCCL refuses several ranks on one device
        print(f"rank {rank}: nccl-unavailable: {e!r}"[:300], flush=True)
        dist.destroy_process_group()
        return
    exp = sum((r + 1) * torch.arange(16, dtype=torch.float64) for r in range(world))
    ok_diag = torch.equal(got.cpu(), exp)
    # migration: each rank owns 64 global cells; ~10% of its particles belong to the other rank
    M, n_live = 64, 20_000
    bounds = ccd.owner_bounds(M * world, world)
    rng = np.random.default_rng(100 + rank)
    g = rng.integers(rank * M, (rank + 1) * M, n_live)
    away = rng.random(n_live) < 0.1
    g[away] = rng.integers(((rank + 1) % world) * M, ((rank + 1) % world + 1) * M, away.sum())
    cap, n = 4096, n_live + 8192
    v0 = np.zeros((3, n)); v0[:, :n_live] = rng.standard_normal((3, n_live))
    c0 = np.full(n, -1, np.int32); c0[:n_live] = g
    diag = torch.zeros(16, dtype=torch.float64, device=dev); diag[0] = n_live
    res = []
    for exch in ("nccl", "torch"):
        v, c = torch.from_numpy(v0.copy()).to(dev), torch.from_numpy(c0.copy()).to(dev)
        dg = diag.clone()
        mig = ccd.Migrator(n, bounds, rank, cap, dev, comm=comm if exch == "nccl" else None,
                           exchange=None if exch == "nccl" else ccd.torch_exchange())
        mig(v, None, c, dg)
        torch.cuda.synchronize()
        res.append((v.cpu(), c.cpu(), mig.status.cpu()))
    same = all(torch.equal(a, b) for a, b in zip(res[0], res[1]))
    arrived = int(res[0][2][3])
    comm.close()
    print(f"rank {rank}: nccl 2 ranks on one GPU OK; diag_reduce rank-ordered sum {'equal' if ok_diag else 'DIFFERENT'}; "
          f"migration via cc_dist_mig_exchange {'bitwise equal to' if same else 'DIFFERENT from'} the gloo path "
          f"({arrived} arrivals, status {res[0][2].tolist()})", flush=True)
    dist.destroy_process_group()
    if not (ok_diag and same):
        sys.exit(1)


if __name__ == "__main__":
    main()
