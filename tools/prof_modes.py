"""Run coulomb_collide on the C4 input in one order mode, for ncu captures of single kernels.
usage: python tools/prof_modes.py cold|warm|steady [calls] [flags]   (the last call is the one to profile;
flags: cc_params.flags, e.g. 2 = CC_NANBU)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import workloads as W  # noqa: E402
import paper_2508_06771_b200 as cc  # noqa: E402


def main():
    mode = sys.argv[1]
    calls = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    flags = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    dev = torch.device("cuda:0")
    w = W.c4()
    v, c = torch.from_numpy(w.v).to(dev), torch.from_numpy(w.cell).to(dev)
    col = cc.Collider(w.n, w.cells, dev, **w.params())
    gen = torch.Generator(device=dev)
    gen.manual_seed(1)
    for s in range(calls):
        o = col.step(v, c, step=s, flags=flags)
        if mode != "cold":
            v, c = o.v_out.clone(), o.cell_out.clone()
            if mode == "steady":
                bench.drift_cells(c, 64, 64, 0.02, gen)
    torch.cuda.synchronize()
    print("done", mode, calls)


if __name__ == "__main__":
    main()
