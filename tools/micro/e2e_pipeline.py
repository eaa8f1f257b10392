"""Round 2: where does the end-to-end path lose against the PCIe duplex bound?  Per step the e2e bench
copies 2.87 GB host->device (v + cell ids) and 2.46 GB device->host (v), with the operator in
between.  Times K steps of (a) the copies alone in the bench's 2-stream / 2-buffer pipeline,
(b) the same with the operator (coulomb_collide_host, CC_PRESERVE_ORDER), (c) (b) with 3 buffers,
(d) (b) with the host buffers split so each step's H2D is issued as 4 chunks."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_2508_06771_b200 as cc  # noqa: E402
from paper_2508_06771_b200 import _lib  # noqa: E402

dev = torch.device("cuda:0")
w = W.c4()
n, M = w.n, w.cells
v_pin = torch.from_numpy(w.v).pin_memory()
c_pin = torch.from_numpy(w.cell).pin_memory()
p = w.params()
K = 6


def run_ordered(nb, compute):
    """H2D of step s+1 waits for the H2D of step s (event), so one H2D and one D2H are in flight at a
    time, each at its full direction rate, instead of two H2Ds sharing the host->device engine."""
    outs = [torch.empty((3, n), dtype=torch.float64).pin_memory() for _ in range(nb)]
    streams = [torch.cuda.Stream(dev) for _ in range(nb)]
    dv = [torch.empty((3, n), dtype=torch.float64, device=dev) for _ in range(nb)]
    dc = [torch.empty(n, dtype=torch.int32, device=dev) for _ in range(nb)]
    bufs = [cc.alloc_host_buffer(n, M, dev) for _ in range(nb)] if compute else None
    h2d_done = [None]

    def step(s):
        k = s % nb
        st = streams[k]
        if h2d_done[0] is not None:
            st.wait_event(h2d_done[0])
        with torch.cuda.stream(st):
            if compute:
                cc.coulomb_collide_host(v_pin, c_pin, M, out_v=outs[k], dev_buffer=bufs[k], stream=st, step=s,
                                        flags=_lib.CC_PRESERVE_ORDER, **p)
            else:
                dc[k].copy_(c_pin, non_blocking=True)
                dv[k].copy_(v_pin, non_blocking=True)
                e = torch.cuda.Event()
                e.record(st)
                h2d_done[0] = e
                outs[k].copy_(dv[k], non_blocking=True)

    step(0)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for s in range(1, K + 1):
        step(s)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / K * 1e3


def run(nb, compute, chunks=1):
    outs = [torch.empty((3, n), dtype=torch.float64).pin_memory() for _ in range(nb)]
    streams = [torch.cuda.Stream(dev) for _ in range(nb)]
    if compute:
        bufs = [cc.alloc_host_buffer(n, M, dev) for _ in range(nb)]
    else:
        dv = [torch.empty((3, n), dtype=torch.float64, device=dev) for _ in range(nb)]
        dc = [torch.empty(n, dtype=torch.int32, device=dev) for _ in range(nb)]

    def step(s):
        k = s % nb
        with torch.cuda.stream(streams[k]):
            if compute:
                cc.coulomb_collide_host(v_pin, c_pin, M, out_v=outs[k], dev_buffer=bufs[k], stream=streams[k],
                                        step=s, flags=_lib.CC_PRESERVE_ORDER, **p)
            else:
                dc[k].copy_(c_pin, non_blocking=True)
                for a in range(chunks):
                    lo, hi = a * n // chunks, (a + 1) * n // chunks
                    dv[k][:, lo:hi].copy_(v_pin[:, lo:hi], non_blocking=True)
                outs[k].copy_(dv[k], non_blocking=True)

    step(0)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for s in range(1, K + 1):
        step(s)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / K * 1e3


print(f"copies only, 2 buffers: {run(2, False):.1f} ms/step")
print(f"copies only, 3 buffers: {run(3, False):.1f} ms/step")
print(f"copies only, 2 buffers, H2D of step s+1 after H2D of step s: {run_ordered(2, False):.1f} ms/step")
print(f"copies only, 3 buffers, H2D of step s+1 after H2D of step s: {run_ordered(3, False):.1f} ms/step")
print(f"operator, 2 buffers: {run(2, True):.1f} ms/step")
print(f"operator, 3 buffers: {run(3, True):.1f} ms/step")
print("bound: 2.87 GB H2D + 2.46 GB D2H at the measured 99 GB/s duplex = 53.8 ms")
