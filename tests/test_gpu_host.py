"""The end-to-end host-buffer entry coulomb_collide_host: identical results to
the device entry (same kernels, copies around them), for pinned and pageable
host memory, strided host rows, optional outputs, and two calls in flight on
two streams (the bench's e2e pattern)."""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2508_06771_b200 as cc  # noqa: E402

DEV = torch.device("cuda:0")


@pytest.mark.parametrize("pinned", [True, False])
@pytest.mark.parametrize("n,M", [(100_001, 97), (3, 1), (0, 4)])
def test_host_entry_equals_device_entry(pinned, n, M):
    w = W.random_cells(n, M, seed=n + M, dead_frac=0.01, skew=True)
    p = w.params()
    ref = cc.coulomb_collide(torch.from_numpy(w.v).to(DEV), torch.from_numpy(w.cell).to(DEV), M, step=5, **p)

    def host(t):
        t = t.clone()
        return t.pin_memory() if pinned else t

    v, c = host(torch.from_numpy(w.v)), host(torch.from_numpy(w.cell))
    ov, oc, op = host(torch.zeros((3, n), dtype=torch.float64)), host(torch.zeros(n, dtype=torch.int32)), \
        host(torch.zeros(n, dtype=torch.int32))
    om, od = host(torch.zeros((M, 7), dtype=torch.float64)), host(torch.zeros(16, dtype=torch.float64))
    buf = cc.alloc_host_buffer(n, M, DEV)
    cc.coulomb_collide_host(v, c, M, out_v=ov, out_cell=oc, out_perm=op, out_moments=om, out_diag=od,
                            dev_buffer=buf, step=5, **p)
    torch.cuda.synchronize()
    assert torch.equal(ov, ref.v_out.cpu()) and torch.equal(oc, ref.cell_out.cpu())
    assert torch.equal(op, ref.perm_out.cpu()) and torch.equal(om, ref.moments.cpu())
    assert torch.equal(od, ref.diag.cpu())


def test_host_entry_strided_rows_and_two_streams():
    n, M = 50_000, 33
    w = W.random_cells(n, M, seed=4, skew=True)
    p = w.params()
    big = torch.zeros((3, n + 5), dtype=torch.float64)
    big[:, :n] = torch.from_numpy(w.v)
    vin = big[:, :n]                                   # ldv = n + 5 on the host
    c = torch.from_numpy(w.cell).pin_memory()
    outs = [(torch.full((3, n + 5), 7.0, dtype=torch.float64), torch.zeros(n, dtype=torch.int32)) for _ in range(2)]
    bufs = [cc.alloc_host_buffer(n, M, DEV) for _ in range(2)]
    sts = [torch.cuda.Stream(DEV) for _ in range(2)]
    for s in range(2):
        cc.coulomb_collide_host(vin, c, M, out_v=outs[s][0][:, :n], out_cell=outs[s][1], dev_buffer=bufs[s],
                                stream=sts[s], step=s, **p)
    torch.cuda.synchronize()
    for s in range(2):
        ref = cc.coulomb_collide(torch.from_numpy(w.v).to(DEV), torch.from_numpy(w.cell).to(DEV), M, step=s, **p)
        assert torch.equal(outs[s][0][:, :n], ref.v_out.cpu())
        assert torch.all(outs[s][0][:, n:] == 7.0)
        assert torch.equal(outs[s][1], ref.cell_out.cpu())


def test_host_entry_preserve_order_velocities_only():
    """The e2e pattern of bench.py: CC_PRESERVE_ORDER, only the velocities copied back."""
    n, M = 80_000, 50
    w = W.random_cells(n, M, seed=8, skew=True)
    p = w.params()
    f = cc._lib.CC_PRESERVE_ORDER
    ref = cc.coulomb_collide(torch.from_numpy(w.v).to(DEV), torch.from_numpy(w.cell).to(DEV), M, step=3, flags=f, **p)
    ov = torch.zeros((3, n), dtype=torch.float64).pin_memory()
    cc.coulomb_collide_host(torch.from_numpy(w.v).pin_memory(), torch.from_numpy(w.cell).pin_memory(), M, out_v=ov,
                            dev_buffer=cc.alloc_host_buffer(n, M, DEV), step=3, flags=f, **p)
    torch.cuda.synchronize()
    assert torch.equal(ov, ref.v_out.cpu())
