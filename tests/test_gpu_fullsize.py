"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

C4 (4096 cells x 25,000 e-, 1.024e8 particles) runs whole on the GPU; the
oracle recomputes sampled cells one by one (a cell's result depends only on
its own particles, its global id and N_j — P:297), and properties that hold
at any size (permutation, sortedness, counts, conservation) are checked on
the full output.
"""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2508_06771_b200 as cc  # noqa: E402

DEV = torch.device("cuda:0")


def sampled_cell_parity(O, w, out, cells_to_check, step, flags=0):
    off = np.concatenate([[0], np.cumsum(np.bincount(w.cell[w.cell >= 0], minlength=w.cells))])
    v_out = out.v_out
    perm = out.perm_out
    worst = 0.0
    for j in cells_to_check:
        idx = np.nonzero(w.cell == j)[0]
        ref = O.coulomb_collide(w.v[:, idx], np.zeros(idx.size, np.int32), 1, dt=w.dt, weight=w.weight,
                                cell_volume=w.cell_volume, ln_lambda=w.ln_lambda,
                                cell_base=w.cell_base + j, seed=w.seed, step=step, want_pairs=False,
                                flags=flags)
        a, b = off[j], off[j + 1]
        g = v_out[:, a:b].cpu().numpy()
        assert np.array_equal(perm[a:b].cpu().numpy(), idx[ref.perm_out])
        scale = np.maximum(np.linalg.norm(ref.v_out, axis=0), 1e-3 * W.sigma_v(2.0))
        err = np.max(np.abs(g - ref.v_out) / scale)
        worst = max(worst, err)
        m = out.moments[j].cpu().numpy()
        r = ref.moments[0]
        assert abs(m[0] - r[0]) <= 1e-15 * r[0]
        assert np.all(np.abs(m[4:7] - r[4:7]) <= 1e-12 * r[4:7])
    assert worst <= 1e-12, worst
    return off


def global_properties(w, out, off):
    n = w.n
    perm = out.perm_out
    s, _ = torch.sort(perm.to(torch.int64))
    assert torch.equal(s, torch.arange(n, device=DEV))
    cell_out = out.cell_out
    L = int(off[-1])
    assert bool((cell_out[1:L] >= cell_out[:L - 1]).all())
    assert torch.equal(torch.bincount(cell_out[:L].to(torch.int64), minlength=w.cells).cpu(),
                       torch.from_numpy(np.diff(off)))
    d = out.diag.cpu().numpy()
    assert d[0] == L and d[2] == np.sum(np.diff(off) // 2)
    assert abs(d[11] - d[7]) <= 1e-13 * d[7]


@pytest.fixture(scope="module")
def O():
    import oracle
    oracle.build()
    return oracle


@pytest.mark.parametrize("maker,step", [(W.c4, 0), (W.c4b, 3)])
def test_full_size_sampled(O, maker, step):
    w = maker()
    out = cc.coulomb_collide(torch.from_numpy(w.v).to(DEV), torch.from_numpy(w.cell).to(DEV), w.cells,
                             step=step, **w.params())
    torch.cuda.synchronize()
    M = w.cells
    off = sampled_cell_parity(O, w, out, [0, 1, 1234, M // 2, M - 1], step)
    global_properties(w, out, off)


def test_c5_shard_equals_global_cells(O):
    """A C5 rank shard (cell_base = 4096 r) reproduces the oracle on global ids."""
    w = W.c5_rank(3, nx=8, ny=16, per_cell=2000)
    out = cc.coulomb_collide(torch.from_numpy(w.v).to(DEV), torch.from_numpy(w.cell).to(DEV), w.cells,
                             step=5, **w.params())
    ref = O.coulomb_collide(w.v, w.cell, w.cells, step=5, want_pairs=False, **w.params())
    assert np.array_equal(out.perm_out.cpu().numpy(), ref.perm_out)
    scale = np.maximum(np.linalg.norm(ref.v_out, axis=0), 1.0)
    assert np.max(np.abs(out.v_out.cpu().numpy() - ref.v_out) / scale) <= 1e-12


@pytest.mark.parametrize("flags", [cc._lib.CC_ODD_TRIPLET, cc._lib.CC_NANBU])
def test_full_size_variants_sampled(O, flags):
    """NEXT f1 variants at full C4 size (odd-count triplet on the C4b profile, whose cells have
    odd and even counts; Nanbu on C4), sampled cells vs the oracle."""
    w = W.c4b() if flags == cc._lib.CC_ODD_TRIPLET else W.c4()
    out = cc.coulomb_collide(torch.from_numpy(w.v).to(DEV), torch.from_numpy(w.cell).to(DEV), w.cells,
                             step=4, flags=flags, **w.params())
    torch.cuda.synchronize()
    counts = np.bincount(w.cell[w.cell >= 0], minlength=w.cells)
    odd = [int(j) for j in np.nonzero(counts % 2 == 1)[0][:3]]
    sampled_cell_parity(O, w, out, sorted(set([0, w.cells // 3, w.cells - 1] + odd)), 4, flags=flags)
