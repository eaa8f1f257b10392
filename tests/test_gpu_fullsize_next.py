"""The NEXT-row kernels at BASELINE.json's full size (C4: 4096 cells x 25,000 e-,
1.024e8 particles), in the configuration bench.py times, checked against the
oracle on samples it can compute one by one: the push is per particle
(bit-exact on 200k sampled particles), recombination per cell (bit-exact on
sampled cells), the atomic P2C per cell (R15 bars on sampled cells)."""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2508_06771_b200 as cc  # noqa: E402

DEV = torch.device("cuda:0")


@pytest.fixture(scope="module")
def O():
    import oracle
    oracle.build()
    return oracle


@pytest.fixture(scope="module")
def c4():
    w = W.c4()
    out = cc.coulomb_collide(torch.from_numpy(w.v).to(DEV), torch.from_numpy(w.cell).to(DEV), w.cells, step=0,
                             **w.params())
    return w, out


def test_push_full_size_sampled(O, c4):
    w, out = c4
    nx = ny = 64
    x = torch.from_numpy(W.positions_in_cells(w.cell, nx, ny, seed=5)).to(DEV)
    E = np.random.default_rng(6).normal(0, 2e3, (3, w.cells))
    v, cell = out.v_out.clone(), out.cell_out.clone()
    g = cc.Grid(2, (nx, ny), (W.PIC_DX, W.PIC_DX), 1)               # x periodic, y absorbing
    xo = cc.cc_push(x, v, cell, g, dt=w.dt, E=torch.from_numpy(E).to(DEV), perm=out.perm_out)
    idx = np.sort(np.random.default_rng(7).choice(w.n, 200_000, replace=False))
    it = torch.from_numpy(idx).to(DEV)
    perm = out.perm_out[it].cpu().numpy()
    xs = x.cpu().numpy()[:, perm]                                    # the sampled particles' input positions
    rx, rv, rc = O.push(xs, out.v_out[:, it].cpu().numpy(), out.cell_out[it].cpu().numpy(), dims=2, nc=[nx, ny],
                        d=[W.PIC_DX, W.PIC_DX], periodic=1, dt=w.dt, E=E)
    assert np.array_equal(xo[:2, it].cpu().numpy(), rx[:2])
    assert np.array_equal(v[:, it].cpu().numpy(), rv)
    assert np.array_equal(cell[it].cpu().numpy(), rc)
    assert (rc == -1).sum() > 0                                      # some crossed the absorbing walls


def test_recombine_full_size_sampled(O, c4):
    w, out = c4
    prob = np.random.default_rng(8).uniform(0, 0.05, w.cells)
    v0, c0 = out.v_out.clone(), out.cell_out.clone()
    st = cc.cc_recombine(v0, c0, torch.from_numpy(prob).to(DEV), eps_bind=2.5e-18, step=0)
    off = np.concatenate([[0], np.cumsum(np.bincount(w.cell, minlength=w.cells))])
    total = 0
    for j in (0, 1, 777, 2048, 4095):
        a, b = off[j], off[j + 1]
        rv, rc, rst = O.recombine(out.v_out[:, a:b].cpu().numpy(), np.zeros(b - a, np.int32), 1, prob[j:j + 1],
                                  eps_bind=2.5e-18, cell_base=j, step=0)
        assert np.array_equal(v0[:, a:b].cpu().numpy(), rv)
        assert np.array_equal(np.where(c0[a:b].cpu().numpy() < 0, -1, 0), rc)
        total += rst[0]
    s = st.cpu().numpy()
    assert s[0] + s[1] == s[2] and total > 0
    assert abs(s[2] - prob.sum() * 25_000) < 5 * np.sqrt(prob.sum() * 25_000)      # binomial


def test_p2c_full_size_sampled(O, c4):
    w, _ = c4
    raw = cc.cc_p2c(torch.from_numpy(w.v).to(DEV), torch.from_numpy(w.cell).to(DEV), w.cells, sub=16)
    m = cc.cc_p2c_moments(raw, weight=w.weight, cell_volume=w.cell_volume).cpu().numpy()
    assert np.array_equal(raw[:, 0].cpu().numpy(), np.bincount(w.cell, minlength=w.cells).astype(np.float64))
    sig = W.sigma_v(2.0)
    for j in (0, 99, 2500, 4095):
        sel = w.cell == j
        r = O.moments(np.ascontiguousarray(w.v[:, sel]), np.array([0, sel.sum()]), w.weight, w.cell_volume)[0]
        assert abs(m[j, 0] - r[0]) <= 1e-15 * r[0]
        assert np.max(np.abs(m[j, 1:4] - r[1:4])) <= 1e-12 * sig
        assert np.all(np.abs(m[j, 4:7] - r[4:7]) <= 1e-12 * r[4:7].sum())
