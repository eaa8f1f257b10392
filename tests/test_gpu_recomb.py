"""NEXT f3 on the GPU: cc_recombine (Table 4 RS0-RS5, readings R25-R28) vs the
oracle on the same collision output — bit-exact (flags from the same Philox
stream, the deterministic rank matching, RS4 evaluated with explicit rounding),
including cells with more matches than one pass window and the forced cases."""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2508_06771_b200 as cc  # noqa: E402

DEV = torch.device("cuda:0")
EB = 15.76 * 1.602176634e-19


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


@pytest.fixture(scope="module")
def O():
    import oracle
    oracle.build()
    return oracle


@pytest.mark.parametrize("n,M,pmax,dead", [(200_000, 300, 0.05, 0.01), (40_000, 2, 0.5, 0.0),
                                          (30_000, 5000, 1.0, 0.02), (1, 1, 1.0, 0.0), (0, 3, 0.5, 0.0),
                                          # many more cells than resident CTAs, half the slots killed: late
                                          # CTAs binary-search an array earlier CTAs are writing
                                          (600_000, 30_000, 0.9, 0.0)])
def test_recombine_bit_exact(O, n, M, pmax, dead):
    w = W.random_cells(n, M, seed=n + M, dead_frac=dead, skew=True)
    p = w.params()
    out = cc.coulomb_collide(to_dev(w.v), to_dev(w.cell), M, step=9, **p)
    prob = np.random.default_rng(M).uniform(0, pmax, M)
    prob[::7] = 0.0
    if M == 2:
        prob[:] = pmax                            # two big cells, half primaries: many windows
    v0, c0 = out.v_out.cpu().numpy(), out.cell_out.cpu().numpy()
    st = cc.cc_recombine(out.v_out, out.cell_out, to_dev(prob), eps_bind=EB, step=9)
    rv, rc, rst = O.recombine(v0, c0, M, prob, eps_bind=EB, step=9)
    assert np.array_equal(st.cpu().numpy(), rst)
    assert np.array_equal(out.cell_out.cpu().numpy(), rc)
    assert np.array_equal(out.v_out.cpu().numpy(), rv)
    if n >= 40_000 and pmax == 0.5:
        assert rst[0] > 4 * 2048                 # several matching windows per cell


def test_recombine_forced():
    w = W.random_cells(10_000, 10, seed=1)
    out = cc.coulomb_collide(to_dev(w.v), to_dev(w.cell), 10, step=0, **w.params())
    v0, c0 = out.v_out.clone(), out.cell_out.clone()
    st = cc.cc_recombine(out.v_out, out.cell_out, torch.ones(10, dtype=torch.float64, device=DEV), eps_bind=EB)
    assert st.tolist() == [0, 10_000, 10_000]       # every particle a primary: no catalyte anywhere
    assert torch.equal(out.v_out, v0) and torch.equal(out.cell_out, c0)
    st = cc.cc_recombine(out.v_out, out.cell_out, torch.zeros(10, dtype=torch.float64, device=DEV), eps_bind=EB)
    assert st.tolist() == [0, 0, 0]
