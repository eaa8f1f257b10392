"""NEXT f2 on the GPU: the push (S2b + S2c) and the subcycled PIC loop.

  - cc_push vs the oracle's push: BIT-exact (x, v, cell) — both evaluate every
    product and sum as written, without FMA contraction (DESIGN R22-R24);
  - cc_params.step_dev: (step = s, *step_dev = d) == (step = s + d) bitwise;
  - PicLoop replayed from a CUDA graph == PicLoop run eagerly, bitwise;
  - PicLoop vs the oracle composed step by step (collide, push, Coulomb-log
    feedback): cell ids equal, velocities and positions within R15's bar.
"""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2508_06771_b200 as cc  # noqa: E402
from paper_2508_06771_b200.pic import PicLoop  # noqa: E402

DEV = torch.device("cuda:0")


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


@pytest.fixture(scope="module")
def O():
    import oracle
    oracle.build()
    return oracle


@pytest.mark.parametrize("dims,periodic", [(1, 1), (2, 3), (2, 1), (3, 5), (3, 0)])
def test_push_bit_exact(O, dims, periodic):
    rng = np.random.default_rng(dims * 10 + periodic)
    n = 200_003
    nc = [16, 8, 4][:dims]
    d = [3e-3, 5e-3, 7e-3][:dims]
    M = int(np.prod(nc))
    x = np.zeros((3, n))
    for a in range(dims):
        x[a] = rng.uniform(0, nc[a] * d[a], n)
    x[dims:] = rng.normal(0, 1, (3 - dims, n))       # rows >= dims: neither read nor written
    v = rng.normal(0, 2e6, (3, n))                    # ~3% cross a cell per step at dt below
    cell = rng.integers(0, M, n).astype(np.int32)
    cell[rng.random(n) < 0.05] = -1
    perm = rng.permutation(n).astype(np.int32)
    E = rng.normal(0, 1e4, (3, M))
    dt = 2e-11
    xo, vo, co = O.push(x, v, cell, dims=dims, nc=nc, d=d, periodic=periodic, dt=dt, E=E, perm=perm)
    gv, gc = to_dev(v), to_dev(cell)
    gx = cc.cc_push(to_dev(x), gv, gc, cc.Grid(dims, tuple(nc), tuple(d), periodic), dt=dt, E=to_dev(E),
                    perm=to_dev(perm), cells=M)
    torch.cuda.synchronize()
    assert np.array_equal(gc.cpu().numpy(), co)
    assert np.array_equal(gv.cpu().numpy(), vo)
    assert np.array_equal(gx.cpu().numpy()[:dims], xo[:dims])
    assert (co == -1).sum() >= (cell == -1).sum()


def test_push_without_field_and_perm(O):
    rng = np.random.default_rng(5)
    n = 1000
    x = rng.uniform(0, 1, (3, n))
    v = rng.normal(0, 1e7, (3, n))
    cell = np.zeros(n, np.int32)
    xo, vo, co = O.push(x, v, cell, dims=2, nc=[10, 10], d=[0.1, 0.1], periodic=2, dt=1e-8)
    gv, gc = to_dev(v), to_dev(cell)
    gx = cc.cc_push(to_dev(x), gv, gc, cc.Grid(2, (10, 10), (0.1, 0.1), 2), dt=1e-8, cells=1)
    assert np.array_equal(gx.cpu().numpy()[:2], xo[:2]) and np.array_equal(gc.cpu().numpy(), co)
    assert np.array_equal(gv.cpu().numpy(), v)


@pytest.mark.parametrize("periodic", [1, 0])
def test_push_far_wrap_and_non_finite(O, periodic):
    """R23 edge cases: positions many periods away (exact remainder, no unbounded
    wrap loop) and +-inf / NaN positions (absorbed) — bit-exact with the oracle, and the kernel
    returns (a hang here would be the old unbounded while-loop)."""
    L = 4.0
    dx = np.array([0.125 + 3 * L, 0.125 + 2 ** 40 * L, -(3 * L) + 0.125, -(2 ** 40) * L + 0.125,
                   np.inf, -np.inf, np.nan, 1e308, 0.3, -0.3])
    n = dx.size
    x = np.zeros((3, n)); x[0, 6:] = 1.0
    v = np.zeros((3, n)); v[0] = dx
    cell = np.zeros(n, np.int32)
    gv, gc = to_dev(v), to_dev(cell)
    gx = cc.cc_push(to_dev(x), gv, gc, cc.Grid(1, (4,), (1.0,), periodic), dt=1.0, cells=1)
    ox, ov, oc = O.push(x, v, cell, dims=1, nc=[4], d=[1.0], periodic=periodic, dt=1.0)
    assert np.array_equal(gc.cpu().numpy(), oc)
    assert np.array_equal(gx.cpu().numpy()[0], ox[0], equal_nan=True)


def test_push_rejects_bad_grid():
    t = torch.zeros((3, 4), dtype=torch.float64, device=DEV)
    c = torch.zeros(4, dtype=torch.int32, device=DEV)
    for g in (cc.Grid(0, (1,), (1.0,)), cc.Grid(1, (0,), (1.0,)), cc.Grid(2, (4, 4), (1.0, -1.0)),
              cc.Grid(3, (2048, 2048, 1024), (1.0, 1.0, 1.0))):
        with pytest.raises(cc._lib.CCError):
            cc.cc_push(t, t.clone(), c, g, dt=1e-10, cells=1)


def test_step_dev_equals_host_step():
    w = W.random_cells(100_000, 50, seed=12, skew=True)
    p = w.params()
    sd = torch.tensor([1234], dtype=torch.int32, device=DEV)
    a = cc.coulomb_collide(to_dev(w.v), to_dev(w.cell), 50, step=7, step_dev=sd, **p)
    b = cc.coulomb_collide(to_dev(w.v), to_dev(w.cell), 50, step=7 + 1234, **p)
    for x, y in ((a.v_out, b.v_out), (a.perm_out, b.perm_out), (a.moments, b.moments)):
        assert torch.equal(x, y)
    cc.cc_step_advance(sd, 10)
    assert int(sd.item()) == 1244


def pic_setup(nx=16, ny=12, per_cell=300, seed=3):
    """2D box, x absorbing (walls), y periodic; Maxwellian 2 eV plus a 1e5 m/s drift
    in x; cell size chosen so that a few % of the electrons change cell per step."""
    rng = np.random.default_rng(seed)
    M = nx * ny
    n = M * per_cell
    d = (2e-4, 2e-4)
    x = np.zeros((3, n))
    x[0] = rng.uniform(0, nx * d[0], n)
    x[1] = rng.uniform(0, ny * d[1], n)
    ix = np.minimum((x[0] / d[0]).astype(int), nx - 1)
    iy = np.minimum((x[1] / d[1]).astype(int), ny - 1)
    cell = (ix + nx * iy).astype(np.int32)
    v = rng.normal(0, W.sigma_v(2.0), (3, n))
    v[0] += 1e5
    E = np.zeros((3, M))
    E[0] = 2e3 * np.sin(np.arange(M) % nx / nx * np.pi)     # a fixed field profile along x
    grid = dict(dims=2, nc=[nx, ny], d=list(d), periodic=2)
    prm = dict(dt=1e-11, weight=W.weight_for(per_cell), cell_volume=W.CELL_VOLUME)
    return x, v, cell, E, grid, prm, M


def oracle_pic(O, x, v, cell, E, grid, prm, M, k, nfield, seed=42):
    lnl = np.full(M, 10.0)
    for f in range(nfield):
        for s in range(k):
            r = O.coulomb_collide(v, cell, M, step=f * k + s, seed=seed, ln_lambda_arr=lnl, want_pairs=False,
                                  dt=prm["dt"], weight=prm["weight"], cell_volume=prm["cell_volume"])
            x, v, cell = O.push(x, r.v_out, r.cell_out, perm=r.perm_out, E=E, dt=prm["dt"], **grid)
        lnl = O.coulomb_log(r.moments)
    return x, v, cell


def make_loop(x, v, cell, E, grid, prm, M, k, graph):
    g = cc.Grid(grid["dims"], tuple(grid["nc"]), tuple(grid["d"]), grid["periodic"])
    return PicLoop(to_dev(x), to_dev(v), to_dev(cell), g, E=to_dev(E), subcycles=k, graph=graph, **prm)


def test_pic_loop_graph_equals_eager():
    x, v, cell, E, grid, prm, M = pic_setup()
    a = make_loop(x, v, cell, E, grid, prm, M, 4, graph=True)
    b = make_loop(x, v, cell, E, grid, prm, M, 4, graph=False)
    for _ in range(3):
        a.field_step()
        b.field_step()
    torch.cuda.synchronize()
    for p, q in zip(a.state, b.state):
        assert torch.equal(p, q)
    assert torch.equal(a.lnl, b.lnl)
    assert int(a.step_dev.item()) == 12


def test_pic_loop_vs_oracle(O):
    x, v, cell, E, grid, prm, M = pic_setup()
    k, nf = 4, 2
    loop = make_loop(x, v, cell, E, grid, prm, M, k, graph=True)
    for _ in range(nf):
        loop.field_step()
    gx, gv, gc = (t.cpu().numpy() for t in loop.state)
    rx, rv, rc = oracle_pic(O, x, v, cell, E, grid, prm, M, k, nf)
    assert np.array_equal(gc, rc)
    scale = np.maximum(np.linalg.norm(rv, axis=0), 1e-3 * W.sigma_v(2.0))
    assert np.max(np.abs(gv - rv) / scale) <= 1e-12
    assert np.max(np.abs(gx - rx)) <= 1e-12 * 16 * 2e-4
    assert (rc < 0).sum() > 0                       # the absorbing walls took some electrons


@pytest.mark.parametrize("flags", [0, 1, 2])
@pytest.mark.parametrize("dims,periodic,field", [(2, 2, True), (1, 0, False), (3, 7, True)])
def test_fused_push_equals_collide_then_push(dims, periodic, field, flags):
    """cc_params.push (the push inside the collision call's output stage) is bit for bit
    coulomb_collide followed by cc_push through perm_out."""
    rng = np.random.default_rng(dims * 7 + periodic + flags)
    nc = [12, 9, 5][:dims]
    d = [2e-4, 3e-4, 5e-4][:dims]
    M = int(np.prod(nc))
    w = W.random_cells(150_001, M, seed=3 + dims, dead_frac=0.02, skew=True)
    x = np.zeros((3, w.n))
    for a in range(dims):
        x[a] = rng.uniform(0, nc[a] * d[a], w.n)
    E = to_dev(rng.normal(0, 3e3, (3, M))) if field else None
    g = cc.Grid(dims, tuple(nc), tuple(d), periodic)
    p = w.params()
    v, c, xin = to_dev(w.v), to_dev(w.cell), to_dev(x)
    ref = cc.coulomb_collide(v, c, M, step=4, flags=flags, **p)
    xr = cc.cc_push(xin, ref.v_out, ref.cell_out, g, dt=w.dt, E=E, perm=ref.perm_out, cells=M)
    xo = torch.zeros((3, w.n), dtype=torch.float64, device=DEV)
    out = cc.coulomb_collide(v, c, M, step=4, flags=flags, push=dict(grid=g, x_in=xin, x_out=xo, E=E), **p)
    assert torch.equal(out.cell_out, ref.cell_out) and torch.equal(out.v_out, ref.v_out)
    assert torch.equal(xo[:dims], xr[:dims]) and torch.equal(out.perm_out, ref.perm_out)
    assert torch.equal(out.moments, ref.moments) and torch.equal(out.diag, ref.diag)


def test_pic_loop_fused_equals_unfused():
    x, v, cell, E, grid, prm, M = pic_setup()
    g = cc.Grid(grid["dims"], tuple(grid["nc"]), tuple(grid["d"]), grid["periodic"])
    a = PicLoop(to_dev(x), to_dev(v), to_dev(cell), g, E=to_dev(E), subcycles=4, graph=True, fused=True, **prm)
    b = PicLoop(to_dev(x), to_dev(v), to_dev(cell), g, E=to_dev(E), subcycles=4, graph=True, fused=False, **prm)
    for _ in range(2):
        a.field_step()
        b.field_step()
    torch.cuda.synchronize()
    for p_, q_ in zip(a.state, b.state):
        assert torch.equal(p_, q_)
