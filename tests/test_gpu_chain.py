"""Chained parity (reading R15's "chained 10-step parity is reported too") and parity on the
bench's steady-state input.

  - C3 in full (256 cells, 2.56e6 e-) and C4 at full size (1.024e8 e- on the GPU, a contiguous
    block of cells re-run by the oracle with the same global ids): 10 steps, each step's output
    feeding the next on both sides (the warm chain of a PIC loop without push).  The pairing
    (perm, cell ids) is integer work and stays bit-exact at every step; the velocity error is
    reported per step (growth), bound at 1e-12 for the first step (R15) and 1e-11 over ten.
  - The bench headline's steady state: C4 after steps with the 2% stand-in drift; one more step
    from that (drifted, nearly sorted) input on sampled cells vs the oracle.
Set CC_REPORT_DIR to write the per-step errors to <dir>/chain_growth.txt.
"""
import os

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


def rel_err(g, r, sigma):
    scale = np.maximum(np.linalg.norm(r, axis=0), 1e-3 * sigma)
    return float(np.max(np.abs(g - r) / scale)) if r.size else 0.0


def report(name, errs):
    d = os.environ.get("CC_REPORT_DIR")
    line = f"{name}: " + " ".join(f"{e:.3e}" for e in errs)
    print(line)
    if d:
        os.makedirs(d, exist_ok=True)
        with open(os.path.join(d, "chain_growth.txt"), "a") as f:
            f.write(line + "\n")


def test_c3_chain_ten_steps(O):
    w = W.c3()
    p = w.params()
    gv, gc = torch.from_numpy(w.v).to(DEV), torch.from_numpy(w.cell).to(DEV)
    rv, rc = w.v, w.cell
    errs = []
    for s in range(10):
        out = cc.coulomb_collide(gv, gc, w.cells, step=s, **p)
        ref = O.coulomb_collide(rv, rc, w.cells, step=s, want_pairs=False, **p)
        assert np.array_equal(out.perm_out.cpu().numpy(), ref.perm_out), s
        assert np.array_equal(out.cell_out.cpu().numpy(), ref.cell_out), s
        errs.append(rel_err(out.v_out.cpu().numpy(), ref.v_out, W.sigma_v(4.0)))
        gv, gc = out.v_out, out.cell_out
        rv, rc = ref.v_out, ref.cell_out
    report("C3 (2.56e6 e-, 256 cells) chained max rel err per step", errs)
    assert errs[0] <= 1e-12 and max(errs) <= 1e-11, errs


def test_c4_chain_sampled_block(O):
    """C4 whole on the GPU for 10 chained steps; the oracle chains cells [1800, 1808) alone (global
    ids via cell_base: a cell's evolution depends only on its own particles, id and count)."""
    w = W.c4()
    p = w.params()
    j0, k = 1800, 8
    sel = (w.cell >= j0) & (w.cell < j0 + k)
    rv = np.ascontiguousarray(w.v[:, sel])
    rc = (w.cell[sel] - j0).astype(np.int32)
    gv, gc = torch.from_numpy(w.v).to(DEV), torch.from_numpy(w.cell).to(DEV)
    errs = []
    for s in range(10):
        out = cc.coulomb_collide(gv, gc, w.cells, step=s, **p)
        ref = O.coulomb_collide(rv, rc, k, step=s, want_pairs=False,
                                **dict(p, cell_base=w.cell_base + j0))
        a = j0 * 25_000                                       # C4: 25,000 e- in every cell, none dead
        b = a + k * 25_000
        assert np.array_equal(out.cell_out[a:b].cpu().numpy(), ref.cell_out + j0), s
        errs.append(rel_err(out.v_out[:, a:b].cpu().numpy(), ref.v_out, W.sigma_v(2.0)))
        gv, gc = out.v_out, out.cell_out
        rv, rc = ref.v_out, ref.cell_out
    report("C4 (1.024e8 e-) cells [1800,1808) chained max rel err per step", errs)
    assert errs[0] <= 1e-12 and max(errs) <= 1e-11, errs


def test_c4_steady_state_input(O):
    """The headline's input: C4 after 4 steps with the bench's 2% stand-in drift; the next step
    on that (nearly sorted, drifted) input vs the oracle on sampled cells of the same input."""
    import bench
    w = W.c4()
    p = w.params()
    gv, gc = torch.from_numpy(w.v).to(DEV), torch.from_numpy(w.cell).to(DEV)
    gen = torch.Generator(device=DEV)
    gen.manual_seed(11)
    for s in range(4):
        out = cc.coulomb_collide(gv, gc, w.cells, step=s, **p)
        gv, gc = out.v_out.clone(), out.cell_out.clone()
        bench.drift_cells(gc, 64, 64, 0.02, gen)
    v_in, c_in = gv.cpu().numpy(), gc.cpu().numpy()
    out = cc.coulomb_collide(gv, gc, w.cells, step=4, **p)
    off = np.concatenate([[0], np.cumsum(np.bincount(c_in[c_in >= 0], minlength=w.cells))])
    worst = 0.0
    for j in (0, 63, 64, 2047, 4095):
        idx = np.nonzero(c_in == j)[0]
        ref = O.coulomb_collide(np.ascontiguousarray(v_in[:, idx]), np.zeros(idx.size, np.int32), 1, step=4,
                                want_pairs=False, **dict(p, cell_base=w.cell_base + j))
        a, b = off[j], off[j + 1]
        assert np.array_equal(out.perm_out[a:b].cpu().numpy(), idx[ref.perm_out])
        worst = max(worst, rel_err(out.v_out[:, a:b].cpu().numpy(), ref.v_out, W.sigma_v(2.0)))
    report("C4 steady-state input (4 drifted steps), sampled cells, max rel err", [worst])
    assert worst <= 1e-12
