"""Pins for the whole operator (Table 5) on tiny and structured inputs."""
import numpy as np
import pytest

import workloads as W


def run(O, w, step=0, **kw):
    p = w.params()
    p.update(kw)
    return O.coulomb_collide(w.v, w.cell, w.cells, step=step, **p)


def check_structure(O, w, r):
    n, M = w.n, w.cells
    cell = w.cell
    perm = r.perm_out
    assert np.array_equal(np.sort(perm), np.arange(n))                 # permutation property
    assert np.array_equal(r.cell_out, cell[perm])
    live = cell >= 0
    L = int(live.sum())
    assert np.all(np.diff(r.cell_out[:L]) >= 0) and np.all(r.cell_out[L:] == -1)
    assert np.array_equal(perm[L:], np.nonzero(~live)[0])               # dead: input order
    counts = np.bincount(cell[live], minlength=M)
    assert r.diag[0] == L and r.diag[1] == n - L
    assert r.diag[2] == np.sum(counts // 2) and r.diag[3] == np.sum(counts % 2)
    # pairs: stable slots, inside their cell, each slot used at most once
    off = np.concatenate([[0], np.cumsum(counts)])
    sl = r.pair_slots.reshape(-1)
    assert len(np.unique(sl)) == sl.size
    g = 0
    for j in range(M):
        for k in range(counts[j] // 2):
            a, b = r.pair_slots[g]
            assert off[j] <= a < off[j + 1] and off[j] <= b < off[j + 1]
            g += 1
    return off, counts


def test_empty_and_single(oracle_mod):
    O = oracle_mod
    w = W.random_cells(0, 3, seed=1)
    r = run(O, w)
    assert r.diag[0] == 0 and np.all(r.moments == 0)
    w = W.random_cells(1, 1, seed=1)
    r = run(O, w)
    assert np.array_equal(r.v_out, w.v) and r.diag[2] == 0 and r.diag[3] == 1


@pytest.mark.parametrize("N", [2, 3, 4, 5])
def test_tiny_cells_bruteforce(oracle_mod, N):
    """A single cell of N particles, evaluated by hand from the components."""
    O = oracle_mod
    w = W.random_cells(N, 1, seed=N)
    G, step, seed = 0, 3, 42
    r = run(O, w, step=step)
    pi = O.cell_perm(N, G, step, seed)
    Cj = O.cell_constant(N, w.weight, w.cell_volume, w.ln_lambda, w.dt)
    expect = np.zeros((3, N))
    for k in range(N // 2):
        a, b = pi[2 * k], pi[2 * k + 1]                      # stable slot = input index here
        u1, u2 = O.pair_uniforms(k, G, step, seed)
        va, vb = O.ta_pair(w.v[:, a], w.v[:, b], Cj, u1, u2)
        expect[:, 2 * k], expect[:, 2 * k + 1] = va, vb
        assert r.perm_out[2 * k] == a and r.perm_out[2 * k + 1] == b
    if N % 2:
        expect[:, N - 1] = w.v[:, pi[N - 1]]
        assert r.perm_out[N - 1] == pi[N - 1]
    assert np.array_equal(r.v_out, expect)


@pytest.mark.parametrize("seed,n,M,dead,skew", [(1, 5000, 7, 0.0, False), (2, 20000, 300, 0.05, True),
                                                (3, 3000, 3000, 0.0, False), (4, 10_000, 50, 0.5, False)])
def test_structure_and_conservation(oracle_mod, seed, n, M, dead, skew):
    O = oracle_mod
    w = W.random_cells(n, M, seed=seed, dead_frac=dead, skew=skew)
    r = run(O, w, step=seed)
    off, counts = check_structure(O, w, r)
    # per-cell conservation of momentum and energy (to rounding)
    vin_sorted = w.v[:, r.perm_out]
    for j in range(M):
        a, b = off[j], off[j + 1]
        if b - a < 2:
            continue
        p0, p1 = vin_sorted[:, a:b].sum(1), r.v_out[:, a:b].sum(1)
        sabs = np.abs(vin_sorted[:, a:b]).sum(1) + np.abs(r.v_out[:, a:b]).sum(1)
        assert np.all(np.abs(p1 - p0) <= 1e-14 * sabs)
        e0, e1 = np.sum(vin_sorted[:, a:b] ** 2), np.sum(r.v_out[:, a:b] ** 2)
        assert abs(e1 - e0) <= 1e-14 * e0
    assert abs(r.diag[11] - r.diag[7]) <= 1e-14 * r.diag[7]


def test_moments_exact_on_dyadic_data(oracle_mod):
    """Integer velocities make every sum exact: moments equal numpy's exact values."""
    O = oracle_mod
    rng = np.random.default_rng(9)
    M, per = 5, 64
    cell = np.repeat(np.arange(M, dtype=np.int32), per)
    v = rng.integers(-1000, 1000, (3, M * per)).astype(np.float64)
    off = np.arange(M + 1) * per
    mom = O.moments(v, off, 2.0, 4.0, mass=3.0, charge=0.5)
    for j in range(M):
        s = v[:, off[j]:off[j + 1]]
        mean = s.sum(1) / per
        T = 3.0 / 0.5 * ((s - mean[:, None]) ** 2).sum(1) / per
        assert mom[j, 0] == per * 2.0 / 4.0
        assert np.array_equal(mom[j, 1:4], mean)
        assert np.allclose(mom[j, 4:7], T, rtol=1e-15, atol=0)


def test_temperature_definition(oracle_mod):
    """T_c = (m/e) <(v_c - <v_c>)^2>: 3 eV monoenergetic isotropic -> 2 eV."""
    O = oracle_mod
    rng = np.random.default_rng(10)
    n = 200_000
    speed = np.sqrt(2 * 3.0 * W.Q_E / W.M_E)
    d = rng.standard_normal((3, n))
    d /= np.linalg.norm(d, axis=0)
    v = d * speed
    mom = O.moments(v, np.array([0, n]), 1.0, 1.0)
    T = mom[0, 4:7].mean()
    assert abs(T - 2.0) < 0.01


def test_determinism_and_shard_invariance(oracle_mod):
    """Same inputs -> identical bytes; running each half of the cells as its own
    shard (cell_base) reproduces the full run (§8e)."""
    O = oracle_mod
    w = W.random_cells(20_000, 64, seed=11)
    r1 = run(O, w, step=4)
    r2 = run(O, w, step=4)
    assert np.array_equal(r1.v_out, r2.v_out) and np.array_equal(r1.perm_out, r2.perm_out)
    for lo, hi in [(0, 32), (32, 64)]:
        sel = (w.cell >= lo) & (w.cell < hi)
        idx = np.nonzero(sel)[0]
        rs = O.coulomb_collide(w.v[:, idx], w.cell[idx] - lo, hi - lo, dt=w.dt, weight=w.weight,
                               cell_volume=w.cell_volume, ln_lambda=w.ln_lambda, cell_base=lo,
                               seed=w.seed, step=4)
        a = np.searchsorted(r1.cell_out, lo)
        b = np.searchsorted(r1.cell_out, hi)
        assert np.array_equal(rs.v_out, r1.v_out[:, a:b])
        assert np.array_equal(idx[rs.perm_out], r1.perm_out[a:b])
        assert np.array_equal(rs.moments, r1.moments[lo:hi])


def test_thread_count_invariance(oracle_mod, tmp_path):
    """OpenMP over cells: results independent of the number of threads."""
    import subprocess, sys, os
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import numpy as np, oracle as O, workloads as W\n"
        "w = W.random_cells(30000, 97, seed=12)\n"
        "r = O.coulomb_collide(w.v, w.cell, w.cells, step=1, **w.params())\n"
        "np.save(sys.argv[1], r.v_out)\n" % os.path.dirname(os.path.dirname(__file__)))
    outs = []
    for t in (1, 4):
        f = str(tmp_path / f"o{t}.npy")
        env = dict(os.environ, OMP_NUM_THREADS=str(t))
        subprocess.check_call([sys.executable, "-c", code, f], env=env)
        outs.append(np.load(f))
    assert np.array_equal(outs[0], outs[1])


def test_preserve_order_is_the_unpermuted_default(oracle_mod):
    """SURVEY §8(b) CC_PRESERVE_ORDER: the same per-particle results in input order —
    v_pres[:, perm_default[p]] == v_default[:, p] exactly, cell_out == the validated input
    ids (invalid -> -1), perm the identity; moments and diagnostics unchanged."""
    O = oracle_mod
    w = W.random_cells(20_000, 37, seed=31, dead_frac=0.05, skew=True)
    cell = w.cell.copy()
    cell[[3, 999]] = [37, -9]                       # invalid ids are treated as dead (R11)
    p = w.params()
    with pytest.raises(ValueError):
        O.coulomb_collide(w.v, cell, 37, step=2, want_pairs=False, **p)   # the oracle rejects invalid ids
    for flags in (0, O.ODD_TRIPLET, O.NANBU):
        d = O.coulomb_collide(w.v, w.cell, 37, step=2, want_pairs=False, flags=flags, **p)
        r = O.coulomb_collide(w.v, w.cell, 37, step=2, want_pairs=False, flags=flags | O.PRESERVE_ORDER, **p)
        assert np.array_equal(r.v_out[:, d.perm_out], d.v_out)
        assert np.array_equal(r.cell_out, np.where(w.cell >= 0, w.cell, -1))
        assert np.array_equal(r.perm_out, np.arange(w.n))
        assert np.array_equal(r.moments, d.moments) and np.array_equal(r.diag, d.diag)
