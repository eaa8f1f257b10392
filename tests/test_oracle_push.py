"""Pins of the oracle's NEXT f2 push (S2b + S2c, Table 2; SPEC push S:204-210).

Each pin comes from outside the oracle's own formula: CODATA's published e/m_e,
the closed-form kick-drift trajectory in a uniform field (which fixes the
operator order "kick then drift"), exact dyadic geometry for the cell
index (compared with numpy.searchsorted / ravel_multi_index), periodic wrap
and absorption conditions evaluated exactly on dyadic numbers.
"""
import numpy as np
import pytest

import oracle

E_OVER_ME = 1.75882001076e11      # CODATA 2018 e/m_e [C/kg], published value (not Q_E/M_E)


def test_spec_example_field_kick():
    """dt = 1e-10 s, E = 3220 V/m on an electron at rest -> dv_x ~ -5.664e4 m/s
    (SPEC's rounding; CODATA e/m_e gives -5.66340e4)."""
    x = np.full((3, 1), 0.5)
    v = np.zeros((3, 1))
    E = np.array([[3220.0], [0.0], [0.0]])
    xo, vo, co = oracle.push(x, v, np.zeros(1, np.int32), dims=1, nc=[1], d=[1.0], periodic=1, dt=1e-10, E=E)
    assert abs(vo[0, 0] / -5.664e4 - 1) < 2e-4
    assert abs(vo[0, 0] - (-E_OVER_ME * 3220.0 * 1e-10)) <= 1e-9 * 5.7e4
    assert vo[1, 0] == 0.0 and vo[2, 0] == 0.0
    assert xo[0, 0] == 0.5 + 1e-10 * vo[0, 0]


def test_uniform_field_trajectory_closed_form():
    """K kick-drift steps in a uniform field: v_K = v0 + K a dt and
    x_K = x0 + K dt v0 + a dt^2 K (K+1) / 2 (kick BEFORE drift; drift-then-kick
    would give K (K-1) / 2)."""
    rng = np.random.default_rng(1)
    n, K, dt = 64, 40, 1e-10
    L = 1e3
    x = np.vstack([rng.uniform(400, 600, n), np.zeros(n), np.zeros(n)])
    v = rng.normal(0, 5e5, (3, n))
    E = np.array([[-150.0], [75.0], [20.0]])
    cell = np.zeros(n, np.int32)
    x0, v0 = x.copy(), v.copy()
    for _ in range(K):
        x, v, cell2 = oracle.push(x, v, cell, dims=1, nc=[1], d=[L], periodic=0, dt=dt, E=E)
        assert np.all(cell2 == 0)
    a = -E_OVER_ME * E[:, 0]
    # K rounded additions (K ulp of max |v|) + the 11-digit CODATA e/m_e (1e-11 of the total kick)
    tol = K * np.spacing(np.abs(v).max()) + 1e-11 * np.abs(K * a * dt)[:, None]
    assert np.all(np.abs(v - (v0 + (K * a * dt)[:, None])) <= tol)
    xk = x0[0] + K * dt * v0[0] + a[0] * dt * dt * K * (K + 1) / 2
    assert np.allclose(x[0], xk, rtol=1e-12, atol=0)
    assert np.all(x[1:] == 0.0)          # rows >= dims are not touched (zero from the wrapper)


def test_cell_index_dyadic_3d():
    """Dyadic grid (d = 2^-k): floor(x/d) is exact, so the cell index equals an
    independent searchsorted over the grid lines, and the global id equals
    numpy.ravel_multi_index in Fortran order (x fastest)."""
    rng = np.random.default_rng(2)
    n = 5000
    nc = [7, 5, 3]
    d = [2.0 ** -3, 2.0 ** -2, 2.0 ** -1]
    L = [nc[a] * d[a] for a in range(3)]
    x = np.vstack([rng.uniform(0, L[a], n) for a in range(3)])
    v = np.zeros((3, n))
    xo, vo, co = oracle.push(x, v, np.zeros(n, np.int32), dims=3, nc=nc, d=d, periodic=0, dt=1e-10)
    idx = [np.searchsorted(np.arange(1, nc[a]) * d[a], x[a], side="right") for a in range(3)]
    G = np.ravel_multi_index(idx, nc, order="F")
    assert np.array_equal(co, G.astype(np.int32))
    assert np.array_equal(xo, x) and np.array_equal(vo, v)


def test_periodic_wrap_and_absorbing_exact():
    """x = L - 1/8 moving +1/4 per step wraps to 1/8 (periodic) or dies (absorbing);
    x = 1/8 moving -1/4 wraps to L - 1/8 — all exact in binary."""
    dt = 2.0 ** -10
    L = 4.0
    x = np.array([[L - 0.125, 0.125, 2.0], [0, 0, 0], [0, 0, 0]])
    v = np.array([[0.25 / dt, -0.25 / dt, 0.25 / dt], [0, 0, 0], [0, 0, 0]])
    cell = np.zeros(3, np.int32)
    xo, _, co = oracle.push(x, v, cell, dims=1, nc=[4], d=[1.0], periodic=1, dt=dt)
    assert list(xo[0]) == [0.125, L - 0.125, 2.25] and list(co) == [0, 3, 2]
    xo, _, co = oracle.push(x, v, cell, dims=1, nc=[4], d=[1.0], periodic=0, dt=dt)
    assert list(co) == [-1, -1, 2]
    assert list(xo[0]) == [L + 0.125, -0.125, 2.25]      # absorbed particles keep the drifted x


def test_far_wrap_and_non_finite():
    """R23: positions many periods away wrap by the exact remainder (dyadic: x = 1/8 + k L lands on
    1/8 for any k, also k ~ 1e12, where repeated subtraction would take 1e12 steps); +-inf and NaN
    positions are absorbed (cell -1) on periodic and absorbing axes alike."""
    dt = 1.0
    L = 4.0
    x0 = np.array([0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 1.0, 1.0])
    dx = np.array([0.125 + 3 * L, 0.125 + 2 ** 40 * L, -(3 * L) + 0.125, -(2 ** 40) * L + 0.125,
                   np.inf, -np.inf, np.nan, 1e308])
    n = x0.size
    x = np.zeros((3, n)); x[0] = x0
    v = np.zeros((3, n)); v[0] = dx / dt
    for per in (1, 0):
        xo, _, co = oracle.push(x, v, np.zeros(n, np.int32), dims=1, nc=[4], d=[1.0], periodic=per, dt=dt)
        if per:
            assert list(xo[0, :4]) == [0.125] * 4 and list(co[:4]) == [0] * 4
            # 1 + 1e308: finite, wrapped by the exact remainder into [0, L)
            assert 0.0 <= xo[0, 7] < L and xo[0, 7] == np.fmod(1.0 + 1e308, L) + (L if np.fmod(1.0 + 1e308, L) < 0 else 0)
        else:
            assert list(co[:4]) == [-1] * 4
        assert list(co[4:7]) == [-1, -1, -1]


def test_dead_untouched_and_perm_gather():
    """Dead particles (cell -1) keep x and v and stay dead; x rows are read through perm."""
    rng = np.random.default_rng(3)
    n = 100
    x = rng.uniform(0, 1, (3, n))
    v = rng.normal(0, 1e5, (3, n))
    perm = rng.permutation(n)
    cell = np.zeros(n, np.int32)
    cell[::7] = -1
    xo, vo, co = oracle.push(x, v, cell, dims=2, nc=[4, 4], d=[0.25, 0.25], periodic=3, dt=1e-10, perm=perm,
                             E=np.ones((3, 1)) * 1e3)
    dead = cell < 0
    assert np.all(co[dead] == -1)
    assert np.array_equal(xo[:2, dead], x[:2, perm[dead]])
    assert np.array_equal(vo[:, dead], v[:, dead])
    # zero field and zero velocity: x_out = x_in[perm] exactly, cells from the gathered positions
    xo, _, co = oracle.push(x, np.zeros((3, n)), np.zeros(n, np.int32), dims=2, nc=[4, 4], d=[0.25, 0.25],
                            periodic=3, dt=1e-10, perm=perm)
    assert np.array_equal(xo[:2], x[:2, perm])
    ix = np.minimum((x[0, perm] * 4).astype(int), 3)
    iy = np.minimum((x[1, perm] * 4).astype(int), 3)
    assert np.array_equal(co, (ix + 4 * iy).astype(np.int32))


def test_momentum_gain_uniform_field():
    """Sum of momentum change over N electrons = N q E dt (Newton, uniform field)."""
    rng = np.random.default_rng(4)
    n = 1000
    v = rng.normal(0, 6e5, (3, n))
    E = np.array([[100.0, 200.0], [0.0, -50.0], [10.0, 0.0]])        # per-cell field, 2 cells
    cell = (rng.random(n) < 0.5).astype(np.int32)
    _, vo, _ = oracle.push(rng.uniform(0, 2, (3, n)), v, cell, dims=1, nc=[2], d=[1.0], periodic=1,
                           dt=1e-10, E=E)
    dv = (vo - v).sum(axis=1)
    expect = -E_OVER_ME * 1e-10 * (E[:, cell]).sum(axis=1)
    assert np.allclose(dv, expect, rtol=1e-10)
