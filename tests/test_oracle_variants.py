"""Pins for the NEXT-f1 collision-model variants of the oracle (DESIGN R19-R21):
Nanbu's cumulative scattering, TA77's odd-count triplet, and the NRL
electron-electron Coulomb logarithm from lagged moments."""
import numpy as np
import pytest

import workloads as W


def test_langevin_series_and_closed_form_agree(oracle_mod):
    O = oracle_mod
    for A in [1e-6, 1e-3, 0.1, 0.2499999, 0.25, 0.5, 1.0, 5.0, 30.0]:
        exact = 1.0 / np.tanh(A) - 1.0 / A if A >= 0.05 else A / 3 - A ** 3 / 45
        assert abs(O.langevin(A) - exact) <= 1e-12 * max(exact, 1e-12)


@pytest.mark.parametrize("s", [1e-9, 1e-4, 1e-2, 0.1, 0.5, 1.0, 2.0, 5.0, 9.0, 20.0])
def test_nanbu_A_inverts_the_langevin_equation(oracle_mod, s):
    """coth A - 1/A = exp(-s) (Nanbu 1997): checked with mpmath at 50 digits."""
    import mpmath as mp
    mp.mp.dps = 50
    A = oracle_mod.nanbu_A(s)
    lhs = mp.coth(mp.mpf(A)) - 1 / mp.mpf(A)
    assert abs(lhs - mp.e ** (-mp.mpf(s))) <= mp.mpf("1e-13") * mp.e ** (-mp.mpf(s)) + mp.mpf("1e-300")
    if s < 1e-3:
        assert abs(A * s - 1.0) < 2 * s          # A ~ 1/s for small s
    if s > 8:
        assert abs(A / (3 * np.exp(-s)) - 1.0) < 1e-3   # A ~ 3 exp(-s) for large s


def test_nanbu_mean_cosine_equals_exp_minus_s(oracle_mod):
    """Nanbu's distribution is built so that <cos chi> = exp(-s) exactly."""
    O = oracle_mod
    va, vb = np.array([3e5, 0, 0]), np.array([-1e5, 2e5, 0])
    u = va - vb
    un = np.linalg.norm(u)
    for s in (0.05, 0.7):
        Cj = 0.5 * s * un ** 3
        cos = []
        for k in range(40_000):
            u1, u2 = O.pair_uniforms(k, 5, 6, 7)
            a, b = O.nanbu_pair(va, vb, Cj, u1, u2)
            up = a - b
            cos.append(u @ up / (un * np.linalg.norm(up)))
        cos = np.array(cos)
        assert abs(cos.mean() - np.exp(-s)) < 3 * cos.std() / np.sqrt(cos.size)


def test_nanbu_pair_conserves(oracle_mod):
    O = oracle_mod
    rng = np.random.default_rng(3)
    s = W.sigma_v(2.0)
    for _ in range(2000):
        va, vb = rng.standard_normal(3) * s, rng.standard_normal(3) * s
        Cj = 10 ** rng.uniform(10, 17)
        a, b = O.nanbu_pair(va, vb, Cj, *rng.random(2))
        vmax = max(np.abs(va).max(), np.abs(vb).max(), np.abs(a).max(), np.abs(b).max())
        assert np.all(np.abs((a + b) - (va + vb)) <= 4 * np.spacing(vmax))
        e0 = va @ va + vb @ vb
        assert abs((a @ a + b @ b) - e0) <= 1e-14 * e0
    v = np.array([1e5, 2e5, 3e5])
    a, b = O.nanbu_pair(v, v, 1e15, 0.3, 0.4)
    assert np.array_equal(a, v) and np.array_equal(b, v)


def test_triplet_is_three_half_step_collisions(oracle_mod):
    """R19 composed from the pinned pair update: (1,2), (2,3), (3,1) at C/2 with
    the purpose-3 Philox randoms; momentum and energy of the three conserved."""
    O = oracle_mod
    rng = np.random.default_rng(4)
    s = W.sigma_v(2.0)
    G, step, seed = 17, 3, 42
    for flags in (0, O.NANBU):
        v = [rng.standard_normal(3) * s for _ in range(3)]
        Cj = 1e15
        t = O.triplet(*v, Cj, G, step, seed, flags)
        e = [x.copy() for x in v]
        for q, (i, k) in enumerate([(0, 1), (1, 2), (2, 0)]):
            w = O.philox4x32_10([q, G, step, 3], [seed & 0xFFFFFFFF, seed >> 32])
            u1, u2 = O.u01(int(w[0]), int(w[1])), O.u01(int(w[2]), int(w[3]))
            f = O.nanbu_pair if flags else O.ta_pair
            e[i], e[k] = f(e[i], e[k], 0.5 * Cj, u1, u2)
        for q in range(3):
            assert np.array_equal(t[q], e[q])
        p0, p1 = sum(v), sum(t)
        assert np.all(np.abs(p1 - p0) <= 8 * np.spacing(np.abs(np.array(v)).max()))
        e0 = sum(x @ x for x in v)
        assert abs(sum(x @ x for x in t) - e0) <= 1e-14 * e0


@pytest.mark.parametrize("flags", [1, 2, 3])
def test_variant_operator_structure_and_conservation(oracle_mod, flags):
    O = oracle_mod
    w = W.random_cells(20_000, 300, seed=31, skew=True)
    r = O.coulomb_collide(w.v, w.cell, w.cells, step=2, flags=flags, want_pairs=False, **w.params())
    assert np.array_equal(np.sort(r.perm_out), np.arange(w.n))
    assert abs(r.diag[11] - r.diag[7]) <= 1e-13 * r.diag[7]
    counts = np.bincount(w.cell, minlength=w.cells)
    off = np.concatenate([[0], np.cumsum(counts)])
    vin = w.v[:, r.perm_out]
    moved = np.any(r.v_out != vin, axis=0)
    for j in range(w.cells):
        N = counts[j]
        if N >= 3 and N % 2 == 1 and (flags & 1):
            assert moved[off[j + 1] - 1]          # with the triplet nobody sits out
        elif N % 2 == 1:
            assert not moved[off[j + 1] - 1]


def test_triplet_mode_on_three_particles(oracle_mod):
    O = oracle_mod
    w = W.random_cells(3, 1, seed=5)
    r = O.coulomb_collide(w.v, w.cell, 1, step=4, flags=O.ODD_TRIPLET, **w.params())
    pi = O.cell_perm(3, 0, 4, 42)
    Cj = O.cell_constant(3, w.weight, w.cell_volume, w.ln_lambda, w.dt)
    t = O.triplet(w.v[:, pi[0]], w.v[:, pi[1]], w.v[:, pi[2]], Cj, 0, 4, 42, 0)
    assert np.array_equal(r.v_out, np.stack(t, axis=1))


def test_nrl_coulomb_log_structure(oracle_mod):
    """lnL_ee = 23.5 - ln(n^1/2 T^-5/4) - sqrt(1e-5 + (ln T - 2)^2/16): exact
    density scaling d lnL / d ln n = -1/2, the T-dependence at fixed n, the floor."""
    O = oracle_mod
    m = np.zeros((5, 7))
    m[:, 0] = [1e19, 1e19 * np.e ** 2, 1e19, 0.0, 1e40]
    m[:, 4:7] = 2.0
    m[2, 4:7] = 2.0 * np.e ** 0.8
    l = O.coulomb_log(m)
    assert abs((l[0] - l[1]) - 1.0) < 1e-12                     # n * e^2 -> lnL - 1
    # T * e^0.8: +1.25*0.8 from the T^-5/4 term, minus the change of the sqrt term
    lt0, lt1 = np.log(2.0), np.log(2.0) + 0.8
    dsq = np.sqrt(1e-5 + (lt1 - 2) ** 2 / 16) - np.sqrt(1e-5 + (lt0 - 2) ** 2 / 16)
    assert abs((l[2] - l[0]) - (1.0 - dsq)) < 1e-12
    assert l[3] == 2.0 and l[4] == 2.0                          # empty cell / floor
    assert 9.0 < l[0] < 9.2                                     # NRL value for 1e19 m^-3, 2 eV


def test_nanbu_relaxation_rate_matches_nrl(oracle_mod):
    """Physics pin of the Nanbu sampler: the same NRL isotropisation rate as TA
    (small-angle limit), within 5% at dt/10."""
    from test_oracle_physics import nrl_ode, temps
    O = oracle_mod
    ncell, per, steps, dt = 16, 100_000, 20, W.DT / 10
    v, cell = W.maxwellian_cells([per] * ncell, 2.5, T_par_eV=1.0, seed=2508_06771 + 12)
    w = W.weight_for(per)
    n = per * w / W.CELL_VOLUME
    tp0, tz0 = temps(O, v, cell, ncell)
    for s in range(steps):
        r = O.coulomb_collide(v, cell, ncell, dt=dt, weight=w, cell_volume=W.CELL_VOLUME,
                              ln_lambda=W.LN_LAMBDA, seed=42, step=s, want_pairs=False, flags=O.NANBU)
        v, cell = r.v_out, r.cell_out
    tp1, tz1 = temps(O, v, cell, ncell)
    ref = np.array([nrl_ode(a, b, n, W.LN_LAMBDA, dt, steps) for a, b in zip(tp0, tz0)])
    ratio = np.mean((tp1 - tz1) - (tp0 - tz0)) / np.mean((ref[:, 0] - ref[:, 1]) - (tp0 - tz0))
    assert abs(ratio - 1.0) < 0.05, ratio
