"""Pins for the TA77 pair update (CCS5; readings R5, R8, R9).

The reference below is written independently of the oracle's TA77 component
formula: it rotates u about an explicit orthonormal frame (e1, e2, u/|u|) by
polar angle Theta (tan(Theta/2) = delta) and azimuth phi, with delta from
scipy's ndtri (not AS241).
"""
import numpy as np
import pytest
import scipy.special as sp

import workloads as W


def frame_rotation(va, vb, Cj, u1, u2):
    va = np.asarray(va, float)
    vb = np.asarray(vb, float)
    u = va - vb
    un = np.linalg.norm(u)
    if un == 0:
        return va.copy(), vb.copy()
    delta = np.sqrt(Cj / un ** 3) * sp.ndtri(u1)
    theta = 2.0 * np.arctan(delta)
    phi = 2.0 * np.pi * u2
    up = np.hypot(u[0], u[1])
    if up == 0:
        e1, e2 = np.array([1.0, 0, 0]) * np.sign(u[2]), np.array([0, 1.0, 0])
        # TA77's u_perp = 0 branch: Delta u = (|u| sin cos, |u| sin sin, -u_z (1-cos))
        du = np.array([un * np.sin(theta) * np.cos(phi), un * np.sin(theta) * np.sin(phi),
                       -u[2] * (1 - np.cos(theta))])
        unew = u + du
    else:
        e1 = np.array([u[0] * u[2], u[1] * u[2], -up * up]) / (up * un)
        e2 = np.array([-u[1], u[0], 0.0]) / up
        unew = u * np.cos(theta) + un * np.sin(theta) * (np.cos(phi) * e1 + np.sin(phi) * e2)
    vcm = 0.5 * (va + vb)
    return vcm + 0.5 * unew, vcm - 0.5 * unew


def _cases(n, seed=0):
    rng = np.random.default_rng(seed)
    s = W.sigma_v(2.0)
    for _ in range(n):
        va = rng.standard_normal(3) * s
        vb = rng.standard_normal(3) * s
        Cj = 10 ** rng.uniform(10, 16)
        u1, u2 = rng.random(2)
        yield va, vb, Cj, u1, u2


def test_ta_matches_independent_frame_rotation(oracle_mod):
    for va, vb, Cj, u1, u2 in _cases(3000):
        a, b = oracle_mod.ta_pair(va, vb, Cj, u1, u2)
        ea, eb = frame_rotation(va, vb, Cj, u1, u2)
        scale = np.linalg.norm(va) + np.linalg.norm(vb)
        assert np.max(np.abs(a - ea)) <= 1e-13 * scale
        assert np.max(np.abs(b - eb)) <= 1e-13 * scale


def test_ta_conservation_to_rounding(oracle_mod):
    for va, vb, Cj, u1, u2 in _cases(3000, seed=1):
        a, b = oracle_mod.ta_pair(va, vb, Cj, u1, u2)
        vmax = max(np.abs(va).max(), np.abs(vb).max(), np.abs(a).max(), np.abs(b).max())
        assert np.all(np.abs((a + b) - (va + vb)) <= 4 * np.spacing(vmax))
        e0 = va @ va + vb @ vb
        assert abs((a @ a + b @ b) - e0) <= 1e-14 * e0
        # |u| preserved and u'.u = |u|^2 cos(Theta) with tan(Theta/2) = delta
        u, un_ = va - vb, a - b
        assert abs(np.linalg.norm(un_) - np.linalg.norm(u)) <= 1e-14 * np.linalg.norm(u)


def test_ta_special_cases(oracle_mod):
    O = oracle_mod
    v = np.array([1.0e5, -2.0e5, 3.0e5])
    a, b = O.ta_pair(v, v, 1e14, 0.3, 0.7)                      # v1 = v2: unchanged
    assert np.array_equal(a, v) and np.array_equal(b, v)
    a, b = O.ta_pair(v, -v, 1e14, 0.3, 0.7)                     # v1 = -v2: total momentum 0
    assert np.array_equal(a + b, np.zeros(3))
    assert abs((a @ a + b @ b) - 2 * (v @ v)) <= 1e-15 * 2 * (v @ v)
    a, b = O.ta_pair(v, -v, 0.0, 0.3, 0.7)                      # C = 0 (delta = 0): identity
    assert np.array_equal(a, v) and np.array_equal(b, -v)
    # u_perp = 0 branch (u along +z and -z): |u| conserved, u'.u = |u|^2 cos(Theta)
    for sgn in (1.0, -1.0):
        va, vb = np.array([3.0, 4.0, 5.0 + sgn * 2e5]), np.array([3.0, 4.0, 5.0])
        u = va - vb
        assert u[0] == 0 and u[1] == 0
        a, b = O.ta_pair(va, vb, 1e15, 0.8, 0.1)
        ea, eb = frame_rotation(va, vb, 1e15, 0.8, 0.1)
        assert np.allclose(a, ea, rtol=0, atol=1e-10 * 2e5)
        un = a - b
        assert abs(np.linalg.norm(un) - 2e5) <= 1e-14 * 2e5
    # huge variance (delta -> inf) gives a finite back-scatter, never NaN
    a, b = O.ta_pair([1e-30, 0, 0], [0, 0, 0], 1e20, 0.9, 0.3)
    assert np.all(np.isfinite(a)) and np.all(np.isfinite(b))


def test_ta_variance_of_tan_half_angle(oracle_mod):
    """E[tan^2(Theta/2)] = <delta^2> = C/|u|^3 at fixed |u|, 3 sigma."""
    O = oracle_mod
    rng = np.random.default_rng(7)
    va, vb = np.array([4e5, 0, 0]), np.array([-2e5, 1e5, 3e5])
    un = np.linalg.norm(va - vb)
    var = 0.01
    Cj = var * un ** 3
    t2 = []
    for k in range(60_000):
        u1, u2 = O.pair_uniforms(k, 1, 2, 3)
        a, b = O.ta_pair(va, vb, Cj, u1, u2)
        u, up = va - vb, a - b
        c = u @ up / (un * np.linalg.norm(up))
        t2.append((1 - c) / (1 + c))
    t2 = np.array(t2)
    # delta^2 = var * z^2, z ~ N(0,1): mean var, sd var*sqrt(2)/sqrt(n)
    assert abs(t2.mean() - var) < 3 * var * np.sqrt(2.0 / t2.size)


def test_cell_constant_si_form(oracle_mod):
    """C_j = e^4 n lnL dt / (8 pi eps0^2 m_r^2), m_r = m/2, n = N w / V (R5, R6)."""
    O = oracle_mod
    Cj = O.cell_constant(1000, 1e10, 1e-6, 10.0, 1e-10)
    n = 1000 * 1e10 / 1e-6
    e = W.Q_E
    expect = e ** 4 * n * 10.0 * 1e-10 / (8 * np.pi * W.EPS0 ** 2 * (W.M_E / 2) ** 2)
    assert abs(Cj - expect) <= 1e-14 * expect
    # <delta^2> at the rms relative speed of a 2 eV plasma is ~0.005 (small angle)
    urms = np.sqrt(6.0) * W.sigma_v(2.0)
    assert 1e-3 < Cj / urms ** 3 < 2e-2
    assert O.cell_constant(1000, 1e10, 1e-6, -1.0, 1e-10) == 0.0


def test_cell_constant_from_rutherford_momentum_transfer(oracle_mod):
    """C_j pinned by a different route than its own formula: TA's small-angle sampler accumulates
    <1 - cos Theta> = 2 <delta^2> per step, and for Coulomb scattering that equals the momentum-
    transfer rate nu_m dt = n sigma_m u dt with the Rutherford cross section integrated over impact
    parameters, sigma_m = int (1 - cos chi) 2 pi b db = 4 pi b90^2 lnL, b90 = e^2 / (4 pi eps0 m_r u^2)
    (tan(chi/2) = b90 / b).  So <delta^2> = n sigma_m u dt / 2 must equal the oracle's C_j / u^3 at
    every u, to rounding; constants from scipy.constants (CODATA 2018, not the oracle's retyped ones).
    Catches any factor of 2, pi, m vs m_r or eps0 power in C_j (the NRL relaxation pin only bounds
    it to 5%)."""
    import scipy.constants as sc
    O = oracle_mod
    N, w, V, lnL, dt = 2500, 3.7e9, 2e-6, 9.3, 7e-11
    n = N * w / V
    mr = sc.m_e / 2
    Cj = O.cell_constant(N, w, V, lnL, dt, mass=sc.m_e, charge=sc.e, eps0=sc.epsilon_0)
    for u in (1e4, 3.3e5, 2e6, 7.5e7):
        b90 = sc.e ** 2 / (4 * np.pi * sc.epsilon_0 * mr * u ** 2)
        sigma_m = 4 * np.pi * b90 ** 2 * lnL
        delta2 = n * sigma_m * u * dt / 2
        assert abs(Cj / u ** 3 - delta2) <= 1e-13 * delta2, (u, Cj / u ** 3, delta2)
