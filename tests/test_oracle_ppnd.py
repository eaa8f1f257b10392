"""Pins for AS241 PPND16 (reading R4): the inverse normal CDF that turns u1 into delta.

Pinned against CPython's ``statistics.NormalDist.inv_cdf`` (an independent
implementation of Wichura's AS241) and scipy's ``ndtri`` (Cephes, a
different algorithm), plus exact antisymmetry on the U grid.
"""
import statistics

import numpy as np
import scipy.special as sp


def _grid():
    rng = np.random.default_rng(1)
    u = list(rng.random(5000))
    u += [2.0 ** -53, 1 - 2.0 ** -53, 1e-300, 1e-20, 1e-10, 0.075, 0.075 + 1e-12, 0.0749999999,
          0.925, 0.5 + 2.0 ** -53, 0.5 - 2.0 ** -53, float(np.exp(-25.0)), float(np.exp(-25.0)) * 1.0001,
          0.25, 0.975]
    return u


def test_ppnd16_matches_cpython_as241(oracle_mod):
    nd = statistics.NormalDist()
    for p in _grid():
        a, b = oracle_mod.ppnd16(p), nd.inv_cdf(p)
        assert abs(a - b) <= 4 * np.spacing(abs(b)), (p, a, b)


def test_ppnd16_matches_ndtri(oracle_mod):
    for p in _grid():
        a, b = oracle_mod.ppnd16(p), float(sp.ndtri(p))
        assert abs(a - b) <= 1e-14 * max(abs(b), 1e-3), (p, a, b)


def test_ppnd16_known_values(oracle_mod):
    assert oracle_mod.ppnd16(0.975) == 1.9599639845400536
    assert oracle_mod.ppnd16(0.25) == -0.6744897501960817


def test_ppnd16_exact_antisymmetry_on_u_grid(oracle_mod):
    O = oracle_mod
    rng = np.random.default_rng(2)
    for hi, lo in rng.integers(0, 2 ** 32, size=(3000, 2)):
        u = O.u01(int(hi), int(lo))
        assert O.ppnd16(1.0 - u) == -O.ppnd16(u)
