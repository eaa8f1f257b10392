"""Pins of the oracle's NEXT f3 recombination (Table 4 RS0-RS5, P:262-290;
SPEC recomb S:271-330; readings R25-R28).  The pins come from the SPEC's worked
examples (1 primary + 1 catalyte, 2 primaries + 1 catalyte, forced pi = 0 / 1,
the binomial count), the energy ledger of the RS4 rule (exact to rounding),
structural invariants (injective, cell-local matching; ledger identities) and
the statistics of the catalyte choice (uniform over the cell's non-primaries,
chi^2 over many steps of a real collision + recombination chain)."""
import numpy as np
import pytest

import oracle
import workloads as W

M_E = oracle.M_E
EB = 15.76 * oracle.Q_E           # argon ionisation energy as the released binding energy [J]


def uniforms(N, G, step, seed=42):
    out = []
    for q in range(N):
        x = oracle.philox4x32_10([q, G, step, 4], [seed & 0xFFFFFFFF, seed >> 32])
        out.append(oracle.u01(int(x[0]), int(x[1])))
    return np.array(out)


def test_one_primary_one_catalyte():
    u = uniforms(2, 7, 3)
    prob = np.array([0.5 * (u.min() + u.max())])
    v = np.array([[1e5, -2e5], [3e5, 1e5], [-4e5, 2e5]])
    v_out, c_out, st = oracle.recombine(v, np.zeros(2, np.int32), 1, prob, eps_bind=EB, cell_base=7, step=3)
    p, c = int(np.argmin(u)), int(np.argmax(u))
    assert list(st) == [1, 0, 1]
    assert c_out[p] == -1 and c_out[c] == 0
    assert np.array_equal(v_out[:, p], v[:, p])                     # the dead primary keeps its v
    expect2 = (v[:, c] ** 2).sum() + (v[:, p] ** 2).sum() + 2 * EB / M_E
    assert abs((v_out[:, c] ** 2).sum() / expect2 - 1) < 1e-15
    assert np.allclose(np.cross(v_out[:, c], v[:, c]), 0, atol=1e-9 * expect2)   # direction kept
    assert np.dot(v_out[:, c], v[:, c]) > 0


def test_two_primaries_one_catalyte_and_forced_probabilities():
    u = np.sort(uniforms(3, 0, 0))
    prob = np.array([0.5 * (u[1] + u[2])])                          # two primaries
    v = np.random.default_rng(1).normal(0, 5e5, (3, 3))
    _, c_out, st = oracle.recombine(v, np.zeros(3, np.int32), 1, prob, eps_bind=EB)
    assert list(st) == [1, 1, 2] and (c_out == -1).sum() == 1
    for pr, expect in ((0.0, [0, 0, 0]), (1.0, [0, 3, 3])):
        v2, c2, st = oracle.recombine(v, np.zeros(3, np.int32), 1, np.array([pr]), eps_bind=EB)
        assert list(st) == expect and np.array_equal(v2, v) and np.all(c2 == 0)


def test_binomial_count():
    """uniform pi = 0.01, N = 1e5 -> 1000 +- 3 sigma (sigma ~ 31.5)."""
    n, M = 100_000, 10
    cell = np.repeat(np.arange(M, dtype=np.int32), n // M)
    v = np.random.default_rng(2).normal(0, 5e5, (3, n))
    _, _, st = oracle.recombine(v, cell, M, np.full(M, 0.01), eps_bind=EB, step=11)
    assert abs(st[2] - 1000) <= 3 * np.sqrt(n * 0.01 * 0.99)
    assert st[0] == st[2] and st[1] == 0


def test_energy_ledger_matching_invariants():
    w = W.random_cells(60_000, 40, seed=3, skew=True, dead_frac=0.01)
    r = oracle.coulomb_collide(w.v, w.cell, 40, step=2, want_pairs=False, **w.params())
    prob = np.random.default_rng(4).uniform(0, 0.3, 40)
    v2, c2, st = oracle.recombine(r.v_out, r.cell_out, 40, prob, eps_bind=EB, step=2)
    live0, live1 = r.cell_out >= 0, c2 >= 0
    assert st[0] + st[1] == st[2]
    assert live0.sum() - live1.sum() == st[0]                      # live count drops by `recombined`
    ke = lambda vv, m: 0.5 * M_E * (vv[:, m] ** 2).sum()
    assert abs(ke(v2, live1) - (ke(r.v_out, live0) + st[0] * EB)) <= 1e-12 * ke(r.v_out, live0)
    changed = np.any(v2 != r.v_out, axis=0)
    killed = live0 & ~live1
    assert changed.sum() == killed.sum() == st[0]                  # one catalyte per primary: injective
    assert not np.any(changed & killed)
    for j in range(40):                                             # cell-local
        sel = r.cell_out == j
        assert (changed & sel).sum() == (killed & sel).sum()


def test_catalyte_uniform_over_non_primaries():
    """N = 5 electrons in one cell, prob 0.2; chain collide -> recombine (primaries
    revived each step) over 6000 steps: every electron is the catalyte equally
    often (chi^2 at alpha = 0.001)."""
    from scipy.stats import chisquare
    rng = np.random.default_rng(5)
    v = rng.normal(0, 5e5, (3, 5))
    cell = np.zeros(5, np.int32)
    hits = np.zeros(5)
    prm = dict(dt=1e-10, weight=1e13, cell_volume=1e-6)
    for s in range(6000):
        r = oracle.coulomb_collide(v, cell, 1, step=s, want_pairs=False, **prm)
        v2, c2, st = oracle.recombine(r.v_out, r.cell_out, 1, np.array([0.2]), eps_bind=0.0, step=s)
        if st[0] == 1:
            changed = np.nonzero(np.any(v2 != r.v_out, axis=0) & (c2 >= 0))[0]
            if changed.size == 1:
                hits[r.perm_out[changed[0]]] += 1
        v = r.v_out[:, np.argsort(r.perm_out)]                      # back to the original labels
        v /= np.sqrt((v ** 2).sum(axis=0) / (3 * 3.5e11))           # keep speeds bounded (eps_bind 0 still heats)
    assert hits.sum() > 1500
    assert chisquare(hits).pvalue > 1e-3
