"""Pins for the in-cell pairing permutation pi_j (reading R1)."""
import itertools

import numpy as np
import pytest
import scipy.stats as st


def test_bijection_bruteforce(oracle_mod):
    O = oracle_mod
    for N in list(range(1, 300)) + [511, 512, 513, 1000, 4096, 4097, 25_000]:
        for G, step in [(0, 0), (5, 17), (123456, 99)]:
            p = O.cell_perm(N, G, step, 42)
            assert np.array_equal(np.sort(p), np.arange(N)), (N, G, step)


def test_feistel_form_is_bijection_for_every_key(oracle_mod):
    O = oracle_mod
    rng = np.random.default_rng(3)
    for N in [65, 66, 100, 127, 128, 129, 1000, 3001]:
        for _ in range(5):
            k = rng.integers(0, 2 ** 32, 4).astype(np.uint32)
            p = [O.feistel_pi(i, N, k) for i in range(N)]
            assert sorted(p) == list(range(N))


@pytest.mark.parametrize("N", [3, 4, 5, 8, 17, 33, 64, 65, 80])
def test_pair_cooccurrence_uniform(oracle_mod, N):
    """Each unordered pair {s,t} is formed with probability 1/(N-1) per member."""
    O = oracle_mod
    S = 6000
    cnt = {}
    first = np.zeros(N)
    for s in range(S):
        p = O.cell_perm(N, 77, s, 42)
        first[p[0]] += 1
        for q in range(N // 2):
            a, b = sorted((int(p[2 * q]), int(p[2 * q + 1])))
            cnt[(a, b)] = cnt.get((a, b), 0) + 1
    obs = np.array([cnt.get(pr, 0) for pr in itertools.combinations(range(N), 2)])
    assert st.chisquare(obs).pvalue > 1e-4
    assert st.chisquare(first).pvalue > 1e-4


@pytest.mark.parametrize("N", [100, 1000, 25_000])
def test_adjacent_slots_get_independent_partners(oracle_mod, N):
    """Slots s, s+1 (a previous step's pair in warm input) must not get adjacent
    partners more often than a uniform matching does: rate*N/2 ~ 1.5."""
    O = oracle_mod
    S = {100: 1500, 1000: 300, 25_000: 20}[N]
    adj = tot = 0
    for s in range(S):
        p = O.cell_perm(N, 9, s, 42)
        partner = np.full(N, -1)
        m = N // 2 * 2
        partner[p[0:m:2]] = p[1:m:2]
        partner[p[1:m:2]] = p[0:m:2]
        i = np.arange(N - 1)
        ok = (partner[i] >= 0) & (partner[i + 1] >= 0)
        adj += int(np.sum(np.abs(partner[i[ok]] - partner[i[ok] + 1]) == 1))
        tot += int(ok.sum())
    rate = adj / tot * N / 2
    assert 1.2 < rate < 1.85, rate


def test_small_cell_form_is_sort_by_philox_key(oracle_mod):
    """N <= 64: pi lists slots by increasing (Philox word, slot) — brute force."""
    O = oracle_mod
    for N in [2, 5, 31, 64]:
        G, step, seed = 3, 8, 42 + (7 << 32)
        keys = []
        for s in range(N):
            w = O.philox4x32_10([s // 4, G, step, 2], [seed & 0xFFFFFFFF, seed >> 32])
            keys.append((int(w[s % 4]), s))
        expect = [s for _, s in sorted(keys)]
        assert list(O.cell_perm(N, G, step, seed)) == expect
