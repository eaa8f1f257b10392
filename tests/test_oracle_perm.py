"""Pins for the in-cell pairing permutation pi_j (readings R1 and R1b).

R1 (CC_CELL_UNIFORM) permutes the whole cell; R1b (the default) permutes random blocks of
whole 32-slot segments and equals R1 for N <= BLOCK = 384."""
import itertools

import numpy as np
import pytest
import scipy.stats as st


def test_bijection_bruteforce(oracle_mod):
    O = oracle_mod
    for N in list(range(1, 300)) + [383, 384, 385, 386, 511, 512, 513, 767, 768, 769, 1000, 2079, 2080, 2081,
                                    4096, 4097, 25_000, 100_003]:
        for G, step in [(0, 0), (5, 17), (123456, 99)]:
            for uniform in (False, True):
                p = O.cell_perm(N, G, step, 42, uniform=uniform)
                assert np.array_equal(np.sort(p), np.arange(N)), (N, G, step, uniform)


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
        p = O.cell_perm(N, 9, s, 42, uniform=True)
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


# ---------------------------------------------------------------- R1b (blocked pairing)
def _blocks(N):
    """Block b's pair-order positions [b*BLOCK, min((b+1)*BLOCK, N))."""
    from oracle import BLOCK
    return [(b * BLOCK, min((b + 1) * BLOCK, N)) for b in range((N + BLOCK - 1) // BLOCK)]


@pytest.mark.parametrize("N", [385, 400, 767, 768, 800, 1000, 2080, 2081, 4097, 25_000])
def test_blocks_are_unions_of_whole_segments(oracle_mod, N):
    """Every block holds whole 32-slot segments: 12 full ones, except the last block, which
    holds the remaining full segments and the tail [32*floor(N/32), N)."""
    O = oracle_mod
    Sf, tail = divmod(N, O.SEG)
    for step in range(3):
        p = O.cell_perm(N, 11, step, 42)
        seen = set()
        blocks = _blocks(N)
        for b, (q0, q1) in enumerate(blocks):
            slots = np.sort(p[q0:q1])
            segs = np.unique(slots // O.SEG)
            # whole segments: the block's slots are exactly the union of the segments it touches
            union = np.concatenate([np.arange(s * O.SEG, min((s + 1) * O.SEG, N)) for s in segs])
            assert np.array_equal(slots, union), (N, b)
            full = [s for s in segs if s < Sf]
            if b < len(blocks) - 1:
                assert len(full) == O.BLOCK_SEGS and (Sf not in segs or tail == 0)
            else:
                assert (tail == 0) or (Sf in segs)
            assert not (set(segs) & seen)
            seen |= set(segs)


def test_segment_to_block_assignment_is_uniform(oracle_mod):
    """A full segment lands in block b with probability (full segments of b) / S_f, for both
    forms of the segment order (sort by key: S_f <= 64; Feistel: S_f > 64)."""
    O = oracle_mod
    for N, steps in [(1000, 3000), (2080, 3000), (3000, 1500)]:
        Sf, tail = divmod(N, O.SEG)
        S = Sf + (tail > 0)
        nb = -(-S // O.BLOCK_SEGS)
        full_in = [O.BLOCK_SEGS] * (nb - 1) + [Sf - O.BLOCK_SEGS * (nb - 1)]
        obs = np.zeros((Sf, nb))
        for step in range(steps):
            p = O.cell_perm(N, 21, step, 42)
            for b, (q0, q1) in enumerate(_blocks(N)):
                for s in np.unique(p[q0:q1] // O.SEG):
                    if s < Sf:
                        obs[s, b] += 1
        exp = np.outer(np.ones(Sf), np.array(full_in) / Sf) * steps
        chi = ((obs - exp) ** 2 / exp).sum()
        dof = (Sf - 1) * (nb - 1)
        assert st.chi2.sf(chi, dof) > 1e-4, (N, chi, dof)


def test_partner_distribution_matches_block_structure(oracle_mod):
    """N = 768: two blocks of 12 random segments.  Slot 0's partner is a given slot of its own
    segment with probability 1/383, a given slot of another segment with (11/23)/383 — the
    probabilities of a uniform matching inside a uniformly random half of the segments."""
    O = oracle_mod
    N, steps = 768, 40_000
    hist = np.zeros(N)
    for step in range(steps):
        p = O.cell_perm(N, 5, step, 42)
        q = int(np.nonzero(p == 0)[0][0])
        hist[p[q ^ 1]] += 1
    exp = np.where(np.arange(N) < 32, 1.0 / 383, (11 / 23) / 383)
    exp[0] = 0.0
    exp *= steps
    # chi^2 over the 31 same-segment slots (pooled) and the 23 other segments (pooled per segment)
    obs_c = [hist[1:32].sum()] + [hist[s * 32:(s + 1) * 32].sum() for s in range(1, 24)]
    exp_c = [exp[1:32].sum()] + [exp[s * 32:(s + 1) * 32].sum() for s in range(1, 24)]
    chi = sum((o - e) ** 2 / e for o, e in zip(obs_c, exp_c))
    assert st.chi2.sf(chi, len(obs_c) - 1) > 1e-4, chi
    # inside the segment: uniform over its 31 other slots
    assert st.chisquare(hist[1:32]).pvalue > 1e-4


@pytest.mark.parametrize("N", [1000, 25_000])
def test_last_steps_partners_repair_at_block_rate(oracle_mod, N):
    """Warm input (stable order = last step's pair order: partners in slots 2k, 2k+1, which
    share a segment and hence a block) re-pairs a last-step pair with probability 1/(n_b - 1)
    per step — 1/383 in full blocks — against 1/(N - 1) for R1 over the whole cell."""
    O = oracle_mod
    steps = {1000: 3000, 25_000: 200}[N]
    hits = tot = 0
    exp = 0.0
    for step in range(steps):
        p = O.cell_perm(N, 3, step, 42)
        for (q0, q1) in _blocks(N):
            nb = q1 - q0
            if nb < 2:
                continue
            blk = p[q0:q1]
            m = nb // 2 * 2
            a, b = blk[0:m:2], blk[1:m:2]
            lo = np.minimum(a, b)
            hits += int(np.sum((np.abs(a - b) == 1) & (lo % 2 == 0)))
            # pairs (2k, 2k+1) wholly inside this block, each re-formed with prob 1/(nb-1)
            slots = np.sort(blk)
            whole = np.sum((slots[:-1] % 2 == 0) & (slots[1:] == slots[:-1] + 1))
            exp += whole / (nb - 1)
            tot += 1
    sigma = np.sqrt(exp)
    assert abs(hits - exp) < 4 * sigma + 1, (hits, exp)


def test_blocked_equals_r1_up_to_block_size(oracle_mod):
    """N <= 384: one block whose slots are the stable slots in order, so R1b is R1."""
    O = oracle_mod
    for N in [2, 63, 64, 65, 200, 383, 384]:
        for step in range(4):
            assert np.array_equal(O.cell_perm(N, 8, step, 42), O.cell_perm(N, 8, step, 42, uniform=True))
