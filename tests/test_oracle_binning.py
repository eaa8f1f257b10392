"""Pins for CCS1-CCS3 (count, prefix sum, stable index order)."""
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_prefix_sum_spec_examples(oracle_mod):
    for line in open(os.path.join(GOLDEN, "spec_prefix_sum.txt")):
        if line.startswith("#") or not line.strip():
            continue
        a, b = line.split("|")
        counts = [int(x) for x in a.split()]
        expect = [int(x) for x in b.split()]
        assert list(oracle_mod.exclusive_scan(counts)) == expect


def test_prefix_sum_random(oracle_mod):
    c = np.random.default_rng(4).integers(0, 1000, 10_000)
    off = oracle_mod.exclusive_scan(c)
    assert off[0] == 0 and np.array_equal(np.diff(off), c)


@pytest.mark.parametrize("n,M,dead", [(0, 1, 0.0), (1, 1, 0.0), (1000, 1, 0.0), (1000, 1000, 0.0),
                                      (100_000, 100, 0.1), (50_000, 4096, 0.0), (7777, 13, 1.0)])
def test_stable_order_equals_numpy_stable_argsort(oracle_mod, n, M, dead):
    rng = np.random.default_rng(n + M)
    cell = rng.integers(0, M, n).astype(np.int32)
    cell[rng.random(n) < dead] = -1
    perm, off = oracle_mod.stable_order(cell, M)
    key = np.where(cell < 0, M, cell)
    assert np.array_equal(perm, np.argsort(key, kind="stable"))
    assert np.array_equal(off[:-1], np.searchsorted(np.sort(key), np.arange(M)))
    assert off[-1] == np.sum(cell >= 0)
    assert np.array_equal(oracle_mod.count(cell, M), np.bincount(cell[cell >= 0], minlength=M))


def test_all_in_one_cell_and_one_per_cell(oracle_mod):
    perm, off = oracle_mod.stable_order(np.zeros(100, np.int32), 1)
    assert np.array_equal(perm, np.arange(100)) and list(off) == [0, 100]
    cell = np.random.default_rng(5).permutation(100).astype(np.int32)
    perm, off = oracle_mod.stable_order(cell, 100)
    assert np.array_equal(cell[perm], np.arange(100))


def test_invalid_cell_id_rejected(oracle_mod):
    with pytest.raises(ValueError):
        oracle_mod.count(np.array([0, 5, 1], np.int32), 5)
    with pytest.raises(ValueError):
        oracle_mod.count(np.array([0, -2], np.int32), 5)
