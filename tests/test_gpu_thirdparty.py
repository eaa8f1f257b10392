"""Third-party cross-checks (SURVEY §8(c) "What pins each part"), on the GPU:

  - binning: cub::DeviceRadixSort::SortPairs — a stable radix sort from the CUDA toolkit that the
    product does not use — of (cell key, input index) gives exactly cc_bin's stable order
    (CCS1-CCS3; dead and invalid ids last, key = cells), at small sizes and at C4's;
  - randoms: cuRAND's device curand_Philox4x32_10 (curand_philox4x32_x.h) on the same counters
    and keys returns cc_philox's words bit for bit (CCS4; reading R3).
The helper library tests/helpers/libthirdparty.so is test infrastructure (built with nvcc)."""
import ctypes as C
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2508_06771_b200 as cc  # noqa: E402
import workloads as W  # noqa: E402

DEV = torch.device("cuda:0")


@pytest.fixture(scope="module")
def TP():
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import helpers
    L = C.CDLL(helpers.build())
    L.tp_sort_temp_bytes.argtypes = [C.c_int]
    L.tp_sort_temp_bytes.restype = C.c_size_t
    L.tp_sort_pairs.argtypes = [C.c_void_p] * 4 + [C.c_int, C.c_int, C.c_void_p, C.c_size_t, C.c_void_p]
    L.tp_philox.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_int64, C.c_void_p]
    return L


def p(t):
    return C.c_void_p(t.data_ptr())


def cub_stable_order(TP, cell, cells):
    n = cell.numel()
    key = torch.where((cell < 0) | (cell >= cells), torch.full_like(cell, cells), cell)
    idx = torch.arange(n, dtype=torch.int32, device=DEV)
    ko, vo = torch.empty_like(key), torch.empty_like(idx)
    tb = TP.tp_sort_temp_bytes(n)
    tmp = torch.empty(max(tb, 1), dtype=torch.uint8, device=DEV)
    end_bit = max(1, int(cells).bit_length())
    st = C.c_void_p(torch.cuda.current_stream(DEV).cuda_stream)
    assert TP.tp_sort_pairs(p(key), p(ko), p(idx), p(vo), n, end_bit, p(tmp), tb, st) == 0
    return ko, vo


@pytest.mark.parametrize("n,M,dead", [(1, 1, 0.0), (1000, 7, 0.1), (300_000, 4096, 0.02), (2_000_000, 32768, 0.0),
                                      (500_000, 3, 0.3)])
def test_cub_sort_pairs_equals_cc_bin(TP, n, M, dead):
    w = W.random_cells(n, M, seed=n + M, dead_frac=dead, skew=True)
    cell = torch.from_numpy(w.cell).to(DEV)
    perm, off = cc.cc_bin(cell, M)
    ko, vo = cub_stable_order(TP, cell, M)
    assert torch.equal(perm, vo)
    counts = torch.bincount(ko.to(torch.int64), minlength=M + 1)[:M]
    assert torch.equal(off[1:].to(torch.int64) - off[:-1].to(torch.int64), counts)


def test_cub_sort_pairs_equals_cc_bin_full_size(TP):
    w = W.c4()
    cell = torch.from_numpy(w.cell).to(DEV)
    perm, off = cc.cc_bin(cell, w.cells)
    _, vo = cub_stable_order(TP, cell, w.cells)
    assert torch.equal(perm, vo)
    assert int(off[-1]) == w.n


def test_curand_philox_equals_cc_philox(TP):
    rng = np.random.default_rng(7)
    m = 1 << 20
    ctr = rng.integers(0, 2 ** 32, (m, 4), dtype=np.uint64).astype(np.uint32)
    ctr[0] = 0
    ctr[1] = 0xFFFFFFFF
    ctr[2] = [0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344]
    # the product's own counter layout too: (k, G, step, purpose)
    ctr[3:1003, 0] = np.arange(1000)
    ctr[3:1003, 1] = 1234
    ctr[3:1003, 2] = 17
    ctr[3:1003, 3] = 0
    c = torch.from_numpy(ctr.view(np.int32)).to(DEV)
    st = C.c_void_p(torch.cuda.current_stream(DEV).cuda_stream)
    for seed in (0, 42, 0xA4093822299F31D0, 0xFFFFFFFFFFFFFFFF, 2508_06771):
        ours = cc.cc_philox(c, seed)
        ref = torch.empty_like(c)
        assert TP.tp_philox(p(c), seed, p(ref), m, st) == 0
        assert torch.equal(ours, ref), hex(seed)
