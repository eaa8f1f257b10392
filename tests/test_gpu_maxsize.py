"""Maximum size: one call with as many particles as the GPU holds (n up to 2^31 - 1, the ABI's
limit; ~98 bytes of device memory per particle: inputs, outputs and workspace), so that every
int32 particle index, int64 byte offset and tile/chunk count runs near its largest value.
Inputs are drawn on the device (workloads.device_random_cells; randomly ordered, 1024 cells of
~1.6e6 e- each, so the keyed Feistel works on its widest halves).  The oracle recomputes sampled
cells one by one; permutation, sortedness, counts and the diagnostics are checked on the whole
output (the properties that hold at any size)."""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2508_06771_b200 as cc  # noqa: E402

DEV = torch.device("cuda:0")
BYTES_PER_PARTICLE = 98          # v_in 24 + cell 4 + v_out 24 + cell_out 4 + perm 4 + workspace ~37 (+ slack)


@pytest.fixture(scope="module")
def O():
    import oracle
    oracle.build()
    return oracle


def _chunks(n, step=1 << 28):
    for a in range(0, n, step):
        yield a, min(n, a + step)


def test_max_size_call(O):
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info(DEV)
    M = 1024
    margin = 12 << 30                 # chunked checks, oracle sample, allocator slack
    n = (1 << 31) - 1
    # inputs v 24 + cell 4, outputs v 24 + cell 4 + perm 4 bytes per particle, plus the workspace
    while n > 0 and 60 * n + cc.cc_workspace_bytes(n, M) + margin > free:
        n = int(n * 0.97)
    n -= n % M
    if n < 500_000_000:
        pytest.skip(f"only {free / 2**30:.0f} GiB free: the maximum-size case needs a B200-class GPU")
    v, cell, p = W.device_random_cells(n, M, seed=W.DATA_SEED_BASE + 99, device=DEV)
    ws = cc.alloc_workspace(n, M, DEV)
    out = cc.coulomb_collide(v, cell, M, step=7, workspace=ws, **p)
    torch.cuda.synchronize()
    assert cc.cc_device_status(ws) == 0
    del ws
    counts = torch.zeros(M, dtype=torch.int64, device=DEV)
    for a, b in _chunks(n):
        counts += torch.bincount(cell[a:b].to(torch.int64), minlength=M)
    off = np.concatenate([[0], np.cumsum(counts.cpu().numpy())])
    # whole-output properties
    d = out.diag.cpu().numpy()
    assert d[0] == n and d[2] == np.sum(np.diff(off) // 2) and d[3] == np.sum(np.diff(off) % 2)
    assert abs(d[11] - d[7]) <= 1e-13 * d[7]                       # energy conserved to rounding
    for q in range(3):                                               # momentum
        assert abs(d[8 + q] - d[4 + q]) <= 1e-12 * float(v[q].abs().sum())
    seen = torch.zeros(n, dtype=torch.bool, device=DEV)
    for a, b in _chunks(n):
        seen[out.perm_out[a:b].to(torch.int64)] = True               # perm is a bijection of [0, n)
    assert bool(seen.all())
    del seen
    ok = True
    for a, b in _chunks(n - 1):
        ok = ok and bool((out.cell_out[a + 1:b + 1] >= out.cell_out[a:b]).all())
    assert ok
    bounds = torch.searchsorted(out.cell_out, torch.arange(M + 1, dtype=torch.int32, device=DEV))
    assert np.array_equal(bounds.cpu().numpy(), off)
    # sampled cells against the oracle (first, a middle one, last)
    worst = 0.0
    for j in (0, M // 2 + 3, M - 1):
        idx = torch.nonzero(cell == j).flatten()
        vj = v[:, idx].cpu().numpy()
        ref = O.coulomb_collide(vj, np.zeros(idx.numel(), np.int32), 1, dt=p["dt"], weight=p["weight"],
                                cell_volume=p["cell_volume"], ln_lambda=p["ln_lambda"], cell_base=j,
                                seed=p["seed"], step=7, want_pairs=False)
        a, b = int(off[j]), int(off[j + 1])
        assert np.array_equal(out.perm_out[a:b].cpu().numpy(), idx.cpu().numpy()[ref.perm_out])
        g = out.v_out[:, a:b].cpu().numpy()
        scale = np.maximum(np.linalg.norm(ref.v_out, axis=0), 1e-3 * W.sigma_v(2.0))
        worst = max(worst, float(np.max(np.abs(g - ref.v_out) / scale)))
        m, r = out.moments[j].cpu().numpy(), ref.moments[0]
        assert abs(m[0] - r[0]) <= 1e-15 * r[0]
        assert np.all(np.abs(m[4:7] - r[4:7]) <= 1e-12 * r[4:7])
    assert worst <= 1e-12, worst
    print(f"max-size call: n = {n} ({n / 2**31:.3f} x 2^31), {M} cells, sampled-cell max rel err {worst:.2e}")
