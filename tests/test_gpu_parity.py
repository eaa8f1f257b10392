"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Bars (BASELINE.json north_star):
  - binning, pairing, perm, cell ids: bit-exact
  - velocities: |v_gpu - v_ref| <= 1e-12 * max(|v_ref|_2, v_floor) per component,
    v_floor = 1e-3 sqrt(kT/m) (reading R15)
  - moments: 1e-12 relative (density exact; mean vs thermal speed; T vs T)
  - diagnostics: counts exact; sums 1e-12 of the sum of magnitudes
"""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2508_06771_b200 as cc  # noqa: E402

DEV = torch.device("cuda:0")
TOL = 1e-12


@pytest.fixture(scope="module")
def O():
    import oracle
    oracle.build()
    return oracle


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def vel_err(v_gpu, v_ref, floor):
    scale = np.maximum(np.linalg.norm(v_ref, axis=0), floor)
    return np.max(np.abs(v_gpu - v_ref) / scale) if v_ref.size else 0.0


def check_collide(O, w, step=0, moments=True, flags=0):
    p = w.params()
    out = cc.coulomb_collide(to_dev(w.v), to_dev(w.cell), w.cells, step=step, flags=flags, **p)
    torch.cuda.synchronize()
    ref = O.coulomb_collide(w.v, w.cell, w.cells, step=step, want_pairs=False, flags=flags, **p)
    assert np.array_equal(out.perm_out.cpu().numpy(), ref.perm_out)
    assert np.array_equal(out.cell_out.cpu().numpy(), ref.cell_out)
    err = vel_err(out.v_out.cpu().numpy(), ref.v_out, 1e-3 * W.sigma_v(2.0))
    assert err <= TOL, err
    if moments:
        check_moments(out.moments.cpu().numpy(), ref.moments, w)
    check_diag(out.diag.cpu().numpy(), ref.diag, ref.v_out)
    return out, ref, err


def check_moments(m, r, w):
    """Density exact to rounding; mean velocity to 1e-12 of max(|mean|, thermal
    speed); each T_c to 1e-12 of the cell's temperature scale T_x+T_y+T_z (the
    magnitude of the summed squares the component is computed from)."""
    assert np.array_equal(m[:, 0] == 0, r[:, 0] == 0)
    nz = r[:, 0] > 0
    if not nz.any():
        assert np.all(m == 0)
        return
    assert np.all(np.abs(m[nz, 0] - r[nz, 0]) <= 1e-15 * r[nz, 0])
    sig = W.sigma_v(2.0)
    assert np.max(np.abs(m[nz, 1:4] - r[nz, 1:4])) <= TOL * max(sig, np.abs(r[nz, 1:4]).max())
    T = r[nz, 4:7]
    scale = T.sum(axis=1, keepdims=True)
    assert np.all(np.abs(m[nz, 4:7] - T) <= TOL * scale + 1e-300)


def check_diag(d, r, v_ref):
    assert np.array_equal(d[[0, 1, 2, 3]], r[[0, 1, 2, 3]])
    sabs = np.abs(v_ref).sum(axis=1)
    for q in range(3):
        assert abs(d[4 + q] - r[4 + q]) <= TOL * sabs[q] + 1e-300
        assert abs(d[8 + q] - r[8 + q]) <= TOL * sabs[q] + 1e-300
    assert abs(d[7] - r[7]) <= TOL * r[7]
    assert abs(d[11] - r[11]) <= TOL * r[11]


# ------------------------------------------------------------------ element functions


def test_philox_matches_oracle_and_kat(O):
    rng = np.random.default_rng(0)
    ctr = rng.integers(0, 2 ** 32, (4096, 4), dtype=np.uint64).astype(np.uint32)
    ctr[0] = [0, 0, 0, 0]
    ctr[1] = [0xFFFFFFFF] * 4
    for seed in (0, 42, (0x299F31D0 << 32) | 0xA4093822, 0xFFFFFFFFFFFFFFFF):
        got = cc.cc_philox(to_dev(ctr.view(np.int32)), seed).cpu().numpy().view(np.uint32)
        key = [seed & 0xFFFFFFFF, seed >> 32]
        for i in range(0, 4096, 97):
            assert np.array_equal(got[i], O.philox4x32_10(ctr[i], key))
    got = cc.cc_philox(to_dev(np.array([[0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344]],
                                       np.uint32).view(np.int32)),
                       (0x299f31d0 << 32) | 0xa4093822).cpu().numpy().view(np.uint32)
    assert [hex(x) for x in got[0]] == ["0xd16cfe09", "0x94fdcceb", "0x5001e420", "0x24126ea1"]


def test_ppnd16_matches_oracle(O):
    rng = np.random.default_rng(1)
    u = np.concatenate([rng.random(20000), [2.0 ** -53, 1 - 2.0 ** -53, 1e-300, 0.075, 0.925,
                                            np.exp(-25.0), 0.5 + 2.0 ** -53]])
    z = cc.cc_ppnd16(to_dev(u)).cpu().numpy()
    ref = np.array([O.ppnd16(x) for x in u])
    assert np.all(np.abs(z - ref) <= 1e-15 * np.maximum(np.abs(ref), 1e-3))


def test_ta_pairs_match_oracle(O):
    rng = np.random.default_rng(2)
    m = 5000
    s = W.sigma_v(2.0)
    va = rng.standard_normal((3, m)) * s
    vb = rng.standard_normal((3, m)) * s
    vb[:, :10] = va[:, :10]                 # identical velocities
    vb[0:2, 10:20] = va[0:2, 10:20]         # u_perp = 0 branch
    C = 10 ** rng.uniform(10, 17, m)
    u1, u2 = rng.random(m), rng.random(m)
    ga, gb = to_dev(va), to_dev(vb)
    cc.cc_ta_pairs(ga, gb, to_dev(C), to_dev(u1), to_dev(u2))
    ga, gb = ga.cpu().numpy(), gb.cpu().numpy()
    for i in range(m):
        ra, rb = O.ta_pair(va[:, i], vb[:, i], C[i], u1[i], u2[i])
        sc = np.linalg.norm(va[:, i]) + np.linalg.norm(vb[:, i])
        assert np.max(np.abs(ga[:, i] - ra)) <= 1e-13 * sc, i
        assert np.max(np.abs(gb[:, i] - rb)) <= 1e-13 * sc, i
    assert np.array_equal(ga[:, :10], va[:, :10]) and np.array_equal(gb[:, :10], vb[:, :10])


# ------------------------------------------------------------------ binning and pairing

BIN_CASES = [(0, 1, 0.0), (1, 1, 0.0), (7, 3, 0.0), (1000, 1, 0.0), (33_000, 1, 0.0),
             (100_000, 100, 0.1), (200_003, 4096, 0.02), (70_001, 32768, 0.0),
             (50_000, 7, 1.0), (300_000, 256, 0.0)]


@pytest.mark.parametrize("n,M,dead", BIN_CASES)
def test_bin_bit_exact(O, n, M, dead):
    w = W.random_cells(n, M, seed=n + M, dead_frac=dead, skew=(M > 50))
    perm, off = cc.cc_bin(to_dev(w.cell), M)
    torch.cuda.synchronize()
    rp, roff = O.stable_order(w.cell, M)
    assert np.array_equal(off.cpu().numpy(), roff)
    assert np.array_equal(perm.cpu().numpy(), rp)


@pytest.mark.parametrize("flags", [0, 8])
@pytest.mark.parametrize("n,M", [(1000, 1), (5000, 3), (20_000, 500), (100_000, 13), (3000, 3000),
                                 (2113, 1), (4097, 1)])
def test_pairs_bit_exact(O, n, M, flags):
    """flags 0: the blocked pairing R1b (segment orders by sort-by-key for <= 64 segments and by
    Feistel above; last blocks of <= 64 slots); 8 = CC_CELL_UNIFORM: R1 over the whole cell."""
    w = W.random_cells(n, M, seed=7 * n + M, skew=True)
    _, off = cc.cc_bin(to_dev(w.cell), M)
    for step in (0, 5):
        pairs = cc.cc_pairs(off, M, cell_base=11, seed=99, step=step, flags=flags).cpu().numpy()
        ref = O.coulomb_collide(w.v, w.cell, M, cell_base=11, seed=99, step=step, flags=flags,
                                dt=w.dt, weight=w.weight, cell_volume=w.cell_volume)
        assert np.array_equal(pairs, ref.pair_slots)


# cell sizes at R1b's edges: one block (384), last blocks of 1-3 slots (385-387: the triplet
# straddles two blocks), whole segments only (768), tails (767, 769, 800), the segment order by
# sort-by-key (2047: 63 segments) vs Feistel (2080: 65, 2113), a 10-slot last block (3850)
R1B_SIZES = [384, 385, 386, 387, 767, 768, 769, 800, 2047, 2080, 2113, 3850, 4097]


@pytest.mark.parametrize("flags", [0, 1, 2])
def test_blocked_pairing_edges(O, flags):
    """Whole operator on single cells of R1b's edge sizes (flags: TA77, odd triplet — whose three
    members straddle blocks when the last block holds 1-2 slots — and Nanbu)."""
    for N in R1B_SIZES:
        w = W.random_cells(N, 1, seed=N + 5 * flags)
        check_collide(O, w, step=3 + N % 7, flags=flags)


@pytest.mark.parametrize("n,M,skew", [(120_007, 64, True), (9000, 2, False), (100_000, 1, False)])
def test_collide_parity_uniform_r1(O, n, M, skew):
    """CC_CELL_UNIFORM keeps R1 (whole-cell permutation, gathered records)."""
    w = W.random_cells(n, M, seed=n + 7 * M, dead_frac=0.02, skew=skew)
    check_collide(O, w, step=11, flags=8)
    check_collide(O, w, step=11, flags=8 | 1)


# ------------------------------------------------------------------ whole operator


@pytest.mark.parametrize("n,M,dead,skew", [(0, 4, 0.0, False), (1, 1, 0.0, False), (2, 1, 0.0, False),
                                           (65, 1, 0.0, False), (1000, 1, 0.0, False),
                                           (50_000, 50, 0.05, True), (120_007, 4096, 0.01, True),
                                           (40_000, 3000, 0.0, False), (9000, 2, 0.0, False),
                                           (100_000, 1, 0.0, False), (20_000, 9, 1.0, False)])
def test_collide_parity(O, n, M, dead, skew):
    w = W.random_cells(n, M, seed=n + 3 * M, dead_frac=dead, skew=skew)
    check_collide(O, w, step=17)


@pytest.mark.parametrize("n,M,dead", [(50_000, 64, 0.0), (80_000, 300, 0.05), (10_000, 5000, 0.1)])
def test_sorted_input_fast_path(O, n, M, dead):
    """Cell-sorted input (dead last): k_count flags it sorted, so (R1b, the default) k_scatter
    moves nothing and the collide copies each block's segments straight from the caller's SoA
    input (kModeSorted); under CC_CELL_UNIFORM k_scatter packs the records in place.  Results
    must equal the oracle's either way."""
    w = W.random_cells(n, M, seed=n + M + 1, dead_frac=dead, skew=True)
    key = np.where(w.cell < 0, M, w.cell)
    order = np.argsort(key, kind="stable")
    w.v = np.ascontiguousarray(w.v[:, order])
    w.cell = np.ascontiguousarray(w.cell[order])
    for flags in (0, 8):
        check_collide(O, w, step=4, flags=flags)
    # one element out of order: the full binning path runs instead (kModePerm: few descents)
    if n > 10:
        w.cell = w.cell.copy()
        w.cell[[1, n // 2]] = w.cell[[n // 2, 1]]
        for flags in (0, 8):
            check_collide(O, w, step=4, flags=flags)


@pytest.mark.parametrize("frac", [0.0, 0.02, 0.1, 0.3, 1.0])
def test_layout_modes_disorder(O, frac):
    """Inputs between sorted and random (sorted input with a fraction `frac` of the particles moved
    to random positions: the PIC steady state is ~0.02): the stable scatter's run structure and
    k_count's order check (4 ids per thread, neighbour-lane predecessor) give the oracle's result."""
    n, M = 200_000, 40
    w = W.random_cells(n, M, seed=77, dead_frac=0.01, skew=True)
    key = np.where(w.cell < 0, M, w.cell)
    order = np.argsort(key, kind="stable")
    rng = np.random.default_rng(5)
    mv = np.flatnonzero(rng.random(n) < frac)
    order[mv] = order[rng.permutation(mv)]
    w.v = np.ascontiguousarray(w.v[:, order])
    w.cell = np.ascontiguousarray(w.cell[order])
    check_collide(O, w, step=6)


def test_c1_chained_ten_steps(O):
    """Config 1 (1 cell, 1,000 e-, Maxwellian 2 eV, 10 steps): each step's GPU
    output feeds the next GPU step, same for the oracle; parity every step."""
    w = W.c1()
    p = w.params()
    gv, gc = to_dev(w.v), to_dev(w.cell)
    rv, rc = w.v, w.cell
    errs = []
    for s in range(10):
        out = cc.coulomb_collide(gv, gc, 1, step=s, **p)
        ref = O.coulomb_collide(rv, rc, 1, step=s, want_pairs=False, **p)
        assert np.array_equal(out.perm_out.cpu().numpy(), ref.perm_out)
        errs.append(vel_err(out.v_out.cpu().numpy(), ref.v_out, 1e-3 * W.sigma_v(2.0)))
        gv, gc = out.v_out.clone(), out.cell_out.clone()
        rv, rc = ref.v_out, ref.cell_out
    assert max(errs) <= TOL, errs


def test_c2_bimaxwellian_full(O):
    w = W.c2()
    check_collide(O, w, step=0)


def test_c3_full(O):
    w = W.c3()
    check_collide(O, w, step=2)


def test_determinism_bitwise(O):
    w = W.random_cells(300_000, 1000, seed=5, skew=True, dead_frac=0.01)
    a = cc.coulomb_collide(to_dev(w.v), to_dev(w.cell), w.cells, step=1, **w.params())
    b = cc.coulomb_collide(to_dev(w.v), to_dev(w.cell), w.cells, step=1, **w.params())
    for x, y in ((a.v_out, b.v_out), (a.perm_out, b.perm_out), (a.moments, b.moments), (a.diag, b.diag)):
        assert torch.equal(x, y)


def test_invalid_cell_ids_flagged(O):
    w = W.random_cells(10_000, 10, seed=6)
    cell = w.cell.copy()
    cell[[5, 77, 9000]] = [10, -7, 123]
    ws = cc.alloc_workspace(w.n, 10, DEV)
    out = cc.coulomb_collide(to_dev(w.v), to_dev(cell), 10, workspace=ws, step=0, **w.params())
    assert cc.cc_device_status(ws) == -4
    assert cc.cc_device_status(ws) == 0          # flag cleared
    # invalid particles are treated as dead: same as the oracle with them marked -1
    cell2 = cell.copy()
    cell2[[5, 77, 9000]] = -1
    ref = O.coulomb_collide(w.v, cell2, 10, step=0, want_pairs=False, **w.params())
    assert np.array_equal(out.perm_out.cpu().numpy(), ref.perm_out)
    assert vel_err(out.v_out.cpu().numpy(), ref.v_out, 1.0) <= TOL


def test_per_cell_arrays(O):
    w = W.random_cells(30_000, 40, seed=8, skew=True)
    rng = np.random.default_rng(8)
    V = rng.uniform(0.5e-6, 2e-6, 40)
    lnL = rng.uniform(5, 15, 40)
    p = w.params()
    out = cc.coulomb_collide(to_dev(w.v), to_dev(w.cell), 40, step=3, cell_volume_arr=to_dev(V),
                             ln_lambda_arr=to_dev(lnL), **p)
    ref = O.coulomb_collide(w.v, w.cell, 40, step=3, cell_volume_arr=V, ln_lambda_arr=lnL,
                            want_pairs=False, **p)
    assert vel_err(out.v_out.cpu().numpy(), ref.v_out, 1.0) <= TOL
    check_moments(out.moments.cpu().numpy(), ref.moments, w)


def test_moments_hook_matches_oracle(O):
    w = W.random_cells(50_000, 100, seed=9, skew=True)
    perm, off = O.stable_order(w.cell, 100)
    vs = np.ascontiguousarray(w.v[:, perm])
    m = cc.cc_moments(to_dev(vs), to_dev(off.astype(np.int32)), 100, weight=w.weight,
                      cell_volume=w.cell_volume).cpu().numpy()
    r = O.moments(vs, off, w.weight, w.cell_volume)
    check_moments(m, r, w)


def test_diag_sum_ranks():
    g = torch.arange(3 * 16, dtype=torch.float64, device=DEV).reshape(3, 16)
    assert torch.equal(cc.cc_diag_sum_ranks(g), g[0] + g[1] + g[2])


def test_steady_state_chain_with_drift(O):
    """The bench headline's input pattern: each step consumes the previous
    step's (cell-sorted, pair-ordered) output after a stand-in drift moved a
    few percent of the particles to another cell; parity every step."""
    w = W.c3(total=300_000, M=64)
    p = w.params()
    rng = np.random.default_rng(21)
    gv, gc = to_dev(w.v), to_dev(w.cell)
    rv, rc = w.v, w.cell
    for s in range(4):
        out = cc.coulomb_collide(gv, gc, w.cells, step=s, **p)
        ref = O.coulomb_collide(rv, rc, w.cells, step=s, want_pairs=False, **p)
        assert np.array_equal(out.perm_out.cpu().numpy(), ref.perm_out)
        assert vel_err(out.v_out.cpu().numpy(), ref.v_out, 1e-3 * W.sigma_v(2.0)) <= TOL
        check_moments(out.moments.cpu().numpy(), ref.moments, w)
        # stand-in drift: 3% of the live particles move to a neighbouring cell
        cell = ref.cell_out.copy()
        mv = (rng.random(cell.size) < 0.03) & (cell >= 0)
        cell[mv] = (cell[mv] + rng.choice([-1, 1], mv.sum())) % w.cells
        gv, gc = out.v_out.clone(), to_dev(cell)
        rv, rc = ref.v_out, cell


def test_strided_rows_ldv_greater_than_n(O):
    """[3][ldv] SoA views with ldv > n (odd and even ldv) are honoured."""
    w = W.random_cells(10_001, 37, seed=23, skew=True)
    for extra in (0, 3, 64):
        ldv = w.n + extra
        big = torch.zeros((3, ldv), dtype=torch.float64, device=DEV)
        big[:, : w.n] = to_dev(w.v)
        vin = big[:, : w.n]
        vout_big = torch.full((3, ldv), 7.0, dtype=torch.float64, device=DEV)
        out = cc.CollideOut(vout_big[:, : w.n], torch.empty(w.n, dtype=torch.int32, device=DEV),
                            torch.empty(w.n, dtype=torch.int32, device=DEV),
                            torch.empty((37, 7), dtype=torch.float64, device=DEV),
                            torch.empty(16, dtype=torch.float64, device=DEV))
        cc.coulomb_collide(vin, to_dev(w.cell), 37, step=2, out=out, **w.params())
        ref = O.coulomb_collide(w.v, w.cell, 37, step=2, want_pairs=False, **w.params())
        assert vel_err(vout_big[:, : w.n].cpu().numpy(), ref.v_out, 1.0) <= TOL
        assert torch.all(vout_big[:, w.n:] == 7.0)          # padding untouched


def test_large_cell_counts_and_max_cells(O):
    """A cell larger than one collide chunk's worth of pairs many times over
    (C2-like, 2e5 particles) and the CC_MAX_CELLS limit."""
    w = W.random_cells(200_001, 1, seed=24)
    check_collide(O, w, step=9)
    w = W.random_cells(100_000, cc._lib.CC_MAX_CELLS, seed=25)
    check_collide(O, w, step=1)


@pytest.mark.parametrize("flags", [1, 2, 3])
@pytest.mark.parametrize("n,M,skew", [(30_001, 7, False), (50_000, 600, True), (999, 1, False), (3, 1, False)])
def test_model_variants_parity(O, flags, n, M, skew):
    """NEXT f1: TA77 odd triplet (1), Nanbu sampler (2), both (3) vs the oracle."""
    w = W.random_cells(n, M, seed=n + M + flags, skew=skew)
    p = w.params()
    out = cc.coulomb_collide(to_dev(w.v), to_dev(w.cell), M, step=5, flags=flags, **p)
    ref = O.coulomb_collide(w.v, w.cell, M, step=5, flags=flags, want_pairs=False, **p)
    assert np.array_equal(out.perm_out.cpu().numpy(), ref.perm_out)
    assert vel_err(out.v_out.cpu().numpy(), ref.v_out, 1e-3 * W.sigma_v(2.0)) <= TOL
    check_moments(out.moments.cpu().numpy(), ref.moments, w)
    check_diag(out.diag.cpu().numpy(), ref.diag, ref.v_out)


def test_coulomb_log_matches_oracle(O):
    w = W.c3(total=500_000, M=64)
    out = cc.coulomb_collide(to_dev(w.v), to_dev(w.cell), w.cells, step=0, **w.params())
    lnl = cc.cc_coulomb_log(out.moments).cpu().numpy()
    ref = O.coulomb_log(out.moments.cpu().numpy())
    assert np.max(np.abs(lnl - ref)) <= 1e-13 * np.max(ref)
    # feed it back as the per-cell Coulomb logarithm of the next step
    out2 = cc.coulomb_collide(out.v_out, out.cell_out, w.cells, step=1, ln_lambda_arr=to_dev(ref), **w.params())
    r2 = O.coulomb_collide(out.v_out.cpu().numpy(), out.cell_out.cpu().numpy(), w.cells, step=1,
                           ln_lambda_arr=ref, want_pairs=False, **w.params())
    assert vel_err(out2.v_out.cpu().numpy(), r2.v_out, 1.0) <= TOL


@pytest.mark.parametrize("flags", [0, 1, 2])
@pytest.mark.parametrize("n,M,dead,skew", [(120_007, 4096, 0.02, True), (50_000, 40, 0.0, False), (999, 1, 0.1, False)])
def test_preserve_order_parity(O, flags, n, M, dead, skew):
    """CC_PRESERVE_ORDER: outputs in input order vs the oracle's un-permute,
    small (N <= 64, warp path) and large cells, dead particles, f1 variants."""
    w = W.random_cells(n, M, seed=n + M + flags, dead_frac=dead, skew=skew)
    p = w.params()
    f = flags | cc._lib.CC_PRESERVE_ORDER
    out = cc.coulomb_collide(to_dev(w.v), to_dev(w.cell), M, step=6, flags=f, **p)
    ref = O.coulomb_collide(w.v, w.cell, M, step=6, flags=f, want_pairs=False, **p)
    assert np.array_equal(out.perm_out.cpu().numpy(), np.arange(n))
    assert np.array_equal(out.cell_out.cpu().numpy(), ref.cell_out)
    assert vel_err(out.v_out.cpu().numpy(), ref.v_out, 1e-3 * W.sigma_v(2.0)) <= TOL
    check_moments(out.moments.cpu().numpy(), ref.moments, w)
    check_diag(out.diag.cpu().numpy(), ref.diag, ref.v_out)


def test_preserve_order_edge_cases(O):
    """CC_PRESERVE_ORDER with no particles, all dead, strided rows (ldv > n) and no perm output."""
    f = cc._lib.CC_PRESERVE_ORDER
    out = cc.coulomb_collide(torch.zeros((3, 0), dtype=torch.float64, device=DEV),
                             torch.zeros(0, dtype=torch.int32, device=DEV), 3, step=0, flags=f, dt=1e-10)
    assert out.v_out.numel() == 0
    w = W.random_cells(5000, 7, seed=3, dead_frac=1.0)
    out = cc.coulomb_collide(to_dev(w.v), to_dev(w.cell), 7, step=0, flags=f, **w.params())
    assert torch.equal(out.v_out.cpu(), torch.from_numpy(w.v)) and bool((out.cell_out == -1).all())
    w = W.random_cells(10_001, 13, seed=4, skew=True, dead_frac=0.1)
    big = torch.zeros((3, w.n + 7), dtype=torch.float64, device=DEV)
    big[:, : w.n] = to_dev(w.v)
    vout = torch.full((3, w.n + 7), 5.0, dtype=torch.float64, device=DEV)
    res = cc.CollideOut(vout[:, : w.n], torch.empty(w.n, dtype=torch.int32, device=DEV), None,
                        torch.empty((13, 7), dtype=torch.float64, device=DEV),
                        torch.empty(16, dtype=torch.float64, device=DEV))
    cc.coulomb_collide(big[:, : w.n], to_dev(w.cell), 13, step=1, out=res, flags=f, **w.params())
    ref = O.coulomb_collide(w.v, w.cell, 13, step=1, flags=f, want_pairs=False, **w.params())
    assert vel_err(vout[:, : w.n].cpu().numpy(), ref.v_out, 1.0) <= TOL
    assert torch.all(vout[:, w.n:] == 5.0)
    assert np.array_equal(res.cell_out.cpu().numpy(), ref.cell_out)
