"""Device-side migration between cell-range shards (cc_mig_pack / cc_mig_unpack),
with P ranks simulated in one process on one GPU: every rank packs, the slots are exchanged by
device copies (what cc_dist_mig_exchange's fixed-size ncclSend / ncclRecv do between GPUs), every
rank unpacks.  Compared BIT-exactly with a numpy statement of the contract: stayers keep their
slot with a LOCAL id, leavers are dead here, arrivals land at [L, L + A) in (source rank, source
order), nothing else changes; status counts arrivals and overflow.  No count reaches the host
inside a migration (the Migrator never calls .cpu() / .item())."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2508_06771_b200 import dist as ccd  # noqa: E402

DEV = torch.device("cuda:0")


def make_rank(rng, n, L, bounds, r, p_leave, xrows, outside=0):
    lo, hi = bounds[r], bounds[r + 1]
    G = bounds[-1]
    cell = np.full(n, -1, np.int32)
    own = rng.integers(lo, hi, L)
    other = rng.integers(0, G, L)
    leave = rng.random(L) < p_leave
    cell[:L] = np.where(leave, other, own)
    cell[:L][rng.random(L) < 0.03] = -1                     # particles absorbed by the push
    if outside:
        cell[rng.choice(L, outside, replace=False)] = G + 5  # ids outside every range
    v = rng.normal(0.0, 1e5, (3, n))
    x = rng.uniform(0.0, 1.0, (3, n))
    return v, x, cell


def owner(c, bounds):
    if c < bounds[0] or c >= bounds[-1]:
        return -1
    return int(np.searchsorted(bounds, c, side="right") - 1)


def expected(ranks, bounds, xrows, n):
    P = len(ranks)
    out = []
    for r in range(P):
        v, x, cell, L = ranks[r]
        v2, x2, c2 = v.copy(), x.copy(), cell.copy()
        for i in range(n):
            c = cell[i]
            if c < 0:
                continue
            o = owner(c, bounds)
            c2[i] = c - bounds[r] if o == r else -1
        pos = L
        for p in range(P):
            if p == r:
                continue
            vp, xp, cp, _ = ranks[p]
            for i in range(n):
                if cp[i] >= 0 and owner(cp[i], bounds) == r:
                    v2[:, pos] = vp[:, i]
                    x2[:xrows, pos] = xp[:xrows, i]
                    c2[pos] = cp[i] - bounds[r]
                    pos += 1
        out.append((v2, x2, c2, pos - L))
    return out


def run_sim(ranks, bounds, cap, xrows, n):
    P = len(ranks)
    migs, dev = [], []
    for r in range(P):
        v, x, cell, L = ranks[r]
        m = ccd.Migrator(n, bounds, r, cap, DEV, xrows=xrows, exchange=lambda *a: None)
        dv, dx, dc = (torch.from_numpy(v.copy()).to(DEV), torch.from_numpy(x.copy()).to(DEV),
                      torch.from_numpy(cell.copy()).to(DEV))
        diag = torch.zeros(16, dtype=torch.float64, device=DEV)
        diag[0] = float(L)
        migs.append(m)
        dev.append((dv, dx, dc, diag))
    for r in range(P):
        migs[r].pack(dev[r][0], dev[r][1], dev[r][2])
    S = migs[0].slot
    for r in range(P):                       # the exchange: my slot p -> rank p's slot r
        for p in range(P):
            if p != r:
                migs[p].recv[r * S:(r + 1) * S].copy_(migs[r].send[p * S:(p + 1) * S])
    for r in range(P):
        migs[r].unpack(*dev[r])
    torch.cuda.synchronize()
    return migs, dev


@pytest.mark.parametrize("P,xrows,p_leave", [(2, 2, 0.05), (4, 3, 0.2), (3, 0, 0.5), (1, 1, 0.0)])
def test_migration_bit_exact(P, xrows, p_leave):
    rng = np.random.default_rng(P * 10 + xrows)
    G, n = 40 * P, 6000
    bounds = ccd.owner_bounds(G, P)
    ranks = []
    for r in range(P):
        L = int(rng.integers(n // 2, 2 * n // 3))
        v, x, cell = make_rank(rng, n, L, bounds, r, p_leave, xrows)
        ranks.append((v, x, cell, L))
    migs, dev = run_sim(ranks, bounds, cap=n, xrows=xrows, n=n)
    exp = expected(ranks, bounds, xrows, n)
    for r in range(P):
        v2, x2, c2, A = exp[r]
        assert np.array_equal(dev[r][2].cpu().numpy(), c2), r
        assert np.array_equal(dev[r][0].cpu().numpy(), v2), r
        if xrows:
            assert np.array_equal(dev[r][1].cpu().numpy()[:xrows], x2[:xrows]), r
        assert migs[r].status.cpu().tolist() == [0, 0, 0, A], r


def test_migration_overflow_and_outside_ids_are_counted():
    rng = np.random.default_rng(3)
    P, G, n = 2, 80, 4000
    bounds = ccd.owner_bounds(G, P)
    ranks = []
    for r in range(P):
        v, x, cell = make_rank(rng, n, 3000, bounds, r, 0.5, 0, outside=7)
        ranks.append((v, x, cell, 3000))
    migs, dev = run_sim(ranks, bounds, cap=100, xrows=0, n=n)
    for r in range(P):
        st = migs[r].status.cpu().tolist()
        leavers = sum(1 for c in ranks[r][2] if c >= 0 and owner(c, bounds) not in (-1, r))
        assert st[0] == leavers - 100 and st[1] == 7 and st[3] == 100
    # arrivals that do not fit into [L, n) are counted, not written past n
    ranks2 = [(v, x, c, n - 10) for (v, x, c, _) in ranks]
    migs, dev = run_sim(ranks2, bounds, cap=100, xrows=0, n=n)
    for r in range(P):
        st = migs[r].status.cpu().tolist()
        assert st[2] == 90 and st[3] == 100
