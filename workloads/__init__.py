"""Seeded synthetic inputs for the e–e Coulomb collision operator.

This module is shared by the oracle side (tests, cpu_baseline) and the CUDA
side (tests, bench, smoke).  It holds NO arithmetic of the method: it draws
velocities and cell ids from plain distributions (numpy PCG64, seeded) and
sets physical parameters.  The recipes follow BASELINE.json's configs and
DESIGN.md §4 ("input recipe"):

  C1  single cell, 1,000 e-, isotropic Maxwellian 2 eV, 10 steps
  C2  single cell, 1e5 e-, bi-Maxwellian T_par (z) = 1 eV, T_perp = 2.5 eV
  C3  1D glow-discharge profile: 256 cells, 2.56e6 e-, density
      0.1 + 0.9 sin(pi (j+1/2)/256), T_j = 2 + 2 (1 - sin(...)) eV, drift
      1e4 m/s along x
  C4  2D discharge: 64 x 64 = 4096 cells x 25,000 e- (1.024e8), Maxwellian 2 eV
  C4b C4 with a 2D sine density profile normalised to the same n
  C5  C4 per GPU, rank r owns global cells [4096 r, 4096 (r+1))

Particle order is a random permutation ("cold": the paper stores particles
unsorted) unless ``sorted_input=True``.  Dead particles (cell id -1)
can be sprinkled in with ``dead_frac``.

Physical parameters (the paper prints none for this operator; DESIGN R5-R7):
m = m_e, CODATA 2018; dt = 1e-10 s; lnL = 10; reference density n_e = 1e19
m^-3 at the mean cell population; cell volume 1e-6 m^3; weight w =
n_ref V / N_mean (uniform weights).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

M_E = 9.1093837015e-31
Q_E = 1.602176634e-19
EPS0 = 8.8541878128e-12

DATA_SEED_BASE = 2508_06771
COLLISION_SEED = 42
DT = 1e-10
LN_LAMBDA = 10.0
N_REF = 1e19
CELL_VOLUME = 1e-6


@dataclass
class Workload:
    name: str
    v: np.ndarray            # [3][n] float64, SoA
    cell: np.ndarray         # [n] int32, -1 = dead
    cells: int               # local cells M
    cell_base: int = 0
    dt: float = DT
    weight: float = 1.0
    cell_volume: float = CELL_VOLUME
    ln_lambda: float = LN_LAMBDA
    seed: int = COLLISION_SEED
    steps: int = 1
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.cell.size)

    def params(self) -> dict:
        return dict(dt=self.dt, weight=self.weight, cell_volume=self.cell_volume,
                    ln_lambda=self.ln_lambda, cell_base=self.cell_base, seed=self.seed)


def sigma_v(T_eV: float, mass: float = M_E) -> float:
    """Thermal speed per component sqrt(kT/m) for T in eV."""
    return float(np.sqrt(T_eV * Q_E / mass))


def weight_for(n_mean: float, n_ref: float = N_REF, volume: float = CELL_VOLUME) -> float:
    return n_ref * volume / n_mean


def _finish(rng, v, cell, sorted_input, dead_frac):
    n = cell.size
    if dead_frac > 0.0:
        dead = rng.random(n) < dead_frac
        cell = cell.copy()
        cell[dead] = -1
    if not sorted_input:
        p = rng.permutation(n)
        v = np.ascontiguousarray(v[:, p])
        cell = np.ascontiguousarray(cell[p])
    return np.ascontiguousarray(v, dtype=np.float64), np.ascontiguousarray(cell, dtype=np.int32)


def maxwellian_cells(counts, T_eV, drift=(0.0, 0.0, 0.0), *, seed, sorted_input=False,
                     dead_frac=0.0, T_par_eV=None):
    """Cells with given populations; per-cell (or scalar) temperature.

    If ``T_par_eV`` is given, the distribution is bi-Maxwellian with T_perp =
    T_eV on x, y and T_par on z.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    counts = np.asarray(counts, dtype=np.int64)
    n = int(counts.sum())
    cell = np.repeat(np.arange(counts.size, dtype=np.int32), counts)
    T = np.broadcast_to(np.asarray(T_eV, dtype=np.float64), (counts.size,))
    s_perp = np.sqrt(T * Q_E / M_E)[cell]
    if T_par_eV is None:
        s_par = s_perp
    else:
        Tp = np.broadcast_to(np.asarray(T_par_eV, dtype=np.float64), (counts.size,))
        s_par = np.sqrt(Tp * Q_E / M_E)[cell]
    v = np.empty((3, n), np.float64)
    v[0] = rng.standard_normal(n) * s_perp + drift[0]
    v[1] = rng.standard_normal(n) * s_perp + drift[1]
    v[2] = rng.standard_normal(n) * s_par + drift[2]
    return _finish(rng, v, cell, sorted_input, dead_frac)


def largest_remainder(total: int, shape) -> np.ndarray:
    shape = np.asarray(shape, dtype=np.float64)
    ideal = total * shape / shape.sum()
    base = np.floor(ideal).astype(np.int64)
    rem = total - int(base.sum())
    order = np.argsort(-(ideal - base), kind="stable")
    base[order[:rem]] += 1
    return base


def c1(seed_offset=1, **kw) -> Workload:
    v, cell = maxwellian_cells([1000], 2.0, seed=DATA_SEED_BASE + seed_offset, **kw)
    return Workload("C1 single cell 1000 e- Maxwellian 2 eV", v, cell, 1,
                    weight=weight_for(1000), steps=10)


def c2(seed_offset=2, n=100_000, T_perp=2.5, T_par=1.0, **kw) -> Workload:
    v, cell = maxwellian_cells([n], T_perp, T_par_eV=T_par, seed=DATA_SEED_BASE + seed_offset, **kw)
    return Workload(f"C2 bi-Maxwellian 1 cell {n} e- Tperp={T_perp} Tpar={T_par}", v, cell, 1,
                    weight=weight_for(n), steps=500,
                    meta=dict(T_perp=T_perp, T_par=T_par))


def c3_counts(M=256, total=2_560_000) -> np.ndarray:
    x = np.sin(np.pi * (np.arange(M) + 0.5) / M)
    return largest_remainder(total, 0.1 + 0.9 * x)


def c3(seed_offset=3, M=256, total=2_560_000, **kw) -> Workload:
    counts = c3_counts(M, total)
    x = np.sin(np.pi * (np.arange(M) + 0.5) / M)
    T = 2.0 + 2.0 * (1.0 - x)
    v, cell = maxwellian_cells(counts, T, drift=(1e4, 0.0, 0.0),
                               seed=DATA_SEED_BASE + seed_offset, **kw)
    return Workload(f"C3 1D discharge {M} cells {total} e-", v, cell, M,
                    weight=weight_for(total / M))


def c4(seed_offset=4, nx=64, ny=64, per_cell=25_000, cell_base=0, **kw) -> Workload:
    M = nx * ny
    counts = np.full(M, per_cell, np.int64)
    v, cell = maxwellian_cells(counts, 2.0, seed=DATA_SEED_BASE + seed_offset, **kw)
    return Workload(f"C4 2D discharge {nx}x{ny} cells x {per_cell} e-", v, cell, M,
                    cell_base=cell_base, weight=weight_for(per_cell))


def c4b(seed_offset=40, nx=64, ny=64, per_cell=25_000, **kw) -> Workload:
    M = nx * ny
    ix, iy = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    shape = (np.sin(np.pi * (ix + 0.5) / nx) * np.sin(np.pi * (iy + 0.5) / ny)).reshape(-1)
    counts = largest_remainder(M * per_cell, shape)
    v, cell = maxwellian_cells(counts, 2.0, seed=DATA_SEED_BASE + seed_offset, **kw)
    return Workload(f"C4b 2D sine profile {nx}x{ny} cells mean {per_cell} e-", v, cell, M,
                    weight=weight_for(per_cell))


def c5_rank(rank: int, nx=64, ny=64, per_cell=25_000, **kw) -> Workload:
    """Rank r's shard of the weak-scaling run: global cells [M r, M (r+1))."""
    w = c4(seed_offset=500 + rank, nx=nx, ny=ny, per_cell=per_cell, cell_base=rank * nx * ny, **kw)
    w.name = f"C5 rank {rank}: " + w.name
    return w


def random_cells(n, M, *, seed, dead_frac=0.0, T_eV=2.0, skew=False) -> Workload:
    """Generic test input: n particles over M cells, uniform or skewed."""
    rng = np.random.Generator(np.random.PCG64(seed))
    if skew:
        p = rng.pareto(1.2, M) + 1e-3
        p /= p.sum()
        cell = rng.choice(M, size=n, p=p).astype(np.int32)
    else:
        cell = rng.integers(0, M, size=n, dtype=np.int32) if M > 0 else np.zeros(n, np.int32)
    if dead_frac > 0:
        cell[rng.random(n) < dead_frac] = -1
    s = sigma_v(T_eV)
    v = rng.standard_normal((3, n)) * s
    return Workload(f"random n={n} M={M}", np.ascontiguousarray(v), np.ascontiguousarray(cell),
                    max(M, 1), weight=weight_for(max(n / max(M, 1), 1.0)))


# NEXT f2 (PIC loop): grid geometry and positions consistent with the cell ids.
PIC_DX = 5e-3            # m; 2D cell 5 mm x 5 mm x 4 cm deep = CELL_VOLUME.  At 2 eV and dt = 1e-10 s
PIC_DEPTH = CELL_VOLUME / (PIC_DX * PIC_DX)   # ~0.95% of the electrons cross each cell face pair per step


def positions_in_cells(cell, nx, ny, dx=PIC_DX, dy=PIC_DX, *, seed) -> np.ndarray:
    """[3][n] positions uniform inside each particle's cell of an nx x ny grid
    (cell = ix + nx iy); dead particles (-1) get x = y = 0.  Row z = 0."""
    rng = np.random.Generator(np.random.PCG64(seed))
    cell = np.asarray(cell)
    n = cell.size
    c = np.where(cell >= 0, cell, 0)
    ix, iy = c % nx, c // nx
    x = np.zeros((3, n), np.float64)
    x[0] = (ix + rng.random(n)) * dx
    x[1] = (iy + rng.random(n)) * dy
    x[0] = np.minimum(x[0], np.nextafter((ix + 1) * dx, 0))
    x[1] = np.minimum(x[1], np.nextafter((iy + 1) * dy, 0))
    x[:, cell < 0] = 0.0
    return x


def device_random_cells(n: int, M: int, *, seed: int, device, T_eV: float = 2.0, chunk: int = 1 << 28):
    """Inputs too large for host memory (the maximum-size parity test): n particles with cell ids
    uniform over M cells (random order, "cold") and Maxwellian velocities, drawn ON THE DEVICE with
    a seeded torch generator in chunks (no temporary larger than `chunk` elements).  Returns
    (v [3][n] float64, cell [n] int32, params dict).  Plain distributions only, like the rest of
    this module."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    v = torch.empty((3, n), dtype=torch.float64, device=device)
    cell = torch.empty(n, dtype=torch.int32, device=device)
    s = sigma_v(T_eV)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        cell[a:b] = torch.randint(0, M, (b - a,), generator=g, device=device, dtype=torch.int32)
        for r in range(3):
            v[r, a:b].normal_(0.0, s, generator=g)
    params = dict(dt=DT, weight=weight_for(max(n / M, 1.0)), cell_volume=CELL_VOLUME, ln_lambda=LN_LAMBDA,
                  cell_base=0, seed=COLLISION_SEED)
    return v, cell, params
