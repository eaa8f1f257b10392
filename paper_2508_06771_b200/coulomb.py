"""Torch-facing binding of the C ABI (same names as include/coulomb.h).

PyTorch supplies device memory and the current CUDA stream; this module only
checks dtypes/devices/layouts and passes raw pointers to ``libcoulomb.so``.
All arithmetic of the operator (arXiv 2508.06771 Table 5, CCS1-CCS5) runs in
the sm_100a kernels of ``csrc/cc_kernels.cu``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import torch

from . import _lib
from ._lib import CC_DIAG_LEN, CC_MOMENTS_LEN, CCParams, check

M_E = 9.1093837015e-31
Q_E = 1.602176634e-19
EPS0 = 8.8541878128e-12


def _stream(dev: torch.device) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _need(t: torch.Tensor, name: str, dtype: torch.dtype, dev: torch.device):
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if t.device != dev:
        raise ValueError(f"{name} must be on {dev}, got {t.device}")


def _soa(v: torch.Tensor, name: str, dev: torch.device) -> int:
    """Checks a [3][n] fp64 SoA view with unit inner stride; returns ldv."""
    _need(v, name, torch.float64, dev)
    if v.dim() != 2 or v.shape[0] != 3 or (v.shape[1] > 1 and v.stride(1) != 1):
        raise ValueError(f"{name} must be [3][n] with contiguous rows")
    return int(v.stride(0)) if v.shape[1] > 0 else 0


def make_params(*, mass=M_E, charge=Q_E, eps0=EPS0, weight=1.0, cell_volume=1.0, ln_lambda=10.0,
                cell_volume_arr: Optional[torch.Tensor] = None,
                ln_lambda_arr: Optional[torch.Tensor] = None, flags: int = 0,
                step_dev: Optional[torch.Tensor] = None) -> CCParams:
    p = CCParams()
    _lib.load().cc_default_params(C.byref(p))
    p.mass, p.charge, p.eps0 = mass, charge, eps0
    p.weight, p.cell_volume, p.ln_lambda = weight, cell_volume, ln_lambda
    p.cell_volume_arr = None if cell_volume_arr is None else cell_volume_arr.data_ptr()
    p.ln_lambda_arr = None if ln_lambda_arr is None else ln_lambda_arr.data_ptr()
    p.flags = flags
    p.step_dev = None if step_dev is None else step_dev.data_ptr()
    return p


def cc_workspace_bytes(n: int, cells: int) -> int:
    return int(_lib.load().cc_workspace_bytes(n, cells))


def cc_strerror(code: int) -> str:
    return _lib.strerror(code)


def cc_device_status(workspace: torch.Tensor) -> int:
    return _lib.load().cc_device_status(_ptr(workspace), C.c_void_p(_stream(workspace.device)))


@dataclass
class CollideOut:
    v_out: torch.Tensor      # [3][n] fp64, cell-major, pair order inside a cell
    cell_out: torch.Tensor   # [n] int32
    perm_out: torch.Tensor   # [n] int32, input index at each output slot
    moments: torch.Tensor    # [cells][7]
    diag: torch.Tensor       # [16]


def alloc_workspace(n: int, cells: int, device) -> torch.Tensor:
    nbytes = cc_workspace_bytes(n, cells)
    ws = torch.empty(nbytes + 256, dtype=torch.uint8, device=device)
    pad = (-ws.data_ptr()) % 256
    ws = ws[pad:pad + nbytes]
    ws[:256].zero_()          # the device error flags (cc_device_status) start clear
    return ws


def coulomb_collide(v: torch.Tensor, cell: torch.Tensor, cells: int, *, dt: float,
                    weight: float = 1.0, cell_volume: float = 1.0, ln_lambda: float = 10.0,
                    cell_volume_arr: Optional[torch.Tensor] = None,
                    ln_lambda_arr: Optional[torch.Tensor] = None, cell_base: int = 0,
                    seed: int = 42, step: int = 0, mass: float = M_E, charge: float = Q_E,
                    eps0: float = EPS0, out: Optional[CollideOut] = None,
                    workspace: Optional[torch.Tensor] = None, moments: bool = True,
                    diag: bool = True, flags: int = 0, step_dev: Optional[torch.Tensor] = None,
                    push: Optional[dict] = None) -> CollideOut:
    """One step of the Coulomb collision operator on CUDA tensors (see coulomb.h)."""
    dev = cell.device
    if dev.type != "cuda":
        raise ValueError("coulomb_collide runs on CUDA tensors only")
    _need(cell, "cell", torch.int32, dev)
    if cell.dim() != 1 or not cell.is_contiguous():
        raise ValueError("cell must be a contiguous 1-D int32 tensor")
    n = cell.numel()
    ldv = _soa(v, "v", dev)
    if v.shape[1] != n:
        raise ValueError("v must be [3][n] with n = cell.numel()")
    if out is None:
        out = CollideOut(torch.empty((3, n), dtype=torch.float64, device=dev),
                         torch.empty(n, dtype=torch.int32, device=dev),
                         torch.empty(n, dtype=torch.int32, device=dev),
                         torch.empty((cells, CC_MOMENTS_LEN), dtype=torch.float64, device=dev),
                         torch.empty(CC_DIAG_LEN, dtype=torch.float64, device=dev))
    ldo = _soa(out.v_out, "v_out", dev)
    if ldo != ldv and n > 0:
        raise ValueError("v and v_out must have the same row stride (ldv)")
    if workspace is None:
        workspace = alloc_workspace(n, cells, dev)
    for arr, nm in ((cell_volume_arr, "cell_volume_arr"), (ln_lambda_arr, "ln_lambda_arr")):
        if arr is not None:
            _need(arr, nm, torch.float64, dev)
            if arr.numel() != cells or not arr.is_contiguous():
                raise ValueError(f"{nm} must be a contiguous [cells] tensor")
    if step_dev is not None:
        _need(step_dev, "step_dev", torch.int32, dev)
    p = make_params(mass=mass, charge=charge, eps0=eps0, weight=weight, cell_volume=cell_volume,
                    ln_lambda=ln_lambda, cell_volume_arr=cell_volume_arr, ln_lambda_arr=ln_lambda_arr,
                    flags=flags, step_dev=step_dev)
    keep = []
    if push is not None:
        # NEXT f2 fused push: dict(grid=Grid, x_in=[3][n] (input order), x_out=[3][n], E=None|[3][cells],
        # q_over_m=-e/m_e); cell_out becomes the post-push GLOBAL cell
        g = push["grid"].c()
        xi, xo, E = push["x_in"], push["x_out"], push.get("E")
        for t, nm in ((xi, "x_in"), (xo, "x_out")):
            _soa(t, nm, dev)
        q = _lib.CCPushParams()
        q.grid = C.pointer(g)
        q.E = None if E is None else E.data_ptr()
        q.ldE = 0 if E is None else _soa(E, "E", dev)
        q.q_over_m = push.get("q_over_m", -Q_E / M_E)
        q.x_in, q.ldx_in = xi.data_ptr(), max(int(xi.stride(0)), n)
        q.x_out, q.ldx_out = xo.data_ptr(), max(int(xo.stride(0)), n)
        p.push = C.pointer(q)
        keep += [g, q]
    rc = _lib.load().coulomb_collide(
        _ptr(v), max(ldv, n), _ptr(cell), _ptr(out.v_out), _ptr(out.cell_out), _ptr(out.perm_out),
        n, cells, cell_base, dt, C.byref(p), seed, step,
        _ptr(out.moments) if moments else None, _ptr(out.diag) if diag else None,
        _ptr(workspace), workspace.numel(), C.c_void_p(_stream(dev)))
    check(rc, "coulomb_collide")
    return out


class Collider:
    """Owns the workspace and ping-pong output buffers for repeated steps.

    ``step()`` enqueues one operator call on the current stream and returns
    the output buffers (valid in stream order).  Feeding the outputs back as
    the next inputs (``chain=True``) is the PIC loop's "warm" case.
    """

    def __init__(self, n: int, cells: int, device="cuda", **params):
        self.n, self.cells = n, cells
        self.device = torch.device(device)
        self.params = params
        self.workspace = alloc_workspace(n, cells, self.device)
        self.bufs = [CollideOut(torch.empty((3, n), dtype=torch.float64, device=self.device),
                                torch.empty(n, dtype=torch.int32, device=self.device),
                                torch.empty(n, dtype=torch.int32, device=self.device),
                                torch.empty((cells, CC_MOMENTS_LEN), dtype=torch.float64,
                                            device=self.device),
                                torch.empty(CC_DIAG_LEN, dtype=torch.float64, device=self.device))
                     for _ in range(2)]
        self._i = 0

    def step(self, v, cell, *, step: int, **kw) -> CollideOut:
        out = self.bufs[self._i]
        self._i ^= 1
        p = dict(self.params)
        p.update(kw)
        return coulomb_collide(v, cell, self.cells, step=step, out=out, workspace=self.workspace, **p)

    def status(self) -> int:
        return cc_device_status(self.workspace)


# ---------------------------------------------------------------- test hooks


def cc_bin(cell: torch.Tensor, cells: int, workspace: Optional[torch.Tensor] = None):
    dev = cell.device
    _need(cell, "cell", torch.int32, dev)
    n = cell.numel()
    perm = torch.empty(n, dtype=torch.int32, device=dev)
    off = torch.empty(cells + 1, dtype=torch.int32, device=dev)
    if workspace is None:
        workspace = alloc_workspace(n, cells, dev)
    rc = _lib.load().cc_bin(_ptr(cell), n, cells, _ptr(perm), _ptr(off), _ptr(workspace),
                            workspace.numel(), C.c_void_p(_stream(dev)))
    check(rc, "cc_bin")
    return perm, off


def cc_pairs(off: torch.Tensor, cells: int, *, cell_base=0, seed=42, step=0, flags=0) -> torch.Tensor:
    dev = off.device
    _need(off, "off", torch.int32, dev)
    cnt = (off[1:] - off[:-1]).to(torch.int64)
    npairs = int((cnt // 2).sum().item())
    out = torch.empty((max(npairs, 1), 2), dtype=torch.int32, device=dev)
    rc = _lib.load().cc_pairs(_ptr(off), cells, cell_base, seed, step, flags, _ptr(out), npairs,
                              C.c_void_p(_stream(dev)))
    check(rc, "cc_pairs")
    return out[:npairs]


def cc_philox(ctr4: torch.Tensor, seed: int) -> torch.Tensor:
    """ctr4: [m][4] int32 tensor holding uint32 bit patterns."""
    dev = ctr4.device
    _need(ctr4, "ctr4", torch.int32, dev)
    out = torch.empty_like(ctr4)
    rc = _lib.load().cc_philox(_ptr(ctr4), seed, _ptr(out), ctr4.shape[0], C.c_void_p(_stream(dev)))
    check(rc, "cc_philox")
    return out


def cc_ppnd16(u: torch.Tensor) -> torch.Tensor:
    dev = u.device
    _need(u, "u", torch.float64, dev)
    z = torch.empty_like(u)
    rc = _lib.load().cc_ppnd16(_ptr(u), _ptr(z), u.numel(), C.c_void_p(_stream(dev)))
    check(rc, "cc_ppnd16")
    return z


def cc_ta_pairs(va: torch.Tensor, vb: torch.Tensor, C_: torch.Tensor, u1: torch.Tensor,
                u2: torch.Tensor):
    """In-place TA77 update of explicit pairs; va, vb are contiguous [3][m]."""
    dev = va.device
    for t, nm in ((va, "va"), (vb, "vb"), (C_, "C"), (u1, "u1"), (u2, "u2")):
        _need(t, nm, torch.float64, dev)
        if not t.is_contiguous():
            raise ValueError(f"{nm} must be contiguous")
    m = u1.numel()
    rc = _lib.load().cc_ta_pairs(_ptr(va), _ptr(vb), _ptr(C_), _ptr(u1), _ptr(u2), m,
                                 C.c_void_p(_stream(dev)))
    check(rc, "cc_ta_pairs")
    return va, vb


def cc_moments(v: torch.Tensor, off: torch.Tensor, cells: int, **params) -> torch.Tensor:
    dev = v.device
    ldv = _soa(v, "v", dev)
    _need(off, "off", torch.int32, dev)
    out = torch.empty((cells, CC_MOMENTS_LEN), dtype=torch.float64, device=dev)
    p = make_params(**params)
    rc = _lib.load().cc_moments(_ptr(v), ldv, _ptr(off), cells, C.byref(p), _ptr(out),
                                C.c_void_p(_stream(dev)))
    check(rc, "cc_moments")
    return out


def cc_gather(v: torch.Tensor, cell: torch.Tensor, idx: torch.Tensor, cell_shift: int = 0):
    """(v[:, idx], cell[idx] - cell_shift (dead stay -1)) on the device (migration pack)."""
    dev = cell.device
    ldv = _soa(v, "v", dev)
    _need(cell, "cell", torch.int32, dev)
    _need(idx, "idx", torch.int32, dev)
    m = idx.numel()
    vo = torch.empty((3, m), dtype=torch.float64, device=dev)
    co = torch.empty(m, dtype=torch.int32, device=dev)
    rc = _lib.load().cc_gather(_ptr(v), max(ldv, 1), _ptr(cell), _ptr(idx.contiguous()), m, cell_shift,
                               _ptr(vo), max(m, 1), _ptr(co), C.c_void_p(_stream(dev)))
    check(rc, "cc_gather")
    return vo, co


def cc_owner(cell_global: torch.Tensor, bounds) -> torch.Tensor:
    """Owner rank of each particle's global cell (-1 dead / out of range)."""
    dev = cell_global.device
    _need(cell_global, "cell", torch.int32, dev)
    b = torch.as_tensor(list(bounds), dtype=torch.int32, device=dev)
    out = torch.empty_like(cell_global)
    rc = _lib.load().cc_owner(_ptr(cell_global), cell_global.numel(), _ptr(b), b.numel() - 1, _ptr(out),
                              C.c_void_p(_stream(dev)))
    check(rc, "cc_owner")
    return out


def cc_coulomb_log(moments: torch.Tensor) -> torch.Tensor:
    """NRL e-e Coulomb logarithm per cell from a [cells][7] moments tensor (R21)."""
    dev = moments.device
    _need(moments, "moments", torch.float64, dev)
    m = moments.contiguous()
    out = torch.empty(m.shape[0], dtype=torch.float64, device=dev)
    rc = _lib.load().cc_coulomb_log(_ptr(m), m.shape[0], _ptr(out), C.c_void_p(_stream(dev)))
    check(rc, "cc_coulomb_log")
    return out


def cc_diag_sum_ranks(gathered: torch.Tensor) -> torch.Tensor:
    dev = gathered.device
    _need(gathered, "gathered", torch.float64, dev)
    out = torch.empty(CC_DIAG_LEN, dtype=torch.float64, device=dev)
    rc = _lib.load().cc_diag_sum_ranks(_ptr(gathered.contiguous()), gathered.shape[0], _ptr(out),
                                       C.c_void_p(_stream(dev)))
    check(rc, "cc_diag_sum_ranks")
    return out


# ---------------------------------------------------------------- NEXT f2: push


@dataclass
class Grid:
    """Regular grid of the push (cc_grid): ``dims`` axes, ``n`` cells and cell size
    ``d`` per axis, ``periodic`` bit a = axis a periodic (else absorbing)."""
    dims: int
    n: tuple
    d: tuple
    periodic: int = 0

    def c(self) -> "_lib.CCGrid":
        g = _lib.CCGrid()
        g.dims = self.dims
        for a in range(3):
            g.n[a] = int(self.n[a]) if a < len(self.n) else 1
            g.d[a] = float(self.d[a]) if a < len(self.d) else 1.0
        g.periodic = self.periodic
        return g

    @property
    def cells(self) -> int:
        c = 1
        for a in range(self.dims):
            c *= int(self.n[a])
        return c


def cc_push(x_in: torch.Tensor, v: torch.Tensor, cell: torch.Tensor, grid: Grid, *, dt: float,
            q_over_m: float = -Q_E / M_E, E: Optional[torch.Tensor] = None, perm: Optional[torch.Tensor] = None,
            x_out: Optional[torch.Tensor] = None, cells: Optional[int] = None, cell_base: int = 0) -> torch.Tensor:
    """Steps S2b + S2c (Table 2): v += dt (q/m) E[cell] and x' = x + dt v' (v, cell in place;
    cell: local in, GLOBAL out).  x_in rows are read through ``perm`` (coulomb_collide's
    perm_out) if given.  Returns x_out [3][n]."""
    dev = cell.device
    _need(cell, "cell", torch.int32, dev)
    n = cell.numel()
    ldx = _soa(x_in, "x_in", dev)
    ldv = _soa(v, "v", dev)
    if x_out is None:
        x_out = torch.empty((3, n), dtype=torch.float64, device=dev)
    ldo = _soa(x_out, "x_out", dev)
    if perm is not None:
        _need(perm, "perm", torch.int32, dev)
    cells = grid.cells if cells is None else cells
    ldE = 0
    if E is not None:
        ldE = _soa(E, "E", dev)
    g = grid.c()
    rc = _lib.load().cc_push(_ptr(x_in), max(ldx, n), _ptr(perm), _ptr(x_out), max(ldo, n), _ptr(v), max(ldv, n),
                             _ptr(cell), n, cells, cell_base, C.byref(g), _ptr(E), max(ldE, cells) if E is not None
                             else 0, q_over_m, dt, C.c_void_p(_stream(dev)))
    check(rc, "cc_push")
    return x_out


def cc_step_advance(step_dev: torch.Tensor, inc: int) -> None:
    _need(step_dev, "step_dev", torch.int32, step_dev.device)
    check(_lib.load().cc_step_advance(_ptr(step_dev), inc, C.c_void_p(_stream(step_dev.device))),
          "cc_step_advance")


# ---------------------------------------------------------------- NEXT f4: atomic P2C


def cc_p2c(v: torch.Tensor, cell: torch.Tensor, cells: int, *, sub: int = 1,
           scratch: Optional[torch.Tensor] = None) -> torch.Tensor:
    """The paper's atomic particle-to-cell block reduction over unsorted
    particles with `sub` sub-bins per cell -> raw sums [cells][7]
    {N, sum v (3), sum v^2 (3)}."""
    dev = cell.device
    _need(cell, "cell", torch.int32, dev)
    n = cell.numel()
    ldv = _soa(v, "v", dev)
    L = _lib.load()
    nb = int(L.cc_p2c_scratch_bytes(cells, sub))
    if scratch is None or scratch.numel() * scratch.element_size() < nb:
        scratch = torch.empty(max(nb // 8, 1), dtype=torch.float64, device=dev)
    raw = torch.empty((cells, 7), dtype=torch.float64, device=dev)
    check(L.cc_p2c(_ptr(v), max(ldv, n), _ptr(cell), n, cells, sub, _ptr(raw), _ptr(scratch),
                   scratch.numel() * scratch.element_size(), C.c_void_p(_stream(dev))), "cc_p2c")
    return raw


def cc_p2c_moments(raw: torch.Tensor, *, weight: float = 1.0, cell_volume: float = 1.0,
                   cell_volume_arr: Optional[torch.Tensor] = None, mass: float = M_E, charge: float = Q_E):
    """Raw P2C sums [cells][7] -> moments [cells][7] (coulomb_collide's layout)."""
    dev = raw.device
    _need(raw, "raw", torch.float64, dev)
    cells = raw.shape[0]
    p = make_params(mass=mass, charge=charge, weight=weight, cell_volume=cell_volume, cell_volume_arr=cell_volume_arr)
    out = torch.empty((cells, CC_MOMENTS_LEN), dtype=torch.float64, device=dev)
    check(_lib.load().cc_p2c_moments(_ptr(raw.contiguous()), cells, C.byref(p), _ptr(out), C.c_void_p(_stream(dev))),
          "cc_p2c_moments")
    return out


# ---------------------------------------------------------------- end-to-end entry with host buffers


def alloc_host_buffer(n: int, cells: int, device) -> torch.Tensor:
    nbytes = int(_lib.load().cc_host_buffer_bytes(n, cells))
    buf = torch.empty(nbytes + 256, dtype=torch.uint8, device=device)
    pad = (-buf.data_ptr()) % 256
    buf = buf[pad:pad + nbytes]
    return buf


def coulomb_collide_host(v: torch.Tensor, cell: torch.Tensor, cells: int, *, dt: float, out_v: torch.Tensor,
                         out_cell: Optional[torch.Tensor] = None, out_perm: Optional[torch.Tensor] = None,
                         out_moments: Optional[torch.Tensor] = None, out_diag: Optional[torch.Tensor] = None,
                         dev_buffer: torch.Tensor, stream: Optional[torch.cuda.Stream] = None, weight: float = 1.0,
                         cell_volume: float = 1.0, ln_lambda: float = 10.0, cell_base: int = 0, seed: int = 42,
                         step: int = 0, mass: float = M_E, charge: float = Q_E, eps0: float = EPS0,
                         flags: int = 0) -> None:
    """coulomb_collide on HOST (CPU, ideally pinned) tensors: copies in, the operator, copies out,
    all enqueued on `stream` (asynchronous; synchronise before reading the outputs)."""
    cpu = torch.device("cpu")
    _need(cell, "cell", torch.int32, cpu)
    n = cell.numel()
    ldv = _soa(v, "v", cpu)
    if _soa(out_v, "out_v", cpu) != ldv and n > 0:
        raise ValueError("v and out_v must have the same row stride")
    for t, nm, dt_ in ((out_cell, "out_cell", torch.int32), (out_perm, "out_perm", torch.int32),
                       (out_moments, "out_moments", torch.float64), (out_diag, "out_diag", torch.float64)):
        if t is not None:
            _need(t, nm, dt_, cpu)
    dev = dev_buffer.device
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    p = make_params(mass=mass, charge=charge, eps0=eps0, weight=weight, cell_volume=cell_volume,
                    ln_lambda=ln_lambda, flags=flags)
    rc = _lib.load().coulomb_collide_host(
        _ptr(v), max(ldv, n), _ptr(cell), _ptr(out_v), _ptr(out_cell), _ptr(out_perm), n, cells, cell_base, dt,
        C.byref(p), seed, step, _ptr(out_moments), _ptr(out_diag), _ptr(dev_buffer), dev_buffer.numel(),
        C.c_void_p(st.cuda_stream))
    check(rc, "coulomb_collide_host")


# ---------------------------------------------------------------- NEXT f3: recombination C5


def cc_recombine(v: torch.Tensor, cell: torch.Tensor, prob: torch.Tensor, *, eps_bind: float, cell_base: int = 0,
                 seed: int = 42, step: int = 0, mass: float = M_E) -> torch.Tensor:
    """Recombination C5 (Table 4) in place on a coulomb_collide output (v_out, cell_out);
    prob [cells] per-cell primary probability.  Returns stats {recombined, starved, primaries}
    (int64 [3], on the device)."""
    dev = cell.device
    _need(cell, "cell", torch.int32, dev)
    _need(prob, "prob", torch.float64, dev)
    n = cell.numel()
    ldv = _soa(v, "v", dev)
    stats = torch.empty(3, dtype=torch.int64, device=dev)
    check(_lib.load().cc_recombine(_ptr(v), max(ldv, n), _ptr(cell), n, prob.numel(), cell_base, _ptr(prob),
                                   eps_bind, mass, seed, step, _ptr(stats), C.c_void_p(_stream(dev))),
          "cc_recombine")
    return stats
