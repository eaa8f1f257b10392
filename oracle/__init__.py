"""CPU oracle for the e–e Coulomb collision operator (arXiv 2508.06771, step S1).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product package ``paper_2508_06771_b200`` never imports it, and
this package never imports the product package; the two share no code.  The
only module both sides use is ``workloads`` (seeded input generators, no
method arithmetic).

The arithmetic lives in ``coulomb_oracle.c`` (plain C, fp64, one loop per step
of the paper's Table 5); this file is ctypes marshalling only.
``build()`` compiles it with gcc (``-ffp-contract=off``: no FMA contraction, so
every operation is the plain IEEE operation written in the source).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "coulomb_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# CODATA 2018 (exact e; m_e and eps0 as published) — DESIGN reading R5.
M_E = 9.1093837015e-31
Q_E = 1.602176634e-19
EPS0 = 8.8541878128e-12


def build(force: bool = False) -> str:
    """Compile the oracle shared library (gcc, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=gnu11", "-fopenmp", "-ffp-contract=off", "-fPIC",
               "-shared", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
        L.or_philox4x32_10.argtypes = [u32p, u32p, u32p]
        L.or_philox4x32_10.restype = None
        L.or_u01.argtypes = [C.c_uint32, C.c_uint32]
        L.or_u01.restype = C.c_double
        L.or_ppnd16.argtypes = [C.c_double]
        L.or_ppnd16.restype = C.c_double
        L.or_fmix32.argtypes = [C.c_uint32]
        L.or_fmix32.restype = C.c_uint32
        L.or_feistel_pi.argtypes = [C.c_int64, C.c_int64, u32p]
        L.or_feistel_pi.restype = C.c_int64
        L.or_cell_perm.argtypes = [C.c_int64, C.c_uint32, C.c_uint32, C.c_uint64, C.c_void_p]
        L.or_cell_perm.restype = None
        L.or_cell_perm_uniform.argtypes = [C.c_int64, C.c_uint32, C.c_uint32, C.c_uint64, C.c_void_p]
        L.or_cell_perm_uniform.restype = None
        L.or_cell_keys.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, u32p]
        L.or_cell_keys.restype = None
        L.or_pair_uniforms.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                       C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.or_pair_uniforms.restype = None
        L.or_count.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p]
        L.or_count.restype = C.c_int
        L.or_exclusive_scan.argtypes = [C.c_void_p, C.c_int32, C.c_void_p]
        L.or_exclusive_scan.restype = None
        L.or_stable_order.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p]
        L.or_stable_order.restype = None
        L.or_cell_constant.argtypes = [C.c_int64] + [C.c_double] * 7
        L.or_cell_constant.restype = C.c_double
        L.or_ta_pair.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_double]
        L.or_ta_pair.restype = None
        L.or_moments.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_double,
                                 C.c_double, C.c_void_p, C.c_double, C.c_double, C.c_void_p]
        L.or_moments.restype = None
        L.or_coulomb_collide.argtypes = [
            C.c_void_p, C.c_int64, C.c_void_p,            # v_in, ldv, cell_in
            C.c_void_p, C.c_void_p, C.c_void_p,           # v_out, cell_out, perm_out
            C.c_int64, C.c_int32, C.c_uint32,             # n, M, cell_base
            C.c_double, C.c_double, C.c_double, C.c_double,   # dt, mass, charge, eps0
            C.c_double, C.c_double, C.c_void_p,           # weight, volume, volume_arr
            C.c_double, C.c_void_p,                       # lnL, lnL_arr
            C.c_uint64, C.c_uint64, C.c_uint32,           # seed, step, flags
            C.c_void_p, C.c_void_p, C.c_void_p]           # moments, diag, pair_slots
        L.or_coulomb_collide.restype = C.c_int
        L.or_nanbu_A.argtypes = [C.c_double]
        L.or_nanbu_A.restype = C.c_double
        L.or_langevin.argtypes = [C.c_double]
        L.or_langevin.restype = C.c_double
        L.or_nanbu_pair.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_double]
        L.or_nanbu_pair.restype = None
        L.or_triplet.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_uint32, C.c_uint32,
                                 C.c_uint64, C.c_uint32]
        L.or_triplet.restype = None
        L.or_coulomb_log.argtypes = [C.c_void_p, C.c_int32, C.c_void_p]
        L.or_coulomb_log.restype = None
        L.or_push.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64,   # x_in, ldx, perm, x_out, ldo
                              C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int32,   # v, ldv, cell, n, dims
                              C.c_void_p, C.c_void_p, C.c_uint32,                        # nc[3], d[3], periodic
                              C.c_void_p, C.c_int64, C.c_double, C.c_double]             # E, ldE, q/m, dt
        L.or_push.restype = None
        L.or_recombine.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int32, C.c_uint32,
                                   C.c_void_p, C.c_double, C.c_double, C.c_uint64, C.c_uint64, C.c_void_p]
        L.or_recombine.restype = None
        L.or_set_num_threads.argtypes = [C.c_int]
        L.or_set_num_threads.restype = None
        L.or_num_threads.argtypes = []
        L.or_num_threads.restype = C.c_int
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# --------------------------------------------------------------------------
# element functions


def philox4x32_10(ctr, key):
    ctr = np.ascontiguousarray(ctr, dtype=np.uint32).reshape(4)
    key = np.ascontiguousarray(key, dtype=np.uint32).reshape(2)
    out = np.zeros(4, np.uint32)
    lib().or_philox4x32_10(ctr, key, out)
    return out


def u01(hi: int, lo: int) -> float:
    return lib().or_u01(hi, lo)


def ppnd16(p: float) -> float:
    return lib().or_ppnd16(p)


def fmix32(h: int) -> int:
    return lib().or_fmix32(h)


def cell_keys(G: int, step: int, seed: int):
    k = np.zeros(4, np.uint32)
    lib().or_cell_keys(G, step, seed, k)
    return k


def feistel_pi(i: int, N: int, keys) -> int:
    """One value of the N > 64 keyed-Feistel permutation (R1)."""
    return lib().or_feistel_pi(i, N, np.ascontiguousarray(keys, dtype=np.uint32))


def cell_perm(N: int, G: int, step: int, seed: int, uniform: bool = False) -> np.ndarray:
    """pi_j as a table: pi[q] = stable slot at pair-order position q.  Default: the
    blocked pairing R1b; uniform=True: R1 over the whole cell
    (CC_CELL_UNIFORM).  The two agree for N <= BLOCK."""
    out = np.zeros(max(N, 0), np.int64)
    if N > 0:
        (lib().or_cell_perm_uniform if uniform else lib().or_cell_perm)(N, G, step, seed, _ptr(out))
    return out


# R1b constants: segment length, segments per block, block size
SEG = 32
BLOCK_SEGS = 12
BLOCK = SEG * BLOCK_SEGS


def pair_uniforms(k: int, G: int, step: int, seed: int):
    a, b = C.c_double(), C.c_double()
    lib().or_pair_uniforms(k, G, step, seed, C.byref(a), C.byref(b))
    return a.value, b.value


def count(cell, M):
    cell = np.ascontiguousarray(cell, dtype=np.int32)
    counts = np.zeros(M, np.int64)
    rc = lib().or_count(_ptr(cell), cell.size, M, _ptr(counts))
    if rc != 0:
        raise ValueError(f"or_count: invalid cell id (rc={rc})")
    return counts


def exclusive_scan(counts):
    counts = np.ascontiguousarray(counts, dtype=np.int64)
    off = np.zeros(counts.size + 1, np.int64)
    lib().or_exclusive_scan(_ptr(counts), counts.size, _ptr(off))
    return off


def stable_order(cell, M):
    cell = np.ascontiguousarray(cell, dtype=np.int32)
    off = exclusive_scan(count(cell, M))
    perm = np.zeros(cell.size, np.int64)
    lib().or_stable_order(_ptr(cell), cell.size, M, _ptr(off), _ptr(perm))
    return perm, off


def cell_constant(Nj, weight, volume, lnL, dt, mass=M_E, charge=Q_E, eps0=EPS0):
    return lib().or_cell_constant(Nj, weight, volume, lnL, dt, mass, charge, eps0)


def ta_pair(va, vb, Cj, u1, u2):
    a = np.array(va, dtype=np.float64)
    b = np.array(vb, dtype=np.float64)
    lib().or_ta_pair(_ptr(a), _ptr(b), Cj, u1, u2)
    return a, b


def moments(v, off, weight, volume, volume_arr=None, mass=M_E, charge=Q_E):
    v = np.ascontiguousarray(v, dtype=np.float64)
    off = np.ascontiguousarray(off, dtype=np.int64)
    M = off.size - 1
    out = np.zeros((M, 7), np.float64)
    va = None if volume_arr is None else np.ascontiguousarray(volume_arr, np.float64)
    lib().or_moments(_ptr(v), v.shape[1], _ptr(off), M, weight, volume, _ptr(va), mass, charge,
                     _ptr(out))
    return out


@dataclass
class OracleResult:
    v_out: np.ndarray       # [3][n] position order (cell-major, pair order in cell)
    cell_out: np.ndarray    # [n] int32
    perm_out: np.ndarray    # [n] int64 input index at each position
    moments: np.ndarray     # [M][7]
    diag: np.ndarray        # [16]
    pair_slots: np.ndarray  # [pairs][2] stable slots


ODD_TRIPLET = 1
NANBU = 2
PRESERVE_ORDER = 4
CELL_UNIFORM = 8


def nanbu_A(s: float) -> float:
    return lib().or_nanbu_A(s)


def langevin(A: float) -> float:
    return lib().or_langevin(A)


def nanbu_pair(va, vb, Cj, u1, u2):
    a = np.array(va, dtype=np.float64)
    b = np.array(vb, dtype=np.float64)
    lib().or_nanbu_pair(_ptr(a), _ptr(b), Cj, u1, u2)
    return a, b


def triplet(v1, v2, v3, Cj, G, step, seed, flags=0):
    a, b, c = (np.array(x, dtype=np.float64) for x in (v1, v2, v3))
    lib().or_triplet(_ptr(a), _ptr(b), _ptr(c), Cj, G, step, seed, flags)
    return a, b, c


def coulomb_log(moments):
    m = np.ascontiguousarray(moments, dtype=np.float64)
    out = np.zeros(m.shape[0], np.float64)
    lib().or_coulomb_log(_ptr(m), m.shape[0], _ptr(out))
    return out


def coulomb_collide(v_in, cell_in, cells, *, dt, weight, cell_volume, ln_lambda=10.0,
                    cell_volume_arr=None, ln_lambda_arr=None, cell_base=0, seed=42, step=0,
                    mass=M_E, charge=Q_E, eps0=EPS0, want_pairs=True, flags=0) -> OracleResult:
    """One call of the whole operator (Table 5 CCS1-CCS5 + moments/diagnostics)."""
    v_in = np.ascontiguousarray(v_in, dtype=np.float64)
    cell_in = np.ascontiguousarray(cell_in, dtype=np.int32)
    n = cell_in.size
    assert v_in.shape == (3, n)
    v_out = np.zeros((3, n), np.float64)
    cell_out = np.zeros(n, np.int32)
    perm_out = np.zeros(n, np.int64)
    mom = np.zeros((cells, 7), np.float64)
    diag = np.zeros(16, np.float64)
    npairs_max = n // 2 + 1
    pairs = np.zeros((npairs_max, 2), np.int64) if want_pairs else None
    va = None if cell_volume_arr is None else np.ascontiguousarray(cell_volume_arr, np.float64)
    la = None if ln_lambda_arr is None else np.ascontiguousarray(ln_lambda_arr, np.float64)
    rc = lib().or_coulomb_collide(_ptr(v_in), n, _ptr(cell_in), _ptr(v_out), _ptr(cell_out),
                                  _ptr(perm_out), n, cells, cell_base, dt, mass, charge, eps0,
                                  weight, cell_volume, _ptr(va), ln_lambda, _ptr(la),
                                  seed, step, flags, _ptr(mom), _ptr(diag), _ptr(pairs))
    if rc == -4:
        raise ValueError("invalid cell id")
    if rc != 0:
        raise ValueError(f"or_coulomb_collide rc={rc}")
    npairs = int(diag[2])
    return OracleResult(v_out, cell_out, perm_out, mom, diag,
                        pairs[:npairs].copy() if want_pairs else None)


def push(x, v, cell, *, dims, nc, d, periodic, dt, q_over_m=-Q_E / M_E, E=None, perm=None):
    """NEXT f2: S2b + S2c (Table 2; SPEC push S:204-210).  Returns
    (x_out [3][n], v_out [3][n], cell_out [n] GLOBAL ids, -1 dead); inputs untouched.
    x rows are indexed through perm (the collision call's perm_out) if given."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    v_out = np.array(v, dtype=np.float64, order="C", copy=True)
    cell_out = np.array(cell, dtype=np.int32, copy=True)
    n = cell_out.size
    assert x.shape[0] == 3 and v_out.shape == (3, n)
    x_out = np.zeros((3, n), np.float64)
    nc3 = np.ones(3, np.int32)
    nc3[:len(nc)] = nc
    d3 = np.ones(3, np.float64)
    d3[:len(d)] = d
    pm = None if perm is None else np.ascontiguousarray(perm, dtype=np.int64)
    Ea = None if E is None else np.ascontiguousarray(E, dtype=np.float64)
    lib().or_push(_ptr(x), x.shape[1], _ptr(pm), _ptr(x_out), n, _ptr(v_out), n, _ptr(cell_out), n, dims,
                  _ptr(nc3), _ptr(d3), periodic, _ptr(Ea), 0 if Ea is None else Ea.shape[1], q_over_m, dt)
    return x_out, v_out, cell_out


def recombine(v, cell, cells, prob, *, eps_bind, cell_base=0, seed=42, step=0, mass=M_E):
    """NEXT f3: recombination C5 (Table 4 RS0-RS5, readings R25-R28) on a collision call's
    cell-sorted output.  Returns (v_out, cell_out, stats {recombined, starved, primaries})."""
    v_out = np.array(v, dtype=np.float64, order="C", copy=True)
    cell_out = np.array(cell, dtype=np.int32, copy=True)
    pr = np.ascontiguousarray(prob, dtype=np.float64)
    st = np.zeros(3, np.int64)
    n = cell_out.size
    lib().or_recombine(_ptr(v_out), n, _ptr(cell_out), n, cells, cell_base, _ptr(pr), eps_bind, mass, seed, step,
                       _ptr(st))
    return v_out, cell_out, st


def set_num_threads(n: int) -> None:
    lib().or_set_num_threads(n)


def num_threads() -> int:
    return lib().or_num_threads()
