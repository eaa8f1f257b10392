"""ctypes binding of ``lib/libcoulomb.so`` (the C ABI declared in include/coulomb.h).

Argument marshalling only: every step of the operator runs in the CUDA
kernels of ``csrc/``.  There is no CPU fallback — if the shared library is
missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libcoulomb.so")

CC_OK = 0
CC_EINVAL = -1
CC_EWORKSPACE = -2
CC_ECUDA = -3
CC_ECELL = -4
CC_ECOUNT = -5
CC_ENCCL = -6
CC_MAX_CELLS = 32768
CC_DIAG_LEN = 16
CC_MOMENTS_LEN = 7
CC_NUM_STAGES = 5
CC_ODD_TRIPLET = 1
CC_NANBU = 2
CC_NCCL_ID_BYTES = 128
CC_PRESERVE_ORDER = 4
CC_CELL_UNIFORM = 8
STAGE_NAMES = ("count", "scan", "scatter", "collide", "finalize")

# every symbol include/coulomb.h declares
EXPORTS = ("cc_default_params", "cc_workspace_bytes", "coulomb_collide", "cc_device_status",
           "cc_strerror", "cc_bin", "cc_pairs", "cc_philox", "cc_ppnd16", "cc_ta_pairs",
           "cc_moments", "cc_coulomb_log", "cc_gather", "cc_owner", "cc_diag_sum_ranks", "cc_push",
           "cc_step_advance", "cc_p2c_scratch_bytes", "cc_p2c", "cc_p2c_moments",
           "cc_host_buffer_bytes", "coulomb_collide_host", "cc_recombine",
           "cc_nccl_get_unique_id", "cc_nccl_comm_init", "cc_nccl_comm_destroy", "cc_dist_diag_reduce",
           "cc_dist_alltoall_counts", "cc_dist_exchange", "cc_mig_slot_bytes", "cc_mig_workspace_bytes",
           "cc_mig_pack", "cc_dist_mig_exchange", "cc_mig_unpack")
CC_MIG_MAX_RANKS = 64


class CCGrid(C.Structure):
    _fields_ = [("dims", C.c_int32), ("n", C.c_int32 * 3), ("d", C.c_double * 3), ("periodic", C.c_uint32)]


class CCPushParams(C.Structure):
    _fields_ = [("grid", C.POINTER(CCGrid)), ("E", C.c_void_p), ("ldE", C.c_int64), ("q_over_m", C.c_double),
                ("x_in", C.c_void_p), ("ldx_in", C.c_int64), ("x_out", C.c_void_p), ("ldx_out", C.c_int64)]


class CCParams(C.Structure):
    _fields_ = [("mass", C.c_double), ("charge", C.c_double), ("eps0", C.c_double),
                ("weight", C.c_double), ("cell_volume", C.c_double),
                ("cell_volume_arr", C.c_void_p), ("ln_lambda", C.c_double),
                ("ln_lambda_arr", C.c_void_p), ("flags", C.c_uint32),
                ("push", C.POINTER(CCPushParams)),
                ("step_dev", C.c_void_p),
                ("stage_events", C.POINTER(C.c_void_p))]


class CCError(RuntimeError):
    def __init__(self, code: int, what: str):
        self.code = code
        super().__init__(f"{what}: {strerror(code)} ({code})")


_lib = None


def load():
    """Load the CUDA library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build the CUDA extension first "
                          "(python -c 'import __graft_entry__ as g; g.build()')")
    L = C.CDLL(LIB_PATH)
    vp, i64, i32, u32, u64, dbl, sz = (C.c_void_p, C.c_int64, C.c_int32, C.c_uint32, C.c_uint64,
                                       C.c_double, C.c_size_t)
    L.cc_default_params.argtypes = [C.POINTER(CCParams)]
    L.cc_default_params.restype = None
    L.cc_workspace_bytes.argtypes = [i64, i32]
    L.cc_workspace_bytes.restype = sz
    L.coulomb_collide.argtypes = [vp, i64, vp, vp, vp, vp, i64, i32, u32, dbl, C.POINTER(CCParams),
                                  u64, u64, vp, vp, vp, sz, vp]
    L.coulomb_collide.restype = C.c_int
    L.cc_device_status.argtypes = [vp, vp]
    L.cc_device_status.restype = C.c_int
    L.cc_strerror.argtypes = [C.c_int]
    L.cc_strerror.restype = C.c_char_p
    L.cc_bin.argtypes = [vp, i64, i32, vp, vp, vp, sz, vp]
    L.cc_bin.restype = C.c_int
    L.cc_pairs.argtypes = [vp, i32, u32, u64, u64, u32, vp, i64, vp]
    L.cc_pairs.restype = C.c_int
    L.cc_philox.argtypes = [vp, u64, vp, i64, vp]
    L.cc_philox.restype = C.c_int
    L.cc_ppnd16.argtypes = [vp, vp, i64, vp]
    L.cc_ppnd16.restype = C.c_int
    L.cc_ta_pairs.argtypes = [vp, vp, vp, vp, vp, i64, vp]
    L.cc_ta_pairs.restype = C.c_int
    L.cc_moments.argtypes = [vp, i64, vp, i32, C.POINTER(CCParams), vp, vp]
    L.cc_moments.restype = C.c_int
    L.cc_coulomb_log.argtypes = [vp, i32, vp, vp]
    L.cc_coulomb_log.restype = C.c_int
    L.cc_gather.argtypes = [vp, i64, vp, vp, i64, i32, vp, i64, vp, vp]
    L.cc_gather.restype = C.c_int
    L.cc_owner.argtypes = [vp, i64, vp, i32, vp, vp]
    L.cc_owner.restype = C.c_int
    L.cc_diag_sum_ranks.argtypes = [vp, i32, vp, vp]
    L.cc_diag_sum_ranks.restype = C.c_int
    L.cc_push.argtypes = [vp, i64, vp, vp, i64, vp, i64, vp, i64, i32, u32, C.POINTER(CCGrid), vp, i64, dbl, dbl, vp]
    L.cc_push.restype = C.c_int
    L.cc_p2c_scratch_bytes.argtypes = [i32, i32]
    L.cc_p2c_scratch_bytes.restype = sz
    L.cc_p2c.argtypes = [vp, i64, vp, i64, i32, i32, vp, vp, sz, vp]
    L.cc_p2c.restype = C.c_int
    L.cc_p2c_moments.argtypes = [vp, i32, C.POINTER(CCParams), vp, vp]
    L.cc_p2c_moments.restype = C.c_int
    L.cc_host_buffer_bytes.argtypes = [i64, i32]
    L.cc_host_buffer_bytes.restype = sz
    L.coulomb_collide_host.argtypes = [vp, i64, vp, vp, vp, vp, i64, i32, u32, dbl, C.POINTER(CCParams),
                                       u64, u64, vp, vp, vp, sz, vp]
    L.coulomb_collide_host.restype = C.c_int
    L.cc_recombine.argtypes = [vp, i64, vp, i64, i32, u32, vp, dbl, dbl, u64, u64, vp, vp]
    L.cc_recombine.restype = C.c_int
    L.cc_nccl_get_unique_id.argtypes = [vp]
    L.cc_nccl_get_unique_id.restype = C.c_int
    L.cc_nccl_comm_init.argtypes = [C.POINTER(C.c_void_p), i32, i32, vp]
    L.cc_nccl_comm_init.restype = C.c_int
    L.cc_nccl_comm_destroy.argtypes = [vp]
    L.cc_nccl_comm_destroy.restype = C.c_int
    L.cc_dist_diag_reduce.argtypes = [vp, vp, vp, vp]
    L.cc_dist_diag_reduce.restype = C.c_int
    L.cc_dist_alltoall_counts.argtypes = [vp, vp, vp, vp]
    L.cc_dist_alltoall_counts.restype = C.c_int
    L.cc_dist_exchange.argtypes = [vp, i64, vp, i64, i32, i32, vp, vp, vp, vp]
    L.cc_dist_exchange.restype = C.c_int
    L.cc_step_advance.argtypes = [vp, u32, vp]
    L.cc_step_advance.restype = C.c_int
    L.cc_mig_slot_bytes.argtypes = [i64, i32]
    L.cc_mig_slot_bytes.restype = sz
    L.cc_mig_workspace_bytes.argtypes = [i64, i32]
    L.cc_mig_workspace_bytes.restype = sz
    L.cc_mig_pack.argtypes = [vp, i64, vp, i64, i32, vp, i64, vp, i32, i32, i64, vp, vp, vp, vp, sz, vp]
    L.cc_mig_pack.restype = C.c_int
    L.cc_dist_mig_exchange.argtypes = [vp, vp, sz, vp, i32, vp, vp]
    L.cc_dist_mig_exchange.restype = C.c_int
    L.cc_mig_unpack.argtypes = [vp, i64, vp, i64, i32, vp, i64, vp, vp, vp, i32, i32, i64, vp, vp]
    L.cc_mig_unpack.restype = C.c_int
    _lib = L
    return L


def strerror(code: int) -> str:
    return load().cc_strerror(code).decode()


def check(code: int, what: str) -> None:
    if code != CC_OK:
        raise CCError(code, what)
