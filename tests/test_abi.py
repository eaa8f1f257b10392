"""CPU-side checks of the boundary: the C-ABI library builds, loads and exports
every symbol include/coulomb.h declares (no compute calls without a GPU)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "coulomb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*([a-z_][a-z0-9_]*)\s*\(",
                                 src, flags=re.M)))


def test_library_builds_and_exports_every_declared_symbol():
    from paper_2508_06771_b200 import build, _lib
    build.build()
    L = _lib.load()
    syms = declared_symbols()
    assert "coulomb_collide" in syms and len(syms) >= 10
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTS)


def test_host_only_entry_points():
    from paper_2508_06771_b200 import _lib
    import ctypes as C
    L = _lib.load()
    p = _lib.CCParams()
    L.cc_default_params(C.byref(p))
    assert p.mass == 9.1093837015e-31 and p.ln_lambda == 10.0
    assert L.cc_workspace_bytes(1000, 1) > 32 * 1000
    assert L.cc_workspace_bytes(-1, 1) == 0
    assert _lib.strerror(-4).startswith("cell id")


def test_argument_errors_are_reported_before_any_launch():
    """Host validation runs without a device: bad arguments return error codes."""
    from paper_2508_06771_b200 import _lib
    import ctypes as C
    L = _lib.load()
    p = _lib.CCParams()
    L.cc_default_params(C.byref(p))
    null = None
    rc = L.coulomb_collide(null, 10, null, null, null, null, 10, 0, 0, 1e-10, C.byref(p), 1, 0,
                           null, null, null, 0, null)
    assert rc == _lib.CC_EINVAL          # cells < 1
    rc = L.coulomb_collide(null, 10, null, null, null, null, 10, 4, 0, -1.0, C.byref(p), 1, 0,
                           null, null, null, 0, null)
    assert rc == _lib.CC_EINVAL          # dt <= 0
    rc = L.coulomb_collide(null, 10, null, null, null, null, 10, 4, 0, 1e-10, C.byref(p), 1, 1 << 32,
                           null, null, null, 0, null)
    assert rc == _lib.CC_EINVAL          # step >= 2^32
    rc = L.coulomb_collide(null, 10, null, null, null, null, 10, 4, 0, 1e-10, C.byref(p), 1, 0,
                           null, null, null, 0, null)
    assert rc == _lib.CC_EWORKSPACE      # no workspace
    rc = L.coulomb_collide(null, 10, null, null, null, null, 10, 40000, 0, 1e-10, C.byref(p), 1, 0,
                           null, null, null, 0, null)
    assert rc == _lib.CC_ECOUNT          # cells > CC_MAX_CELLS


def test_next_row_entry_points_validate_arguments():
    """NEXT-row and multi-GPU entries reject bad arguments host-side (no device needed)."""
    from paper_2508_06771_b200 import _lib
    import ctypes as C
    L = _lib.load()
    null = None
    g = _lib.CCGrid()
    g.dims = 4                                             # invalid dims
    assert L.cc_push(null, 0, null, null, 0, null, 0, null, 10, 1, 0, C.byref(g), null, 0, -1.0, 1e-10,
                     null) == _lib.CC_EINVAL
    g.dims, g.n[0], g.d[0] = 1, 0, 1.0                     # zero cells on an axis
    assert L.cc_push(null, 0, null, null, 0, null, 0, null, 10, 1, 0, C.byref(g), null, 0, -1.0, 1e-10,
                     null) == _lib.CC_EINVAL
    assert L.cc_recombine(null, 0, null, -1, 1, 0, null, 0.0, 1.0, 0, 0, null, null) == _lib.CC_EINVAL
    assert L.cc_p2c(null, 0, null, 10, 4, 0, null, null, 0, null) == _lib.CC_EINVAL          # sub < 1
    assert L.cc_p2c_scratch_bytes(4096, 16) == 4096 * 16 * 7 * 8
    assert L.cc_host_buffer_bytes(1000, 4) > L.cc_workspace_bytes(1000, 4)
    assert L.coulomb_collide_host(null, 10, null, null, null, null, 10, 0, 0, 1e-10, null, 0, 0, null, null,
                                  null, 0, null) == _lib.CC_EINVAL                      # cells < 1
    # host entry: a bad dt / flag is reported before any copy is enqueued (here the device buffer is
    # missing too: the argument error must win over CC_EWORKSPACE)
    import numpy as np
    hv, hc = np.zeros((3, 10)), np.zeros(10, np.int32)
    ptr = lambda a: C.c_void_p(a.ctypes.data)  # noqa: E731
    assert L.coulomb_collide_host(ptr(hv), 10, ptr(hc), ptr(hv), null, null, 10, 1, 0, -1.0, null, 0, 0, null,
                                  null, null, 0, null) == _lib.CC_EINVAL                # dt <= 0
    bad = _lib.CCParams()
    L.cc_default_params(C.byref(bad))
    bad.flags = 1 << 20
    assert L.coulomb_collide_host(ptr(hv), 10, ptr(hc), ptr(hv), null, null, 10, 1, 0, 1e-10, C.byref(bad), 0, 0,
                                  null, null, null, 0, null) == _lib.CC_EINVAL          # unknown flag
    assert L.cc_nccl_comm_init(null, 2, 0, null) == _lib.CC_EINVAL
    assert L.cc_dist_exchange(null, 0, null, 0, 1, 3, null, null, null, null) == _lib.CC_EINVAL   # elem 3
    assert L.cc_step_advance(null, 1, null) == _lib.CC_EINVAL


def test_product_package_never_imports_oracle():
    """The product path must not route through the oracle (or any CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2508_06771_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liboracle" not in txt and "coulomb_oracle" not in txt, f


def test_oracle_never_imports_product():
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c", ".h")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert not re.search(r"^\s*(import|from)\s+paper_2508_06771_b200", txt, flags=re.M), f
            assert "#include" not in txt or "cc_device" not in txt, f


def test_flag_constants_agree_across_header_binding_and_oracle():
    """The cc_params.flags bits (include/coulomb.h) equal the binding's and the oracle's, and an
    unknown bit is rejected on the host before any launch."""
    from paper_2508_06771_b200 import _lib
    import ctypes as C
    import oracle
    src = open(os.path.join(ROOT, "include", "coulomb.h")).read()
    hdr = {k: int(v) for k, v in re.findall(r"#define (CC_[A-Z_]+) (\d+)u", src)}
    for name in ("CC_ODD_TRIPLET", "CC_NANBU", "CC_PRESERVE_ORDER", "CC_CELL_UNIFORM"):
        assert getattr(_lib, name) == hdr[name], name
        assert getattr(oracle, name[3:]) == hdr[name], name
    L = _lib.load()
    p = _lib.CCParams()
    L.cc_default_params(C.byref(p))
    p.flags = 16
    null = None
    rc = L.coulomb_collide(null, 10, null, null, null, null, 10, 4, 0, 1e-10, C.byref(p), 1, 0,
                           null, null, null, 0, null)
    assert rc == _lib.CC_EINVAL
