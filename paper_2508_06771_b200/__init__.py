"""B200-native electron–electron Coulomb collision operator (arXiv 2508.06771, step S1).

C ABI: include/coulomb.h -> lib/libcoulomb.so (sm_100a CUDA).  This package is
the thin torch binding; see DESIGN.md.
"""
from ._lib import CC_NANBU, CC_ODD_TRIPLET  # noqa: F401
from .coulomb import (Collider, CollideOut, alloc_workspace, cc_bin, cc_device_status,  # noqa: F401
                      cc_diag_sum_ranks, cc_moments, cc_pairs, cc_philox, cc_ppnd16, cc_strerror,
                      cc_ta_pairs, cc_workspace_bytes, coulomb_collide, make_params, cc_gather, cc_owner, cc_coulomb_log,
                      Grid, cc_push, cc_step_advance, cc_p2c, cc_p2c_moments, alloc_host_buffer,
                      coulomb_collide_host, cc_recombine)
