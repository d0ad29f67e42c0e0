"""paper_2506_15976_b200 — B200-native locally bi-directional (LBMamba) selective scan.

Drop-in for the reference's scan path (lbscan: block._run_scan / engine /
autodiff).  Compute runs in hand-written sm_100a kernels behind the C ABI in
``include/lbscan_b200.h`` (``liblbscan_b200.so``); there is no CPU fallback.
"""

from .errors import NonFiniteError, ShapeError
from .tiling import TilePlan, select_tile_len

__all__ = ["ShapeError", "NonFiniteError", "TilePlan", "select_tile_len",
           "lbm_selective_scan", "selective_scan", "global_bidir_selective_scan"]


def __getattr__(name):
    # torch-dependent API is imported lazily so `import paper_2506_15976_b200`
    # stays cheap for the C-ABI tests
    if name in ("lbm_selective_scan", "selective_scan", "lbm_selective_scan_fwd", "lbm_selective_scan_bwd",
                "global_bidir_selective_scan"):
        from . import scan
        return getattr(scan, name)
    raise AttributeError(name)
