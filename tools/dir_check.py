"""Forward vs reverse direction, accumulate on/off, at cfg2/cfg4 (dev tool)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from kbench import CFGS, make, time_fn  # noqa: E402

from paper_2506_15976_b200.scan import lbm_selective_scan_fwd  # noqa: E402

flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for name in ("cfg2", "cfg4"):
    Bt, L, E, N, M, io, bc = CFGS[name]
    x = make(Bt, L, E, N, io, bc)
    out = torch.empty(Bt, L, E, device="cuda", dtype=io)
    for lb in (True, False):
        for w in (8, 16):
            for rev in (False, True):
                for acc in ((False, True) if not lb else (False,)):
                    ms = time_fn(lambda: lbm_selective_scan_fwd(**x, window=w, lb=lb, reverse=rev, out=out,
                                                                accumulate=acc), 5, flush)
                    print(name, "lb" if lb else "fwd", "w", w, "rev" if rev else "fwd-dir", "acc" if acc else "", round(ms, 4))
