"""Launch the fused scan a few times at one BASELINE shape (target for ncu).

    ncu --set full -k regex:fwd_kernel -s 2 -c 1 python tools/prof_fwd.py --cfg cfg2
"""

import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from kbench import CFGS, make  # noqa: E402

from paper_2506_15976_b200.scan import lbm_selective_scan_bwd, lbm_selective_scan_fwd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="cfg2")
ap.add_argument("--iters", type=int, default=4)
ap.add_argument("--fwd-only", action="store_true")
ap.add_argument("--bwd", action="store_true")
a = ap.parse_args()
Bt, L, E, N, M, io, bc = CFGS[a.cfg]
x = make(Bt, L, E, N, io, bc)
out = torch.empty(Bt, L, E, device="cuda", dtype=io)
if a.bwd:
    dout = torch.randn(Bt, L, E, device="cuda").to(io)
    _, ck = lbm_selective_scan_fwd(**x, window=M, save_checkpoints=True)
for _ in range(a.iters):
    if a.bwd:
        lbm_selective_scan_bwd(dout, **x, window=M, checkpoints=ck)
    else:
        lbm_selective_scan_fwd(**x, window=M, lb=not a.fwd_only, out=out)
torch.cuda.synchronize()
print("done", a.cfg)
