"""Backward launches at one config with a forced split (ncu launch-list target)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from kbench import CFGS, make  # noqa: E402

from paper_2506_15976_b200.scan import lbm_selective_scan_bwd, lbm_selective_scan_fwd  # noqa: E402

name, S = sys.argv[1], int(sys.argv[2])
Bt, L, E, N, M, io, bc = CFGS[name]
x = make(Bt, L, E, N, io, bc)
dout = torch.randn(Bt, L, E, device="cuda").to(io)
_, ck = lbm_selective_scan_fwd(**x, window=M, save_checkpoints=True)
for _ in range(3):
    lbm_selective_scan_bwd(dout, **x, window=M, checkpoints=ck, seg_hint=S)
torch.cuda.synchronize()
