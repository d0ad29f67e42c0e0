"""Launch the fused forward a few times at one config with a forced split (ncu target)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from kbench import CFGS, make  # noqa: E402

from paper_2506_15976_b200.scan import lbm_selective_scan_fwd  # noqa: E402

name, S = sys.argv[1], int(sys.argv[2])
Bt, L, E, N, M, io, bc = CFGS[name]
x = make(Bt, L, E, N, io, bc)
out = torch.empty(Bt, L, E, device="cuda", dtype=io)
for _ in range(3):
    lbm_selective_scan_fwd(**x, window=M, out=out, seg_hint=S)
torch.cuda.synchronize()
