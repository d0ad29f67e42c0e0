"""Launch the fused scan (fwd) a few times at one BASELINE config inside a
profiler range (ncu --profile-from-start off)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from kbench import CFGS, make  # noqa: E402

from paper_2506_15976_b200.scan import lbm_selective_scan_fwd  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5s"
Bt, L, E, N, M, io, bc = CFGS[name]
x = make(Bt, L, E, N, io, bc)
out = torch.empty(Bt, L, E, device="cuda", dtype=io)
for _ in range(2):
    lbm_selective_scan_fwd(**x, window=M, out=out)
torch.cuda.synchronize()
torch.cuda.profiler.start()
lbm_selective_scan_fwd(**x, window=M, out=out)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
