"""Launch the conv1d+SiLU backward and RMSNorm backward at the LBVim-S training shape (ncu target)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_15976_b200.conv import causal_conv1d_silu_bwd  # noqa: E402
from paper_2506_15976_b200.norm import rms_norm_bwd  # noqa: E402

B, L, D = 128, 197, 384
E = 2 * D
x = torch.randn(B, L, E, device="cuda")
g = torch.randn(B, L, E, device="cuda")
w = torch.randn(E, 4, device="cuda")
t = torch.randn(B, L, D, device="cuda")
dt = torch.randn(B, L, D, device="cuda")
s = torch.randn(D, device="cuda")
for _ in range(3):
    causal_conv1d_silu_bwd(x, w, None, g)
    rms_norm_bwd(t, s, dt)
torch.cuda.synchronize()
