"""Launch the conv1d+SiLU forward a few times at the LBVim-Ti shape (ncu target)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_15976_b200.conv import causal_conv1d_silu_fwd  # noqa: E402

B, L, D = 256, 197, 192
E = 2 * D
xz = torch.randn(B, L, 2 * E, device="cuda").to(torch.bfloat16)
w = torch.randn(E, 4, device="cuda")
out = torch.empty(B, L, E, device="cuda", dtype=torch.bfloat16)
for _ in range(4):
    causal_conv1d_silu_fwd(xz[..., :E], w, out=out)
torch.cuda.synchronize()
