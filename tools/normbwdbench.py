"""RMSNorm backward timing at the LBVim training shapes (dev tool)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from kbench import peak_gbs, time_fn  # noqa: E402

from paper_2506_15976_b200.norm import rms_norm_bwd  # noqa: E402

flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for rows, D, dt in ((128 * 197, 384, torch.float32), (128 * 197, 384, torch.bfloat16), (256 * 197, 192, torch.bfloat16)):
    x = torch.randn(rows, D, device="cuda").to(dt)
    g = torch.randn(rows, D, device="cuda").to(dt)
    s = torch.randn(D, device="cuda")
    ms = time_fn(lambda: rms_norm_bwd(x, s, g), 20, flush)
    nb = 3 * x.element_size() * rows * D
    print(f"rows={rows} D={D} {dt}: {ms * 1e3:.1f} us  {nb / ms / 1e6 / peak_gbs():.3f} of HBM")
