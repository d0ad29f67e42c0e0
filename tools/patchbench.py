"""Patchify copy variants at the LBVim-Ti input shape (dev tool)."""
import torch
import sys, os
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from kbench import time_fn
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
B, H, p, C = 256, 224, 16, 3
g = H // p
img = torch.randn(B, H, H, C, device="cuda").to(torch.bfloat16)
v = {
    "6d_permute": lambda: img.reshape(B, g, p, g, p, C).permute(0, 1, 3, 2, 4, 5).reshape(B, g * g, p * p * C),
    "4d_transpose": lambda: img.reshape(B * g, p, g, p * C).transpose(1, 2).contiguous(),
    "copy_into_view": lambda: torch.empty(B * g, g, p, p * C, device="cuda", dtype=img.dtype).copy_(
        img.reshape(B * g, p, g, p * C).transpose(1, 2)),
    "u64_4d": lambda: img.reshape(B * g, p, g, p * C).view(torch.int64).transpose(1, 2).contiguous().view(torch.bfloat16),
    "u32_4d": lambda: img.reshape(B * g, p, g, p * C).view(torch.int32).transpose(1, 2).contiguous().view(torch.bfloat16),
}
ref = v["6d_permute"]().reshape(-1)
for k, fn in v.items():
    out = fn()
    same = torch.equal(out.reshape(-1), ref)
    ms = time_fn(fn, 20, flush)
    print(f"{k:16s} {ms*1e3:7.1f} us  same={same}")
