"""LBVim-Ti projection GEMM shapes with alternative weight layouts / padding (dev tool)."""
import torch
import sys, os
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from kbench import time_fn

flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
M = 256 * 197
bf = torch.bfloat16
for name, K, N in (("in_proj", 192, 768), ("x_proj", 384, 416), ("x_proj_pad448", 384, 448),
                   ("x_proj_pad512", 384, 512), ("out_proj", 384, 192)):
    a = torch.randn(M, K, device="cuda", dtype=bf)
    w = torch.randn(K, N, device="cuda", dtype=bf)
    wt = w.t().contiguous()
    o = torch.empty(M, N, device="cuda", dtype=bf)
    for lay, fn in (("NN", lambda: torch.matmul(a, w, out=o)), ("NT", lambda: torch.matmul(a, wt.t(), out=o))):
        ms = time_fn(fn, 20, flush)
        nb = 2 * (M * K + K * N + M * N)
        print(f"{name:14s} {lay} {ms*1e3:7.1f} us  {nb/ms/1e6:7.0f} GB/s  {2*M*K*N/ms/1e9:6.0f} TFLOP/s", flush=True)
