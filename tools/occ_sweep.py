"""Per-channel throughput of the fused LB forward vs the number of channels B*E
(dev tool): is a shape latency-bound by parallelism?   python tools/occ_sweep.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from kbench import gpu_warmup, make, time_fn  # noqa: E402

from paper_2506_15976_b200.scan import lbm_selective_scan_fwd  # noqa: E402

gpu_warmup()
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
rows = [("cfg4", 4096, 768, 16, torch.bfloat16, [8, 16, 24, 32, 48, 64, 96]),
        ("cfg3", 197, 768, 8, torch.float32, [8, 16, 32, 64, 128, 256]),
        ("cfg2", 197, 384, 8, torch.bfloat16, [32, 64, 128, 256, 512])]
for name, L, E, M, dt, bs in rows:
    for Bt in bs:
        x = make(Bt, L, E, 16, dt, dt)
        out = torch.empty(Bt, L, E, device="cuda", dtype=dt)
        ms = time_fn(lambda: lbm_selective_scan_fwd(**x, window=M, out=out), 10, flush, graph=True)
        print(f"{name} B={Bt:4d} chans={Bt * E:7d} ms={ms:.4f} ns_per_chan_step={ms * 1e6 / (Bt * E * L) * 1e3:.3f}",
              flush=True)
        del x, out
