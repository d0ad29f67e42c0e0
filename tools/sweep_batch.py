"""Kernel time vs batch (number of CTAs) at the LBVim-Ti layer shape: tells a
wave-quantised kernel (steps at multiples of the resident-CTA capacity) from a
throughput-bound one (linear).  Dev tool."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from kbench import make, time_fn  # noqa: E402

from paper_2506_15976_b200.scan import lbm_selective_scan_fwd  # noqa: E402

flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
E = int(os.environ.get("SWEEP_E", 384))
io = torch.bfloat16 if os.environ.get("SWEEP_DT", "bf16") == "bf16" else torch.float32
for Bt in [int(x) for x in os.environ.get("SWEEP_B", "16,32,49,64,98,128,148,197,246,256,296,394").split(",")]:
    x = make(Bt, 197, E, 16, io, io)
    out = torch.empty(Bt, 197, E, device="cuda", dtype=io)
    ms = time_fn(lambda: lbm_selective_scan_fwd(**x, window=8, out=out), 10, flush)
    ctas = Bt * ((E + 127) // 128)
    print(json.dumps(dict(B=Bt, ctas=ctas, ms=round(ms, 4), us_per_cta_wave=round(ms * 1e3 * 592 / ctas, 2))), flush=True)
