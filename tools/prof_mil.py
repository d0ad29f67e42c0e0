"""One MambaMIL-style bag forward (L = 100k, bf16) in a profiler range (ncu launch-list target)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_15976_b200.mil import MILBag, MILConfig, init_mil_params  # noqa: E402

cfg = MILConfig()
bag = MILBag(cfg, init_mil_params(cfg, seed=0, device="cuda"), dtype=torch.bfloat16)
X = torch.randn(100000, cfg.d_in, device="cuda").to(torch.bfloat16)
for _ in range(2):
    bag(X)
torch.cuda.synchronize()
torch.cuda.profiler.start()
bag(X)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
