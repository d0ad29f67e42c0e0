"""One LBVim-S training step (batch 128, fp32) inside a profiler range (ncu launch-list target)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_15976_b200 import model as M  # noqa: E402

cfg = M.lbvim_small()
tr = M.LBVimTrainer(cfg, M.init_params(cfg, seed=0, device="cuda"), lr=1e-4, amp=bool(int(os.environ.get("AMP", 0))))
x = torch.randn(int(os.environ.get("BATCH", 128)), 224, 224, 3, device="cuda")
y = torch.randint(0, cfg.num_classes, (x.shape[0],), device="cuda")
for _ in range(2):
    tr.step(x, y)
torch.cuda.synchronize()
torch.cuda.profiler.start()
tr.step(x, y)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
