"""torch.profiler attribution of the LBVim-S training step's device time to aten ops
and input shapes (dev tool): which glue kernels come from where.
    AMP=1 python tools/prof_train_ops.py"""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_15976_b200 import model as M  # noqa: E402

cfg = M.lbvim_small()
tr = M.LBVimTrainer(cfg, M.init_params(cfg, seed=0, device="cuda"), lr=1e-4,
                    amp=bool(int(os.environ.get("AMP", 1))))
if int(os.environ.get("FUSED", 0)):
    tr.fused = True
x = torch.randn(128, 224, 224, 3, device="cuda")
y = torch.randint(0, cfg.num_classes, (128,), device="cuda")
for _ in range(2):
    tr.step(x, y)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], record_shapes=True) as prof:
    tr.step(x, y)
    torch.cuda.synchronize()
print(prof.key_averages(group_by_input_shape=True).table(sort_by="self_cuda_time_total", row_limit=45,
                                                          max_name_column_width=40, max_shapes_column_width=70))
