"""One eager LBVim-Ti forward at batch 256 bf16 inside a cudaProfilerStart/Stop
range (target for an ncu launch list: ncu --profile-from-start off ...)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_15976_b200 import model as M  # noqa: E402

cfg = M.lbvim_tiny()
net = M.LBVim(cfg, M.init_params(cfg, seed=0), dtype=torch.bfloat16)
x = torch.randn(int(os.environ.get("BATCH", 256)), 224, 224, 3, device="cuda").to(torch.bfloat16)
for _ in range(int(os.environ.get("ITERS", 2))):
    net(x)
torch.cuda.synchronize()
torch.cuda.profiler.start()
net(x)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
