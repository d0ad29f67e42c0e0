"""Host overhead of the eager LBVim-S training step vs its CUDA-graph replay (dev tool).

    python tools/train_overhead.py [--amp]

Eager: device time (CUDA events around the step) and host wall time of issuing
it (perf_counter around step() without a sync, i.e. how long Python/ctypes/
autograd take to enqueue the ~1,000 launches); graphed: device time per replay."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_15976_b200 import model as M  # noqa: E402

amp = "--amp" in sys.argv
cfg = M.lbvim_small()
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(128, 224, 224, 3, generator=g, device="cuda")
y = torch.randint(0, cfg.num_classes, (128,), generator=g, device="cuda")
tr = M.LBVimTrainer(cfg, M.init_params(cfg, seed=0, device="cuda"), lr=1e-4, amp=amp)
for _ in range(3):
    tr.step(x, y)
torch.cuda.synchronize()
dev, host = [], []
for _ in range(5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    t0 = time.perf_counter()
    tr.step(x, y)
    host.append((time.perf_counter() - t0) * 1e3)
    e.record()
    torch.cuda.synchronize()
    dev.append(s.elapsed_time(e))
run = tr.graphed(x, y)
for _ in range(3):
    run(x, y)
torch.cuda.synchronize()
gdev = []
for _ in range(5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    run(x, y)
    e.record()
    torch.cuda.synchronize()
    gdev.append(s.elapsed_time(e))
med = lambda v: sorted(v)[len(v) // 2]
print(json.dumps({"amp": amp, "batch": 128, "eager_device_ms": med(dev), "eager_host_issue_ms": med(host),
                  "graphed_device_ms": med(gdev), "images_per_s_eager": 128 / med(dev) * 1e3,
                  "images_per_s_graphed": 128 / med(gdev) * 1e3}))
