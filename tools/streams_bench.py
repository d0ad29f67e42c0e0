"""LBVim-Ti forward graph replay with the batch split over 1..4 capture streams (dev tool)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from kbench import time_fn  # noqa: E402

from paper_2506_15976_b200 import model as M  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
cfg = M.lbvim_tiny() if name == "tiny" else M.lbvim_small(image_size=1024)
B = 256 if name == "tiny" else 32
net = M.LBVim(cfg, M.init_params(cfg, seed=0), dtype=torch.bfloat16)
g = torch.Generator(device="cuda").manual_seed(0)
imgs = torch.randn(B, cfg.image_size, cfg.image_size, 3, generator=g, device="cuda").to(torch.bfloat16)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
ref = None
ks = [int(v) for v in os.environ.get("STREAMS", "1,2,3,4").split(",")]
for k in ks:
    run = net.graphed(imgs, streams=k)
    ms = time_fn(run, 10, flush)
    out = run().float()
    if ref is None:
        ref = out.clone()
    print(json.dumps(dict(model=name, streams=k, ms=round(ms, 4), images_per_s=round(B / ms * 1e3, 1),
                          max_abs_diff_vs_1=float((out - ref).abs().max()))), flush=True)
    del run
    torch.cuda.empty_cache()
