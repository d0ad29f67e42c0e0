"""Dump backward outputs for a fixed set of shapes (dev tool: bitwise A/B of two library builds).
    [DT=f32] python tools/dump_bwd.py out.pt"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from kbench import make  # noqa: E402

from paper_2506_15976_b200.scan import lbm_selective_scan_bwd, lbm_selective_scan_fwd  # noqa: E402

dt = torch.float32 if os.environ.get("DT") == "f32" else torch.bfloat16
out = {}
for (Bt, L, E, M, seg) in [(4, 197, 384, 8, 0), (3, 50, 256, 4, 0), (2, 300, 128, 16, 0), (2, 700, 192, 8, 3),
                           (1, 33, 64, 5, 0), (5, 17, 200, 3, 0), (16, 197, 768, 8, 0), (1, 3000, 64, 16, 0)]:
    x = make(Bt, L, E, 16, dt, dt, seed=L + E)
    g = torch.Generator(device="cuda").manual_seed(E)
    dout = torch.randn(Bt, L, E, device="cuda", generator=g).to(dt)
    for rev in (False, True):
        for lb in (True, False):
            _, ck = lbm_selective_scan_fwd(**x, window=M, reverse=rev, lb=lb, save_checkpoints=True)
            r = lbm_selective_scan_bwd(dout, **x, window=M, reverse=rev, lb=lb, checkpoints=ck, seg_hint=seg)
            out[(Bt, L, E, M, seg, rev, lb)] = {k: (None if v is None else v.cpu()) for k, v in r.items()}
torch.save(out, sys.argv[1])
