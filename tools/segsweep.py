"""Sequence-split sweep (dev tool).   python tools/segsweep.py [cfg,cfg...] [S,S,...]  (S = seg_hint, 0 = auto)"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from kbench import CFGS, make, time_fn  # noqa: E402

from paper_2506_15976_b200.scan import lbm_selective_scan_bwd, lbm_selective_scan_fwd  # noqa: E402

flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["cfg4", "cfg5", "cfg5s"]
segs = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 1, 2, 3, 4, 8, 16, 64, 256]
for name in names:
    Bt, L, E, N, M, io, bc = CFGS[name]
    x = make(Bt, L, E, N, io, bc)
    out = torch.empty(Bt, L, E, device="cuda", dtype=io)
    bwd = "--bwd" in sys.argv
    if bwd:
        dout = torch.randn(Bt, L, E, device="cuda").to(io)
        _, ck = lbm_selective_scan_fwd(**x, window=M, save_checkpoints=True)
    for S in segs:
        if bwd:
            fn = lambda: lbm_selective_scan_bwd(dout, **x, window=M, checkpoints=ck, seg_hint=S)
        else:
            fn = lambda: lbm_selective_scan_fwd(**x, window=M, out=out, seg_hint=S)
        ms = time_fn(fn, 10, flush, graph=True)
        print(json.dumps(dict(cfg=name, pass_="bwd" if bwd else "fwd", seg_hint=S, ms=round(ms, 4))), flush=True)
