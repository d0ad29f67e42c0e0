"""Kernel timing of the conv1d+SiLU front end and RMSNorm at the LBVim shapes (dev tool).

    python tools/convbench.py [--iters 20]
Bytes: conv 2*s*B*L*E (+ weights), norm 2*s*B*L*D; L2 flushed between launches.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from kbench import peak_gbs, time_fn  # noqa: E402

from paper_2506_15976_b200.conv import causal_conv1d_silu_fwd  # noqa: E402
from paper_2506_15976_b200.norm import rms_norm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
peak = peak_gbs()
for name, (B, L, D) in {"cfg2": (256, 197, 192), "cfg4": (32, 4097, 384)}.items():
    E = 2 * D
    xz = torch.randn(B, L, 2 * E, device="cuda").to(torch.bfloat16)
    x = xz[..., :E]  # the model's strided view of the in-projection
    w = torch.randn(E, 4, device="cuda")
    bias = torch.randn(E, device="cuda")
    out = torch.empty(B, L, E, device="cuda", dtype=torch.bfloat16)
    for rev in (False, True):
        ms = time_fn(lambda: causal_conv1d_silu_fwd(x, w, bias, reverse=rev, out=out), a.iters, flush)
        nb = 2 * 2 * B * L * E
        print(json.dumps(dict(cfg=name, kernel="conv_fwd", reverse=rev, ms=round(ms, 4),
                              gbs=round(nb / ms / 1e6, 1), frac=round(nb / ms / 1e6 / peak, 3))), flush=True)
    t = torch.randn(B, L, D, device="cuda").to(torch.bfloat16)
    sc = torch.randn(D, device="cuda")
    o2 = torch.empty_like(t)
    ms = time_fn(lambda: rms_norm(t, sc, out=o2), a.iters, flush)
    nb = 2 * 2 * B * L * D
    print(json.dumps(dict(cfg=name, kernel="rms_norm", ms=round(ms, 4), gbs=round(nb / ms / 1e6, 1),
                          frac=round(nb / ms / 1e6 / peak, 3))), flush=True)

# backward (training shapes): reads x, dout, writes dx (+ weight-grad partials)
from paper_2506_15976_b200.conv import causal_conv1d_silu_bwd  # noqa: E402
for name, (B, L, E, dt) in {"cfg3_bwd_f32": (128, 197, 768, torch.float32),
                            "cfg2_bwd_bf16": (256, 197, 384, torch.bfloat16)}.items():
    x = torch.randn(B, L, E, device="cuda").to(dt)
    g = torch.randn(B, L, E, device="cuda").to(dt)
    w = torch.randn(E, 4, device="cuda")
    bias = torch.randn(E, device="cuda")
    s = torch.tensor([], dtype=dt).element_size()
    for rev in (False, True):
        ms = time_fn(lambda: causal_conv1d_silu_bwd(x, w, bias, g, reverse=rev), a.iters, flush)
        nb = 3 * s * B * L * E
        print(json.dumps(dict(cfg=name, kernel="conv_bwd", reverse=rev, ms=round(ms, 4),
                              gbs=round(nb / ms / 1e6, 1), frac=round(nb / ms / 1e6 / peak, 3))), flush=True)
