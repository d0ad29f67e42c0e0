"""Write-flush vs read-flush of L2 before a small HBM-bound kernel (dev tool): a
256 MiB zero-fill leaves ~126 MB of dirty lines whose write-back lands in the
next kernel's time."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_15976_b200.conv import causal_conv1d_silu_fwd  # noqa: E402
from paper_2506_15976_b200.norm import rms_norm  # noqa: E402

buf = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
bufr = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device="cuda")


def timed(fn, flush, iters=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(iters):
        flush()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


B, L, D = 256, 197, 192
E = 2 * D
t = torch.randn(B, L, D, device="cuda").to(torch.bfloat16)
sc = torch.randn(D, device="cuda")
o = torch.empty_like(t)
xz = torch.randn(B, L, 2 * E, device="cuda").to(torch.bfloat16)
w = torch.randn(E, 4, device="cuda")
oc = torch.empty(B, L, E, device="cuda", dtype=torch.bfloat16)
for name, fn, nb in (("rms_norm", lambda: rms_norm(t, sc, out=o), 2 * 2 * B * L * D),
                     ("conv_fwd", lambda: causal_conv1d_silu_fwd(xz[..., :E], w, out=oc), 2 * 2 * B * L * E)):
    for fname, fl in (("write", lambda: buf.zero_()), ("read", lambda: bufr.sum())):
        ms = timed(fn, fl)
        print(json.dumps(dict(kernel=name, flush=fname, us=round(ms * 1e3, 2), gbs=round(nb / ms / 1e6))), flush=True)
