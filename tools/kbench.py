"""Kernel-level timing of the fused LB scan at the BASELINE shapes (dev tool).

    python tools/kbench.py [--iters 20] [--only cfg2,cfg4]

Prints one line per (config, variant): ms per launch (CUDA events, L2 flushed
between launches), algorithmic GB/s (SURVEY.md §8d formula) and fraction of
the measured HBM peak.
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_15976_b200.scan import lbm_selective_scan_bwd, lbm_selective_scan_fwd  # noqa: E402

CFGS = {
    # name: (Bt, L, E, N, M, io dtype, bc dtype)
    "cfg1": (2, 197, 192, 16, 8, torch.float32, torch.float32),
    "cfg2": (256, 197, 384, 16, 8, torch.bfloat16, torch.bfloat16),
    "cfg3": (128, 197, 768, 16, 8, torch.float32, torch.float32),
    "cfg4": (32, 4096, 768, 16, 16, torch.bfloat16, torch.bfloat16),
    "cfg5": (1, 100000, 512, 16, 16, torch.float32, torch.float32),
    "cfg5s": (1, 100000, 64, 16, 16, torch.float32, torch.float32),
    "cfg3s": (16, 197, 768, 16, 8, torch.float32, torch.float32),  # configs[2] per-GPU shard at 8 GPUs
    "cfg3b": (128, 197, 768, 16, 8, torch.bfloat16, torch.bfloat16),  # configs[2] shape, bf16 I/O (amp training)
}


def peak_gbs():
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        return json.load(open(p))["hbm_gbs"]
    except Exception:
        return 6650.0


def alg_bytes(Bt, L, E, N, s_in, s_bc, s_out, last_state=False):
    # s_in*B*L*(3E) + s_bc*B*L*2N + s_out*B*L*E + 4*(E*N + 2E)
    b = s_in * Bt * L * 3 * E + s_bc * Bt * L * 2 * N + s_out * Bt * L * E + 4 * (E * N + 2 * E)
    if last_state:
        b += 4 * Bt * E * N
    return b


def bwd_alg_bytes(Bt, L, E, N, s_in, s_bc, s_g):
    # SURVEY §8d bwd: s_in*B*L*(3E+2N) + s_g*B*L*E (dout) + s_g*B*L*3E (du, ddelta, dz)
    #                 + 4*B*L*2N (dB, dC fp32) + 4*(E*N + 2E)
    return (s_in * Bt * L * 3 * E + s_bc * Bt * L * 2 * N + s_g * Bt * L * E + s_g * Bt * L * 3 * E
            + 4 * Bt * L * 2 * N + 4 * (E * N + 2 * E))


def make(Bt, L, E, N, io, bc, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    r = lambda *s, dt=io: torch.randn(*s, generator=g, device="cuda", dtype=torch.float32).to(dt)
    A = -torch.arange(1, N + 1, device="cuda", dtype=torch.float32).repeat(E, 1)
    dtv = torch.exp(torch.empty(E, device="cuda").uniform_(-6.9, -2.3, generator=g))
    bias = dtv + torch.log(-torch.expm1(-dtv))
    return dict(u=r(Bt, L, E), delta=0.5 * r(Bt, L, E), A=A, B=r(Bt, L, N, dt=bc), C=r(Bt, L, N, dt=bc),
                D=torch.ones(E, device="cuda"), z=r(Bt, L, E), delta_bias=bias)


def time_fn(fn, iters, flush, graph=False):
    """Median device time of fn (CUDA events, L2 flushed before each launch).  With
    graph=True fn is captured once into a CUDA graph and replayed, so the host-side
    wrapper cost (ctypes, allocations) cannot stretch the device timeline of the
    small configs."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        fn = g.replay
        fn()
        torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


def gpu_warmup(seconds=0.5):
    """Spin the GPU so its clocks have ramped before the first timed config."""
    import time
    a = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        for _ in range(20):
            a = (a @ a).clamp_(-1, 1)
        torch.cuda.synchronize()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--only", default="")
    ap.add_argument("--bwd", default="cfg1,cfg3,cfg3s,cfg3b", help="configs that also time the backward")
    a = ap.parse_args()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    peak = peak_gbs()
    gpu_warmup()
    names = [n for n in CFGS if not a.only or n in a.only.split(",")]
    for name in names:
        Bt, L, E, N, M, io, bc = CFGS[name]
        x = make(Bt, L, E, N, io, bc)
        out = torch.empty(Bt, L, E, device="cuda", dtype=io)
        s = torch.tensor([], dtype=io).element_size()
        sbc = torch.tensor([], dtype=bc).element_size()
        nbytes = alg_bytes(Bt, L, E, N, s, sbc, s)
        for variant, lb in (("lbm", True), ("fwd", False)):
            ms = time_fn(lambda: lbm_selective_scan_fwd(**x, window=M, lb=lb, out=out), a.iters, flush, graph=True)
            gbs = nbytes / ms / 1e6
            print(json.dumps(dict(cfg=name, variant=variant, ms=round(ms, 4), gbs=round(gbs, 1),
                                  frac=round(gbs / peak, 3), elems_per_s=Bt * L * E / ms * 1e3,
                                  lanes_per_s=Bt * L * E * N / ms * 1e3)), flush=True)
        if a.bwd and name in a.bwd.split(","):
            dout = torch.randn(Bt, L, E, device="cuda").to(io)
            _, ck = lbm_selective_scan_fwd(**x, window=M, save_checkpoints=True)
            nb = bwd_alg_bytes(Bt, L, E, N, s, sbc, s)
            for variant, kw in (("bwd_ckpt", dict(checkpoints=ck)), ("bwd_recompute", {})):
                ms = time_fn(lambda: lbm_selective_scan_bwd(dout, **x, window=M, **kw), a.iters, flush, graph=True)
                gbs = nb / ms / 1e6
                print(json.dumps(dict(cfg=name, variant=variant, ms=round(ms, 4), gbs=round(gbs, 1),
                                      frac=round(gbs / peak, 3), lanes_per_s=Bt * L * E * N / ms * 1e3)),
                      flush=True)
            ms = time_fn(lambda: lbm_selective_scan_fwd(**x, window=M, save_checkpoints=True), a.iters, flush, graph=True)
            print(json.dumps(dict(cfg=name, variant="lbm_fwd_with_ckpt", ms=round(ms, 4))), flush=True)


if __name__ == "__main__":
    main()
