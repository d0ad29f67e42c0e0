"""Benchmark: LBVim-Ti forward (BASELINE configs[1]) on the fused LB-scan kernels.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one LBVim-Ti forward (24 layers, dim 192, 224^2 patch 16, L=197,
alternating scan direction) over a batch of 256 synthetic images in bf16 with
fp32 scan state, random-init weights of the reference architecture.  N GPUs
run one process each (torchrun) with the batch per GPU fixed (weak scaling,
pure data parallel: no collective on the data path).

Printed JSON (rank 0): ``value`` = images/s over all ranks, device-timed with
CUDA events per step (L2 flushed between steps, outside the events), max over
ranks; ``e2e`` = the same metric through the public API with pinned host
images copied in and logits copied out every step (double-buffered on a copy
stream); ``roofline`` = the fused scan kernel's algorithmic GB/s vs the
measured HBM peak; ``cpu_baseline`` = the reference CPU path (oracle port:
numpy + the engine restated in C/OpenMP, bitwise equal to the reference
engine) on a bounded sample on this host.
``--impl reference`` times only that CPU path (rank 0) on the same metric.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "LB selective-scan GB/s (% of HBM peak); LBVim-T images/sec at 1/2/4/8 B200"
UNIT = "images/s"
GLOBAL_BATCH_PER_GPU = 256
CPU_SAMPLE_BATCH = 2


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def _workload_config(n, batch, extra=None):
    c = {"workload": "LBVim-Ti forward, 224^2 patch16, L=197 (middle class token), 24 layers, "
                     "D=192, E=384, N=16, window M=8, alternating direction",
         "model": "LBVim-Ti", "global_batch": batch * n, "batch_per_gpu": batch, "seq_len": 197,
         "parallelism": f"dp{n} (batch-sharded, weights replicated, no collective)",
         "l2": "flushed between timed steps (256 MiB write, outside the timed events)"}
    if extra:
        c.update(extra)
    return c


# ---------------------------------------------------------------------------
# clocks sampling (nvidia-smi during the timed region)

class NvmlClockSampler:
    """SM clock and clock-event (throttle) reasons polled through NVML every ~2 ms
    during the timed region (nvidia-smi's 100 ms loop gives one sample per 60 ms
    step block).  Falls back to ``ClockSampler`` when NVML is unavailable."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, index):
        import pynvml
        self.nv = pynvml
        pynvml.nvmlInit()
        self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        self.samples, self.reasons = [], set()
        self.stop = threading.Event()

    def _poll(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, const in self.REASONS:
                    if r & getattr(nv, const):
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        self.t = threading.Thread(target=self._poll, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=1)

    def summary(self):
        nv = self.nv
        try:
            mx = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
        except Exception:
            mx = None
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0, "source": "nvml"}
        sm = sorted(float(v) for v in self.samples)
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(self.reasons),
                "samples": len(sm), "source": "nvml"}


def clock_sampler(index):
    try:
        return NvmlClockSampler(index)
    except Exception:
        return ClockSampler(index)


class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baseline (reference CPU path, oracle port)

def _cpu_params(seed=0):
    import numpy as np
    rng = np.random.default_rng(seed)
    D, E, N = 192, 384, 16
    f = np.float32
    p = {"patch_w": (rng.standard_normal((768, D)) / np.sqrt(768)).astype(f), "patch_b": np.zeros(D, f),
         "pos": (0.02 * rng.standard_normal((197, D))).astype(f), "cls": (0.02 * rng.standard_normal((1, D))).astype(f)}
    for i in range(24):
        dt = np.exp(rng.uniform(np.log(1e-3), np.log(1e-1), E))
        w = dict(norm_scale=np.ones(D), w_x=rng.standard_normal((D, E)) / np.sqrt(D),
                 w_z=rng.standard_normal((D, E)) / np.sqrt(D), conv_kernel=rng.uniform(-1, 1, (E, 4)) / 2,
                 w_b=rng.standard_normal((E, N)) / np.sqrt(E), w_c=rng.standard_normal((E, N)) / np.sqrt(E),
                 w_delta=rng.standard_normal((E, E)) * 0.1 / np.sqrt(E), delta_bias=dt + np.log(-np.expm1(-dt)),
                 a_log=np.tile(np.log(np.arange(1, N + 1)), (E, 1)), d_param=np.ones(E),
                 w_out=rng.standard_normal((E, D)) / np.sqrt(E))
        for k, v in w.items():
            p[f"blocks.{i}.{k}"] = v.astype(f)
    p.update({"head.mlp_w1": (rng.standard_normal((D, 4 * D)) / np.sqrt(D)).astype(f),
              "head.mlp_b1": np.zeros(4 * D, f),
              "head.mlp_w2": (rng.standard_normal((4 * D, 1000)) / np.sqrt(4 * D)).astype(f),
              "head.mlp_b2": np.zeros(1000, f)})
    return p


def cpu_reference_run(steps, warmup, batch=CPU_SAMPLE_BATCH):
    """Time the reference's CPU path (port) on `batch` images per step."""
    import numpy as np
    from oracle import cpu_port
    cpu_port.build()
    threads = os.cpu_count() or 1
    cfg = dict(image_size=224, patch_size=16, in_channels=3, embed_dim=192, inner_dim=384, state_dim=16,
               depth=24, tile_len=None, class_token="middle")
    params = _cpu_params()
    imgs = np.random.default_rng(1).standard_normal((batch, 224, 224, 3)).astype(np.float32)
    for _ in range(warmup):
        cpu_port.model_forward(imgs, cfg, params, threads=threads)
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        cpu_port.model_forward(imgs, cfg, params, threads=threads)
        ts.append(time.perf_counter() - t0)
    total = sum(ts)
    return {"value": batch * steps / total, "unit": UNIT, "cores": threads, "kind": "port",
            "ms_per_step": total / steps * 1e3,
            "sample": f"LBVim-Ti fp32 forward on {batch} images per step x {steps} steps (+{warmup} warm-up), "
                      f"numpy + engine restated in C/OpenMP ({threads} threads; bitwise equal to the "
                      f"reference numba engine on its verification grid)"}


def cpu_op_baseline(reps=7):
    """BASELINE.md §4 op-level CPU leg: the reference's fused-op composition on the
    host (numpy discretisation block.py:90-98 + the engine restated in C/OpenMP +
    the gate block.py:177-178, all cores), and the engine alone on pre-discretised
    inputs (lbm_scan_par and forward_scan_par, engine.py:294-302), at the configs[0]
    shape and on a batch sample of the configs[1] layer shape.  Median of ``reps``
    after one warm-up (the method of cli/__init__.py:166-179); lanes/s and
    algorithmic GB/s (SURVEY.md §8d fused-op bytes, fp32)."""
    import numpy as np
    from oracle import cpu_port
    cpu_port.build()
    threads = os.cpu_count() or 1
    out = {}
    for name, (Bt, L, E, N, M, scale_to) in {"cfg1": (2, 197, 192, 16, 8, 2),
                                             "cfg2": (8, 197, 384, 16, 8, 256)}.items():
        rng = np.random.default_rng(0)
        f = np.float32
        u, z = rng.standard_normal((Bt, L, E)).astype(f), rng.standard_normal((Bt, L, E)).astype(f)
        delta = (0.5 * rng.standard_normal((Bt, L, E))).astype(f)
        Bm, Cm = rng.standard_normal((Bt, L, N)).astype(f), rng.standard_normal((Bt, L, N)).astype(f)
        A = -np.tile(np.arange(1, N + 1, dtype=f), (E, 1))
        D = np.ones(E, f)
        dt = np.exp(rng.uniform(np.log(1e-3), np.log(1e-1), E))
        bias = (dt + np.log(-np.expm1(-dt))).astype(f)
        dl = np.logaddexp(f(0), delta + bias)
        abar = np.exp(dl[..., None] * A).astype(f)
        bx = (dl[..., None] * Bm[:, :, None, :] * u[..., None]).astype(f)

        def med(fn):
            fn()
            ts = []
            for _ in range(reps):
                t0 = time.perf_counter()
                fn()
                ts.append(time.perf_counter() - t0)
            return sorted(ts)[len(ts) // 2] * 1e3

        fused = med(lambda: cpu_port.fused_op(u, delta, A, Bm, Cm, D, z, bias, M, threads=threads))
        lbm = med(lambda: cpu_port.scan_par(abar, bx, Cm, D * u, M, True, threads=threads))
        fwd = med(lambda: cpu_port.scan_par(abar, bx, Cm, D * u, M, False, threads=threads))
        lanes = Bt * L * E * N
        nb = scan_alg_bytes(Bt, L, E, N, 4, 4)
        out[name] = {"sample": f"B={Bt} of {scale_to}, L={L}, E={E}, N={N}, M={M}, fp32",
                     "fused_op_ms": fused, "fused_op_ms_scaled": fused * scale_to / Bt,
                     "fused_lanes_per_s": lanes / fused * 1e3, "fused_gbs": nb / fused / 1e6,
                     "engine_lbm_ms": lbm, "engine_fwd_ms": fwd, "engine_lbm_over_fwd": lbm / fwd,
                     "engine_lbm_lanes_per_s": lanes / lbm * 1e3}
    return {"cores": threads, "kind": "port", "rows": out}


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    steps = max(1, min(args.steps, 20))  # ~0.4 s per 2-image step on 16 cores
    warm = max(1, min(args.warmup, 5))
    r = cpu_reference_run(steps, warm)
    line = {"metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": args.gpus, "steps": steps,
            "warmup": warm, "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (N(0,1) images, random-init weights)",
            "config": _workload_config(1, CPU_SAMPLE_BATCH, {"note": "bounded CPU sample, scaled to images/s"}),
            "impl": "reference",
            "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm

def xu_roofline(B, L, E, N, ms, clocks):
    """The binding pipe of the fused scan: MUFU (XU) ops per launch = (N state exps +
    2 softplus + 2 SiLU) per (b, l, e), against 16 MUFU lanes/clk/SM x 148 SMs at the
    SM clock sampled during the timed region."""
    ops = (N + 4) * B * L * E
    mhz = (clocks or {}).get("sm_mhz") or 1965.0
    peak = 16 * 148 * mhz * 1e6 / 1e9  # G MUFU ops/s
    achieved = ops / (ms / 1e3) / 1e9
    return {"bound": "mufu", "ops_per_launch": ops, "achieved": achieved, "peak": peak,
            "unit": "Gop/s", "frac": achieved / peak,
            "peak_source": "16 MUFU.EX2 lanes/clk/SM (measured, tools/micro) x 148 SMs x sampled SM clock"}


def scan_alg_bytes(B, L, E, N, s_io, s_bc):
    """s_in*B*L*(3E + 2N) + s_out*B*L*E + 4*(E*N + 2E)."""
    return s_io * B * L * 3 * E + s_bc * B * L * 2 * N + s_io * B * L * E + 4 * (E * N + 2 * E)


def measure_ops(peak, iters=10):
    """Kernel-level numbers for every BASELINE config on this GPU (rank 0): fused
    LB fwd, forward-only fwd (the LB/fwd cost ratio of the north star) and, for
    configs[2], the backward with training checkpoints.  CUDA events on the
    launching stream, L2 flushed between launches, median of ``iters``; the scan
    launches are replayed from a CUDA graph so host-side wrapper time cannot stretch
    the device timeline of the small configs."""
    import torch
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from kbench import CFGS, alg_bytes, bwd_alg_bytes, gpu_warmup, make, time_fn

    from paper_2506_15976_b200.scan import lbm_selective_scan_bwd, lbm_selective_scan_fwd
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    gpu_warmup()
    names = {"cfg1": "configs[0] op fwd fp32 B=2 E=192 L=197", "cfg2": "configs[1] LBVim-Ti layer scan bf16 B=256 E=384",
             "cfg3": "configs[2] LBVim-S scan fp32 B=128 E=768 fwd+bwd", "cfg4": "configs[3] LBVim-S 1024^2 layer scan bf16 "
             "B=32 L=4096 E=768", "cfg5": "configs[4] MIL bag fp32 B=1 L=100k E=512 (1 GPU)",
             "cfg5s": "configs[4] one 8-way channel shard (E=64)",
             "cfg3s": "configs[2] per-GPU batch shard at 8 GPUs (B=16) fwd+bwd",
             "cfg3b": "configs[2] shape with bf16 I/O (the amp training path) fwd+bwd"}
    res = {}
    for name, (Bt, L, E, N, M, io, bc) in CFGS.items():
        if name not in names:
            continue
        x = make(Bt, L, E, N, io, bc)
        out = torch.empty(Bt, L, E, device="cuda", dtype=io)
        s_io = torch.tensor([], dtype=io).element_size()
        s_bc = torch.tensor([], dtype=bc).element_size()
        nb = alg_bytes(Bt, L, E, N, s_io, s_bc, s_io)
        lb_ms = time_fn(lambda: lbm_selective_scan_fwd(**x, window=M, out=out), iters, flush, graph=True)
        fw_ms = time_fn(lambda: lbm_selective_scan_fwd(**x, window=M, lb=False, out=out), iters, flush, graph=True)
        from paper_2506_15976_b200.scan import global_bidir_selective_scan
        bi_ms = time_fn(lambda: global_bidir_selective_scan(**x), iters, flush, graph=True) if name in ("cfg2", "cfg4") else None
        r = {"what": names[name], "window": M, "lbm_fwd_ms": lb_ms, "fwd_only_ms": fw_ms,
             "global_bidir_ms": bi_ms, "lb_over_bidir": (lb_ms / bi_ms) if bi_ms else None,
             "lb_over_fwd": lb_ms / fw_ms, "bytes": nb, "gbs": nb / lb_ms / 1e6, "frac": nb / lb_ms / 1e6 / peak,
             "lanes_per_s": Bt * L * E * N / lb_ms * 1e3}
        if name in ("cfg3", "cfg3s", "cfg3b"):
            dout = torch.randn(Bt, L, E, device="cuda").to(io)
            _, ck = lbm_selective_scan_fwd(**x, window=M, save_checkpoints=True)
            nbb = bwd_alg_bytes(Bt, L, E, N, s_io, s_bc, s_io)
            bw_ms = time_fn(lambda: lbm_selective_scan_bwd(dout, **x, window=M, checkpoints=ck), iters, flush, graph=True)
            fck_ms = time_fn(lambda: lbm_selective_scan_fwd(**x, window=M, save_checkpoints=True), iters, flush, graph=True)
            r.update({"bwd_ms": bw_ms, "bwd_bytes": nbb, "bwd_gbs": nbb / bw_ms / 1e6,
                      "bwd_frac": nbb / bw_ms / 1e6 / peak, "fwd_with_ckpt_ms": fck_ms,
                      "fwd_bwd_ms": fck_ms + bw_ms, "fwd_bwd_gbs": (nb + nbb) / (fck_ms + bw_ms) / 1e6})
            del dout, ck
        res[name] = r
        del x, out
    # configs[1] model in fp32 (activations, weights, scan I/O): the precision of the
    # reference's CPU arm, so the GPU/CPU ratio can be read like for like
    from paper_2506_15976_b200 import model as M
    tcfg = M.lbvim_tiny()
    net = M.LBVim(tcfg, M.init_params(tcfg, seed=0), dtype=torch.float32)
    g = torch.Generator(device="cuda").manual_seed(7)
    imgs = torch.randn(256, 224, 224, 3, generator=g, device="cuda")
    run = net.graphed(imgs)
    ms = time_fn(run, 5, flush)
    res["lbvim_t_fp32"] = {"what": "configs[1] LBVim-Ti forward in fp32 (fp32 scan I/O, fp32 GEMMs), batch 256",
                           "ms_per_batch": ms, "images_per_s": 256 / ms * 1e3}
    del net, imgs, run
    torch.cuda.empty_cache()
    # configs[3] at model level: LBVim-S 1024^2 (L = 4096 + class token), batch 32, bf16 forward
    cfg = M.lbvim_small(image_size=1024)
    net = M.LBVim(cfg, M.init_params(cfg, seed=0), dtype=torch.bfloat16)
    imgs = torch.randn(32, 1024, 1024, 3, generator=g, device="cuda").to(torch.bfloat16)
    run = net.graphed(imgs)
    ms = time_fn(run, 3, flush)
    res["cfg4_model"] = {"what": "configs[3] LBVim-S 1024^2 patch16 forward, batch 32, bf16, 24 layers, L=4097",
                         "ms_per_batch": ms, "images_per_s": 32 / ms * 1e3}
    del net, imgs, run
    torch.cuda.empty_cache()
    # the other hand-written kernels of the block at the LBVim shapes (HBM-bound):
    # conv1d+SiLU fwd (2 s B L E bytes) and bwd (3 s B L E), RMSNorm (2 s B L D)
    from paper_2506_15976_b200.conv import causal_conv1d_silu_bwd, causal_conv1d_silu_fwd
    from paper_2506_15976_b200.norm import rms_norm
    kern = {}
    for tag, (Bk, Lk, Dk, dt) in {"lbvim_t": (256, 197, 192, torch.bfloat16),
                                  "lbvim_s_1024": (32, 4097, 384, torch.bfloat16),
                                  "lbvim_s_train_f32": (128, 197, 384, torch.float32)}.items():
        Ek = 2 * Dk
        sz = torch.tensor([], dtype=dt).element_size()
        xz = torch.randn(Bk, Lk, 2 * Ek, generator=g, device="cuda").to(dt)
        wk = torch.randn(Ek, 4, generator=g, device="cuda")
        ok = torch.empty(Bk, Lk, Ek, device="cuda", dtype=dt)
        ms_f = time_fn(lambda: causal_conv1d_silu_fwd(xz[..., :Ek], wk, out=ok), iters, flush)
        gk = torch.randn(Bk, Lk, Ek, generator=g, device="cuda").to(dt)
        ms_b = time_fn(lambda: causal_conv1d_silu_bwd(xz[..., :Ek], wk, None, gk), iters, flush)
        tk = torch.randn(Bk, Lk, Dk, generator=g, device="cuda").to(dt)
        sk = torch.randn(Dk, generator=g, device="cuda")
        on = torch.empty_like(tk)
        ms_n = time_fn(lambda: rms_norm(tk, sk, out=on), iters, flush)
        nb_c, nb_n = 2 * sz * Bk * Lk * Ek, 2 * sz * Bk * Lk * Dk
        kern[tag] = {"shape": [Bk, Lk, Ek], "dtype": str(dt).replace("torch.", ""),
                     "conv_fwd_ms": ms_f, "conv_fwd_frac": nb_c / ms_f / 1e6 / peak,
                     "conv_bwd_ms": ms_b, "conv_bwd_frac": 1.5 * nb_c / ms_b / 1e6 / peak,
                     "rms_norm_ms": ms_n, "rms_norm_frac": nb_n / ms_n / 1e6 / peak}
        del xz, ok, gk, tk, on
    res["block_kernels"] = kern
    torch.cuda.empty_cache()
    # configs[4] as a workload: one MambaMIL-style bag (mil.py) on one GPU, bf16
    from paper_2506_15976_b200.mil import MILBag, MILConfig, init_mil_params
    mcfg = MILConfig(d_in=1024, dim=512, state_dim=16, dt_rank=32, num_classes=2)
    bag = MILBag(mcfg, init_mil_params(mcfg, seed=0, device="cuda"), dtype=torch.bfloat16)
    X = torch.randn(100000, 1024, generator=g, device="cuda").to(torch.bfloat16)
    ms = time_fn(lambda: bag(X), 5, flush)
    res["cfg5_model"] = {"what": "configs[4] MambaMIL-style bag forward (fc 1024->512, RMSNorm, in-proj, conv, "
                                 "x_proj, LB scan E=512 N=16 M=16, mean pool, head), L=100k, bf16, 1 GPU",
                         "ms_per_bag": ms, "bags_per_s": 1e3 / ms}
    del bag, X
    torch.cuda.empty_cache()
    # configs[2] as a workload: one LBVim-S training step (fwd + bwd through the fused
    # scan / conv kernels, cuBLAS fp32 GEMMs, AdamW), batch 128, fp32
    from paper_2506_15976_b200 import model as M
    tcfg = M.lbvim_small()
    tr = M.LBVimTrainer(tcfg, M.init_params(tcfg, seed=0, device="cuda"), lr=1e-4)
    ti = torch.randn(128, 224, 224, 3, generator=g, device="cuda")
    tl = torch.randint(0, tcfg.num_classes, (128,), generator=g, device="cuda")
    ms = time_fn(lambda: tr.step(ti, tl), 3, flush)
    res["cfg3_train"] = {"what": "configs[2] LBVim-S training step (fwd+bwd+AdamW), batch 128, fp32, 24 layers, "
                                 "fused scan fwd/bwd + conv fwd/bwd, cuBLAS fp32 GEMMs",
                         "ms_per_step": ms, "images_per_s": 128 / ms * 1e3}
    del tr
    torch.cuda.empty_cache()
    tr = M.LBVimTrainer(tcfg, M.init_params(tcfg, seed=0, device="cuda"), lr=1e-4, amp=True)
    ms = time_fn(lambda: tr.step(ti, tl), 3, flush)
    res["cfg3_train_bf16"] = {"what": "configs[2] LBVim-S training step, bf16 autocast projections (tensor cores), "
                                      "bf16-I/O fused scan / conv kernels with fp32 state, fp32 master weights + AdamW, "
                                      "batch 128",
                              "ms_per_step": ms, "images_per_s": 128 / ms * 1e3}
    # the same step captured once into a CUDA graph (LBVimTrainer.graphed: forward,
    # fused-kernel backward and capturable AdamW replayed as one graph launch)
    run = tr.graphed(ti, tl)
    ms = time_fn(lambda: run(ti, tl), 5, flush)
    res["cfg3_train_bf16_graphed"] = {"what": "configs[2] LBVim-S bf16-autocast training step as one CUDA graph replay",
                                      "ms_per_step": ms, "images_per_s": 128 / ms * 1e3}
    del run
    del tr, ti, tl, flush
    torch.cuda.empty_cache()
    return res


def strong_scaling(world, rank, dev, iters=10):
    """Fixed-total-work rows for the BASELINE configs that shard (run on every rank,
    device time per iteration = max over ranks of CUDA-event time on the launching
    stream, L2 flushed outside the events):
      * configs[2]: global batch 128 (LBVim-S scan shape, fp32) split over the ranks,
        fused fwd with training checkpoints + fused bwd per rank, no collective;
      * configs[4]: one bag, L=100k, E=512 split by channel (E/world per rank, B and C
        replicated), the scan alone, then the all_gather of the (1, L, E/world) outputs
        timed separately;
      * configs[1]: LBVim-Ti forward with a global batch of 256 split over the ranks."""
    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from kbench import make

    from paper_2506_15976_b200 import model as M
    from paper_2506_15976_b200.scan import lbm_selective_scan_bwd, lbm_selective_scan_fwd
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def timed(fn, n=iters):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ts = []
        for _ in range(n):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            e.synchronize()
            ts.append(s.elapsed_time(e))
        ms = sorted(ts)[len(ts) // 2]
        t = torch.tensor([ms], device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    rows = {}
    Bl = 128 // world
    x = make(Bl, 197, 768, 16, torch.float32, torch.float32, seed=rank)
    dout = torch.randn(Bl, 197, 768, device=dev)

    def step():
        _, ck = lbm_selective_scan_fwd(**x, window=8, save_checkpoints=True)
        lbm_selective_scan_bwd(dout, **x, window=8, checkpoints=ck)
    ms = timed(step)
    rows["cfg3_fwd_bwd"] = {"global_batch": 128, "batch_per_rank": Bl, "ms": ms,
                            "images_per_s": 128 / ms * 1e3, "what": "fused LB scan fwd (checkpoints) + bwd, "
                            "LBVim-S scan shape L=197 E=768 N=16 M=8 fp32"}
    del x, dout
    El = 512 // world
    x = make(1, 100000, El, 16, torch.float32, torch.float32, seed=rank)
    out = torch.empty(1, 100000, El, device=dev)
    ms = timed(lambda: lbm_selective_scan_fwd(**x, window=16, out=out))
    r = {"E": 512, "E_per_rank": El, "scan_ms": ms, "scan_instances_per_s": 1e5 / ms * 1e3}
    if world > 1:
        full = torch.empty(world, 1, 100000, El, device=dev)
        r["all_gather_ms"] = timed(lambda: dist.all_gather_into_tensor(full, out))
        r["all_gather_bytes_per_rank"] = out.numel() * 4 * (world - 1)
    rows["cfg5_bag_scan"] = r
    del x, out
    torch.cuda.empty_cache()
    cfg = M.lbvim_tiny()
    Bl = 256 // world
    net = M.LBVim(cfg, M.init_params(cfg, seed=0, device=dev), dtype=torch.bfloat16)
    g = torch.Generator(device=dev).manual_seed(99 + rank)
    run = net.graphed(torch.randn(Bl, 224, 224, 3, generator=g, device=dev).to(torch.bfloat16))
    ms = timed(run)
    rows["lbvim_t_global256"] = {"global_batch": 256, "batch_per_rank": Bl, "ms": ms,
                                 "images_per_s": 256 / ms * 1e3}
    del net, run, flush
    torch.cuda.empty_cache()
    return {"note": "strong scaling: total work fixed as N grows; ms = median per iteration, max over ranks",
            "n_gpus": world, "rows": rows}


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2506_15976_b200 import model as M
    from paper_2506_15976_b200 import scan as S

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    B = args.batch
    cfg = M.lbvim_tiny()
    params = M.init_params(cfg, seed=0, device=dev)
    net = M.LBVim(cfg, params, dtype=torch.bfloat16)
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    images = torch.randn(B, 224, 224, 3, generator=g, device=dev).to(torch.bfloat16)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    # ---- device-timed steps (inputs resident) -------------------------------
    run = net.graphed(images)
    for _ in range(args.warmup):
        run()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with clock_sampler(local_rank) as clk:
        t_wall = time.perf_counter()
        for s, e in evs:
            flush.zero_()
            s.record()
            run()
            e.record()
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    dev_ms = sum(s.elapsed_time(e) for s, e in evs)
    t = torch.tensor([dev_ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms = float(t.item())
    value = world * B * args.steps / (dev_ms / 1e3)

    # ---- end to end through the public API: pinned host in, logits out ------
    host_imgs = [images.cpu().pin_memory() for _ in range(2)]
    runs = [run, net.graphed(images)]
    outs = [torch.empty((B, cfg.num_classes), dtype=torch.float32).pin_memory() for _ in range(2)]
    copy = torch.cuda.Stream(device=dev)
    comp = torch.cuda.current_stream()
    h2d_done = [torch.cuda.Event() for _ in range(2)]
    comp_done = [torch.cuda.Event() for _ in range(2)]
    e2e_steps = args.steps

    e2e_ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))

    def e2e_loop(n):
        with torch.cuda.stream(copy):
            e2e_ev[0].record(copy)  # before the first host->device copy
            runs[0].static_in.copy_(host_imgs[0], non_blocking=True)
            h2d_done[0].record(copy)
        for i in range(n):
            k = i % 2
            comp.wait_event(h2d_done[k])
            runs[k].graph.replay()
            comp_done[k].record(comp)
            with torch.cuda.stream(copy):
                if i + 1 < n:
                    kn = (i + 1) % 2
                    if i >= 1:
                        copy.wait_event(comp_done[kn])
                    runs[kn].static_in.copy_(host_imgs[kn], non_blocking=True)
                    h2d_done[kn].record(copy)
                copy.wait_event(comp_done[k])
                outs[k].copy_(runs[k].static_out, non_blocking=True)
        with torch.cuda.stream(copy):
            e2e_ev[1].record(copy)  # after the last device->host copy
        torch.cuda.synchronize()

    e2e_loop(2)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_loop(e2e_steps)
    e2e_wall_s = time.perf_counter() - t0
    # device time from before the first H2D to after the last D2H (CUDA events on the
    # copy stream, max over ranks); the host wall clock is reported beside it
    e2e_s = e2e_ev[0].elapsed_time(e2e_ev[1]) / 1e3
    t = torch.tensor([e2e_s], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_value = world * B * e2e_steps / float(t.item())
    h2d_bytes = host_imgs[0].numel() * host_imgs[0].element_size()
    d2h_bytes = outs[0].numel() * outs[0].element_size()

    # ---- roofline: the fused scan kernel, timed live per launch -------------
    scan_evs = []
    orig = S.lbm_selective_scan_fwd

    def timed_scan(*a, **kw):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        r = orig(*a, **kw)
        e.record()
        scan_evs.append((s, e))
        return r

    M.lbm_selective_scan_fwd = timed_scan
    try:
        for _ in range(2):
            net.forward(images)
        torch.cuda.synchronize()
        scan_evs.clear()
        for _ in range(max(2, args.steps // 2)):
            flush.zero_()
            net.forward(images)
        torch.cuda.synchronize()
    finally:
        M.lbm_selective_scan_fwd = orig
    scan_ms = sum(s.elapsed_time(e) for s, e in scan_evs) / len(scan_evs)
    E, N, L = cfg.inner_dim, cfg.state_dim, cfg.seq_len
    nbytes = scan_alg_bytes(B, L, E, N, 2, 2)
    achieved = nbytes / (scan_ms / 1e3) / 1e9
    peaks = _peaks()
    peak = peaks.get("hbm_gbs")
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if peak else "fallback 6650 GB/s (B200_PROFILING.md)"
    peak = peak or 6650.0
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        traffic = tr.get("lbvim_t_scan_bytes_per_launch")
    except Exception:
        pass
    step_ms = dev_ms / args.steps
    scan_share = cfg.depth * scan_ms / step_ms

    ops = None
    if rank == 0 and not args.no_ops:
        ops = measure_ops(peak)
    if world > 1:
        dist.barrier()
    strong = None if args.no_strong else strong_scaling(world, rank, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = cpu_reference_run(steps=10, warmup=1)
        cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}
        cpu["op_level"] = cpu_op_baseline()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (N(0,1) images, random-init weights of the reference architecture)",
            "config": _workload_config(world, B),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d_bytes,
                    "d2h_bytes_per_step": d2h_bytes,
                    "note": "graph replay per step; pinned host images H2D and logits D2H every step on a "
                            "copy stream, double-buffered; CUDA events from before the first H2D to after "
                            "the last D2H, max over ranks",
                    "wall_s": e2e_wall_s},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "lbs::fwd_kernel (fused discretize + LB scan + D skip + SiLU gate)",
                         "bytes_per_launch": nbytes, "ms_per_launch": scan_ms, "peak_source": peak_src,
                         "share_of_step": scan_share,
                         "note": "MUFU/issue-bound: 1 ex2 + ~3.5 packed FP32 ops per state-step (DESIGN.md)",
                         "xu": xu_roofline(B, 197, cfg.inner_dim, cfg.state_dim, scan_ms, clk.summary())},
            "cpu_baseline": cpu,
            "ops": ops,
            "strong_scaling": strong,
            "gpu_launches": 3 * cfg.depth * args.steps,  # rms_norm + conv1d+SiLU + fused scan per block
            "clocks": clk.summary(),
            "wall_s_timed_region": t_wall,
        }
        print(json.dumps(line), flush=True)
    return 0


def _free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _self_launch(n):
    """``--gpus N`` outside torchrun: start N ranks (one per GPU) with
    torch.distributed.run on 127.0.0.1 and pass their output through."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=GLOBAL_BATCH_PER_GPU)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ops", action="store_true", help="skip the per-config kernel table")
    ap.add_argument("--no-strong", action="store_true", help="skip the strong-scaling rows")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _self_launch(args.gpus)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        return run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
