"""Generate golden vectors by running the UNMODIFIED reference (test infrastructure).

Run in the build container, where /root/reference exists:

    python oracle/gen_golden.py

It imports ``lbscan`` read-only from /root/reference/pkg/src with numba's cache
and Python bytecode redirected away from the read-only tree (SURVEY.md §0
gotcha), and writes small compressed fixtures to ``tests/golden/``.  The
fixtures travel with the repo; nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_lbscan")
os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
sys.dont_write_bytecode = True
REF = os.environ.get("LBSCAN_REFERENCE", "/root/reference/pkg/src")
sys.path.insert(0, REF)

import numpy as np  # noqa: E402

from lbscan import autodiff, block, engine, model, nn, oracle  # noqa: E402
from lbscan.core import random_scan_params, seeded_rng  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")

GRID_L = (1, 5, 31, 128, 129, 197, 256, 257)  # cli/__init__.py:25 (+197 = LBVim L)
GRID_M = (1, 3, 4, 8, 16)  # cli/__init__.py:26
DIMS = (2, 3, 4)  # cli/__init__.py:82


def scan_grid():
    """Pre-discretised scans on the reference verification grid
    (cli/__init__.py:75-120): oracle fp64 + engine fp32, forward/lbm/reverse."""
    out = {}
    B, E, N = DIMS
    for L in GRID_L:
        p = random_scan_params(seeded_rng(L), B, L, E, N)
        out[f"L{L}_abar"], out[f"L{L}_bx"], out[f"L{L}_c"], out[f"L{L}_dx"] = p.abar, p.bx, p.c, p.dx
        f = oracle.forward_scan_seq(p.abar, p.bx, p.c, p.dx)
        out[f"L{L}_fwd_y"], out[f"L{L}_fwd_h"] = f.y, f.h_final
        p32 = random_scan_params(seeded_rng(L), B, L, E, N, dtype=np.float32)
        for M in GRID_M:
            r = oracle.lbm_scan_seq(p.abar, p.bx, p.c, p.dx, M)
            out[f"L{L}_M{M}_lbm_y"] = r.y
            plan = engine.TilePlan.for_length(L, M)
            e32 = engine.lbm_scan_par(p32.abar, p32.bx, p32.c, p32.dx, plan, workers=2)
            out[f"L{L}_M{M}_engine32_y"] = e32.y
            out[f"L{L}_M{M}_engine32_h"] = e32.h_final
            # private reverse flag: flip-on-load scan (engine.py:89,133,183)
            rv = engine._run(p.abar, p.bx, p.c, p.dx, plan, 1, True, True, "lbm")
            out[f"L{L}_M{M}_rev_y"] = rv.y
            out[f"L{L}_M{M}_rev_h"] = rv.h_final
    return out


def scan_grads():
    """autodiff.lbm_scan_grad / forward_scan_grad (autodiff.py:192-201)."""
    out = {}
    cases = [(12, 3, 2, 2, 2, 0), (11, 4, 2, 2, 2, 3), (197, 8, 2, 3, 4, 5), (40, 16, 1, 2, 3, 7)]
    for i, (L, M, B, E, N, seed) in enumerate(cases):
        p = random_scan_params(seeded_rng(seed), B, L, E, N)
        gy = seeded_rng(seed + 1).standard_normal((B, L, E))
        g = autodiff.lbm_scan_grad(p.abar, p.bx, p.c, p.dx, gy, M)
        gf = autodiff.forward_scan_grad(p.abar, p.bx, p.c, p.dx, gy)
        out[f"c{i}_meta"] = np.array([L, M, B, E, N, seed])
        for k, v in (("abar", p.abar), ("bx", p.bx), ("c", p.c), ("dx", p.dx), ("gy", gy)):
            out[f"c{i}_{k}"] = v
        for k in ("abar", "bx", "c", "dx"):
            out[f"c{i}_g_{k}"] = getattr(g, k)
            out[f"c{i}_gf_{k}"] = getattr(gf, k)
    return out


def block_cases():
    """LBVim block forward + backward (block.py:141-220), exp and linear modes,
    both directions.  The cache exposes the fused-op inputs (xs, z) so the
    op-level oracle is pinned, and block_backward's weight grads pin the
    fused-op adjoint (w_b = xs^T dB, a_log = dA*A, ...)."""
    out = {}
    cases = [
        # D, E, N, L, B, M, k, mode, reverse, seed
        (6, 8, 4, 9, 2, 3, 4, "exp", True, 29),
        (5, 6, 3, 13, 2, 4, 3, "exp", False, 20),
        (8, 12, 16, 40, 2, 8, 4, "exp", True, 11),
        (4, 5, 2, 6, 1, 3, 2, "linear", True, 21),
    ]
    for i, (D, E, N, L, B, M, k, mode, rev, seed) in enumerate(cases):
        rng = seeded_rng(seed)
        w = block.init_block_weights(rng, D, E, N, conv_width=k)
        dt = rng.uniform(0.15, 0.5, size=E)  # test_autodiff.py:123-129 conditioning
        w.delta_bias[:] = dt + np.log(-np.expm1(-dt))
        T = rng.standard_normal((B, L, D))
        gout = rng.standard_normal((B, L, D))
        o, cache = block.block_forward_cached(T, w, M, scan_impl="seq", reverse=rev, discretize_mode=mode)
        grads, g_in = block.block_backward(cache, w, gout)
        pre = f"b{i}_"
        out[pre + "meta"] = np.array([D, E, N, L, B, M, k, int(mode == "linear"), int(rev), seed])
        out[pre + "T"], out[pre + "gout"], out[pre + "out"], out[pre + "g_in"] = T, gout, o, g_in
        for name in ("xs", "z", "y", "yg", "x", "xc"):
            out[pre + "cache_" + name] = cache[name]
        for f in oracle_fields():
            out[pre + "w_" + f] = getattr(w, f)
            out[pre + "g_" + f] = getattr(grads, f)
    return out


def oracle_fields():
    return ("norm_scale", "w_x", "w_z", "conv_kernel", "w_b", "w_c", "w_delta",
            "delta_bias", "a_log", "d_param", "w_out")


def conv_cases():
    out = {}
    rng = seeded_rng(77)
    x = rng.standard_normal((2, 11, 5))
    kern = rng.standard_normal((5, 4))
    g = rng.standard_normal((2, 11, 5))
    out["x"], out["k"], out["g"] = x, kern, g
    out["y"] = nn.causal_conv1d(x, kern)
    out["gx"], out["gk"] = nn.causal_conv1d_grad(x, kern, g)
    return out


def model_cases():
    """model_forward (model.py:287-325) on desk-scale configs."""
    out = {}
    cfgs = [
        dict(image_size=16, patch_size=4, embed_dim=8, inner_dim=12, state_dim=4, depth=2,
             tile_len=4, head="gap", class_token="none", num_classes=3),
        dict(image_size=16, patch_size=4, embed_dim=8, inner_dim=16, state_dim=16, depth=3,
             tile_len=None, head="gap", class_token="middle", num_classes=5),
        dict(image_size=8, patch_size=2, embed_dim=8, inner_dim=12, state_dim=4, depth=3,
             tile_len=3, head="map", map_heads=2, class_token="none", num_classes=4),
    ]
    for i, cfg in enumerate(cfgs):
        mc = model.ModelConfig(**cfg)
        params = model.init_model_weights(mc, seed=40 + i)
        imgs = seeded_rng(50 + i).standard_normal((2, mc.image_size, mc.image_size, 1))
        logits = model.model_forward(imgs, mc, params, scan_impl="seq")
        logits_par = model.model_forward(imgs, mc, params, scan_impl="par")
        pre = f"m{i}_"
        out[pre + "images"] = imgs
        out[pre + "logits"] = logits
        out[pre + "logits_par"] = logits_par
        for k, v in params.items():
            out[pre + "p_" + k] = v
        for k, v in mc.to_dict().items():
            out[pre + "cfg_" + k] = np.array(v)
    return out


def bidir_cases():
    """global_bidir_seq / global_backward_scan_seq (oracle.py:55-77)."""
    out = {}
    pf = random_scan_params(seeded_rng(8), 2, 5, 2, 3)
    pb = random_scan_params(seeded_rng(9), 2, 5, 2, 3)
    r = oracle.global_bidir_seq(pf, pb)
    gb = oracle.global_backward_scan_seq(pb.abar, pb.bx, pb.c, pb.dx)
    for tag, p in (("f", pf), ("b", pb)):
        out[tag + "_abar"], out[tag + "_bx"], out[tag + "_c"], out[tag + "_dx"] = p.abar, p.bx, p.c, p.dx
    out["y"], out["h"] = r.y, r.h_final
    out["gb_y"], out["gb_h"] = gb.y, gb.h_final
    return out


def cost_cases():
    """costmodel.count_scan_cost / count_model_cost / reports_to_csv / format_table
    (costmodel.py:90-227) and the counters the engine tallies at run time
    (engine.py:290), which the reference asserts equal to the closed form."""
    from lbscan import costmodel

    out = {}
    dims, counters, variants = [], [], []
    for variant in ("forward", "lbm", "global_bidir"):
        for (B, L, E, N, M) in ((1, 1, 1, 1, 1), (2, 300, 4, 8, 8), (1, 100, 3, 4, 1), (1, 64, 2, 4, 4),
                                (2, 197, 3, 16, 8), (1, 4096, 2, 16, 16), (3, 257, 5, 4, 3), (1, 129, 2, 2, 16),
                                (256, 197, 384, 16, 8), (1, 100000, 512, 16, 16)):
            r = costmodel.count_scan_cost(variant, B, L, E, N, M)
            dims.append((B, L, E, N, M))
            variants.append(variant)
            counters.append([r.flops, r.hbm_reads, r.hbm_writes, r.tile_exchanges, r.register_ops])
    out["scan_dims"] = np.array(dims, dtype=np.int64)
    out["scan_variants"] = np.array(variants)
    out["scan_counters"] = np.array(counters, dtype=np.int64)
    # engine-tallied counters on a small run (engine.py:290 vs the closed form)
    p = random_scan_params(seeded_rng(3), 2, 37, 3, 4)
    plan = engine.TilePlan.for_length(37, 8)
    tallied = []
    for fn in (engine.forward_scan_par, engine.lbm_scan_par):
        c = fn(p.abar, p.bx, p.c, p.dx, plan).cost
        tallied.append([c.flops, c.hbm_reads, c.hbm_writes, c.tile_exchanges, c.register_ops])
    out["engine_counters"] = np.array(tallied, dtype=np.int64)
    cfgs = [dict(), dict(inner_dim=64), dict(head="map", class_token="head"),
            dict(image_size=224, patch_size=16, in_channels=3, embed_dim=192, inner_dim=384, state_dim=16,
                 depth=24, class_token="middle", num_classes=1000),
            dict(scan_variant="forward", tile_len=4)]
    mc = []
    for kw in cfgs:
        r = costmodel.count_model_cost(model.ModelConfig(**kw))
        mc.append([r.flops, r.hbm_reads, r.hbm_writes, r.tile_exchanges, r.register_ops])
    out["model_cfgs"] = np.array([repr(kw) for kw in cfgs])
    out["model_counters"] = np.array(mc, dtype=np.int64)
    reps = [costmodel.count_scan_cost(v, 2, 300, 4, 8, 8) for v in ("forward", "lbm", "global_bidir")]
    out["csv"] = np.array(costmodel.reports_to_csv(reps))
    out["table"] = np.array(costmodel.format_table(reps))
    return out


CASES = (("scan_grid", scan_grid), ("scan_grads", scan_grads), ("block", block_cases),
         ("conv", conv_cases), ("model", model_cases), ("bidir", bidir_cases), ("costs", cost_cases))


def main(only=()):
    os.makedirs(OUT, exist_ok=True)
    for name, fn in CASES:
        if only and name not in only:
            continue
        data = fn()
        path = os.path.join(OUT, f"{name}.npz")
        np.savez_compressed(path, **data)
        print(f"wrote {path}: {len(data)} arrays, {os.path.getsize(path) / 1e3:.0f} kB")


if __name__ == "__main__":
    main(tuple(sys.argv[1:]))  # e.g. python oracle/gen_golden.py costs
