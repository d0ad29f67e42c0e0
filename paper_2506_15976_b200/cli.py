"""Command-line front end mirroring the reference's ``lbscan verify``, ``lbscan
bench`` and ``lbscan flops`` (cli/__init__.py:75-139, 159-218, 326-341) on the
B200 kernels.

    python -m paper_2506_15976_b200.cli verify [--l 1,5,...] [--m 1,3,...] [--variants forward,lbm,global_bidir]
                                               [--precision single,double] [--seed 0] [--fused]
    python -m paper_2506_15976_b200.cli bench [--l 4096] [--m 16] [--reps 20] [--ben 65536] [--out f.csv]
    python -m paper_2506_15976_b200.cli flops [--config key=value-file] [--out f.csv]

``bench`` prints the reference's CSV schema (variant, L, M, workers, median_ns,
flops, hbm_elems, tile_exchanges) for the forward / lbm / global_bidir scans of
the pre-discretised contract (engine.py:294-327) on the same synthetic
distribution (cli/__init__.py:143-154), timed with CUDA events on the device
(inputs resident, interleaved repetitions, median), followed by the same three
ratio lines.  ``--fused`` adds rows for the fused B200 operator (discretise +
scan + gate from u/delta/B/C in one launch) at the same B*E*N lanes.
``verify`` sweeps the engine against the sequential definition (verify.py) over
the reference's default grid, fp32 at 1e-5 and fp64 at 1e-12, with bitwise
equality across repeated launches in place of worker counts; ``--fused`` adds
the fused operator (both directions).
Exit codes as the reference: 0 ok, 1 check failure / runtime / shape error, 2 bad flags.
"""

from __future__ import annotations

import argparse
import sys

import numpy as np

from .costmodel import VARIANTS, count_model_cost, count_scan_cost, format_table, reports_to_csv
from .errors import ShapeError
from .model import ModelConfig

_HEADER = ("variant", "L", "M", "workers", "median_ns", "flops", "hbm_elems", "tile_exchanges")


def _device_median_ns(fns: dict, reps: int) -> dict:
    import torch

    for fn in fns.values():  # untimed warm-up (cli/__init__.py:161-162)
        fn()
    torch.cuda.synchronize()
    times = {k: [] for k in fns}
    for _ in range(reps):  # interleaved (cli/__init__.py:163-170)
        for k, fn in fns.items():
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            e.synchronize()
            times[k].append(s.elapsed_time(e) * 1e6)
    return {k: int(np.median(v)) for k, v in times.items()}


def run_bench(L: int, M: int, workers: int, reps: int, ben: int = 1 << 16, seed: int = 0, fused: bool = False):
    """cli/__init__.py:143-179 on the GPU: {variant: {"median_ns", "cost"}}."""
    import torch

    from . import engine
    from .scan import global_bidir_selective_scan, lbm_selective_scan_fwd
    from .tiling import TilePlan

    if min(L, M, reps) < 1:
        raise ShapeError("L, M and reps must be >= 1")
    N = 16
    E = max(1, ben // N)
    rng = np.random.default_rng(np.random.PCG64(seed))  # core.seeded_rng
    abar = rng.random((1, L, E, N), dtype=np.float32) * 0.6 + 0.35
    bx = rng.standard_normal((1, L, E, N), dtype=np.float32)
    c = rng.standard_normal((1, L, N), dtype=np.float32)
    dx = rng.standard_normal((1, L, E), dtype=np.float32)
    dev = [torch.from_numpy(a).cuda() for a in (abar, bx, c, dx)]
    plan = TilePlan.for_length(L, M)
    fns = {
        "forward": lambda: engine.forward_scan_par(*dev, plan, workers),
        "lbm": lambda: engine.lbm_scan_par(*dev, plan, workers),
        "global_bidir": lambda: engine.global_bidir_par(dev, dev, plan, workers),
    }
    if fused:
        g = torch.Generator(device="cuda").manual_seed(seed)
        x = dict(u=torch.randn(1, L, E, device="cuda", generator=g),
                 delta=0.5 * torch.randn(1, L, E, device="cuda", generator=g),
                 A=-torch.arange(1, N + 1, device="cuda", dtype=torch.float32).repeat(E, 1),
                 B=torch.randn(1, L, N, device="cuda", generator=g), C=torch.randn(1, L, N, device="cuda", generator=g),
                 D=torch.ones(E, device="cuda"), z=torch.randn(1, L, E, device="cuda", generator=g),
                 delta_bias=torch.full((E,), -4.0, device="cuda"))
        out = torch.empty(1, L, E, device="cuda")
        fns["fused_forward"] = lambda: lbm_selective_scan_fwd(**x, window=M, lb=False, out=out)
        fns["fused_lbm"] = lambda: lbm_selective_scan_fwd(**x, window=M, lb=True, out=out)
        # parameter reuse for the backward sweep, as the reference's bench does (cli/__init__.py:161-163)
        fns["fused_global_bidir"] = lambda: global_bidir_selective_scan(**x)
    med = _device_median_ns(fns, reps)
    res = {}
    for k, ns in med.items():
        base = k.replace("fused_", "")
        res[k] = {"median_ns": ns, "cost": count_scan_cost(base, 1, L, E, N, M)}
    return res


def bench_rows(results, L, M, workers):
    """cli/__init__.py:182-197."""
    rows = []
    for variant, r in results.items():
        cost = r["cost"]
        rows.append(dict(zip(_HEADER, (variant, L, M, workers, r["median_ns"], cost.flops,
                                       cost.hbm_reads + cost.hbm_writes, cost.tile_exchanges))))
    return rows


def _int_list(text: str) -> list[int]:
    return [int(tok) for tok in text.split(",") if tok]


def cmd_verify(args) -> int:
    """cli/__init__.py:123-139."""
    from .verify import TOLERANCE, VerificationError, run_verification
    try:
        worst = run_verification(grid_l=args.l, grid_m=args.m, variants=args.variants, precisions=args.precision,
                                 seed=args.seed, fused=args.fused)
    except VerificationError as exc:
        print(f"FAIL: {exc}")
        return 1
    for variant, errs in worst.items():
        for precision, err in errs.items():
            print(f"{variant:13s} {precision:6s} max rel err {err:.3e}  (tol {TOLERANCE[precision]:.0e})")
    print("ok")
    return 0


def cmd_bench(args) -> int:
    res = run_bench(args.l, args.m, args.workers, args.reps, ben=args.ben, seed=args.seed, fused=args.fused)
    rows = bench_rows(res, args.l, args.m, args.workers)
    print(",".join(_HEADER))
    for row in rows:
        print(",".join(str(row[k]) for k in _HEADER))
    t = {k: v["median_ns"] for k, v in res.items()}
    print(f"# lbm/forward time ratio:      {t['lbm'] / t['forward']:.3f}")
    print(f"# lbm/global_bidir time ratio: {t['lbm'] / t['global_bidir']:.3f}")
    print(f"# lbm/forward flop ratio:      {res['lbm']['cost'].flops / res['forward']['cost'].flops:.3f}")
    if "fused_lbm" in t:
        print(f"# fused lbm/forward time ratio: {t['fused_lbm'] / t['fused_forward']:.3f}")
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(",".join(_HEADER) + "\n")
            for row in rows:
                fh.write(",".join(str(row[k]) for k in _HEADER) + "\n")
    return 0


def read_config_file(path: str) -> ModelConfig:
    """key=value lines, '#' comments -> ModelConfig (cli/io.py:77-92 and
    ModelConfig.from_dict, model.py:100-115: tile_len "auto" or an int, booleans 0/1)."""
    fields = ModelConfig.__dataclass_fields__
    kw = {}
    for lineno, raw in enumerate(open(path, encoding="utf-8").read().splitlines(), 1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        if "=" not in line:
            raise ShapeError(f"config line {lineno} is not key=value: {line!r}")
        k, _, v = (s.strip() for s in line.partition("="))
        if k not in fields:
            raise ShapeError(f"unknown config key {k!r}")
        default = fields[k].default
        if k == "tile_len":
            kw[k] = None if v == "auto" else int(v)
        elif isinstance(default, bool):
            kw[k] = bool(int(v))
        elif isinstance(default, int):
            kw[k] = int(v)
        else:
            kw[k] = v
    return ModelConfig(**kw)


def cmd_flops(args) -> int:
    """cli/__init__.py:326-341."""
    cfg = read_config_file(args.config) if args.config else ModelConfig()
    reports = [count_model_cost(cfg)]
    scans = [count_scan_cost(v, 1, cfg.seq_len, cfg.inner_dim, cfg.state_dim, cfg.resolved_tile_len)
             for v in VARIANTS]
    print("model total (per image):")
    print(format_table(reports))
    print("\nscan kernel per block:")
    print(format_table(scans))
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(reports_to_csv(reports + scans))
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2506_15976_b200.cli", description=__doc__,
                                 formatter_class=argparse.RawDescriptionHelpFormatter)
    sub = ap.add_subparsers(dest="command", required=True)
    from .verify import DEFAULT_GRID_L, DEFAULT_GRID_M, VARIANTS as VERIFY_VARIANTS
    p = sub.add_parser("verify", help="engine-vs-sequential equivalence sweep")
    p.add_argument("--l", type=_int_list, default=list(DEFAULT_GRID_L))
    p.add_argument("--m", type=_int_list, default=list(DEFAULT_GRID_M))
    p.add_argument("--variants", type=lambda s: s.split(","), default=list(VERIFY_VARIANTS))
    p.add_argument("--precision", type=lambda s: s.split(","), default=["single", "double"])
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--fused", action="store_true", help="also verify the fused operator (fp32, both directions)")
    p.set_defaults(fn=cmd_verify)
    p = sub.add_parser("bench", help="device-timed scan variants + counters (reference CSV schema)")
    p.add_argument("--l", type=int, default=4096)
    p.add_argument("--m", type=int, default=16)
    p.add_argument("--workers", type=int, default=1, help="accepted for compatibility; results do not depend on it")
    p.add_argument("--reps", type=int, default=20)
    p.add_argument("--ben", type=int, default=1 << 16, help="B*E*N work lanes")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--out", default=None, help="CSV output path")
    p.add_argument("--fused", action="store_true", help="also time the fused operator at the same lanes")
    p.set_defaults(fn=cmd_bench)
    p = sub.add_parser("flops", help="analytic cost tables")
    p.add_argument("--config", default=None)
    p.add_argument("--out", default=None, help="CSV output path")
    p.set_defaults(fn=cmd_flops)
    return ap


def main(argv=None) -> int:
    ap = build_parser()
    args = ap.parse_args(argv)
    if args.command == "verify":  # cli/__init__.py:398-406
        from .verify import TOLERANCE, VARIANTS as VV
        if any(L < 1 for L in args.l) or any(M < 1 for M in args.m):
            ap.error("--l and --m entries must be >= 1")
        bad = set(args.variants) - set(VV)
        if bad:
            ap.error(f"unknown variants: {sorted(bad)}")
        bad = set(args.precision) - set(TOLERANCE)
        if bad:
            ap.error(f"unknown precisions: {sorted(bad)}")
    if args.command == "bench" and (args.l < 1 or args.m < 1 or args.reps < 1 or args.workers < 1):
        ap.error("--l, --m, --reps and --workers must be >= 1")
    try:
        return args.fn(args)
    except ShapeError as exc:
        print(f"error: {exc}")
        return 1


if __name__ == "__main__":
    sys.exit(main())
