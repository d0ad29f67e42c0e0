"""``verify``: equivalence sweep of the B200 engine against the sequential
definition of every scan variant — the B200 counterpart of the reference's
``lbscan verify`` (cli/__init__.py:25-29 grid, :75-120 run_verification,
:123-139 cmd_verify).

What is compared: the pre-discretised engine entry points (``engine.forward_scan_par``,
``lbm_scan_par``, ``global_bidir_par`` -> ``lbs_prediscretized_fwd``) in fp32
("single", 1e-5) and fp64 ("double", 1e-12), and — with ``fused=True`` — the
fused operator (``lbs_scan_fwd``: discretise + scan + D skip + gate, both
directions) in fp32 at 1e-5.  The reference checks bitwise equality across
numba worker counts; the B200 equivalent is bitwise equality across repeated
launches (the kernels are deterministic; ``workers`` has no effect on them).

The sequential definition below is the verification tool's own restatement of
the reference's oracle.py:39-129 (plain float64 loops, like the reference's
``oracle`` module that its ``verify`` uses).  It is a checker: no product op
calls it.  tests/test_verify.py pins it against the repo's golden-vector-pinned
oracle.
"""

from __future__ import annotations

import numpy as np

DEFAULT_GRID_L = (1, 5, 31, 128, 129, 256, 257, 1024, 4096)
DEFAULT_GRID_M = (1, 3, 4, 8, 16)
DEFAULT_GRID_WORKERS = (1, 2, 4, 8)
VARIANTS = ("forward", "lbm", "global_bidir")
TOLERANCE = {"single": 1e-5, "double": 1e-12}


class VerificationError(AssertionError):
    pass


# ---------------------------------------------------------------------------
# sequential definition (float64)


def _seq_states(abar, bx, reverse=False):
    B, L, E, N = abar.shape
    h = np.zeros((B, E, N))
    states = np.empty((B, L, E, N))
    order = range(L - 1, -1, -1) if reverse else range(L)
    for t in order:
        h = abar[:, t] * h + bx[:, t]
        states[:, t] = h
    return states, h


def _seq_local_record(abar, bx, M):
    B, L, E, N = abar.shape
    rec = np.empty((B, L, E, N))
    r = np.zeros((B, E, N))
    for i in range(L - 1, -1, -1):
        r = np.zeros((B, E, N)) if (i + 1) % M == 0 else abar[:, i] * r
        rec[:, i] = r
        r = r + bx[:, i]
    return rec


def seq_scan(variant, abar, bx, c, dx, M=1):
    """(y, h_final) of ``variant`` on one parameter set (global_bidir uses it for
    both directions, as cli/__init__.py:64-65 does)."""
    abar, bx, c, dx = (np.asarray(a, np.float64) for a in (abar, bx, c, dx))
    st, hf = _seq_states(abar, bx)
    if variant == "forward":
        return np.einsum("blen,bln->ble", st, c) + dx, hf
    if variant == "lbm":
        st = st + _seq_local_record(abar, bx, M)
        return np.einsum("blen,bln->ble", st, c) + dx, hf
    if variant == "global_bidir":
        sb, hb = _seq_states(abar, bx, reverse=True)
        y = np.einsum("blen,bln->ble", st, c) + np.einsum("blen,bln->ble", sb, c) + 2 * dx
        return y, hf + hb
    raise ValueError(f"unknown variant {variant!r}")


def _softplus(x):
    return np.logaddexp(0.0, x)


def seq_fused(u, delta, A, Bm, Cm, D, z, bias, M, reverse):
    """block.py:90-98 discretisation + lbm scan + gate (block.py:177-178), float64."""
    u, delta, A, Bm, Cm, D, z, bias = (np.asarray(a, np.float64) for a in (u, delta, A, Bm, Cm, D, z, bias))
    if reverse:
        u, delta, Bm, Cm, z = (a[:, ::-1] for a in (u, delta, Bm, Cm, z))
    dl = _softplus(delta + bias)
    abar = np.exp(dl[..., None] * A)
    bx = (dl * u)[..., None] * Bm[:, :, None, :]
    y, _ = seq_scan("lbm", abar, bx, Cm, D * u, M)
    out = y * z / (1.0 + np.exp(-z))
    return out[:, ::-1] if reverse else out


def max_rel_err(got, ref):
    """core.py:149-156: max |got - ref| / max |ref|."""
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    if ref.size == 0:
        return 0.0
    return float(np.max(np.abs(got - ref)) / max(float(np.max(np.abs(ref))), 1e-30))


def _params(rng, B, L, E, N, dtype):
    """core.random_scan_params (core.py:131-146): same draw order."""
    abar = rng.uniform(0.2, 0.99, size=(B, L, E, N)).astype(dtype)
    bx = rng.standard_normal((B, L, E, N)).astype(dtype)
    c = rng.standard_normal((B, L, N)).astype(dtype)
    dx = rng.standard_normal((B, L, E)).astype(dtype)
    return abar, bx, c, dx


# ---------------------------------------------------------------------------
# sweep


def _engine(variant, prm, plan, workers):
    from . import engine
    if variant == "forward":
        return engine.forward_scan_par(*prm, plan, workers)
    if variant == "lbm":
        return engine.lbm_scan_par(*prm, plan, workers)
    return engine.global_bidir_par(prm, prm, plan, workers)


def run_verification(grid_l=DEFAULT_GRID_L, grid_m=DEFAULT_GRID_M, grid_workers=DEFAULT_GRID_WORKERS,
                     variants=VARIANTS, precisions=("single", "double"), seed=0, dims=(2, 3, 4),
                     fused=False, log=None):
    """Engine-vs-sequential sweep; returns {variant: {precision: worst max_rel_err}}.
    Raises VerificationError on the first tolerance or determinism failure."""
    from .tiling import TilePlan
    B, E, N = dims
    worst = {v: {p: 0.0 for p in precisions} for v in variants}
    for precision in precisions:
        dtype = np.float32 if precision == "single" else np.float64
        tol = TOLERANCE[precision]
        for L in grid_l:
            prm = _params(np.random.default_rng(np.random.PCG64(seed + L)), B, L, E, N, dtype)
            refs = {}
            for M in grid_m:
                plan = TilePlan.for_length(L, M)
                for variant in variants:
                    key = (variant, M if variant == "lbm" else None)
                    if key not in refs:
                        refs[key] = seq_scan(variant, *prm, M)
                    ry, rh = refs[key]
                    base = None
                    for workers in grid_workers:
                        got = _engine(variant, prm, plan, workers)
                        err = max(max_rel_err(got.y, ry), max_rel_err(got.h_final, rh))
                        worst[variant][precision] = max(worst[variant][precision], err)
                        if err > tol:
                            raise VerificationError(f"{variant} {precision} L={L} M={M} workers={workers}: "
                                                    f"rel err {err:.3e} > {tol:.0e}")
                        if base is None:
                            base = got.y
                        elif not np.array_equal(base, got.y):
                            raise VerificationError(f"{variant} {precision} L={L} M={M}: outputs differ "
                                                    f"across repeated launches")
            if log:
                log(f"  {precision} L={L}: ok")
    if fused:
        worst["fused_lbm"] = {"single": _verify_fused(grid_l, grid_m, seed, log)}
    return worst


def _verify_fused(grid_l, grid_m, seed, log):
    import torch

    from .scan import lbm_selective_scan_fwd
    B, E, N = 2, 40, 16
    tol = TOLERANCE["single"]
    worst = 0.0
    for L in grid_l:
        rng = np.random.default_rng(np.random.PCG64(seed + 7 * L))
        u, z = rng.standard_normal((B, L, E)), rng.standard_normal((B, L, E))
        delta = 0.5 * rng.standard_normal((B, L, E))
        Bm, Cm = rng.standard_normal((B, L, N)), rng.standard_normal((B, L, N))
        A = -rng.uniform(0.5, N, size=(E, N))
        D = 1.0 + 0.1 * rng.standard_normal(E)
        dt = np.exp(rng.uniform(np.log(1e-3), np.log(1e-1), size=E))
        bias = dt + np.log(-np.expm1(-dt))
        t = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float32, device="cuda")  # noqa: E731
        for M in grid_m:
            for reverse in (False, True):
                ref = seq_fused(u, delta, A, Bm, Cm, D, z, bias, M, reverse)
                outs = [lbm_selective_scan_fwd(t(u), t(delta), t(A), t(Bm), t(Cm), D=t(D), z=t(z), delta_bias=t(bias),
                                               window=M, reverse=reverse).cpu().numpy() for _ in range(2)]
                err = max_rel_err(outs[0], ref)
                worst = max(worst, err)
                if err > tol:
                    raise VerificationError(f"fused_lbm single L={L} M={M} reverse={reverse}: rel err {err:.3e} > "
                                            f"{tol:.0e}")
                if not np.array_equal(outs[0], outs[1]):
                    raise VerificationError(f"fused_lbm L={L} M={M} reverse={reverse}: repeated launches differ")
        if log:
            log(f"  fused L={L}: ok")
    return worst
