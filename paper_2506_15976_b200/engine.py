"""GPU mirror of the reference engine's pre-discretised entry points
(engine.py:221-327): ``lbm_scan_par``, ``forward_scan_par``,
``global_bidir_par`` on (abar, bx, c, dx).

This is the debug/parity boundary: it lets the
reference's own verification grid (cli/__init__.py:25-29) and test_engine.py
vectors run unchanged on the B200.  Arguments may be numpy arrays (results come
back as numpy, like the reference) or CUDA tensors (results stay on device).
``workers`` is accepted for signature compatibility; the kernel is
deterministic, so results are bit-identical for any value
(test_engine.py:78-86).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .costmodel import count_scan_cost
from .errors import ShapeError
from .tiling import TilePlan, select_tile_len  # noqa: F401  (re-export, engine.py:54-85)


@dataclass
class ScanOutput:
    """Mirror of core.OracleOutput (core.py:120-128); ``cost`` carries the
    reference's counters for the call (costmodel.count_scan_cost, which the
    reference engine's run-time tallies equal, engine.py:290)."""

    y: object
    h_final: object
    cost: object = None


def _to_dev(x, dtype):
    if isinstance(x, torch.Tensor):
        return x.to(device="cuda", dtype=dtype).contiguous(), True
    return torch.as_tensor(np.ascontiguousarray(x), dtype=dtype, device="cuda"), False


def _run(abar, bx, c, dx, plan, workers, do_backward, reverse, variant):
    if workers < 1:
        raise ShapeError(f"workers must be >= 1, got {workers}")  # engine.py:239-242
    is_t = isinstance(abar, torch.Tensor)
    dt = (abar.dtype if is_t else np.asarray(abar).dtype)
    f64 = dt in (np.float64, torch.float64) or dt not in (np.float32, torch.float32)
    tdt = torch.float64 if f64 else torch.float32
    abar_t, _ = _to_dev(abar, tdt)
    if abar_t.dim() != 4:
        raise ShapeError(f"abar must be (B, L, E, N), got {tuple(abar_t.shape)}")
    B, L, E, N = abar_t.shape
    bx_t, _ = _to_dev(bx, tdt)
    c_t, _ = _to_dev(c, tdt)
    dx_t, _ = _to_dev(dx, tdt)
    for name, t, shp in (("bx", bx_t, (B, L, E, N)), ("c", c_t, (B, L, N)), ("dx", dx_t, (B, L, E))):
        if tuple(t.shape) != shp:
            raise ShapeError(f"{name} has shape {tuple(t.shape)}, expected {shp}")
    plan.check(L)
    y = torch.empty((B, L, E), dtype=tdt, device="cuda")
    hf = torch.empty((B, E, N), dtype=tdt, device="cuda")
    a = _lib.PrediscretizedArgs()
    a.batch, a.seqlen, a.dim, a.dstate, a.window = B, L, E, N, plan.tile_len
    a.flags = (_lib.FLAG_LB if do_backward else 0) | (_lib.FLAG_REVERSE if reverse else 0)
    a.dtype = _lib.LBS_F64 if f64 else _lib.LBS_F32
    a.abar, a.bx, a.c, a.dx = abar_t.data_ptr(), bx_t.data_ptr(), c_t.data_ptr(), dx_t.data_ptr()
    a.y, a.h_final = y.data_ptr(), hf.data_ptr()
    rc = _lib.lib().lbs_prediscretized_fwd(ctypes.byref(a), torch.cuda.current_stream().cuda_stream)
    _lib.check(rc, "lbm_scan_par")
    cost = count_scan_cost(variant, B, L, E, N, plan.tile_len)
    if variant == "global_bidir":  # one of the two sweeps (engine.py:316-326)
        cost = count_scan_cost("forward", B, L, E, N, plan.tile_len)
        cost.variant = variant
    if is_t:
        return ScanOutput(y=y, h_final=hf, cost=cost)
    return ScanOutput(y=y.cpu().numpy(), h_final=hf.cpu().numpy(), cost=cost)


def forward_scan_par(abar, bx, c, dx, plan: TilePlan, workers: int = 1) -> ScanOutput:
    """engine.py:294-296."""
    return _run(abar, bx, c, dx, plan, workers, False, False, "forward")


def lbm_scan_par(abar, bx, c, dx, plan: TilePlan, workers: int = 1) -> ScanOutput:
    """engine.py:299-302."""
    return _run(abar, bx, c, dx, plan, workers, True, False, "lbm")


def lbm_scan_par_reverse(abar, bx, c, dx, plan: TilePlan, workers: int = 1) -> ScanOutput:
    """engine._run(..., do_backward=True, reverse=True) (engine.py:265-291, 133, 183)."""
    return _run(abar, bx, c, dx, plan, workers, True, True, "lbm")


def _fields(p):
    """(abar, bx, c, dx) of a reference ``core.ScanParams`` (a plain dataclass,
    core.py:89-108) or of any 4-sequence."""
    if hasattr(p, "abar"):
        return p.abar, p.bx, p.c, p.dx
    return tuple(p)


def global_bidir_par(params_f, params_b, plan: TilePlan, workers: int = 1) -> ScanOutput:
    """engine.py:305-327: two full sweeps (the second flip-on-load), summed.
    ``params_f`` / ``params_b`` are ``ScanParams`` like the reference's
    (test_engine.py:64,73) or (abar, bx, c, dx) tuples."""
    f = _run(*_fields(params_f), plan, workers, False, False, "global_bidir")
    b = _run(*_fields(params_b), plan, workers, False, True, "global_bidir")
    return ScanOutput(y=f.y + b.y, h_final=f.h_final + b.h_final, cost=f.cost + b.cost)
