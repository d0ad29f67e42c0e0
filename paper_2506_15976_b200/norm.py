"""RMSNorm (nn.rms_norm, nn.py:55-58) on the C ABI — the LBVim block's first op."""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .errors import ShapeError
from .scan import _DT, _ptr, _stream

RMS_EPS = 1e-6


def rms_norm(x, scale, eps: float = RMS_EPS, out=None):
    if not x.is_cuda:
        raise ShapeError("x must be a CUDA tensor (no CPU fallback)")
    D = x.shape[-1]
    if x.stride(-1) != 1:
        x = x.contiguous()
    x2 = x.reshape(-1, D)
    if out is None:
        out = torch.empty_like(x)
    o2 = out.view(-1, D)
    scale = scale.to(torch.float32).contiguous()
    a = _lib.NormArgs()
    a.rows, a.dim, a.io_dtype, a.eps = x2.shape[0], D, _DT[x.dtype], eps
    a.x, a.x_row_stride = _ptr(x2), x2.stride(0)
    a.scale = _ptr(scale)
    a.out, a.out_row_stride = _ptr(o2), o2.stride(0)
    _lib.check(_lib.lib().lbs_rms_norm_fwd(ctypes.byref(a), _stream()), "rms_norm")
    return out
