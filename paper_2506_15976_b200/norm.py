"""RMSNorm (nn.rms_norm, nn.py:55-58) on the C ABI — the LBVim block's first op —
and its adjoint (block_backward, block.py:193-220) for the training path."""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .errors import ShapeError
from .scan import _DT, _ptr, _stream

RMS_EPS = 1e-6


def rms_norm(x, scale, eps: float = RMS_EPS, out=None, out_dtype=None):
    """``out_dtype=torch.bfloat16`` with fp32 ``x``: the normalised rows leave as bf16 (the
    input of a bf16 projection on an fp32 residual stream) in the same pass."""
    if not x.is_cuda:
        raise ShapeError("x must be a CUDA tensor (no CPU fallback)")
    D = x.shape[-1]
    if x.stride(-1) != 1:
        x = x.contiguous()
    x2 = x.reshape(-1, D)
    if out is None:
        out = torch.empty(x.shape, dtype=out_dtype or x.dtype, device=x.device)
    o2 = out.view(-1, D)
    scale = scale.to(torch.float32).contiguous()
    a = _lib.NormArgs()
    a.rows, a.dim, a.io_dtype, a.eps = x2.shape[0], D, _DT[x.dtype], eps
    if out.dtype not in _DT:
        raise ShapeError(f"unsupported output dtype {out.dtype}")
    a.out_dtype = _DT[out.dtype]
    a.x, a.x_row_stride = _ptr(x2), x2.stride(0)
    a.scale = _ptr(scale)
    a.out, a.out_row_stride = _ptr(o2), o2.stride(0)
    _lib.check(_lib.lib().lbs_rms_norm_fwd(ctypes.byref(a), _stream()), "rms_norm")
    return out


def rms_norm_bwd(x, scale, dout, eps: float = RMS_EPS, dres=None):
    """-> (dx in x's dtype, dscale fp32 (D,)).  dx = r g - x r^3 mean(g x) with
    g = dout * scale, r = 1/sqrt(mean(x^2) + eps); dscale = sum over rows of dout x r
    (deterministic fixed-order reduction).  ``dres`` (x's shape): a residual branch's
    gradient added to dx in the same pass."""
    if not x.is_cuda:
        raise ShapeError("x must be a CUDA tensor (no CPU fallback)")
    D = x.shape[-1]
    x2 = x.reshape(-1, D) if x.stride(-1) == 1 else x.contiguous().reshape(-1, D)
    g2 = dout.to(x.dtype).reshape(-1, D).contiguous()
    dx = torch.empty_like(x2)
    dscale = torch.zeros(D, dtype=torch.float32, device=x.device)
    scale = scale.to(torch.float32).contiguous()
    a = _lib.NormBwdArgs()
    a.rows, a.dim, a.io_dtype, a.eps = x2.shape[0], D, _DT[x.dtype], eps
    a.x, a.x_row_stride = _ptr(x2), x2.stride(0)
    a.scale = _ptr(scale)
    a.dout, a.dout_row_stride = _ptr(g2), g2.stride(0)
    a.dx, a.dx_row_stride = _ptr(dx), dx.stride(0)
    a.dscale = _ptr(dscale)
    if dres is not None:
        r2 = dres.to(x.dtype).reshape(-1, D)
        if r2.stride(-1) != 1:
            r2 = r2.contiguous()
        a.dres, a.dres_row_stride = _ptr(r2), r2.stride(0)
    L = _lib.lib()
    nws = L.lbs_rms_norm_bwd_workspace_bytes(ctypes.byref(a))
    ws = torch.empty(max(nws, 1), dtype=torch.uint8, device=x.device)
    _lib.check(L.lbs_rms_norm_bwd(ctypes.byref(a), ws.data_ptr(), nws, _stream()), "rms_norm_bwd")
    return dx.reshape(x.shape), dscale


class RMSNormFn(torch.autograd.Function):
    """Fused RMSNorm forward (lbs_rms_norm_fwd) with the fused adjoint (lbs_rms_norm_bwd)."""

    @staticmethod
    def forward(ctx, x, scale, eps=RMS_EPS):
        ctx.save_for_backward(x, scale)
        ctx.eps = eps
        return rms_norm(x, scale, eps=eps)

    @staticmethod
    def backward(ctx, dout):
        x, scale = ctx.saved_tensors
        dx, ds = rms_norm_bwd(x, scale, dout, eps=ctx.eps)
        return dx, ds.to(scale.dtype), None


def rms_norm_train(x, scale, eps: float = RMS_EPS):
    """Differentiable RMSNorm on the fused kernels."""
    return RMSNormFn.apply(x, scale, eps)
