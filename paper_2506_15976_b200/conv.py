"""Fused depthwise causal conv1d + SiLU (nn.causal_conv1d + nn.silu,
nn.py:87-99,25-26) on the C ABI, with flip-on-load for reverse layers.

``weight`` is (E, K) in the reference's tap order (kernel[e, q] multiplies
x[l-q]); a torch Conv1d weight w[e, 0, j] corresponds to kernel[e, K-1-j].
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .errors import ShapeError
from .scan import _DT, _ptr, _stream, _strides


def _conv_args(x, weight, bias, reverse, silu):
    if not x.is_cuda:
        raise ShapeError("x must be a CUDA tensor (no CPU fallback)")
    if x.dim() != 3:
        raise ShapeError(f"x must be (B, L, E), got {tuple(x.shape)}")
    Bt, L, E = x.shape
    if weight.dim() != 2 or weight.shape[0] != E:
        raise ShapeError(f"weight must be (E, K) = ({E}, K), got {tuple(weight.shape)}")
    a = _lib.ConvArgs()
    a.batch, a.seqlen, a.dim, a.width = Bt, L, E, weight.shape[1]
    if x.dtype not in _DT:
        raise ShapeError(f"unsupported dtype {x.dtype}")
    a.io_dtype = _DT[x.dtype]
    a.flags = (_lib.FLAG_REVERSE if reverse else 0) | (_lib.CONV_SILU if silu else 0)
    a.x, a.x_stride = _ptr(x), _strides(x)
    a.weight = _ptr(weight)
    a.bias = _ptr(bias)
    return a


def causal_conv1d_silu_fwd(x, weight, bias=None, reverse=False, silu=True, out=None):
    weight = weight.to(torch.float32).contiguous()
    bias = None if bias is None else bias.to(torch.float32).contiguous()
    a = _conv_args(x, weight, bias, reverse, silu)
    if out is None:
        out = torch.empty(x.shape, dtype=x.dtype, device=x.device)
    a.out, a.out_stride = _ptr(out), _strides(out)
    _lib.check(_lib.lib().lbs_causal_conv1d_fwd(ctypes.byref(a), _stream()), "causal_conv1d_silu")
    return out


def causal_conv1d_silu_bwd(x, weight, bias, dout, reverse=False, silu=True, dx=None, dweight=None):
    """-> (dx, dweight (E,K) fp32, dbias (E,) fp32 or None).  ``dx``: optional output
    view (x's shape and dtype, any strides); ``dweight``: optional fp32 (E, K) buffer
    accumulated into (+=)."""
    weight = weight.to(torch.float32).contiguous()
    bias_f = None if bias is None else bias.to(torch.float32).contiguous()
    a = _conv_args(x, weight, bias_f, reverse, silu)
    dout = dout.to(x.dtype)
    if dx is None:
        dx = torch.empty(x.shape, dtype=x.dtype, device=x.device)
    elif tuple(dx.shape) != tuple(x.shape) or dx.dtype != x.dtype:
        raise ShapeError(f"dx must be a {x.dtype} tensor of shape {tuple(x.shape)}")
    dw = torch.zeros(weight.shape, dtype=torch.float32, device=x.device) if dweight is None else dweight
    db = torch.zeros(weight.shape[0], dtype=torch.float32, device=x.device) if bias is not None else None
    a.dout, a.dout_stride = _ptr(dout), _strides(dout)
    a.dx, a.dx_stride = _ptr(dx), _strides(dx)
    a.dweight, a.dbias = _ptr(dw), _ptr(db)
    L_ = _lib.lib()
    nws = L_.lbs_causal_conv1d_bwd_workspace_bytes(ctypes.byref(a))
    ws = torch.empty(max(nws, 1), dtype=torch.uint8, device=x.device)
    _lib.check(L_.lbs_causal_conv1d_bwd(ctypes.byref(a), _ptr(ws), nws, _stream()), "causal_conv1d_silu_bwd")
    return dx, dw, db


class CausalConv1dSiluFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, weight, bias, reverse, silu):
        ctx.save_for_backward(x, weight, bias)
        ctx.reverse, ctx.silu = reverse, silu
        return causal_conv1d_silu_fwd(x, weight, bias, reverse, silu)

    @staticmethod
    def backward(ctx, dout):
        x, weight, bias = ctx.saved_tensors
        dx, dw, db = causal_conv1d_silu_bwd(x, weight, bias, dout.contiguous(), ctx.reverse, ctx.silu)
        return dx, dw.to(weight.dtype), (None if db is None else db.to(bias.dtype)), None, None


def causal_conv1d_silu(x, weight, bias=None, reverse=False, silu=True):
    """Differentiable fused conv (+SiLU)."""
    if torch.is_grad_enabled() and (x.requires_grad or weight.requires_grad or
                                    (bias is not None and bias.requires_grad)):
        return CausalConv1dSiluFn.apply(x, weight, bias, reverse, silu)
    return causal_conv1d_silu_fwd(x, weight, bias, reverse, silu)
