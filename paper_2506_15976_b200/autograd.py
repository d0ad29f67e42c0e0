"""autograd.Function for the fused LB selective scan.

Forward = lbs_scan_fwd with training checkpoints (the state entering every
backward chunk, fp32, ~N/ckpt_len floats per (b, l, e)); backward =
lbs_scan_bwd, i.e. the reference's autodiff.lbm_scan_grad (autodiff.py:192-195)
chained through block._discretize_backward (block.py:106-129) and the gate
adjoint (block.py:199-200) in one launch.  Gradients come back in each input's
dtype.
"""

from __future__ import annotations

import torch

from .scan import lbm_selective_scan_bwd, lbm_selective_scan_fwd


def _cast_like(g, ref):
    if g is None or ref is None or not isinstance(ref, torch.Tensor):
        return None
    return g.to(ref.dtype).reshape(ref.shape)


class LbmSelectiveScanFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, u, delta, A, B, C, D, z, delta_bias, delta_softplus, window, reverse, lb,
                discretize_mode):
        # parameters given as arrays / lists are tensors from here on (save_for_backward
        # takes tensors only); their gradients are not returned (no tensor to own them)
        A, D, delta_bias = (t if t is None or isinstance(t, torch.Tensor) else torch.as_tensor(t, device=u.device)
                            for t in (A, D, delta_bias))
        out, ck = lbm_selective_scan_fwd(u, delta, A, B, C, D, z, delta_bias, delta_softplus, window,
                                         reverse, False, lb, discretize_mode, save_checkpoints=True)
        ctx.save_for_backward(u, delta, A, B, C, D, z, delta_bias, ck)
        ctx.cfg = (delta_softplus, window, reverse, lb, discretize_mode)
        return out

    @staticmethod
    def backward(ctx, dout):
        u, delta, A, B, C, D, z, delta_bias, ck = ctx.saved_tensors
        delta_softplus, window, reverse, lb, mode = ctx.cfg
        g = lbm_selective_scan_bwd(dout.contiguous(), u, delta, A, B, C, D, z, delta_bias, delta_softplus,
                                   window, reverse, lb, mode, checkpoints=ck)
        return (_cast_like(g["du"], u), _cast_like(g["ddelta"], delta), _cast_like(g["dA"], A),
                _cast_like(g["dB"], B), _cast_like(g["dC"], C), _cast_like(g["dD"], D),
                _cast_like(g["dz"], z), _cast_like(g["ddelta_bias"], delta_bias),
                None, None, None, None, None)
