"""``torch.library`` registration of the fused LB selective scan (SURVEY.md §8b:
"torch.library custom op plus autograd.Function"): ``torch.ops.lbscan.lbm_selective_scan``
with a fake (meta) implementation, so the op can sit inside traced / exported
PyTorch programs, and an autograd formula on the fused backward kernel.

The eager hot path is ``scan.lbm_selective_scan`` (autograd.LbmSelectiveScanFn keeps
the forward's chunk checkpoints for the backward); this op saves only its inputs
and lets ``lbs_scan_bwd`` recompute the chunk states (the reference's own
``lbm_scan_grad`` also recomputes them, autodiff.py:48-195).
"""

from __future__ import annotations

from typing import Optional

import torch

from .scan import lbm_selective_scan_bwd, lbm_selective_scan_fwd


@torch.library.custom_op("lbscan::lbm_selective_scan", mutates_args=())
def lbm_selective_scan_op(u: torch.Tensor, delta: torch.Tensor, A: torch.Tensor, B: torch.Tensor,
                          C: torch.Tensor, D: Optional[torch.Tensor], z: Optional[torch.Tensor],
                          delta_bias: Optional[torch.Tensor], delta_softplus: bool, window: int,
                          reverse: bool) -> torch.Tensor:
    """block._discretize_cached + engine.lbm_scan_par + gate (block.py:87-103,132-138,177-178)."""
    return lbm_selective_scan_fwd(u, delta, A, B, C, D, z, delta_bias, delta_softplus,
                                  window if window > 0 else None, reverse)


@lbm_selective_scan_op.register_fake
def _(u, delta, A, B, C, D, z, delta_bias, delta_softplus, window, reverse):
    # the real op computes in fp32 or bf16 I/O; any other input dtype comes back fp32
    dt = u.dtype if u.dtype in (torch.float32, torch.bfloat16) else torch.float32
    return torch.empty(u.shape, dtype=dt, device=u.device)


def _setup_context(ctx, inputs, output):
    u, delta, A, B, C, D, z, delta_bias, delta_softplus, window, reverse = inputs
    ctx.save_for_backward(u, delta, A, B, C, D, z, delta_bias)
    ctx.cfg = (delta_softplus, window if window > 0 else None, reverse)


def _backward(ctx, dout):
    u, delta, A, B, C, D, z, delta_bias = ctx.saved_tensors
    softplus, window, reverse = ctx.cfg
    g = lbm_selective_scan_bwd(dout.contiguous(), u, delta, A, B, C, D, z, delta_bias, softplus, window,
                               reverse)

    def like(k, ref):
        return None if ref is None or g.get(k) is None else g[k].to(ref.dtype).reshape(ref.shape)

    return (like("du", u), like("ddelta", delta), like("dA", A), like("dB", B), like("dC", C), like("dD", D),
            like("dz", z), like("ddelta_bias", delta_bias), None, None, None)


lbm_selective_scan_op.register_autograd(_backward, setup_context=_setup_context)
