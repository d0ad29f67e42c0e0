"""One LBVim block as a single autograd node with a hand-written backward (training).

The reference's block forward / backward pair (block.py:158-190, block.py:193-220)
on the fused kernels, with the glue between them removed:

* forward: RMSNorm (lbs_rms_norm_fwd) -> one in-projection GEMM for x|z -> fused
  conv1d+SiLU on the x column block -> one GEMM for delta|B|C -> fused LB scan (with
  training checkpoints) on column views of those buffers -> out-projection GEMM with
  the residual added in its epilogue (``addmm`` with an fp32 output for bf16 operands);
* backward: the scan adjoint writes ``ddelta`` and ``dz`` straight into column blocks
  of the two projection gradients and ``du`` into the conv-output gradient, which the
  x|dt|B|C GEMM then accumulates into (``addmm_``, beta = 1); the conv adjoint writes
  ``dx`` into the x|z gradient's first column block; weight gradients and the
  normalised-input gradient come out of the GEMMs in fp32; the RMSNorm forward writes
  its bf16 GEMM input directly and its adjoint adds the residual branch's gradient.
  No concatenation of gradient slices, no separate residual / branch additions or
  casts, one zero-fill.

Used by :class:`paper_2506_15976_b200.model.LBVimTrainer` (default); the plain
autograd composition ``model.block_forward_train`` stays as the reference for tests.
``cdt`` is the compute dtype of the GEMMs and the fused kernels' I/O (bf16 under
amp, else fp32); the residual stream and all parameters stay fp32.
"""

from __future__ import annotations

import torch

from .conv import causal_conv1d_silu_bwd, causal_conv1d_silu_fwd
from .norm import RMS_EPS, rms_norm, rms_norm_bwd
from .scan import lbm_selective_scan_bwd, lbm_selective_scan_fwd


def _mm(a, b, dtype):
    """a @ b with a ``dtype`` output (fp32 out of bf16 operands: cuBLAS fp32 epilogue)."""
    return a @ b if a.dtype == dtype else torch.mm(a, b, out_dtype=dtype)


class LBVimBlockFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, T, norm_scale, w_x, w_z, conv_kernel, w_delta, w_b, w_c, delta_bias, a_log, d_param,
                w_out, M, reverse, mode, lb, cdt, eps):
        Bt, L, Dm = T.shape
        E, N = w_x.shape[1], w_b.shape[1]
        rows = Bt * L
        xn_c = rms_norm(T, norm_scale, eps=eps, out_dtype=cdt).reshape(rows, Dm)  # cast in the norm pass
        w_in = torch.cat([w_x, w_z], 1).to(cdt)                    # (D, 2E)
        xz = (xn_c @ w_in).view(Bt, L, 2 * E)
        xs = causal_conv1d_silu_fwd(xz[..., :E], conv_kernel, None, reverse)
        w_xp = torch.cat([w_delta, w_b, w_c], 1).to(cdt)           # (E, E + 2N)
        dbc = (xs.view(rows, E) @ w_xp).view(Bt, L, E + 2 * N)
        A = -torch.exp(a_log.float())
        yg, ck = lbm_selective_scan_fwd(xs, dbc[..., :E], A, dbc[..., E:E + N], dbc[..., E + N:], d_param,
                                        xz[..., E:], delta_bias, True, M, reverse, False, lb, mode,
                                        save_checkpoints=True)
        w_out_c = w_out.to(cdt)
        T2 = T.reshape(rows, Dm)
        if cdt == T.dtype:
            out = torch.addmm(T2, yg.view(rows, E), w_out_c)
        else:
            out = torch.addmm(T2, yg.view(rows, E), w_out_c, out_dtype=T.dtype)
        ctx.save_for_backward(T, norm_scale, xn_c, w_in, xz, conv_kernel, xs, w_xp, dbc, A, d_param, delta_bias,
                              yg, w_out_c, ck)
        ctx.cfg = (M, reverse, mode, lb, eps, E, N)
        return out.view(Bt, L, Dm)

    @staticmethod
    def backward(ctx, dOut):
        (T, norm_scale, xn_c, w_in, xz, conv_kernel, xs, w_xp, dbc, A, d_param, delta_bias, yg, w_out_c,
         ck) = ctx.saved_tensors
        M, reverse, mode, lb, eps, E, N = ctx.cfg
        Bt, L, Dm = T.shape
        rows = Bt * L
        with torch.autocast("cuda", enabled=False):
            return LBVimBlockFn._backward(ctx, dOut, T, norm_scale, xn_c, w_in, xz, conv_kernel, xs, w_xp, dbc, A,
                                          d_param, delta_bias, yg, w_out_c, ck, M, reverse, mode, lb, eps, E, N,
                                          Bt, L, Dm, rows)

    @staticmethod
    def _backward(ctx, dOut, T, norm_scale, xn_c, w_in, xz, conv_kernel, xs, w_xp, dbc, A, d_param, delta_bias, yg,
                  w_out_c, ck, M, reverse, mode, lb, eps, E, N, Bt, L, Dm, rows):
        cdt, f32 = xs.dtype, torch.float32
        dO = dOut.reshape(rows, Dm)
        dO_c = dO.to(cdt)
        # out-projection
        dyg = (dO_c @ w_out_c.t()).view(Bt, L, E)
        dw_out = _mm(yg.view(rows, E).t(), dO_c, f32)
        # fused scan adjoint, straight into the projection gradients' column blocks
        dbc_g = torch.empty(Bt, L, E + 2 * N, dtype=cdt, device=T.device)
        dxz = torch.empty(Bt, L, 2 * E, dtype=cdt, device=T.device)
        small = torch.zeros(E * N + 2 * E + conv_kernel.numel(), dtype=f32, device=T.device)  # one fill
        dA = small[:E * N].view(E, N)
        dD = small[E * N:E * N + E]
        dbias = small[E * N + E:E * N + 2 * E]
        dconv = small[E * N + 2 * E:].view(conv_kernel.shape)
        g = lbm_selective_scan_bwd(dyg, xs, dbc[..., :E], A, dbc[..., E:E + N], dbc[..., E + N:], d_param,
                                   xz[..., E:], delta_bias, True, M, reverse, lb, mode, checkpoints=ck,
                                   grads=dict(ddelta=dbc_g[..., :E], dz=dxz[..., E:], dA=dA, dD=dD,
                                              ddelta_bias=dbias))
        dbc_g[..., E:E + N].copy_(g["dB"])
        dbc_g[..., E + N:].copy_(g["dC"])
        dbc2 = dbc_g.view(rows, E + 2 * N)
        # x|dt|B|C projection: its input gradient accumulates into the scan's du (beta = 1)
        dxs = g["du"]
        dxs.view(rows, E).addmm_(dbc2, w_xp.t())
        dw_xp = _mm(xs.view(rows, E).t(), dbc2, f32)
        # conv1d + SiLU adjoint, dx into the x column block of the in-projection gradient
        causal_conv1d_silu_bwd(xz[..., :E], conv_kernel, None, dxs, reverse, True, dx=dxz[..., :E], dweight=dconv)
        dxz2 = dxz.view(rows, 2 * E)
        dxn = _mm(dxz2, w_in.t(), T.dtype).view(Bt, L, Dm)
        dw_in = _mm(xn_c.t(), dxz2, f32)
        dT, dscale = rms_norm_bwd(T, norm_scale, dxn, eps=eps, dres=dOut)  # + the residual branch
        d_alog = dA * A  # A = -exp(a_log)
        return (dT, dscale, dw_in[:, :E], dw_in[:, E:], dconv, dw_xp[:, :E], dw_xp[:, E:E + N], dw_xp[:, E + N:],
                dbias, d_alog, dD, dw_out, None, None, None, None, None, None)


def block_forward_fused(T, w: dict, M: int, reverse: bool = False, discretize_mode: str = "exp",
                        lb: bool = True, eps: float = RMS_EPS, compute_dtype=None):
    """Differentiable LBVim block as one autograd node (see module docstring).
    ``compute_dtype`` defaults to bf16 inside an enabled CUDA autocast region, else
    T's dtype.  ``w`` holds the reference's weight names (model.BLOCK_FIELDS)."""
    if compute_dtype is None:
        compute_dtype = torch.bfloat16 if torch.is_autocast_enabled("cuda") else T.dtype
    with torch.autocast("cuda", enabled=False):
        return LBVimBlockFn.apply(T, w["norm_scale"], w["w_x"], w["w_z"], w["conv_kernel"], w["w_delta"], w["w_b"],
                                  w["w_c"], w["delta_bias"], w["a_log"], w["d_param"], w["w_out"], M, reverse,
                                  discretize_mode, lb, compute_dtype, eps)
