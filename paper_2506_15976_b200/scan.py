"""Host side of the fused LB selective scan (PyTorch tensors -> C ABI).

North-star operator API:

    lbm_selective_scan(u, delta, A, B, C, D=None, z=None, delta_bias=None,
                       delta_softplus=True, window=None, reverse=False,
                       return_last_state=False)

in the reference's channel-last layout (core.py:8-14): ``u``, ``delta``, ``z``
are (B, L, E); ``B``, ``C`` are (B, L, N); ``A`` is (E, N); ``D`` and
``delta_bias`` are (E,).  The composition it computes is exactly
block.py:90-98 + engine.lbm_scan_par + block.py:177-178:

    dl = softplus(delta + delta_bias);  abar = exp(dl (x) A);  bx = (dl*u) (x) B
    y  = lbm(abar, bx, C, D*u, M);      out = y * silu(z)

``window`` defaults to ``select_tile_len(L)`` (engine.py:54-62); ``reverse``
scans right-to-left by flip-on-load (no copies).  Any strides are accepted
(e.g. B and C as column slices of one fused projection output).
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import FLAG_LB, FLAG_LINEAR, FLAG_REVERSE, FLAG_SOFTPLUS
from .errors import ShapeError
from .tiling import select_tile_len

_DT = {torch.float32: _lib.LBS_F32, torch.bfloat16: _lib.LBS_BF16, torch.float16: _lib.LBS_F16}


def _ptr(t):
    return None if t is None else t.data_ptr()


def _strides(t):
    return _lib.I64x3(*t.stride()) if t is not None else _lib.I64x3(0, 0, 0)


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _need_cuda(name, t):
    if t is not None and not t.is_cuda:
        raise ShapeError(f"{name} must be a CUDA tensor (the product path has no CPU fallback)")


def _vec(name, t, E, device):
    if t is None:
        return None
    t = torch.as_tensor(t, device=device)
    if t.shape != (E,):
        raise ShapeError(f"{name} has shape {tuple(t.shape)}, expected {(E,)}")
    return t.to(torch.float32).contiguous()


def _prepare(u, delta, A, B, C_, D, z, delta_bias, window):
    for name, t in (("u", u), ("delta", delta), ("B", B), ("C", C_), ("z", z)):
        _need_cuda(name, t)
    if u.dim() != 3:
        raise ShapeError(f"u must be (B, L, E), got {tuple(u.shape)}")
    Bt, L, E = u.shape
    if min(Bt, L, E) < 1:
        raise ShapeError(f"u has a zero-length dimension: {tuple(u.shape)}")
    if delta.shape != u.shape:
        raise ShapeError(f"delta has shape {tuple(delta.shape)}, expected {tuple(u.shape)}")
    if z is not None and z.shape != u.shape:
        raise ShapeError(f"z has shape {tuple(z.shape)}, expected {tuple(u.shape)}")
    A = torch.as_tensor(A, device=u.device)
    if A.dim() != 2 or A.shape[0] != E:
        raise ShapeError(f"A must be (E, N) = ({E}, N), got {tuple(A.shape)}")
    N = A.shape[1]
    for name, t in (("B", B), ("C", C_)):
        if t.shape != (Bt, L, N):
            raise ShapeError(f"{name} has shape {tuple(t.shape)}, expected {(Bt, L, N)}")
    if u.dtype not in (torch.float32, torch.bfloat16):
        u = u.to(torch.float32)
    io = u.dtype
    delta = delta.to(io)
    if z is not None:
        z = z.to(io)
    bc = B.dtype if B.dtype in (torch.float32, torch.bfloat16) else torch.float32
    if bc != io and not (io == torch.bfloat16 and bc == torch.float32):
        bc = io
    B = B.to(bc)
    C_ = C_.to(bc)
    M = select_tile_len(L) if window in (None, "auto") else int(window)
    if M < 1:
        raise ShapeError(f"tile length must be >= 1, got {M}")
    A = A.to(torch.float32).contiguous()
    D = _vec("D", D, E, u.device)
    delta_bias = _vec("delta_bias", delta_bias, E, u.device)
    return u, delta, A, B, C_, D, z, delta_bias, M, (Bt, L, E, N)


def _fwd_args(u, delta, A, B, C_, D, z, delta_bias, M, dims, flags, out, last_state, seg_hint=0):
    Bt, L, E, N = dims
    a = _lib.ScanFwdArgs()
    a.batch, a.seqlen, a.dim, a.dstate, a.window = Bt, L, E, N, M
    a.io_dtype = _DT[u.dtype]
    a.bc_dtype = _DT[B.dtype]
    a.flags = flags
    a.seg_hint = seg_hint
    a.u, a.u_stride = _ptr(u), _strides(u)
    a.delta, a.delta_stride = _ptr(delta), _strides(delta)
    a.A = _ptr(A)
    a.B, a.B_stride = _ptr(B), _strides(B)
    a.C, a.C_stride = _ptr(C_), _strides(C_)
    a.D = _ptr(D)
    a.delta_bias = _ptr(delta_bias)
    a.z, a.z_stride = _ptr(z), _strides(z)
    a.out, a.out_stride = _ptr(out), _strides(out)
    a.last_state = _ptr(last_state)
    a.checkpoints = None
    a.ckpt_len = 0
    return a


def _flags(delta_softplus, reverse, lb, mode):
    if mode not in ("exp", "linear"):
        raise ShapeError(f"unknown discretize mode {mode!r}")  # block.py:88-89
    f = 0
    if delta_softplus:
        f |= FLAG_SOFTPLUS
    if reverse:
        f |= FLAG_REVERSE
    if lb:
        f |= FLAG_LB
    if mode == "linear":
        f |= FLAG_LINEAR
    return f


def lbm_selective_scan_fwd(u, delta, A, B, C, D=None, z=None, delta_bias=None,
                           delta_softplus=True, window=None, reverse=False,
                           return_last_state=False, lb=True, discretize_mode="exp",
                           out=None, seg_hint=0, save_checkpoints=False, accumulate=False,
                           tma=True):
    """Forward launch (no autograd).  Returns ``out`` or ``(out, last_state)``;
    with ``save_checkpoints`` a trailing fp32 checkpoint buffer for
    :func:`lbm_selective_scan_bwd` is appended (None for shapes on the generic
    path, N > 16 or a window > 16, whose backward recomputes the states).
    ``tma=False`` stages the inputs with cp.async rows instead of TMA tensor copies
    (testing: the results are bitwise equal)."""
    u, delta, A, B, C, D, z, delta_bias, M, dims = _prepare(u, delta, A, B, C, D, z, delta_bias, window)
    Bt, L, E, N = dims
    if out is None:
        out = torch.empty((Bt, L, E), dtype=u.dtype, device=u.device)
    last = torch.empty((Bt, E, N), dtype=torch.float32, device=u.device) if return_last_state else None
    flags = _flags(delta_softplus, reverse, lb, discretize_mode)
    if accumulate:
        flags |= _lib.FLAG_ACCUM
    if not tma:
        flags |= _lib.FLAG_NO_TMA
    args = _fwd_args(u, delta, A, B, C, D, z, delta_bias, M, dims, flags, out, last, seg_hint)
    L_ = _lib.lib()
    ck = None
    if save_checkpoints:
        # None for the generic path (N > 16 or a window > 16), whose backward recomputes
        nck = L_.lbs_scan_ckpt_bytes(ctypes.byref(args))
        if nck:
            ck = torch.empty(nck // 4, dtype=torch.float32, device=u.device)
            args.checkpoints = ck.data_ptr()
            args.ckpt_len = L_.lbs_scan_ckpt_len(L, M)
    nws = L_.lbs_scan_fwd_workspace_bytes(ctypes.byref(args))
    ws = torch.empty(max(nws, 1), dtype=torch.uint8, device=u.device) if nws else None
    rc = L_.lbs_scan_fwd(ctypes.byref(args), _ptr(ws), nws, _stream())
    _lib.check(rc, "lbm_selective_scan")
    res = (out, last) if return_last_state else (out,)
    if save_checkpoints:
        res = res + (ck,)
    return res if len(res) > 1 else res[0]


def lbm_selective_scan_bwd(dout, u, delta, A, B, C, D=None, z=None, delta_bias=None,
                           delta_softplus=True, window=None, reverse=False, lb=True,
                           discretize_mode="exp", checkpoints=None, seg_hint=0, grads=None):
    """Backward launch (lbs_scan_bwd): the adjoint of :func:`lbm_selective_scan_fwd`
    (autodiff.lbm_scan_grad, autodiff.py:192-195, chained through
    block._discretize_backward, block.py:106-129, and the gate).

    Returns a dict ``du, ddelta, dz`` (io dtype, ``dz`` None without ``z``),
    ``dA`` (E, N), ``dD``, ``ddelta_bias`` (E,) and ``dB``, ``dC`` (B, L, N), all
    fp32.  ``checkpoints`` is the buffer from ``save_checkpoints=True`` (else the
    states are recomputed by a checkpoint-only forward sweep).  ``seg_hint`` > 0
    forces that many sequence segments (testing; 0 = the launch plan's choice).
    ``grads``: optional dict of preallocated outputs by the same keys (any subset; views
    with any strides, e.g. column blocks of a fused projection's gradient); a given
    ``dA`` / ``dD`` / ``ddelta_bias`` is accumulated into (+=), as by the C ABI."""
    u, delta, A, B, C, D, z, delta_bias, M, dims = _prepare(u, delta, A, B, C, D, z, delta_bias, window)
    Bt, L, E, N = dims
    _need_cuda("dout", dout)
    if dout.shape != u.shape:
        raise ShapeError(f"dout has shape {tuple(dout.shape)}, expected {tuple(u.shape)}")
    dout = dout.to(u.dtype)
    flags = _flags(delta_softplus, reverse, lb, discretize_mode)
    dev = u.device
    a = _lib.ScanBwdArgs()
    a.fwd = _fwd_args(u, delta, A, B, C, D, z, delta_bias, M, dims, flags, None, None, seg_hint)
    L_ = _lib.lib()
    if checkpoints is not None:
        a.fwd.checkpoints = checkpoints.data_ptr()
        a.fwd.ckpt_len = L_.lbs_scan_ckpt_len(L, M)
    g = grads or {}

    def out(key, shape, dtype, make):
        t = g.get(key)
        if t is None:
            return make(shape, dtype=dtype, device=dev)
        if tuple(t.shape) != tuple(shape) or t.dtype != dtype or not t.is_cuda:
            raise ShapeError(f"grads[{key!r}] must be a CUDA {dtype} tensor of shape {tuple(shape)}")
        return t

    du = out("du", (Bt, L, E), u.dtype, torch.empty)
    ddelta = out("ddelta", (Bt, L, E), u.dtype, torch.empty)
    dz = out("dz", (Bt, L, E), u.dtype, torch.empty) if z is not None else None
    dA = out("dA", (E, N), torch.float32, torch.zeros)
    dD = out("dD", (E,), torch.float32, torch.zeros) if D is not None else None
    dbias = out("ddelta_bias", (E,), torch.float32, torch.zeros) if delta_bias is not None else None
    dB = out("dB", (Bt, L, N), torch.float32, torch.empty)
    dC = out("dC", (Bt, L, N), torch.float32, torch.empty)
    a.dout, a.dout_stride = _ptr(dout), _strides(dout)
    a.du, a.du_stride = _ptr(du), _strides(du)
    a.ddelta, a.ddelta_stride = _ptr(ddelta), _strides(ddelta)
    a.dz, a.dz_stride = _ptr(dz), _strides(dz)
    a.dA, a.dD, a.ddelta_bias = _ptr(dA), _ptr(dD), _ptr(dbias)
    a.dB, a.dB_stride = _ptr(dB), _strides(dB)
    a.dC, a.dC_stride = _ptr(dC), _strides(dC)
    nws = L_.lbs_scan_bwd_workspace_bytes(ctypes.byref(a))
    ws = torch.empty(max(nws, 1), dtype=torch.uint8, device=dev)
    rc = L_.lbs_scan_bwd(ctypes.byref(a), _ptr(ws), nws, _stream())
    _lib.check(rc, "lbm_selective_scan_bwd")
    return dict(du=du, ddelta=ddelta, dA=dA, dB=dB, dC=dC, dD=dD, dz=dz, ddelta_bias=dbias)


def _needs_grad(*ts):
    return torch.is_grad_enabled() and any(
        t is not None and isinstance(t, torch.Tensor) and t.requires_grad for t in ts)


def lbm_selective_scan(u, delta, A, B, C, D=None, z=None, delta_bias=None,
                       delta_softplus=True, window=None, reverse=False,
                       return_last_state=False, discretize_mode="exp", lb=True):
    """The north-star fused operator (LB scan).  Differentiable when any input
    requires grad (backward = lbs_scan_bwd, one fused launch + a reduction)."""
    if _needs_grad(u, delta, A, B, C, D, z, delta_bias):
        if return_last_state:
            raise NotImplementedError("return_last_state is not differentiable (the reference's "
                                      "h_final has no adjoint either, autodiff.py:192-195)")
        from .autograd import LbmSelectiveScanFn
        return LbmSelectiveScanFn.apply(u, delta, A, B, C, D, z, delta_bias, delta_softplus,
                                        window, reverse, lb, discretize_mode)
    return lbm_selective_scan_fwd(u, delta, A, B, C, D, z, delta_bias, delta_softplus, window,
                                  reverse, return_last_state, lb, discretize_mode)


def selective_scan(u, delta, A, B, C, D=None, z=None, delta_bias=None, delta_softplus=True,
                   reverse=False, return_last_state=False):
    """Plain unidirectional selective scan (engine.forward_scan_par semantics,
    engine.py:294) — the same kernels with the LB pass compiled out."""
    # the window is irrelevant without the LB pass; 8-step tiles keep the
    # forward-only kernel on its fast full-tile path
    return lbm_selective_scan(u, delta, A, B, C, D, z, delta_bias, delta_softplus, 8, reverse,
                              return_last_state, "exp", lb=False)


def global_bidir_selective_scan(u, delta, A, B, C, D=None, z=None, delta_bias=None, *,
                                delta_b=None, A_b=None, B_b=None, C_b=None, D_b=None,
                                delta_bias_b=None, delta_softplus=True, return_last_state=False):
    """Vim-style globally bi-directional selective scan — the baseline LBMamba is
    measured against (engine.global_bidir_par, engine.py:305-327; oracle.py:71-77):
    a full forward sweep with (delta, A, B, C, D, delta_bias) plus a full
    right-to-left sweep (flip-on-load) with the ``*_b`` parameters, summed, gated
    by silu(z).  Two launches of the forward-only kernel, the second accumulating
    into the first's output; ``last_state`` is h_f + h_b like the reference.
    Differentiable when an input requires grad (autodiff.global_bidir_grad,
    autodiff.py:204-236): the sum of two autograd scans, each backward one fused
    lbs_scan_bwd launch."""
    pb = dict(delta=delta if delta_b is None else delta_b, A=A if A_b is None else A_b,
              B=B if B_b is None else B_b, C=C if C_b is None else C_b, D=D if D_b is None else D_b,
              delta_bias=delta_bias if delta_bias_b is None else delta_bias_b)
    if _needs_grad(u, delta, A, B, C, D, z, delta_bias, *pb.values()):
        if return_last_state:
            raise NotImplementedError("return_last_state is not differentiable")
        yf = lbm_selective_scan(u, delta, A, B, C, D, z, delta_bias, delta_softplus, 8, False, lb=False)
        yb = lbm_selective_scan(u, pb["delta"], pb["A"], pb["B"], pb["C"], pb["D"], z, pb["delta_bias"],
                                delta_softplus, 8, True, lb=False)
        return yf + yb
    out, hf = lbm_selective_scan_fwd(u, delta, A, B, C, D, z, delta_bias, delta_softplus, 8, False,
                                     True, False)
    _, hb = lbm_selective_scan_fwd(u, pb["delta"], pb["A"], pb["B"], pb["C"], pb["D"], z, pb["delta_bias"],
                                   delta_softplus, 8, True, True, False, out=out, accumulate=True)
    return (out, hf + hb) if return_last_state else out
