"""MambaMIL-style whole-slide bag classifier on the channel-sharded LB scan
(BASELINE configs[4]) — cfg 5 as an end-to-end
workload instead of a bare op.

One bag = L instance features X (L, d_in).  Forward, with the scan's E channels
partitioned over the ranks of ``group`` (rank r owns the block [lo, hi)):

  1. H  = relu(X W_fc + b_fc)                 (L, D)   replicated (contracts over d_in)
  2. Hn = rms_norm(H)                                   replicated
  3. x_r, z_r = Hn W_in[:, block]             (L, E_r) local column block, no exchange
  4. u_r = silu(causal_conv1d(x_r))                     local (channels independent)
  5. P_r = u_r W_xproj[block, :]              (L, R+2N) partial over this rank's channels
     P   = all_reduce_sum(P_r)                          <- exchange 1 (x_proj contracts over E)
  6. dt, B, C = split(P);  delta_r = dt W_dt[:, block]  local
  7. y_r = LB scan(u_r, delta_r, A_r, B, C, D_r, z_r, dt_bias_r)  local
  8. m_r = mean_L(y_r)                         (E_r,)
     m   = all_gather(m_r)                     (E,)     <- exchange 2 (E floats per rank)
  9. o = m W_out + mean_L(H);  logits = o W_cls + b_cls
     (mean pooling commutes with the out projection and the residual, so the
     (L, D) block output is never formed or exchanged)

The two collectives move (L, R + 2N) and (E,) values — for L = 100 k, R = 32,
N = 16: 25.6 MB fp32 once per layer, against 205 MB for gathering the scan
output.  ``scan_fn`` / ``conv_fn`` / ``norm_fn`` default to the fused CUDA
kernels; they are parameters only so the partitioning logic can run in
world-size-2 gloo tests on a CPU-only machine.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.distributed as dist

from .errors import ShapeError
from .sharding import shard_range
from .tiling import select_tile_len

RMS_EPS = 1e-6


@dataclass
class MILConfig:
    d_in: int = 1024        # instance feature width (e.g. a ResNet-50 trunc. / UNI embedding)
    dim: int = 512          # D: the scan's channel count (BASELINE configs[4] "D=512")
    state_dim: int = 16     # N
    dt_rank: int = 32       # R = ceil(D / 16), Mamba's low-rank delta projection
    conv_width: int = 4
    num_classes: int = 2
    tile_len: int | None = None  # LB window; None -> select_tile_len(L)

    def __post_init__(self):
        if min(self.d_in, self.dim, self.state_dim, self.dt_rank, self.conv_width, self.num_classes) < 1:
            raise ShapeError("all MIL dimensions must be >= 1")


def init_mil_params(cfg: MILConfig, seed: int = 0, device="cpu") -> dict:
    """fp32 parameters (Mamba-style init: A = -(1..N), dt in [1e-3, 1e-1], D = 1)."""
    g = torch.Generator().manual_seed(seed)
    D, E, N, R = cfg.dim, cfg.dim, cfg.state_dim, cfg.dt_rank

    def lin(i, o):
        return torch.randn(i, o, generator=g) / math.sqrt(i)

    dt = torch.exp(torch.rand(E, generator=g) * (math.log(1e-1) - math.log(1e-3)) + math.log(1e-3))
    p = {
        "w_fc": lin(cfg.d_in, D), "b_fc": torch.zeros(D),
        "norm_scale": torch.ones(D),
        "w_in": lin(D, 2 * E),
        "conv_w": torch.randn(E, cfg.conv_width, generator=g) / math.sqrt(cfg.conv_width),
        "conv_b": torch.zeros(E),
        "w_xproj": lin(E, R + 2 * N),
        "w_dt": lin(R, E),
        "dt_bias": dt + torch.log(-torch.expm1(-dt)),  # softplus^-1(dt)
        "A": -torch.arange(1, N + 1, dtype=torch.float32).repeat(E, 1),
        "D": torch.ones(E),
        "w_out": lin(E, D),
        "w_cls": lin(D, cfg.num_classes), "b_cls": torch.zeros(cfg.num_classes),
    }
    return {k: v.to(device) for k, v in p.items()}


def _default_scan(**kw):
    from .scan import lbm_selective_scan
    return lbm_selective_scan(**kw)


def _default_conv(x, w, b):
    from .conv import causal_conv1d_silu_fwd
    return causal_conv1d_silu_fwd(x, w, b)


def _default_norm(x, scale):
    from .norm import rms_norm
    return rms_norm(x, scale, eps=RMS_EPS)


def _col_mean(t: torch.Tensor, acc) -> torch.Tensor:
    """Mean over rows of an (L, E) tensor as a GEMV (cuBLAS, fp32 accumulation and an
    fp32 result for 16-bit inputs): torch's strided column reduction over the (L, E)
    activations cost ~4x the HBM time of reading them once."""
    ones = torch.ones(1, t.shape[0], dtype=t.dtype, device=t.device)
    if t.is_cuda and t.dtype in (torch.bfloat16, torch.float16):
        s = torch.mm(ones, t, out_dtype=torch.float32)
    else:
        s = (ones @ t).to(acc)
    return s[0].to(acc) / t.shape[0]


class MILBag:
    """Bag classifier; ``forward(X)`` -> logits (num_classes,) on every rank.

    ``X`` is (L, d_in) (or (1, L, d_in)), replicated on the ranks.  ``dtype``
    is the activation dtype of the projections / conv / scan I/O (bf16 on the
    GPU); the scan state is always fp32.
    """

    def __init__(self, cfg: MILConfig, params: dict, *, group=None, dtype=torch.float32,
                 scan_fn=None, conv_fn=None, norm_fn=None):
        self.cfg, self.group, self.dtype = cfg, group, dtype
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.lo, self.hi = shard_range(cfg.dim, self.world, self.rank)
        self.sizes = [shard_range(cfg.dim, self.world, r)[1] - shard_range(cfg.dim, self.world, r)[0]
                      for r in range(self.world)]
        self.scan_fn = scan_fn or _default_scan
        self.conv_fn = conv_fn or _default_conv
        self.norm_fn = norm_fn or _default_norm
        E, lo, hi = cfg.dim, self.lo, self.hi
        # fp32 (fp64 for an fp64 model) for the x_proj partials, scan parameters and the pooled head
        self.acc = torch.float64 if dtype == torch.float64 else torch.float32
        a = lambda t: t.to(dtype).contiguous()     # noqa: E731  (projection weights in the activation dtype)
        f = lambda t: t.to(self.acc).contiguous()  # noqa: E731
        self.w_fc, self.b_fc = a(params["w_fc"]), a(params["b_fc"])
        self.norm_scale = f(params["norm_scale"])
        # this rank's x and z column blocks of the in-projection, fused into one GEMM
        self.w_in = a(torch.cat([params["w_in"][:, lo:hi], params["w_in"][:, E + lo:E + hi]], dim=1))
        self.conv_w, self.conv_b = f(params["conv_w"][lo:hi]), f(params["conv_b"][lo:hi])
        self.w_xproj = a(params["w_xproj"][lo:hi])
        self.w_dt = a(params["w_dt"][:, lo:hi])
        self.dt_bias, self.A, self.Dp = f(params["dt_bias"][lo:hi]), f(params["A"][lo:hi]), f(params["D"][lo:hi])
        self.w_out = f(params["w_out"])
        self.w_cls, self.b_cls = f(params["w_cls"]), f(params["b_cls"])

    def forward(self, X: torch.Tensor) -> torch.Tensor:
        cfg = self.cfg
        if X.dim() == 3:
            if X.shape[0] != 1:
                raise ShapeError("one bag per call (batch 1, as MambaMIL)")
            X = X[0]
        if X.dim() != 2 or X.shape[1] != cfg.d_in:
            raise ShapeError(f"bag must be (L, {cfg.d_in}), got {tuple(X.shape)}")
        L, E_r, R, N = X.shape[0], self.hi - self.lo, cfg.dt_rank, cfg.state_dim
        X = X.to(self.dtype)
        if X.is_cuda:  # bias + ReLU in the cuBLASLt epilogue (one kernel)
            H = torch._addmm_activation(self.b_fc, X, self.w_fc)                    # (L, D)
        else:
            H = torch.relu(torch.addmm(self.b_fc, X, self.w_fc))
        Hn = self.norm_fn(H, self.norm_scale)
        xz = Hn @ self.w_in                                                         # (L, 2 E_r)
        x, z = xz[:, :E_r], xz[:, E_r:]
        u = self.conv_fn(x[None], self.conv_w, self.conv_b)                         # (1, L, E_r)
        P = (u[0] @ self.w_xproj).to(self.acc)                                           # (L, R + 2N) partial
        if self.world > 1:
            dist.all_reduce(P, group=self.group)                                    # exchange 1
        dt, Bm, Cm = P[:, :R], P[:, R:R + N], P[:, R + N:]
        delta = (dt.to(self.dtype) @ self.w_dt)[None]                               # (1, L, E_r)
        window = cfg.tile_len or select_tile_len(L)
        y = self.scan_fn(u=u, delta=delta, A=self.A, B=Bm[None].to(self.dtype).contiguous(),
                         C=Cm[None].to(self.dtype).contiguous(), D=self.Dp, z=z[None], delta_bias=self.dt_bias,
                         window=window, reverse=False, delta_softplus=True)          # (1, L, E_r)
        m = _col_mean(y[0], self.acc)                                               # (E_r,)
        if self.world > 1:                                                          # exchange 2
            smax = max(self.sizes)
            buf = torch.zeros(self.world * smax, dtype=m.dtype, device=m.device)
            dist.all_gather_into_tensor(buf, torch.nn.functional.pad(m, (0, smax - E_r)), group=self.group)
            m = torch.cat([buf[r * smax:r * smax + s] for r, s in enumerate(self.sizes)])
        o = m @ self.w_out + _col_mean(H, self.acc)                                 # pooled block output
        return o @ self.w_cls + self.b_cls

    __call__ = forward
