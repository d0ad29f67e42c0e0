"""LBVim backbone on the B200 path — the caller of the fused LB scan.

Mirrors the reference model (model.py:25-325) and block (block.py:141-190):

    patchify -> linear -> [class token] -> +pos -> U x block -> head
    block: RMSNorm -> x = xn W_x, z = xn W_z -> causal conv1d + SiLU ->
           [delta | B | C] = xs [W_delta | W_b | W_c] -> LB scan (+D skip,
           x SiLU(z) gate) -> out = yg W_out + residual -> (sequence reversal)

B200 design:
  * the per-block sequence reversal (block.py:180-181, model.py:216-218) is
    never materialised: tokens stay in input order and block i runs its conv
    and scan in direction (-1)^i by flip-on-load (LBS_FLAG_REVERSE), which is
    exactly equivalent;
  * W_delta, W_b, W_c are one fused GEMM; delta, B and C are strided column
    views of its output, and z is a strided view of the in-projection output,
    passed straight to the scan kernel (no copies);
  * GEMMs stay on stock torch/cuBLAS (north star); conv+SiLU and the scan
    are the hand-written sm_100a kernels;
  * the whole forward can be captured in one CUDA graph (``LBVim.graphed``).

Weights follow the reference's shapes and initialisation (block.py:52-73,
model.py:118-148) including the full-rank E x E delta projection.  The
reference's conv tap order is kept: kernel[e, q] multiplies x[l - q].
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch
import torch.nn.functional as F

from .block_train import block_forward_fused
from .conv import causal_conv1d_silu, causal_conv1d_silu_fwd
from .errors import ShapeError
from .norm import rms_norm, rms_norm_train
from .scan import lbm_selective_scan, lbm_selective_scan_fwd
from .tiling import select_tile_len

RMS_EPS = 1e-6  # nn.py:13
CLASS_TOKENS = {"none": 0, "head": 1, "middle": 1, "double": 2}  # model.py:22


@dataclass
class ModelConfig:
    """model.py:25-115 (same fields and defaults)."""

    image_size: int = 32
    patch_size: int = 4
    in_channels: int = 1
    embed_dim: int = 64
    inner_dim: int = 128
    state_dim: int = 16
    depth: int = 4
    tile_len: int | None = None
    head: str = "gap"
    map_heads: int = 4
    class_token: str = "none"
    num_classes: int = 2
    conv_width: int = 4
    reverse_between_blocks: bool = True
    unreverse_output: bool = True
    discretize_mode: str = "exp"
    scan_variant: str = "lbm"

    def __post_init__(self):
        if self.image_size % self.patch_size:
            raise ShapeError(f"image size {self.image_size} not divisible by patch size {self.patch_size}")
        if self.depth < 1:
            raise ShapeError("depth must be >= 1")
        if self.head not in ("gap", "map"):
            raise ShapeError(f"unknown head {self.head!r}")
        if self.class_token not in CLASS_TOKENS:
            raise ShapeError(f"unknown class token mode {self.class_token!r}")
        if self.scan_variant not in ("forward", "lbm"):
            raise ShapeError(f"unsupported scan variant {self.scan_variant!r}")

    @property
    def num_patches(self) -> int:
        return (self.image_size // self.patch_size) ** 2

    @property
    def seq_len(self) -> int:
        return self.num_patches + CLASS_TOKENS[self.class_token]

    @property
    def resolved_tile_len(self) -> int:
        return select_tile_len(self.seq_len) if self.tile_len in (None, "auto") else int(self.tile_len)


def lbvim_tiny(**kw) -> ModelConfig:
    """LBVim-Ti at 224^2, patch 16 (BASELINE configs[1]): D=192, E=384, N=16,
    24 layers, L = 196 patches + 1 middle class token = 197."""
    base = dict(image_size=224, patch_size=16, in_channels=3, embed_dim=192, inner_dim=384,
                state_dim=16, depth=24, head="gap", class_token="middle", num_classes=1000)
    base.update(kw)
    return ModelConfig(**base)


def lbvim_small(**kw) -> ModelConfig:
    """LBVim-S: D=384, E=768 (BASELINE configs[2], [3])."""
    base = dict(image_size=224, patch_size=16, in_channels=3, embed_dim=384, inner_dim=768,
                state_dim=16, depth=24, head="gap", class_token="middle", num_classes=1000)
    base.update(kw)
    return ModelConfig(**base)


BLOCK_FIELDS = ("norm_scale", "w_x", "w_z", "conv_kernel", "w_b", "w_c",
                "w_delta", "delta_bias", "a_log", "d_param", "w_out")


def init_params(cfg: ModelConfig, seed: int = 0, device="cuda", dtype=torch.float32) -> dict:
    """Random init with the reference's distributions (block.py:52-73,
    model.py:118-148), drawn from a seeded torch generator on the device."""
    g = torch.Generator(device=device).manual_seed(seed)
    D, E, N, k = cfg.embed_dim, cfg.inner_dim, cfg.state_dim, cfg.conv_width
    patch_in = cfg.patch_size ** 2 * cfg.in_channels

    def randn(*s, scale=1.0):
        return torch.randn(*s, generator=g, device=device, dtype=torch.float32) * scale

    def unif(lo, hi, *s):
        return torch.empty(*s, device=device, dtype=torch.float32).uniform_(lo, hi, generator=g)

    p = {
        "patch_w": randn(patch_in, D, scale=1 / math.sqrt(patch_in)),
        "patch_b": torch.zeros(D, device=device),
        "pos": randn(cfg.seq_len, D, scale=0.02),
    }
    if CLASS_TOKENS[cfg.class_token]:
        p["cls"] = randn(CLASS_TOKENS[cfg.class_token], D, scale=0.02)
    for i in range(cfg.depth):
        dt = torch.exp(unif(math.log(1e-3), math.log(1e-1), E))
        blk = {
            "norm_scale": torch.ones(D, device=device),
            "w_x": randn(D, E, scale=1 / math.sqrt(D)),
            "w_z": randn(D, E, scale=1 / math.sqrt(D)),
            "conv_kernel": unif(-1, 1, E, k) / math.sqrt(k),
            "w_b": randn(E, N, scale=1 / math.sqrt(E)),
            "w_c": randn(E, N, scale=1 / math.sqrt(E)),
            "w_delta": randn(E, E, scale=0.1 / math.sqrt(E)),
            "delta_bias": dt + torch.log(-torch.expm1(-dt)),
            "a_log": torch.log(torch.arange(1, N + 1, device=device, dtype=torch.float32)).repeat(E, 1),
            "d_param": torch.ones(E, device=device),
            "w_out": randn(E, D, scale=1 / math.sqrt(E)),
        }
        for f, v in blk.items():
            p[f"blocks.{i}.{f}"] = v
    if cfg.head == "map":
        p["head.q"] = randn(D, scale=1 / math.sqrt(D))
        p["head.wk"] = randn(D, D, scale=1 / math.sqrt(D))
        p["head.wv"] = randn(D, D, scale=1 / math.sqrt(D))
    hidden = 4 * D
    p["head.mlp_w1"] = randn(D, hidden, scale=1 / math.sqrt(D))
    p["head.mlp_b1"] = torch.zeros(hidden, device=device)
    p["head.mlp_w2"] = randn(hidden, cfg.num_classes, scale=1 / math.sqrt(hidden))
    p["head.mlp_b2"] = torch.zeros(cfg.num_classes, device=device)
    return {k: v.to(dtype) for k, v in p.items()}


def _pad_cols(w: torch.Tensor, mult: int) -> torch.Tensor:
    """Zero-pad the columns of a (K, N) weight to a multiple of ``mult``."""
    pad = (-w.shape[1]) % mult
    return torch.nn.functional.pad(w, (0, pad)) if pad else w


class LBVim:
    """Inference-time LBVim on the fused kernels.  ``dtype`` is the activation
    / weight dtype (bf16 for throughput, fp32 for parity); scan state is fp32."""

    def __init__(self, cfg: ModelConfig, params: dict, dtype=torch.bfloat16):
        self.cfg = cfg
        self.dtype = dtype
        D, E, N = cfg.embed_dim, cfg.inner_dim, cfg.state_dim
        self.M = cfg.resolved_tile_len
        cast = lambda t: t.to(dtype).contiguous()
        f32 = lambda t: t.to(torch.float32).contiguous()
        self.patch_w, self.patch_b = cast(params["patch_w"]), cast(params["patch_b"])
        self.pos = cast(params["pos"])
        self.cls = cast(params["cls"]) if "cls" in params else None
        self.blocks = []
        for i in range(cfg.depth):
            w = {f: params[f"blocks.{i}.{f}"] for f in BLOCK_FIELDS}
            self.blocks.append(dict(
                norm_scale=cast(w["norm_scale"]), norm_f32=f32(w["norm_scale"]),
                w_in=cast(torch.cat([w["w_x"], w["w_z"]], dim=1)),                  # (D, 2E)
                conv_kernel=f32(w["conv_kernel"]),                                    # (E, k)
                # (E, E+2N) padded to a multiple of 64 columns and stored transposed:
                # cuBLAS runs the x-projection ~15 % faster on that shape (N=448 "NT"
                # vs N=416 "NN" at the LBVim-Ti shape, tools/gemmbench.py); the scan
                # reads delta / B / C as strided column views either way
                w_xpT=_pad_cols(cast(torch.cat([w["w_delta"], w["w_b"], w["w_c"]], dim=1)), 64).t().contiguous(),
                A=f32(-torch.exp(w["a_log"].float())),
                D=f32(w["d_param"]), delta_bias=f32(w["delta_bias"]),
                w_outT=cast(w["w_out"]).t().contiguous(),  # "NT" out-projection (~4 % faster)
            ))
        self.head = {k: cast(v) for k, v in params.items() if k.startswith("head.")}
        # the head runs in fp32 (model.py:238-325); its weights are cast once here, not per forward
        self.head32 = {k: v.float().contiguous() for k, v in self.head.items()}
        self._graph = None

    # -- pieces -----------------------------------------------------------------
    def patch_embed(self, images):
        """model.py:190-201; images (B, H, W, C) channel-last like the reference."""
        cfg = self.cfg
        B, H, W, C = images.shape
        if H != cfg.image_size or W != cfg.image_size or C != cfg.in_channels:
            raise ShapeError(f"image shape {tuple(images.shape[1:])} does not match config")
        p, g = cfg.patch_size, cfg.image_size // cfg.patch_size
        # (a channels_last stride-p cuDNN convolution instead of this patchify copy measured
        # 12x slower: cuDNN converted to NCHW and ran an SIMT kernel)
        xi = images.to(self.dtype).reshape(B * g, p, g, p * C)  # (b gi) pi gj (pj c)
        if (p * C * xi.element_size()) % 8 == 0:
            # move each patch row segment as 8-byte words: the gi/pj transpose copy runs
            # 2.3x faster than the element-wise permute (tools/patchbench.py)
            x = xi.view(torch.int64).transpose(1, 2).contiguous().view(xi.dtype).reshape(B, g * g, p * p * C)
        else:
            x = xi.transpose(1, 2).reshape(B, g * g, p * p * C)
        tok = torch.addmm(self.patch_b, x.reshape(-1, x.shape[-1]), self.patch_w).reshape(B, g * g, -1)
        ct = cfg.class_token
        D = tok.shape[-1]
        if ct == "none":
            return (tok + self.pos).contiguous()
        # class token(s) and the position add written straight into the token buffer
        L = self.pos.shape[0]
        out = torch.empty(B, L, D, dtype=tok.dtype, device=tok.device)
        pos = self.pos  # (L, D)
        if ct == "head":
            spans = [(1, 0, g * g)]
            cls_at = [(0, 0)]
        elif ct == "middle":
            mid = (g * g) // 2
            spans = [(0, 0, mid), (mid + 1, mid, g * g)]
            cls_at = [(mid, 0)]
        else:
            spans = [(1, 0, g * g)]
            cls_at = [(0, 0), (L - 1, 1)]
        for dst, lo, hi in spans:
            torch.add(tok[:, lo:hi], pos[dst:dst + hi - lo], out=out[:, dst:dst + hi - lo])
        for dst, k in cls_at:
            torch.add(self.cls[k].expand(B, D), pos[dst], out=out[:, dst])
        return out

    def block(self, T, w, reverse: bool):
        """block.py:158-190 with the output reversal replaced by direction."""
        B, L, D = T.shape
        E, N = w["A"].shape
        xn = rms_norm(T, w["norm_f32"], eps=RMS_EPS)
        xz = (xn.reshape(-1, D) @ w["w_in"]).reshape(B, L, 2 * E)
        x, z = xz[..., :E], xz[..., E:]
        xs = causal_conv1d_silu_fwd(x, w["conv_kernel"], reverse=reverse)
        proj = (xs.reshape(-1, E) @ w["w_xpT"].t()).reshape(B, L, -1)
        yg = lbm_selective_scan_fwd(
            xs, proj[..., :E], w["A"], proj[..., E:E + N], proj[..., E + N:E + 2 * N], D=w["D"], z=z,
            delta_bias=w["delta_bias"], window=self.M, reverse=reverse,
            lb=self.cfg.scan_variant == "lbm", discretize_mode=self.cfg.discretize_mode)
        return torch.addmm(T.reshape(-1, D), yg.reshape(-1, E), w["w_outT"].t()).reshape(B, L, D)

    def run_blocks(self, tok):
        """model.py:204-222.  Returns tokens in original order; the number of
        reference reversals applied is tracked only for the head's index map."""
        rev = self.cfg.reverse_between_blocks
        for i, w in enumerate(self.blocks):
            tok = self.block(tok, w, reverse=rev and (i % 2 == 1))
        return tok

    def head_forward(self, tok):
        """model.py:238-325 heads.  Tokens arrive in original order here.  The
        reference reads class tokens at p or L-1-p depending on how many
        reversals are left (model.py:225-229,307-312) — both are original
        position p — and its GAP / MAP pools are order-invariant."""
        pooled = pool_tokens(tok.float(), self.cfg, self.head32)
        h1 = F.gelu(pooled @ self.head32["head.mlp_w1"] + self.head32["head.mlp_b1"],
                    approximate="tanh")
        return h1 @ self.head32["head.mlp_w2"] + self.head32["head.mlp_b2"]

    @torch.no_grad()
    def forward(self, images):
        return self.head_forward(self.run_blocks(self.patch_embed(images)))

    __call__ = forward

    # -- CUDA graph ---------------------------------------------------------------
    @torch.no_grad()
    def graphed(self, example_images, streams: int = 1):
        """Capture forward() for a fixed input shape; returns a callable that
        copies new images into the static input and replays the graph.

        ``streams`` > 1 splits the batch into that many slices whose forwards are
        captured on separate streams (forked from and joined to the capture
        stream), so the graph can run one slice's latency-bound scan next to
        another slice's tensor-core GEMMs and HBM-bound conv / RMSNorm."""
        static_in = example_images.clone()
        B = static_in.shape[0]
        k = max(1, min(int(streams), B))
        cuts = [B * i // k for i in range(k + 1)]
        side = [torch.cuda.Stream() for _ in range(k)]

        def fwd_split(x):
            if k == 1:
                return self.forward(x)
            main = torch.cuda.current_stream()
            outs = []
            for i, st in enumerate(side):
                st.wait_stream(main)
                with torch.cuda.stream(st):
                    outs.append(self.forward(x[cuts[i]:cuts[i + 1]]))
            for st in side:
                main.wait_stream(st)
            return torch.cat(outs, 0)

        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(2):
                fwd_split(static_in)
        torch.cuda.current_stream().wait_stream(s)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            static_out = fwd_split(static_in)

        def run(images=None):
            if images is not None:
                static_in.copy_(images, non_blocking=True)
            graph.replay()
            return static_out

        run.graph, run.static_in, run.static_out = graph, static_in, static_out
        return run


# ---------------------------------------------------------------------------
# training path (autograd through the fused kernels)


def pool_tokens(tok, cfg: ModelConfig, head: dict):
    """Head pooling of model.py:238-325, shared by inference and training.  Tokens
    arrive in original order: class tokens are read at their original position
    (the reference's p / L-1-p index map, model.py:225-229,307-312); GAP is the
    token mean; MAP is single-query multi-head attention pooling over the tokens
    with ``head.wk``, ``head.wv``, ``head.q`` (model.py:260-290).  Differentiable."""
    ct = cfg.class_token
    if ct != "none":
        pos = {"head": [0], "middle": [cfg.num_patches // 2], "double": [0, cfg.seq_len - 1]}[ct]
        return torch.stack([tok[:, q] for q in pos], 1).mean(1)  # graph-capturable
    if cfg.head == "gap":
        return tok.mean(1)
    B, L, D = tok.shape
    nh = cfg.map_heads
    dh = D // nh
    K = (tok @ head["head.wk"]).reshape(B, L, nh, dh)
    V = (tok @ head["head.wv"]).reshape(B, L, nh, dh)
    q = head["head.q"].reshape(nh, dh)
    att = torch.softmax(torch.einsum("blhd,hd->blh", K, q) / math.sqrt(dh), dim=1)
    return torch.einsum("blh,blhd->bhd", att, V).reshape(B, D)



def block_forward_train(T, w: dict, M: int, reverse: bool = False, discretize_mode: str = "exp",
                        lb: bool = True, eps: float = RMS_EPS):
    """Differentiable LBVim block (block.py:158-190 forward, block.py:193-220 backward)
    on the fused kernels: conv1d+SiLU (lbs_causal_conv1d_fwd/bwd) and the LB scan
    (lbs_scan_fwd with checkpoints / lbs_scan_bwd) carry their own adjoints;
    RMSNorm and the projections are stock torch autograd.  ``w`` holds the
    reference's weight names (BLOCK_FIELDS).  As in ``LBVim.block`` the output is
    NOT reversed: ``reverse`` selects the scan direction (flip-on-load)."""
    xn = rms_norm_train(T, w["norm_scale"], eps)  # fused fwd / bwd kernels
    E, N = w["w_x"].shape[1], w["w_b"].shape[1]
    # one GEMM per projection group (x|z and delta|B|C): torch.split's backward
    # concatenates the slice gradients in one kernel, and under autocast the shared
    # input is cast once
    x, z = torch.split(xn @ torch.cat([w["w_x"], w["w_z"]], dim=1), [E, E], dim=-1)
    xs = causal_conv1d_silu(x, w["conv_kernel"], reverse=reverse)
    delta, Bm, Cm = torch.split(xs @ torch.cat([w["w_delta"], w["w_b"], w["w_c"]], dim=1), [E, N, N], dim=-1)
    A = -torch.exp(w["a_log"].float())
    yg = lbm_selective_scan(xs, delta, A, Bm, Cm, D=w["d_param"], z=z, delta_bias=w["delta_bias"],
                            window=M, reverse=reverse, discretize_mode=discretize_mode, lb=lb)
    return yg @ w["w_out"] + T


class LBVimTrainer:
    """LBVim training step on the fused kernels: forward with autograd, cross
    entropy, backward (lbs_scan_bwd / lbs_causal_conv1d_bwd + cuBLAS), AdamW.
    Mirrors autodiff.train_step (autodiff.py:293-314) for the class-token, GAP and
    MAP heads; blocks alternate direction by flip-on-load as in ``LBVim``."""

    def __init__(self, cfg: ModelConfig, params: dict, lr: float = 1e-3, weight_decay: float = 0.05,
                 amp: bool = False, fused_block: bool = True):
        """``amp=True``: bf16 autocast for the projections (tensor cores), so the fused
        scan / conv kernels run their bf16-I/O variants (fp32 state, fp32 master
        weights and optimizer); default fp32 throughout, like the reference.
        ``fused_block``: each block is one autograd node with a hand-written backward
        (block_train.LBVimBlockFn: no gradient concatenations or separate residual
        adds); False = the plain autograd composition ``block_forward_train``."""
        self.cfg = cfg
        self.amp = amp
        self.fused_block = fused_block
        self.M = cfg.resolved_tile_len
        self.params = {k: v.detach().clone().float().requires_grad_(True) for k, v in params.items()}
        # one fused multi-tensor AdamW kernel per step on CUDA (the foreach form is ~3x the launches)
        fused = all(p_.is_cuda for p_ in self.params.values())
        self.opt = torch.optim.AdamW(self.params.values(), lr=lr, weight_decay=weight_decay, fused=fused)

    def forward(self, images):
        cfg, p = self.cfg, self.params
        B = images.shape[0]
        g, ps = cfg.image_size // cfg.patch_size, cfg.patch_size
        x = images.float().reshape(B, g, ps, g, ps, cfg.in_channels).permute(0, 1, 3, 2, 4, 5)
        tok = x.reshape(B, g * g, -1) @ p["patch_w"] + p["patch_b"]
        ct = cfg.class_token
        if ct == "head":
            tok = torch.cat([p["cls"][0].expand(B, 1, -1), tok], 1)
        elif ct == "middle":
            mid = tok.shape[1] // 2
            tok = torch.cat([tok[:, :mid], p["cls"][0].expand(B, 1, -1), tok[:, mid:]], 1)
        elif ct == "double":
            tok = torch.cat([p["cls"][0].expand(B, 1, -1), tok, p["cls"][1].expand(B, 1, -1)], 1)
        tok = tok + p["pos"]
        rev = cfg.reverse_between_blocks
        for i in range(cfg.depth):
            w = {f: p[f"blocks.{i}.{f}"] for f in BLOCK_FIELDS}
            blk = block_forward_fused if self.fused_block else block_forward_train
            tok = blk(tok, w, self.M, reverse=rev and i % 2 == 1, discretize_mode=cfg.discretize_mode,
                      lb=cfg.scan_variant == "lbm")
        pooled = pool_tokens(tok, cfg, p)
        h1 = F.gelu(pooled @ p["head.mlp_w1"] + p["head.mlp_b1"], approximate="tanh")
        return h1 @ p["head.mlp_w2"] + p["head.mlp_b2"]

    def step(self, images, labels):
        """One optimisation step; returns the loss tensor (no host sync)."""
        self.opt.zero_grad(set_to_none=True)
        with torch.autocast("cuda", dtype=torch.bfloat16, enabled=self.amp):
            logits = self.forward(images)
        loss = F.cross_entropy(logits.float(), labels)
        loss.backward()
        self.opt.step()
        return loss.detach()

    def graphed(self, images, labels, warmup: int = 3):
        """The whole training step (forward, cross entropy, backward through the
        fused kernels, AdamW) captured once into a CUDA graph: each call of the
        returned function copies a batch into the static inputs and replays the
        graph — one launch instead of ~1,000 Python-issued kernels and ctypes
        calls per step.  The optimizer is rebuilt with ``capturable=True`` (step
        counts on the device) and its state carried over.  Runs ``warmup`` eager
        steps on a side stream first (they update the parameters, as real steps
        would).  Returns ``run(images, labels) -> loss``."""
        d = self.opt.defaults
        opt = torch.optim.AdamW(self.params.values(), lr=d["lr"], betas=d["betas"], eps=d["eps"],
                                weight_decay=d["weight_decay"], amsgrad=d["amsgrad"], capturable=True,
                                fused=bool(d.get("fused")))
        for p_, st in self.opt.state.items():
            opt.state[p_] = {k: (v.to(p_.device) if torch.is_tensor(v) else torch.tensor(float(v), device=p_.device))
                             for k, v in st.items()}
        self.opt = opt
        static_x = images.clone()
        static_y = labels.clone()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                self.step(static_x, static_y)
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        self.opt.zero_grad(set_to_none=True)
        with torch.cuda.graph(g):
            with torch.autocast("cuda", dtype=torch.bfloat16, enabled=self.amp):
                logits = self.forward(static_x)
            static_loss = F.cross_entropy(logits.float(), static_y)
            static_loss.backward()
            self.opt.step()

        def run(images, labels):
            static_x.copy_(images, non_blocking=True)
            static_y.copy_(labels, non_blocking=True)
            g.replay()
            return static_loss

        run.graph = g
        return run
