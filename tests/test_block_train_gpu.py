"""The LBVim block as one autograd node (block_train.LBVimBlockFn, hand-written backward
with the gradient glue removed) against the UNMODIFIED reference's block_backward
golden vectors and against the plain autograd composition.  -m gpu."""

import os

import numpy as np
import pytest

from oracle import lbscan_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2506_15976_b200.block_train import block_forward_fused  # noqa: E402
from paper_2506_15976_b200.model import (BLOCK_FIELDS, LBVimTrainer, ModelConfig,  # noqa: E402
                                         block_forward_train, init_params)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("i", range(4))
def test_fused_block_backward_matches_reference_golden(i):
    """fp32: all 11 weight gradients and the input gradient of the reference's
    block.block_backward (block.py:193-220) within 1e-4."""
    g = np.load(os.path.join(GOLD, "block.npz"))
    D, E, N, L, B, M, k, linear, rev, seed = [int(v) for v in g[f"b{i}_meta"]]
    w = {f: torch.tensor(g[f"b{i}_w_{f}"], dtype=torch.float32, device="cuda").requires_grad_(True)
         for f in BLOCK_FIELDS}
    T = torch.tensor(g[f"b{i}_T"], dtype=torch.float32, device="cuda").requires_grad_(True)
    out = block_forward_fused(T, w, M, reverse=False, discretize_mode="linear" if linear else "exp")
    gout = g[f"b{i}_gout"]
    gout = gout[:, ::-1] if rev else gout  # the reference reverses its block output
    out.backward(torch.tensor(np.ascontiguousarray(gout), dtype=torch.float32, device="cuda"))
    for f in BLOCK_FIELDS:
        err = O.max_rel_err(w[f].grad.cpu().numpy(), g[f"b{i}_g_{f}"])
        assert err <= 1e-4, (f, err)
    assert O.max_rel_err(T.grad.cpu().numpy(), g[f"b{i}_g_in"]) <= 1e-4


def _block_case(seed, Bt=4, L=197, D=96, E=192, N=16):
    cfg = ModelConfig(image_size=32, patch_size=4, in_channels=3, embed_dim=D, inner_dim=E, state_dim=N, depth=1,
                      class_token="none", num_classes=10)
    p = init_params(cfg, seed=seed)
    w = {f: p[f"blocks.0.{f}"].detach().clone() for f in BLOCK_FIELDS}
    gen = torch.Generator(device="cuda").manual_seed(seed)
    T = torch.randn(Bt, L, D, device="cuda", generator=gen)
    gout = torch.randn(Bt, L, D, device="cuda", generator=gen)
    return w, T, gout


def _grads(fn, w, T, gout, amp, **kw):
    w = {k: v.clone().requires_grad_(True) for k, v in w.items()}
    T = T.clone().requires_grad_(True)
    with torch.autocast("cuda", dtype=torch.bfloat16, enabled=amp):
        out = fn(T, w, 8, **kw)
    out.backward(gout)
    return out.detach(), T.grad, {k: v.grad for k, v in w.items()}


@pytest.mark.parametrize("reverse", [False, True])
@pytest.mark.parametrize("amp", [False, True])
def test_fused_block_matches_autograd_block(amp, reverse):
    """Same outputs and gradients as the autograd composition (model.block_forward_train):
    fp32 1e-5 relative; bf16 autocast to bf16 rounding (the fused node keeps the GEMM
    epilogues, weight gradients and the normalised-input gradient in fp32, where the
    autograd path rounds them to bf16 first)."""
    w, T, gout = _block_case(3 + reverse)
    o1, dT1, g1 = _grads(block_forward_train, w, T, gout, amp, reverse=reverse)
    o2, dT2, g2 = _grads(block_forward_fused, w, T, gout, amp, reverse=reverse)
    tol = 2e-2 if amp else 1e-5
    rel = lambda a, b: ((a.float() - b.float()).abs().max() / b.float().abs().max()).item()
    assert o2.dtype == torch.float32 and rel(o2, o1) <= tol
    assert rel(dT2, dT1) <= tol
    for f in BLOCK_FIELDS:
        assert g2[f].shape == w[f].shape
        assert rel(g2[f], g1[f]) <= tol, (f, rel(g2[f], g1[f]))


def test_trainer_fused_vs_autograd_blocks():
    """LBVimTrainer with fused_block=True (default) and False take the same fp32 steps."""
    cfg = ModelConfig(image_size=32, patch_size=4, in_channels=3, embed_dim=64, inner_dim=128, state_dim=16,
                      depth=4, class_token="middle", num_classes=10)
    gen = torch.Generator(device="cuda").manual_seed(5)
    batches = [(torch.randn(16, 32, 32, 3, device="cuda", generator=gen),
                torch.randint(0, 10, (16,), device="cuda", generator=gen)) for _ in range(4)]
    a = LBVimTrainer(cfg, init_params(cfg, seed=0), lr=3e-3, fused_block=True)
    b = LBVimTrainer(cfg, init_params(cfg, seed=0), lr=3e-3, fused_block=False)
    for x, y in batches:
        la, lb = a.step(x, y).item(), b.step(x, y).item()
        assert abs(la - lb) <= 1e-5 * max(1.0, abs(lb)), (la, lb)
    for k in ("blocks.0.w_x", "blocks.1.w_delta", "blocks.2.a_log", "blocks.3.conv_kernel", "patch_w"):
        x, y = a.params[k].detach(), b.params[k].detach()
        assert ((x - y).abs().max() / y.abs().max()).item() < 1e-5, k
