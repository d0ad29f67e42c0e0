"""LBVim block/model on the fused kernels vs the reference's own outputs
(golden vectors) and the oracle.  -m gpu."""

import os

import numpy as np
import pytest

from oracle import lbscan_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2506_15976_b200.model import BLOCK_FIELDS, LBVim, ModelConfig, init_params  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _model_from_golden(i):
    g = np.load(os.path.join(GOLD, "model.npz"))
    pre = f"m{i}_"
    cfg = {k[len(pre) + 4:]: g[k].item() for k in g.files if k.startswith(pre + "cfg_")}
    cfg["tile_len"] = None if cfg["tile_len"] in (None, "auto") else int(cfg["tile_len"])
    for k in ("reverse_between_blocks", "unreverse_output"):
        cfg[k] = bool(cfg[k])
    for k in ("image_size", "patch_size", "in_channels", "embed_dim", "inner_dim", "state_dim", "depth",
              "map_heads", "num_classes", "conv_width"):
        cfg[k] = int(cfg[k])
    params = {k[len(pre) + 2:]: torch.tensor(g[k], dtype=torch.float32, device="cuda")
              for k in g.files if k.startswith(pre + "p_")}
    return ModelConfig(**cfg), params, g[pre + "images"], g[pre + "logits"]


@pytest.mark.parametrize("i", range(3))
def test_model_forward_matches_reference_golden(i):
    cfg, params, images, ref = _model_from_golden(i)
    m = LBVim(cfg, params, dtype=torch.float32)
    got = m(torch.tensor(images, dtype=torch.float32, device="cuda")).cpu().numpy()
    assert O.max_rel_err(got, ref) <= 1e-4


@pytest.mark.parametrize("i", range(4))
def test_block_matches_reference_golden(i):
    g = np.load(os.path.join(GOLD, "block.npz"))
    D, E, N, L, B, M, k, linear, rev, seed = [int(v) for v in g[f"b{i}_meta"]]
    cfg = ModelConfig(image_size=4, patch_size=4, embed_dim=D, inner_dim=E, state_dim=N, depth=1,
                      tile_len=M, conv_width=k, discretize_mode="linear" if linear else "exp")
    params = {f"blocks.0.{f}": torch.tensor(g[f"b{i}_w_{f}"], dtype=torch.float32, device="cuda")
              for f in BLOCK_FIELDS}
    params.update(patch_w=torch.zeros(16, D), patch_b=torch.zeros(D), pos=torch.zeros(1, D))
    m = LBVim(cfg, {k: v.cuda() for k, v in params.items()}, dtype=torch.float32)
    T = torch.tensor(g[f"b{i}_T"], dtype=torch.float32, device="cuda")
    out = m.block(T, m.blocks[0], reverse=False).cpu().numpy()
    ref = g[f"b{i}_out"]
    ref = ref[:, ::-1] if rev else ref  # the reference reverses the block output
    assert O.max_rel_err(out, ref) <= 1e-5
    # flip-on-load: a reverse-direction block on the reversed sequence equals
    # the reversed forward-direction block
    Tr = torch.flip(T, dims=[1])
    out_r = m.block(Tr, m.blocks[0], reverse=True).cpu().numpy()
    assert O.max_rel_err(out_r[:, ::-1], ref) <= 1e-5


def test_lbvim_tiny_bf16_vs_fp32_and_graph():
    """Full-size LBVim-Ti (24 layers, L=197) at a small batch: bf16 path vs the
    fp32 path of the same weights, and the CUDA-graph replay is identical."""
    from paper_2506_15976_b200.model import lbvim_tiny
    cfg = lbvim_tiny()
    params = init_params(cfg, seed=0)
    imgs = torch.randn(4, 224, 224, 3, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
    m32 = LBVim(cfg, params, dtype=torch.float32)
    m16 = LBVim(cfg, params, dtype=torch.bfloat16)
    l32 = m32(imgs)
    l16 = m16(imgs)
    assert torch.isfinite(l16).all()
    rel = (l16 - l32).abs().max() / l32.abs().max()
    assert rel.item() <= 5e-2
    run = m16.graphed(imgs)
    torch.testing.assert_close(run(imgs), l16, rtol=0, atol=0)


def test_lbvim_tiny_fp32_vs_oracle_subsample():
    """LBVim-Ti structure (24 layers) with the CPU oracle on one image, fp32."""
    from paper_2506_15976_b200.model import lbvim_tiny
    cfg = lbvim_tiny(depth=4)
    params = init_params(cfg, seed=3)
    imgs = torch.randn(1, 224, 224, 3, device="cuda", generator=torch.Generator(device="cuda").manual_seed(2))
    got = LBVim(cfg, params, dtype=torch.float32)(imgs).cpu().numpy()
    npp = {k: v.double().cpu().numpy() for k, v in params.items()}
    ocfg = dict(image_size=224, patch_size=16, in_channels=3, embed_dim=192, inner_dim=384, state_dim=16,
                depth=4, tile_len=None, head="gap", class_token="middle")
    ref = O.model_forward(imgs.double().cpu().numpy(), ocfg, npp)
    assert O.max_rel_err(got, ref) <= 1e-4


@pytest.mark.parametrize("i", range(4))
def test_block_backward_matches_reference_golden(i):
    """Autograd through the fused kernels reproduces the UNMODIFIED reference's
    block.block_backward (all 11 weight gradients and the input gradient)."""
    from paper_2506_15976_b200.model import block_forward_train
    g = np.load(os.path.join(GOLD, "block.npz"))
    D, E, N, L, B, M, k, linear, rev, seed = [int(v) for v in g[f"b{i}_meta"]]
    w = {f: torch.tensor(g[f"b{i}_w_{f}"], dtype=torch.float32, device="cuda").requires_grad_(True)
         for f in BLOCK_FIELDS}
    T = torch.tensor(g[f"b{i}_T"], dtype=torch.float32, device="cuda").requires_grad_(True)
    out = block_forward_train(T, w, M, reverse=False, discretize_mode="linear" if linear else "exp")
    gout = g[f"b{i}_gout"]
    gout = gout[:, ::-1] if rev else gout  # the reference reverses its block output
    out.backward(torch.tensor(np.ascontiguousarray(gout), dtype=torch.float32, device="cuda"))
    for f in BLOCK_FIELDS:
        err = O.max_rel_err(w[f].grad.cpu().numpy(), g[f"b{i}_g_{f}"])
        assert err <= 1e-4, (f, err)
    assert O.max_rel_err(T.grad.cpu().numpy(), g[f"b{i}_g_in"]) <= 1e-4


def test_lbvim_trainer_steps():
    """A few LBVim training steps (small config): finite loss that decreases on a
    fixed batch; reverse-direction blocks are exercised (depth 4)."""
    from paper_2506_15976_b200.model import LBVimTrainer
    cfg = ModelConfig(image_size=32, patch_size=4, in_channels=3, embed_dim=64, inner_dim=128, state_dim=16,
                      depth=4, class_token="middle", num_classes=10)
    tr = LBVimTrainer(cfg, init_params(cfg, seed=0), lr=3e-3)
    gen = torch.Generator(device="cuda").manual_seed(0)
    imgs = torch.randn(16, 32, 32, 3, device="cuda", generator=gen)
    labels = torch.randint(0, 10, (16,), device="cuda", generator=gen)
    losses = [tr.step(imgs, labels).item() for _ in range(8)]
    assert all(np.isfinite(losses))
    assert losses[-1] < losses[0]


def test_lbvim_trainer_bf16_autocast():
    """amp=True: bf16 projections, the fused kernels' bf16-I/O variants in forward and
    backward; gradients of one step agree with the fp32 trainer to bf16 accuracy and
    the loss decreases over a few steps."""
    from paper_2506_15976_b200.model import LBVimTrainer
    cfg = ModelConfig(image_size=32, patch_size=4, in_channels=3, embed_dim=64, inner_dim=128, state_dim=16,
                      depth=4, class_token="middle", num_classes=10)
    gen = torch.Generator(device="cuda").manual_seed(1)
    imgs = torch.randn(16, 32, 32, 3, device="cuda", generator=gen)
    labels = torch.randint(0, 10, (16,), device="cuda", generator=gen)
    grads = []
    for amp in (False, True):
        tr = LBVimTrainer(cfg, init_params(cfg, seed=0), lr=3e-3, amp=amp)
        tr.opt.zero_grad(set_to_none=True)
        with torch.autocast("cuda", dtype=torch.bfloat16, enabled=amp):
            logits = tr.forward(imgs)
        torch.nn.functional.cross_entropy(logits.float(), labels).backward()
        grads.append({k: v.grad.detach().clone() for k, v in tr.params.items() if v.grad is not None})
    for k in ("blocks.1.w_x", "blocks.2.a_log", "blocks.3.delta_bias", "blocks.0.conv_kernel", "head.mlp_w2"):
        ref, got = grads[0][k], grads[1][k]
        assert ((got - ref).abs().max() / ref.abs().max()).item() < 0.1, k
    tr = LBVimTrainer(cfg, init_params(cfg, seed=0), lr=3e-3, amp=True)
    losses = [tr.step(imgs, labels).item() for _ in range(8)]
    assert all(np.isfinite(losses)) and losses[-1] < losses[0]


@pytest.mark.parametrize("amp", [False, True])
def test_lbvim_trainer_graphed_matches_eager(amp):
    """The CUDA-graph-captured training step (forward + fused-kernel backward +
    capturable AdamW, one replay per step) follows the eager trainer: same losses
    and parameters after the same steps on the same batches."""
    from paper_2506_15976_b200.model import LBVimTrainer
    cfg = ModelConfig(image_size=32, patch_size=4, in_channels=3, embed_dim=64, inner_dim=128, state_dim=16,
                      depth=4, class_token="middle", num_classes=10)
    gen = torch.Generator(device="cuda").manual_seed(2)
    batches = [(torch.randn(16, 32, 32, 3, device="cuda", generator=gen),
                torch.randint(0, 10, (16,), device="cuda", generator=gen)) for _ in range(6)]
    eager = LBVimTrainer(cfg, init_params(cfg, seed=0), lr=3e-3, amp=amp)
    graphed = LBVimTrainer(cfg, init_params(cfg, seed=0), lr=3e-3, amp=amp)
    run = graphed.graphed(*batches[0], warmup=2)   # the 2 warm-up steps train on batches[0]
    for _ in range(2):
        eager.step(*batches[0])
    # fp32: the same kernels in the same order; bf16 autocast: cuBLAS may pick other
    # bf16 GEMM algorithms under capture, so bf16-rounding-level differences remain
    tol = 3e-3 if amp else 1e-4
    for x, y in batches[1:]:
        le = eager.step(x, y).item()
        lg = run(x, y).item()
        assert abs(le - lg) <= tol * max(1.0, abs(le)), (le, lg)
    for k in ("blocks.0.w_x", "blocks.3.a_log", "head.mlp_w2", "patch_w"):
        a, b = eager.params[k].detach(), graphed.params[k].detach()
        assert ((a - b).abs().max() / a.abs().max()).item() < tol, k


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_lbvim_tiny_full_depth_vs_oracle(dtype):
    """The headline model at full depth (LBVim-Ti, 24 layers, 224^2, L=197) against the
    CPU oracle on two images: fp32 at 1e-4; bf16 (the benchmarked dtype) at 5e-2 with
    the oracle fed the same bf16-rounded weights and images (activations between
    layers are bf16 on the GPU, fp64 in the oracle)."""
    from paper_2506_15976_b200.model import lbvim_tiny
    cfg = lbvim_tiny()
    params = init_params(cfg, seed=5)
    imgs = torch.randn(2, 224, 224, 3, device="cuda", generator=torch.Generator(device="cuda").manual_seed(6))
    tdt = torch.float32 if dtype == "fp32" else torch.bfloat16
    got = LBVim(cfg, params, dtype=tdt)(imgs.to(tdt)).float().cpu().numpy()
    rnd = (lambda t: t) if dtype == "fp32" else (lambda t: t.to(torch.bfloat16))
    npp = {k: rnd(v).double().cpu().numpy() for k, v in params.items()}
    # the GPU model keeps A, D, delta_bias and the conv taps in fp32 (model.py: f32 casts)
    for k in params:
        if k.endswith(("a_log", "d_param", "delta_bias", "conv_kernel", "norm_scale")):
            npp[k] = params[k].double().cpu().numpy()
    ocfg = dict(image_size=224, patch_size=16, in_channels=3, embed_dim=192, inner_dim=384, state_dim=16,
                depth=24, tile_len=None, head="gap", class_token="middle")
    ref = O.model_forward(rnd(imgs).double().cpu().numpy(), ocfg, npp)
    assert O.max_rel_err(got, ref) <= (1e-4 if dtype == "fp32" else 5e-2)
