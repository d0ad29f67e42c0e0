"""Operator-API edge cases on the GPU: bf16 B/C rows narrower than a 16-byte
piece, the reference engine's ScanParams dataclass arguments, the MAP head in
training, autograd through the global bi-directional baseline."""

from dataclasses import dataclass

import numpy as np
import pytest

from helpers import TOL_BF16, TOL_F32, TOL_GRAD, op_inputs
from oracle import lbscan_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2506_15976_b200.scan import (  # noqa: E402
    global_bidir_selective_scan, lbm_selective_scan_bwd, lbm_selective_scan_fwd)

SEQ = ("u", "delta", "z", "B", "C")


def dev(x, dtype=torch.float32):
    return None if x is None else torch.as_tensor(np.ascontiguousarray(x), dtype=dtype, device="cuda")


@pytest.mark.parametrize("reverse", [False, True])
def test_bf16_state4_aligned_slices(reverse):
    """B, C = 16-byte aligned (B, L, 4) bf16 slices of a (B, L, 8) buffer: rows of 8
    bytes cannot go through the 16-byte cp.async B/C stager."""
    Bt, L, E, N = 2, 70, 64, 4
    inp = op_inputs(31, Bt, L, E, N)
    q = {k: (dev(v, torch.bfloat16).float().cpu().numpy() if k in SEQ else v) for k, v in inp.items()}
    buf = torch.zeros(Bt, L, 8, dtype=torch.bfloat16, device="cuda")
    buf[..., :4] = dev(q["B"], torch.bfloat16)
    buf2 = torch.zeros(Bt, L, 8, dtype=torch.bfloat16, device="cuda")
    buf2[..., :4] = dev(q["C"], torch.bfloat16)
    t = {k: (dev(v, torch.bfloat16) if k in SEQ else dev(v)) for k, v in q.items()}
    t["B"], t["C"] = buf[..., :4], buf2[..., :4]
    got = lbm_selective_scan_fwd(**t, window=8, reverse=reverse).float().cpu().numpy()
    ref = O.lbm_selective_scan(**q, window=8, reverse=reverse)
    assert O.max_rel_err(got, ref) <= TOL_BF16
    dout = O.seeded_rng(2).standard_normal((Bt, L, E))
    dq = dev(dout, torch.bfloat16)
    g = lbm_selective_scan_bwd(dq, **t, window=8, reverse=reverse)
    rg = O.lbm_selective_scan_bwd(dq.float().cpu().numpy(), **q, window=8, reverse=reverse)
    for k in ("dB", "dC", "dA"):
        assert O.max_rel_err(g[k].float().cpu().numpy(), rg[k]) <= TOL_BF16, k


@dataclass
class ScanParams:  # the shape of the reference's core.ScanParams (core.py:89-108)
    abar: np.ndarray
    bx: np.ndarray
    c: np.ndarray
    dx: np.ndarray


def test_engine_global_bidir_takes_scan_params_dataclass():
    from paper_2506_15976_b200 import engine
    rng = O.seeded_rng(4)
    pf = ScanParams(*O.random_scan_params(rng, 2, 33, 3, 4))
    pb = ScanParams(*O.random_scan_params(rng, 2, 33, 3, 4))
    plan = engine.TilePlan.for_length(33)
    got = engine.global_bidir_par(pf, pb, plan)
    ref_y, ref_h = O.global_bidir_scan((pf.abar, pf.bx, pf.c, pf.dx), (pb.abar, pb.bx, pb.c, pb.dx))
    assert O.max_rel_err(got.y, ref_y) <= 1e-12
    assert O.max_rel_err(got.h_final, ref_h) <= 1e-12
    tup = engine.global_bidir_par((pf.abar, pf.bx, pf.c, pf.dx), (pb.abar, pb.bx, pb.c, pb.dx), plan)
    assert np.array_equal(tup.y, got.y)


def test_trainer_map_head_matches_inference():
    """LBVimTrainer pools with the MAP head (model.py:260-290) like LBVim does."""
    from paper_2506_15976_b200 import model as Mdl
    cfg = Mdl.ModelConfig(image_size=16, patch_size=4, in_channels=1, embed_dim=16, inner_dim=32, state_dim=4,
                          depth=2, head="map", map_heads=4, class_token="none", num_classes=3)
    params = Mdl.init_params(cfg, seed=3)
    imgs = torch.randn(2, 16, 16, 1, device="cuda")
    net = Mdl.LBVim(cfg, params, dtype=torch.float32)
    tr = Mdl.LBVimTrainer(cfg, params)
    want = net(imgs)
    got = tr.forward(imgs)
    assert torch.allclose(got, want, rtol=1e-4, atol=1e-5), (got - want).abs().max()
    loss = torch.nn.functional.cross_entropy(got, torch.tensor([0, 2], device="cuda"))
    loss.backward()
    for k in ("head.q", "head.wk", "head.wv"):
        assert tr.params[k].grad is not None and tr.params[k].grad.abs().sum() > 0, k


def test_global_bidir_autograd():
    """Gradients of the baseline (autodiff.global_bidir_grad, autodiff.py:204-236):
    the sum of a forward-only scan and a flip-on-load forward-only scan, each of
    which is the oracle's M = 1 adjoint."""
    Bt, L, E, N = 2, 45, 24, 16
    inp = op_inputs(77, Bt, L, E, N)
    t = {k: dev(v).requires_grad_(True) for k, v in inp.items()}
    out = global_bidir_selective_scan(**t)
    ref_f = O.lbm_selective_scan(**inp, window=1)
    ref_b = O.lbm_selective_scan(**inp, window=1, reverse=True)
    assert O.max_rel_err(out.detach().cpu().numpy(), ref_f + ref_b) <= TOL_F32
    dout = O.seeded_rng(8).standard_normal((Bt, L, E))
    out.backward(dev(dout))
    gf = O.lbm_selective_scan_bwd(dout, **inp, window=1)
    gb = O.lbm_selective_scan_bwd(dout, **inp, window=1, reverse=True)
    names = {"u": "du", "delta": "ddelta", "A": "dA", "B": "dB", "C": "dC", "D": "dD", "z": "dz",
             "delta_bias": "ddelta_bias"}
    for k, gk in names.items():
        err = O.max_rel_err(t[k].grad.cpu().numpy(), gf[gk] + gb[gk])
        assert err <= TOL_GRAD, (k, err)
