"""Parity at every BASELINE.json config's FULL size (-m gpu).

The GPU runs the whole configured shape (the sequence split, CTA-width plan
and vectorised staging paths the benchmarks use); the CPU oracle checks a
deterministic subsample of batch rows and channels, which is exact because
lanes (b, e, n) are independent (engine.py:94-99) and B, C are shared per
(b, l).  Tolerances from the north star (tests/helpers.py)."""

import numpy as np
import pytest

from helpers import TOL_BF16, TOL_F32, TOL_GRAD
from oracle import lbscan_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2506_15976_b200.scan import lbm_selective_scan_bwd, lbm_selective_scan_fwd  # noqa: E402

# name: (B, L, E, N, window, dtype)
CONFIGS = {
    "configs[0] op fwd fp32": (2, 197, 192, 16, 8, torch.float32),
    "configs[1] LBVim-Ti layer bf16": (256, 197, 384, 16, 8, torch.bfloat16),
    "configs[2] LBVim-S layer fp32": (128, 197, 768, 16, 8, torch.float32),
    "configs[3] LBVim-S 1024^2 layer bf16": (32, 4096, 768, 16, 16, torch.bfloat16),
    "configs[4] MIL bag fp32": (1, 100000, 512, 16, 16, torch.float32),
    "configs[4] one 8-way channel shard": (1, 100000, 64, 16, 16, torch.float32),
}


def make_inputs(Bt, L, E, N, dtype, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    r = lambda *s: torch.randn(*s, generator=g, device="cuda").to(dtype)  # noqa: E731
    A = -torch.empty(E, N, device="cuda").uniform_(0.5, float(N), generator=g)
    dt = torch.exp(torch.empty(E, device="cuda").uniform_(np.log(1e-3), np.log(1e-1), generator=g))
    return dict(u=r(Bt, L, E), delta=0.5 * r(Bt, L, E), A=A, B=r(Bt, L, N), C=r(Bt, L, N),
                D=1.0 + 0.1 * torch.randn(E, generator=g, device="cuda"), z=r(Bt, L, E),
                delta_bias=dt + torch.log(-torch.expm1(-dt)))


def subsample(x, bsel, esel):
    """numpy fp64 oracle inputs for batch rows bsel and channels esel."""
    n = lambda t: t.double().cpu().numpy()  # noqa: E731
    return dict(u=n(x["u"][bsel][:, :, esel]), delta=n(x["delta"][bsel][:, :, esel]), A=n(x["A"][esel]),
                B=n(x["B"][bsel]), C=n(x["C"][bsel]), D=n(x["D"][esel]), z=n(x["z"][bsel][:, :, esel]),
                delta_bias=n(x["delta_bias"][esel]))


@pytest.mark.parametrize("name", list(CONFIGS))
def test_config_forward_full_size(name):
    Bt, L, E, N, M, dtype = CONFIGS[name]
    x = make_inputs(Bt, L, E, N, dtype)
    out, hf = lbm_selective_scan_fwd(**x, window=M, return_last_state=True)
    bsel = sorted({0, Bt - 1})
    esel = sorted({0, 1, E // 3, E // 2 + 1, E - 1})
    ref, rhf = O.lbm_selective_scan(**subsample(x, bsel, esel), window=M, return_last_state=True)
    tol = TOL_F32 if dtype == torch.float32 else TOL_BF16
    got = out[bsel][:, :, esel].float().cpu().numpy()
    assert O.max_rel_err(got, ref) <= tol
    assert O.max_rel_err(hf[bsel][:, esel].cpu().numpy(), rhf) <= tol
    assert torch.isfinite(out).all()


def test_config2_backward_full_size():
    """configs[2] (LBVim-S scan fwd+bwd, B=128, L=197, E=768, fp32): the training
    path (forward with checkpoints + fused backward) at full size; per-channel
    gradients checked on a subsample, dB/dC (sums over ALL channels) on sampled rows."""
    Bt, L, E, N, M, dtype = CONFIGS["configs[2] LBVim-S layer fp32"]
    x = make_inputs(Bt, L, E, N, dtype, seed=1)
    dout = torch.randn(Bt, L, E, device="cuda", generator=torch.Generator(device="cuda").manual_seed(2))
    _, ck = lbm_selective_scan_fwd(**x, window=M, save_checkpoints=True)
    g = lbm_selective_scan_bwd(dout, **x, window=M, checkpoints=ck)
    bsel, esel = [0, Bt - 1], [0, 5, E // 2, E - 1]
    sub = subsample(x, bsel, esel)
    ref = O.lbm_selective_scan_bwd(dout[bsel][:, :, esel].double().cpu().numpy(), **sub, window=M)
    for k in ("du", "ddelta", "dz"):
        assert O.max_rel_err(g[k][bsel][:, :, esel].cpu().numpy(), ref[k]) <= TOL_GRAD, k
    # dB, dC sum over all E channels: oracle over every channel of two batch rows
    full = subsample(x, bsel, list(range(E)))
    reff = O.lbm_selective_scan_bwd(dout[bsel].double().cpu().numpy(), **full, window=M)
    for k in ("dB", "dC"):
        assert O.max_rel_err(g[k][bsel].cpu().numpy(), reff[k]) <= TOL_GRAD, k
    assert all(torch.isfinite(v).all() for v in g.values() if v is not None)


@pytest.mark.parametrize("name,Bt,dtype,tol", [
    ("configs[2] shape, bf16 I/O (the amp training path)", 128, torch.bfloat16, TOL_BF16),
    ("configs[2] 8-GPU batch shard (B=16: sequence-split backward)", 16, torch.float32, TOL_GRAD),
])
def test_config2_backward_variants_full_size(name, Bt, dtype, tol):
    """The other two backward launches the benchmarks report at full size: the bf16-I/O
    training path (fp32 state, bf16 du/ddelta/dz) and one GPU's share of the 8-way batch
    split, whose plan cuts the sequence into segments joined by the adjoint carry."""
    _, L, E, N, M, _ = CONFIGS["configs[2] LBVim-S layer fp32"]
    x = make_inputs(Bt, L, E, N, dtype, seed=3)
    dout = torch.randn(Bt, L, E, device="cuda", generator=torch.Generator(device="cuda").manual_seed(4)).to(dtype)
    _, ck = lbm_selective_scan_fwd(**x, window=M, save_checkpoints=True)
    g = lbm_selective_scan_bwd(dout, **x, window=M, checkpoints=ck)
    bsel, esel = [0, Bt - 1], [0, 7, E // 2, E - 1]
    ref = O.lbm_selective_scan_bwd(dout[bsel][:, :, esel].double().cpu().numpy(), **subsample(x, bsel, esel), window=M)
    for k in ("du", "ddelta", "dz"):
        assert O.max_rel_err(g[k][bsel][:, :, esel].float().cpu().numpy(), ref[k]) <= tol, (name, k)
    reff = O.lbm_selective_scan_bwd(dout[bsel].double().cpu().numpy(), **subsample(x, bsel, list(range(E))),
                                    window=M)
    for k in ("dB", "dC"):
        assert O.max_rel_err(g[k][bsel].cpu().numpy(), reff[k]) <= tol, (name, k)
    assert all(torch.isfinite(v).all() for v in g.values() if v is not None)
