"""Parity of the generic fused path (csrc/lbs_generic.cu) with the CPU oracle (-m gpu).

The register-resident kernels cover N <= 16 and windows min(M, L) <= 16; the
reference accepts any M >= 1 and any N (engine.py:65-85, test_oracle.py:221-226),
so larger shapes take a state-outer kernel pair behind the same entry points.
Same bars as the fast path: fp32 outputs 1e-5, fp32 gradients 1e-4, bf16 2e-2,
M=1 and tile ends bitwise equal to the forward-only scan (test_engine.py:98-114)."""

import numpy as np
import pytest

from helpers import TOL_BF16, TOL_F32, TOL_GRAD, op_inputs
from oracle import lbscan_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2506_15976_b200.scan import (  # noqa: E402
    lbm_selective_scan, lbm_selective_scan_bwd, lbm_selective_scan_fwd)

SEQ = ("u", "delta", "z", "B", "C")
GRADS = ("du", "ddelta", "dA", "dB", "dC", "dD", "dz", "ddelta_bias")


def dev(x, dtype=torch.float32):
    return None if x is None else torch.as_tensor(np.ascontiguousarray(x), dtype=dtype, device="cuda")


def tens(inp, dtype=torch.float32):
    return {k: (dev(v, dtype) if k in SEQ else dev(v)) for k, v in inp.items()}


@pytest.mark.parametrize("N,M,L", [(17, 8, 97), (32, 4, 50), (64, 16, 197), (4, 17, 60), (16, 32, 197),
                                   (8, 100, 230), (33, 40, 81)])
def test_generic_forward(N, M, L):
    inp = op_inputs(N * 7 + M, 2, L, 45, N)
    t = tens(inp)
    for reverse in (False, True):
        y, hf = lbm_selective_scan_fwd(**t, window=M, reverse=reverse, return_last_state=True)
        ref, rhf = O.lbm_selective_scan(**inp, window=M, reverse=reverse, return_last_state=True)
        assert O.max_rel_err(y.cpu().numpy(), ref) <= TOL_F32, (N, M, L, reverse)
        assert O.max_rel_err(hf.cpu().numpy(), rhf) <= TOL_F32, (N, M, L, reverse)


@pytest.mark.parametrize("N,M,L", [(17, 8, 61), (24, 3, 40), (4, 20, 75), (20, 33, 90)])
def test_generic_backward(N, M, L):
    inp = op_inputs(N + 3 * M, 2, L, 37, N)
    dout = O.seeded_rng(N + M).standard_normal((2, L, 37))
    for reverse in (False, True):
        g = lbm_selective_scan_bwd(dev(dout), **tens(inp), window=M, reverse=reverse)
        ref = O.lbm_selective_scan_bwd(dout, **inp, window=M, reverse=reverse)
        for k in GRADS:
            err = O.max_rel_err(g[k].cpu().numpy(), ref[k])
            assert err <= TOL_GRAD, f"N={N} M={M} L={L} rev={reverse} {k}: {err:.3e}"


def test_generic_options_and_bf16():
    inp = op_inputs(5, 2, 70, 24, 20)
    dout = O.seeded_rng(6).standard_normal((2, 70, 24))
    for drop in ("z", "delta_bias", "D"):
        x = dict(inp)
        x[drop] = None
        y = lbm_selective_scan_fwd(**tens(x), window=24).cpu().numpy()
        assert O.max_rel_err(y, O.lbm_selective_scan(**x, window=24)) <= TOL_F32, drop
        g = lbm_selective_scan_bwd(dev(dout), **tens(x), window=24)
        ref = O.lbm_selective_scan_bwd(dout, **x, window=24)
        for k in GRADS:
            if ref[k] is None:
                assert g[k] is None
                continue
            assert O.max_rel_err(g[k].cpu().numpy(), ref[k]) <= TOL_GRAD, (drop, k)
    x = dict(inp)
    x["A"] = -np.abs(inp["A"]) * 0.05  # linear mode, contractive (block.py:94)
    y = lbm_selective_scan_fwd(**tens(x), window=20, discretize_mode="linear").cpu().numpy()
    assert O.max_rel_err(y, O.lbm_selective_scan(**x, window=20, mode="linear")) <= TOL_F32
    g = lbm_selective_scan_bwd(dev(dout), **tens(x), window=20, discretize_mode="linear")
    ref = O.lbm_selective_scan_bwd(dout, **x, window=20, mode="linear")
    for k in GRADS:
        assert O.max_rel_err(g[k].cpu().numpy(), ref[k]) <= TOL_GRAD, ("linear", k)
    # bf16 I/O with fp32 state: the oracle sees the same bf16-rounded inputs
    tb = tens(inp, torch.bfloat16)
    rounded = {k: (v.float().cpu().numpy() if k in SEQ and v is not None else inp[k]) for k, v in tb.items()}
    y = lbm_selective_scan_fwd(**tb, window=24).float().cpu().numpy()
    assert O.max_rel_err(y, O.lbm_selective_scan(**rounded, window=24)) <= TOL_BF16


def test_generic_bitwise_identities():
    """M=1 and tile-end outputs bitwise the forward-only scan's (same plan), N=32."""
    inp = op_inputs(8, 2, 50, 30, 32)
    t = tens(inp)
    for M in (1, 5, 20):
        lb = lbm_selective_scan_fwd(**t, window=M).cpu().numpy()
        fw = lbm_selective_scan_fwd(**t, window=M, lb=False).cpu().numpy()
        ends = [i for i in range(50) if (i + 1) % M == 0 or i == 49]
        np.testing.assert_array_equal(lb[:, ends], fw[:, ends])


def test_generic_autograd():
    """torch autograd through the generic path (no training checkpoints)."""
    inp = op_inputs(2, 2, 40, 16, 24)
    t = tens(inp)
    for k in ("u", "delta", "A", "B", "C", "D", "z", "delta_bias"):
        t[k].requires_grad_(True)
    y = lbm_selective_scan(**t, window=18)
    dout = O.seeded_rng(1).standard_normal(y.shape)
    y.backward(dev(dout))
    ref = O.lbm_selective_scan_bwd(dout, **inp, window=18)
    for k, r in (("u", "du"), ("delta", "ddelta"), ("A", "dA"), ("B", "dB"), ("C", "dC"), ("D", "dD"),
                 ("z", "dz"), ("delta_bias", "ddelta_bias")):
        assert O.max_rel_err(t[k].grad.cpu().numpy(), ref[r]) <= TOL_GRAD, k
