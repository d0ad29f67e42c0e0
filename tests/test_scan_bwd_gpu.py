"""Parity of the sm_100a fused backward (lbs_scan_bwd) with the CPU oracle's
adjoint (oracle.lbm_selective_scan_bwd = autodiff.lbm_scan_grad chained through
block._discretize_backward and the gate, pinned to the reference by
tests/test_oracle_golden.py).  North-star bar: fp32 gradients within 1e-4
max_rel_err (core.py:149-156).  Runs on the B200 box: -m gpu."""

import numpy as np
import pytest

from helpers import TOL_BF16, TOL_GRAD, op_inputs
from oracle import lbscan_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2506_15976_b200.scan import (  # noqa: E402
    lbm_selective_scan, lbm_selective_scan_bwd, lbm_selective_scan_fwd, selective_scan)

SEQ = ("u", "delta", "z", "B", "C")
GRADS = ("du", "ddelta", "dA", "dB", "dC", "dD", "dz", "ddelta_bias")


def dev(x, dtype=torch.float32):
    return None if x is None else torch.as_tensor(np.ascontiguousarray(x), dtype=dtype, device="cuda")


def gpu_bwd(inp, dout, dtype=torch.float32, **kw):
    t = {k: (dev(v, dtype) if k in SEQ else dev(v)) for k, v in inp.items()}
    g = lbm_selective_scan_bwd(dev(dout, dtype), **t, **kw)
    return {k: (None if v is None else v.float().cpu().numpy()) for k, v in g.items()}


def check(got, ref, tol, what=""):
    for k in GRADS:
        if ref[k] is None:
            assert got[k] is None, (what, k)
            continue
        err = O.max_rel_err(got[k], ref[k])
        assert err <= tol, f"{what} {k}: max rel err {err:.3e} > {tol}"


def case(seed, Bt, L, E, N, **drop):
    inp = op_inputs(seed, Bt, L, E, N)
    for k, v in drop.items():
        if v:
            inp[k] = None
    dout = O.seeded_rng(seed + 1000).standard_normal((Bt, L, E))
    return inp, dout


@pytest.mark.parametrize("L", [1, 5, 31, 128, 129, 197, 257])
@pytest.mark.parametrize("M", [1, 3, 4, 8, 16])
@pytest.mark.parametrize("reverse", [False, True])
def test_bwd_fp32_grid(L, M, reverse):
    inp, dout = case(200 + L + M, 2, L, 5, 4)
    got = gpu_bwd(inp, dout, window=M, reverse=reverse)
    ref = O.lbm_selective_scan_bwd(dout, **inp, window=M, reverse=reverse)
    check(got, ref, TOL_GRAD, f"L={L} M={M} rev={reverse}")


@pytest.mark.parametrize("N", [1, 3, 4, 7, 16])
@pytest.mark.parametrize("E", [37, 130])
def test_bwd_state_and_channel_sizes(N, E):
    inp, dout = case(7 + N + E, 2, 97, E, N)
    for M in (4, 8):
        got = gpu_bwd(inp, dout, window=M)
        ref = O.lbm_selective_scan_bwd(dout, **inp, window=M)
        check(got, ref, TOL_GRAD, f"N={N} E={E} M={M}")


def test_bwd_cfg1_shape():
    """BASELINE configs[0] shape (B=2, D=192, L=197, N=16, window 8), both directions."""
    inp, dout = case(0, 2, 197, 192, 16)
    for reverse in (False, True):
        got = gpu_bwd(inp, dout, window=8, reverse=reverse)
        ref = O.lbm_selective_scan_bwd(dout, **inp, window=8, reverse=reverse)
        check(got, ref, TOL_GRAD, f"cfg1 rev={reverse}")


def test_bwd_cfg3_channels_subsample():
    """BASELINE configs[2] channel width (E=768, L=197, N=16, window 8) on a
    batch subsample (lanes are independent, so the check is exact per row)."""
    inp, dout = case(3, 3, 197, 768, 16)
    got = gpu_bwd(inp, dout, window=8)
    ref = O.lbm_selective_scan_bwd(dout, **inp, window=8)
    check(got, ref, TOL_GRAD, "cfg3-sub")


@pytest.mark.parametrize("drop", ["z", "D", "delta_bias"])
def test_bwd_optional_inputs(drop):
    inp, dout = case(11, 2, 50, 9, 4, **{drop: True})
    got = gpu_bwd({k: v for k, v in inp.items() if v is not None}, dout, window=4)
    ref = O.lbm_selective_scan_bwd(dout, **inp, window=4)
    check(got, ref, TOL_GRAD, drop)


def test_bwd_modes():
    inp, dout = case(12, 2, 70, 11, 8)
    # no softplus: positive step
    x = dict(inp)
    x["delta"] = np.abs(inp["delta"]) * 0.2
    x["delta_bias"] = np.abs(inp["delta_bias"]) * 0.01
    check(gpu_bwd(x, dout, window=4, delta_softplus=False),
          O.lbm_selective_scan_bwd(dout, **x, window=4, delta_softplus=False), TOL_GRAD, "no-softplus")
    # discretize_mode="linear" (block.py:94)
    x = dict(inp)
    x["A"] = -np.abs(inp["A"]) * 0.05
    check(gpu_bwd(x, dout, window=4, discretize_mode="linear"),
          O.lbm_selective_scan_bwd(dout, **x, window=4, mode="linear"), TOL_GRAD, "linear")
    # forward-only scan (engine.forward_scan_par) gradient
    for reverse in (False, True):
        check(gpu_bwd(inp, dout, window=8, lb=False, reverse=reverse),
              O.lbm_selective_scan_bwd(dout, **inp, window=8, lb=False, reverse=reverse), TOL_GRAD,
              f"forward-only rev={reverse}")


def test_bwd_m1_equals_forward_only():
    """M=1 LB == forward-only (test_autodiff.py:99-106).  The two are separate
    template instantiations (LB terms compiled in / out), so ptxas may order
    the FP32 ops differently: equal to fp32 rounding, not bitwise."""
    inp, dout = case(13, 2, 45, 20, 16)
    a = gpu_bwd(inp, dout, window=1)
    b = gpu_bwd(inp, dout, window=8, lb=False)
    for k in GRADS:
        assert O.max_rel_err(a[k], b[k]) <= 1e-6, k


def test_bwd_checkpoints_equal_recompute_and_deterministic():
    inp, dout = case(14, 3, 300, 140, 16)
    t = {k: (dev(v) if v is not None else None) for k, v in inp.items()}
    for M in (3, 8, 16):
        for reverse in (False, True):
            out, ck = lbm_selective_scan_fwd(**t, window=M, reverse=reverse, save_checkpoints=True)
            ref_out = lbm_selective_scan_fwd(**t, window=M, reverse=reverse)
            torch.testing.assert_close(out, ref_out, rtol=0, atol=0)
            g1 = lbm_selective_scan_bwd(dev(dout), **t, window=M, reverse=reverse, checkpoints=ck)
            g2 = lbm_selective_scan_bwd(dev(dout), **t, window=M, reverse=reverse)
            g3 = lbm_selective_scan_bwd(dev(dout), **t, window=M, reverse=reverse)
            for k in GRADS:
                torch.testing.assert_close(g1[k], g2[k], rtol=0, atol=0)
                torch.testing.assert_close(g2[k], g3[k], rtol=0, atol=0)


def test_bwd_zero_upstream_gives_zero():
    """test_autodiff.py:93-97."""
    inp, _ = case(15, 2, 40, 8, 4)
    got = gpu_bwd(inp, np.zeros((2, 40, 8)), window=4)
    for k in GRADS:
        assert not np.any(got[k]), k


@pytest.mark.parametrize("reverse", [False, True])
def test_bwd_bf16(reverse):
    inp, dout = case(16, 4, 197, 384, 16)
    q = {k: (dev(v, torch.bfloat16).float().cpu().numpy().astype(np.float64) if k in SEQ else v)
         for k, v in inp.items()}
    dq = dev(dout, torch.bfloat16).float().cpu().numpy().astype(np.float64)
    got = gpu_bwd(q, dq, dtype=torch.bfloat16, window=8, reverse=reverse)
    ref = O.lbm_selective_scan_bwd(dq, **q, window=8, reverse=reverse)
    check(got, ref, TOL_BF16, f"bf16 rev={reverse}")


def test_autograd_function_matches_direct_bwd():
    inp, dout = case(17, 2, 64, 33, 16)
    leaves = {k: dev(v).requires_grad_(True) for k, v in inp.items()}
    out = lbm_selective_scan(**leaves, window=8, reverse=True)
    out.backward(dev(dout))
    ref = O.lbm_selective_scan_bwd(dout, **inp, window=8, reverse=True)
    names = {"u": "du", "delta": "ddelta", "A": "dA", "B": "dB", "C": "dC", "D": "dD", "z": "dz",
             "delta_bias": "ddelta_bias"}
    for k, g in names.items():
        err = O.max_rel_err(leaves[k].grad.cpu().numpy(), ref[g])
        assert err <= TOL_GRAD, (k, err)
    # forward-only operator is differentiable too
    leaves2 = {k: dev(v).requires_grad_(True) for k, v in inp.items()}
    selective_scan(**leaves2).backward(dev(dout))
    ref2 = O.lbm_selective_scan_bwd(dout, **inp, window=8, lb=False)
    assert O.max_rel_err(leaves2["u"].grad.cpu().numpy(), ref2["du"]) <= TOL_GRAD


def test_strided_views_like_the_block():
    """B, C and delta as column slices of one projection, z a slice of the
    in-projection (model.py layout): no copies, same gradients."""
    inp, dout = case(18, 2, 80, 24, 16)
    Bt, L, E, N = 2, 80, 24, 16
    proj = torch.cat([dev(inp["delta"]), dev(inp["B"]), dev(inp["C"])], -1)
    xz = torch.cat([dev(inp["u"]), dev(inp["z"])], -1)
    t = dict(u=dev(inp["u"]), delta=proj[..., :E], A=dev(inp["A"]), B=proj[..., E:E + N],
             C=proj[..., E + N:], D=dev(inp["D"]), z=xz[..., E:], delta_bias=dev(inp["delta_bias"]))
    g = lbm_selective_scan_bwd(dev(dout), **t, window=8)
    got = {k: (None if v is None else v.cpu().numpy()) for k, v in g.items()}
    check(got, O.lbm_selective_scan_bwd(dout, **inp, window=8), TOL_GRAD, "strided")


@pytest.mark.parametrize("i", range(4))
def test_bwd_reproduces_reference_block_backward_golden(i):
    """The GPU adjoint mapped onto the block's weights reproduces the UNMODIFIED
    reference's block.block_backward (tests/golden/block.npz, made by
    oracle/gen_golden.py) to the fp32-gradient bar — no oracle in between."""
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "block.npz"))
    D, E, N, L, B, M, k, linear, rev, seed = [int(v) for v in g[f"b{i}_meta"]]
    w = {f: g[f"b{i}_w_{f}"] for f in O.BLOCK_FIELDS}
    mode = "linear" if linear else "exp"
    T = g[f"b{i}_T"]
    gout = g[f"b{i}_gout"]
    if rev:
        gout = gout[:, ::-1]
    xs, z, x, xc = (g[f"b{i}_cache_{k}"] for k in ("xs", "z", "x", "xc"))
    A = -np.exp(w["a_log"])
    dout = gout @ w["w_out"].T
    inp = dict(u=xs, delta=xs @ w["w_delta"], A=A, B=xs @ w["w_b"], C=xs @ w["w_c"], D=w["d_param"], z=z,
               delta_bias=w["delta_bias"])
    r = gpu_bwd(inp, dout, window=M, discretize_mode=mode)
    r = {kk: (None if v is None else v.astype(np.float64)) for kk, v in r.items()}
    xT = lambda a, b: np.tensordot(a, b, axes=((0, 1), (0, 1)))
    xn = O.rms_norm(T, w["norm_scale"])
    got = {"d_param": r["dD"], "delta_bias": r["ddelta_bias"], "a_log": r["dA"] * A,
           "w_b": xT(xs, r["dB"]), "w_c": xT(xs, r["dC"]), "w_delta": xT(xs, r["ddelta"]),
           "w_z": xT(xn, r["dz"])}
    g_xs = r["du"] + r["ddelta"] @ w["w_delta"].T + r["dB"] @ w["w_b"].T + r["dC"] @ w["w_c"].T
    _, got["conv_kernel"] = O.causal_conv1d_grad(x, w["conv_kernel"], g_xs * O.silu_grad(xc))
    for name, v in got.items():
        err = O.max_rel_err(v, g[f"b{i}_g_{name}"])
        assert err <= TOL_GRAD, (name, err)


@pytest.mark.parametrize("N", [4, 16])
@pytest.mark.parametrize("M", [3, 8])
def test_bwd_vectorised_path_small_state(N, M):
    """E multiple of 4 and 16-byte aligned rows -> the cp.async staging path;
    N = 4 makes the B/C table smaller than the CTA (regression: out-of-table
    writes clobbered the staged checkpoints)."""
    inp, dout = case(19 + N + M, 2, 40, 16, N)
    for ck in (False, True):
        t = {k: dev(v) for k, v in inp.items()}
        c = lbm_selective_scan_fwd(**t, window=M, save_checkpoints=True)[1] if ck else None
        g = lbm_selective_scan_bwd(dev(dout), **t, window=M, checkpoints=c)
        got = {k: (None if v is None else v.cpu().numpy()) for k, v in g.items()}
        check(got, O.lbm_selective_scan_bwd(dout, **inp, window=M), TOL_GRAD, f"vec N={N} M={M} ck={ck}")
