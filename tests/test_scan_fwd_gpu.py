"""Parity of the sm_100a forward kernels with the CPU oracle (pinned to the
reference by tests/test_oracle_golden.py).  Runs on the B200 box: -m gpu."""

import os

import numpy as np
import pytest

from helpers import TOL_BF16, TOL_F32, op_inputs
from oracle import lbscan_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2506_15976_b200 import engine  # noqa: E402
from paper_2506_15976_b200.scan import lbm_selective_scan, lbm_selective_scan_fwd, selective_scan  # noqa: E402
from paper_2506_15976_b200.tiling import TilePlan  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def dev(x, dtype=torch.float32):
    return torch.as_tensor(np.ascontiguousarray(x), dtype=dtype, device="cuda")


def run_gpu(inp, dtype=torch.float32, **kw):
    t = {k: (dev(v, dtype) if k in ("u", "delta", "z", "B", "C") else dev(v)) for k, v in inp.items()}
    out = lbm_selective_scan_fwd(**t, **kw)
    if isinstance(out, tuple):
        return tuple(o.float().cpu().numpy() for o in out)
    return out.float().cpu().numpy()


def quantize(inp, dtype):
    """Round the sequence inputs to ``dtype`` so the oracle sees what the GPU sees."""
    return {k: (dev(v, dtype).float().cpu().numpy().astype(np.float64)
                if k in ("u", "delta", "z", "B", "C") else v) for k, v in inp.items()}


# --- fused operator -----------------------------------------------------------

@pytest.mark.parametrize("L", [1, 5, 31, 128, 129, 197, 256, 257])
@pytest.mark.parametrize("M", [1, 3, 4, 8, 16])
@pytest.mark.parametrize("reverse", [False, True])
def test_fused_fp32_grid(L, M, reverse):
    inp = op_inputs(100 + L + M, 2, L, 5, 4)
    got = run_gpu(inp, window=M, reverse=reverse)
    ref = O.lbm_selective_scan(**inp, window=M, reverse=reverse)
    assert O.max_rel_err(got, ref) <= TOL_F32


@pytest.mark.parametrize("N", [1, 3, 4, 7, 8, 16])
def test_fused_state_sizes(N):
    inp = op_inputs(7 + N, 2, 97, 37, N)
    got, hf = run_gpu(inp, window=8, return_last_state=True)
    ref, rhf = O.lbm_selective_scan(**inp, window=8, return_last_state=True)
    assert O.max_rel_err(got, ref) <= TOL_F32
    assert O.max_rel_err(hf, rhf) <= TOL_F32


def test_cfg1_shape_fp32():
    """BASELINE configs[0]: B=2 D=192 L=197 N=16 window 8, fp32."""
    inp = op_inputs(0, 2, 197, 192, 16, random_A=False)
    for reverse in (False, True):
        got, hf = run_gpu(inp, window=8, reverse=reverse, return_last_state=True)
        ref, rhf = O.lbm_selective_scan(**inp, window=8, reverse=reverse, return_last_state=True)
        assert O.max_rel_err(got, ref) <= TOL_F32
        assert O.max_rel_err(hf, rhf) <= TOL_F32


@pytest.mark.parametrize("reverse", [False, True])
def test_fused_bf16(reverse):
    inp = quantize(op_inputs(3, 4, 197, 384, 16, random_A=False), torch.bfloat16)
    got = run_gpu(inp, dtype=torch.bfloat16, window=8, reverse=reverse)
    ref = O.lbm_selective_scan(**inp, window=8, reverse=reverse)
    assert O.max_rel_err(got, ref) <= TOL_BF16


def test_optional_inputs_and_modes():
    inp = op_inputs(11, 2, 50, 9, 4)
    for drop in ("z", "D", "delta_bias"):
        x = dict(inp)
        x[drop] = None
        got = run_gpu({k: v for k, v in x.items() if v is not None}, window=4)
        ref = O.lbm_selective_scan(**x, window=4)
        assert O.max_rel_err(got, ref) <= TOL_F32, drop
    # without softplus the step must already be positive for a contractive decay
    x = dict(inp)
    x["delta"] = np.abs(inp["delta"]) * 0.2
    x["delta_bias"] = np.abs(inp["delta_bias"]) * 0.01
    got = run_gpu(x, window=4, delta_softplus=False)
    ref = O.lbm_selective_scan(**x, window=4, delta_softplus=False)
    assert O.max_rel_err(got, ref) <= TOL_F32
    # discretize_mode="linear" (block.py:94) with a contractive decay
    x = dict(inp)
    x["A"] = -np.abs(inp["A"]) * 0.05
    got = run_gpu(x, window=4, discretize_mode="linear")
    ref = O.lbm_selective_scan(**x, window=4, mode="linear")
    assert O.max_rel_err(got, ref) <= TOL_F32


def test_window_longer_than_sequence_is_one_tile():
    inp = op_inputs(5, 1, 5, 3, 4)
    a = run_gpu(inp, window=16)
    b = run_gpu(inp, window=5)
    np.testing.assert_array_equal(a, b)
    assert O.max_rel_err(a, O.lbm_selective_scan(**inp, window=5)) <= TOL_F32


@pytest.mark.parametrize("seg_hint", [0, 1, 3])
def test_m1_equals_forward_bitwise_and_tile_ends(seg_hint):
    """test_engine.py:98-114 on the fused kernel: with the same tile plan, LB with
    M=1 and LB outputs at tile ends are bitwise the forward-only scan's (under
    the automatic launch plan, which splits this low-parallelism shape, and
    with forced segment counts)."""
    inp = op_inputs(21, 2, 61, 40, 16)
    t = {k: dev(v) for k, v in inp.items()}
    fwd_for = lambda M: lbm_selective_scan_fwd(**t, window=M, lb=False, seg_hint=seg_hint).cpu().numpy()
    fwd = fwd_for(1)
    m1 = lbm_selective_scan_fwd(**t, window=1, seg_hint=seg_hint).cpu().numpy()
    np.testing.assert_array_equal(m1, fwd)
    for M in (3, 4, 8, 16):
        lb = lbm_selective_scan_fwd(**t, window=M, seg_hint=seg_hint).cpu().numpy()
        fw = fwd_for(M)
        for i in range(61):
            if (i + 1) % M == 0 or i == 60:
                np.testing.assert_array_equal(lb[:, i], fw[:, i])
    assert O.max_rel_err(fwd, O.lbm_selective_scan(**inp, window=1)) <= TOL_F32
    assert O.max_rel_err(selective_scan(**t).cpu().numpy(), O.lbm_selective_scan(**inp, window=1)) <= TOL_F32


@pytest.mark.parametrize("S", [2, 3, 7])
def test_sequence_split_matches_unsplit(S):
    inp = op_inputs(33, 2, 777, 70, 16)
    for reverse in (False, True):
        got, hf = run_gpu(inp, window=16, reverse=reverse, return_last_state=True, seg_hint=S)
        ref, rhf = O.lbm_selective_scan(**inp, window=16, reverse=reverse, return_last_state=True)
        assert O.max_rel_err(got, ref) <= TOL_F32
        assert O.max_rel_err(hf, rhf) <= TOL_F32


def test_long_sequence_auto_split_fp32():
    """cfg-5-like: few channels, long L -> the launcher splits L; compare a
    (b, e) subsample with the oracle (lanes are independent, so exact)."""
    inp = op_inputs(44, 1, 20000, 64, 16)
    got = run_gpu(inp, window=16)
    sub = {k: (v[:, :, :8] if k in ("u", "delta", "z") else v[:8] if k in ("A", "D", "delta_bias") else v)
           for k, v in inp.items()}
    ref = O.lbm_selective_scan(**sub, window=16)
    assert O.max_rel_err(got[:, :, :8], ref) <= TOL_F32


def test_strided_views_of_fused_projection():
    """B and C as column slices of one (B, L, E+2N) projection output, u as a
    transposed view: strides go straight to the kernel, no copies."""
    inp = op_inputs(9, 2, 64, 24, 16)
    Bt, L, E = inp["u"].shape
    proj = np.concatenate([inp["delta"], inp["B"], inp["C"]], axis=-1)
    P = dev(proj)
    uT = dev(np.ascontiguousarray(inp["u"].transpose(0, 2, 1))).transpose(1, 2)
    got = lbm_selective_scan(uT, P[..., :E], dev(inp["A"]), P[..., E:E + 16], P[..., E + 16:],
                             D=dev(inp["D"]), z=dev(inp["z"]), delta_bias=dev(inp["delta_bias"]),
                             window=4).cpu().numpy()
    ref = O.lbm_selective_scan(**inp, window=4)
    assert O.max_rel_err(got, ref) <= TOL_F32


# --- pre-discretised entry: the reference's own grid and fixtures ---------------

@pytest.fixture(scope="module")
def grid():
    return np.load(os.path.join(GOLD, "scan_grid.npz"))


@pytest.mark.parametrize("L", [1, 5, 31, 128, 129, 197, 256, 257])
def test_prediscretized_grid_vs_reference(grid, L):
    p = [grid[f"L{L}_{k}"] for k in ("abar", "bx", "c", "dx")]
    p32 = [a.astype(np.float32) for a in p]
    for M in (1, 3, 4, 8, 16):
        plan = TilePlan.for_length(L, M)
        ref = grid[f"L{L}_M{M}_lbm_y"]
        g64 = engine.lbm_scan_par(*p, plan)
        assert O.max_rel_err(g64.y, ref) <= 1e-12
        assert O.max_rel_err(g64.h_final, grid[f"L{L}_fwd_h"]) <= 1e-12
        g32 = engine.lbm_scan_par(*p32, plan)
        assert O.max_rel_err(g32.y, ref) <= TOL_F32
        rv = engine.lbm_scan_par_reverse(*p, plan)
        assert O.max_rel_err(rv.y, grid[f"L{L}_M{M}_rev_y"]) <= 1e-12
        assert O.max_rel_err(rv.h_final, grid[f"L{L}_M{M}_rev_h"]) <= 1e-12
    f = engine.forward_scan_par(*p, TilePlan.for_length(L, 4))
    assert O.max_rel_err(f.y, grid[f"L{L}_fwd_y"]) <= 1e-12


def test_prediscretized_bitwise_identities():
    """test_engine.py:98-114, fp64."""
    p = O.random_scan_params(O.seeded_rng(12), 2, 29, 2, 3)
    fwd = engine.forward_scan_par(*p, TilePlan.for_length(29, 4))
    lbm = engine.lbm_scan_par(*p, TilePlan.for_length(29, 4))
    for i in range(29):
        if (i + 1) % 4 == 0 or i == 28:
            np.testing.assert_array_equal(lbm.y[:, i], fwd.y[:, i])
    m1 = engine.lbm_scan_par(*p, TilePlan.for_length(29, 1))
    np.testing.assert_array_equal(m1.y, engine.forward_scan_par(*p, TilePlan.for_length(29, 1)).y)


def test_prediscretized_large_window_and_bidir():
    p = O.random_scan_params(O.seeded_rng(3), 2, 300, 3, 4)
    got = engine.lbm_scan_par(*p, TilePlan.for_length(300, 100))
    assert O.max_rel_err(got.y, O.lbm_scan(*p, 100)[0]) <= 1e-12
    pb = O.random_scan_params(O.seeded_rng(4), 2, 300, 3, 4)
    bid = engine.global_bidir_par(p, pb, TilePlan.for_length(300, 8))
    ry, rh = O.global_bidir_scan(p, pb)
    assert O.max_rel_err(bid.y, ry) <= 1e-12
    assert O.max_rel_err(bid.h_final, rh) <= 1e-12


def test_plan_consistency_checked():
    from paper_2506_15976_b200.errors import ShapeError
    p = O.random_scan_params(O.seeded_rng(0), 1, 8, 2, 2, dtype=np.float32)
    with pytest.raises(ShapeError):
        engine.forward_scan_par(*p, TilePlan(tile_len=4, num_tiles=7))


# --- conv ----------------------------------------------------------------------

@pytest.mark.parametrize("reverse", [False, True])
@pytest.mark.parametrize("K", [2, 3, 4])
def test_conv_fwd_bwd(reverse, K):
    from paper_2506_15976_b200.conv import causal_conv1d_silu_bwd, causal_conv1d_silu_fwd
    rng = O.seeded_rng(K + 10 * reverse)
    x = rng.standard_normal((2, 77, 50))
    w = rng.standard_normal((50, K)) * 0.5
    g = rng.standard_normal((2, 77, 50))
    flip = (lambda a: a[:, ::-1]) if reverse else (lambda a: a)
    xc = O.causal_conv1d(flip(x), w)
    ref = flip(O.silu(xc))
    got = causal_conv1d_silu_fwd(dev(x), dev(w), reverse=reverse).cpu().numpy()
    assert O.max_rel_err(got, ref) <= TOL_F32
    gx_ref, gw_ref = O.causal_conv1d_grad(flip(x), w, flip(g) * O.silu_grad(xc))
    dx, dw, _ = causal_conv1d_silu_bwd(dev(x), dev(w), None, dev(g), reverse=reverse)
    assert O.max_rel_err(dx.cpu().numpy(), flip(gx_ref)) <= TOL_F32
    assert O.max_rel_err(dw.cpu().numpy(), gw_ref) <= TOL_F32


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("K", [2, 4, 6])
@pytest.mark.parametrize("reverse", [False, True])
def test_conv_fwd_vectorised(dtype, K, reverse):
    """16-byte channel-group path (E % 8 == 0, aligned rows), input a column view of
    a wider projection output like the block's x = xz[..., :E]; L spans several
    64-step chunks plus a ragged one."""
    from paper_2506_15976_b200.conv import causal_conv1d_silu_fwd
    rng = O.seeded_rng(K + 7 * reverse)
    Bt, L, E = 3, 150, 64
    xz = dev(rng.standard_normal((Bt, L, 2 * E)), dtype)
    x = xz[..., :E]
    w = rng.standard_normal((E, K)) * 0.5
    xq = x.double().cpu().numpy()
    flip = (lambda a: a[:, ::-1]) if reverse else (lambda a: a)
    ref = flip(O.silu(O.causal_conv1d(flip(xq), w)))
    got = causal_conv1d_silu_fwd(x, dev(w), reverse=reverse).float().cpu().numpy()
    assert O.max_rel_err(got, ref) <= (TOL_F32 if dtype == torch.float32 else 1e-2)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("E", [256, 96])
@pytest.mark.parametrize("reverse", [False, True])
def test_conv_tile_kernels_fwd_bwd(dtype, E, reverse):
    """The 128-channel pair forward kernel (E % 128 == 0) / single-channel tile kernel
    (E = 96), and the tile-staged backward (K = 4, 64-channel tiles, partial tile at
    E = 96), on column views of a wider projection, L with a ragged 32-step chunk,
    with a bias; against the oracle on the same (rounded) inputs."""
    from paper_2506_15976_b200.conv import causal_conv1d_silu_bwd, causal_conv1d_silu_fwd
    rng = O.seeded_rng(E + 3 * reverse)
    Bt, L, K = 2, 101, 4
    xz = dev(rng.standard_normal((Bt, L, 2 * E)), dtype)
    x = xz[..., :E]
    gz = dev(rng.standard_normal((Bt, L, 2 * E)), dtype)
    g = gz[..., E:]
    w = rng.standard_normal((E, K)) * 0.5
    bias = rng.standard_normal(E) * 0.1
    xq, gq = x.double().cpu().numpy(), g.double().cpu().numpy()
    flip = (lambda a: a[:, ::-1]) if reverse else (lambda a: a)
    xc = O.causal_conv1d(flip(xq), w) + bias
    tol = TOL_F32 if dtype == torch.float32 else 1e-2
    got = causal_conv1d_silu_fwd(x, dev(w), dev(bias), reverse=reverse).double().cpu().numpy()
    assert O.max_rel_err(got, flip(O.silu(xc))) <= tol
    gpre = flip(gq) * O.silu_grad(xc)
    gx_ref, gw_ref = O.causal_conv1d_grad(flip(xq), w, gpre)
    dx, dw, db = causal_conv1d_silu_bwd(x, dev(w), dev(bias), g, reverse=reverse)
    assert O.max_rel_err(dx.double().cpu().numpy(), flip(gx_ref)) <= tol
    assert O.max_rel_err(dw.cpu().numpy(), gw_ref) <= (1e-4 if dtype == torch.float32 else 1e-2)
    assert O.max_rel_err(db.cpu().numpy(), gpre.sum((0, 1))) <= (1e-4 if dtype == torch.float32 else 1e-2)


def test_conv_golden():
    from paper_2506_15976_b200.conv import causal_conv1d_silu_bwd, causal_conv1d_silu_fwd
    g = np.load(os.path.join(GOLD, "conv.npz"))
    y = causal_conv1d_silu_fwd(dev(g["x"]), dev(g["k"]), silu=False).cpu().numpy()
    assert O.max_rel_err(y, g["y"]) <= TOL_F32
    dx, dw, _ = causal_conv1d_silu_bwd(dev(g["x"]), dev(g["k"]), None, dev(g["g"]), silu=False)
    assert O.max_rel_err(dx.cpu().numpy(), g["gx"]) <= TOL_F32
    assert O.max_rel_err(dw.cpu().numpy(), g["gk"]) <= TOL_F32


@pytest.mark.parametrize("dtype,D", [(torch.float32, 192), (torch.bfloat16, 192), (torch.bfloat16, 384),
                                     (torch.float32, 8), (torch.bfloat16, 1024)])
@pytest.mark.parametrize("rows", [1, 3 * 37, 4 * 64 + 3])
def test_rms_norm(dtype, D, rows):
    from paper_2506_15976_b200.norm import rms_norm
    rng = O.seeded_rng(D + rows)
    x = rng.standard_normal((1, rows, D))
    s = rng.uniform(0.5, 1.5, D)
    got = rms_norm(dev(x, dtype), dev(s)).float().cpu().numpy()
    xq = dev(x, dtype).double().cpu().numpy()
    ref = O.rms_norm(xq, s)
    assert O.max_rel_err(got, ref) <= (TOL_F32 if dtype == torch.float32 else 1e-2)


@pytest.mark.parametrize("N", [4, 8, 16])
def test_fused_vectorised_path_state_sizes(N):
    """E multiple of 8 (bf16) / 4 (fp32) with aligned rows -> cp.async staging path."""
    inp = op_inputs(40 + N, 2, 99, 16, N)
    for reverse in (False, True):
        got, hf = run_gpu(inp, window=8, reverse=reverse, return_last_state=True)
        ref, rhf = O.lbm_selective_scan(**inp, window=8, reverse=reverse, return_last_state=True)
        assert O.max_rel_err(got, ref) <= TOL_F32
        assert O.max_rel_err(hf, rhf) <= TOL_F32


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_global_bidir_fused(dtype):
    """Vim-style global bi-directional baseline (engine.global_bidir_par,
    engine.py:305-327) on the fused op: forward sweep + flip-on-load backward
    sweep with separate parameters, summed, gated."""
    from paper_2506_15976_b200.scan import global_bidir_selective_scan
    inp = op_inputs(50, 2, 150, 64, 16)
    pb = op_inputs(51, 2, 150, 64, 16)
    if dtype != torch.float32:
        inp = quantize(inp, dtype)
        pb = quantize(pb, dtype)
    t = {k: (dev(v, dtype) if k in ("u", "delta", "z", "B", "C") else dev(v)) for k, v in inp.items()}
    tb = {k: (dev(v, dtype) if k in ("delta", "B", "C") else dev(v)) for k, v in pb.items()}
    out, h = global_bidir_selective_scan(**t, delta_b=tb["delta"], A_b=tb["A"], B_b=tb["B"], C_b=tb["C"],
                                         D_b=tb["D"], delta_bias_b=tb["delta_bias"], return_last_state=True)
    fb = dict(inp, delta=pb["delta"], A=pb["A"], B=pb["B"], C=pb["C"], D=pb["D"], delta_bias=pb["delta_bias"])
    rf, hf = O.lbm_selective_scan(**inp, lb=False, return_last_state=True)
    rb, hb = O.lbm_selective_scan(**fb, lb=False, reverse=True, return_last_state=True)
    tol = TOL_F32 if dtype == torch.float32 else TOL_BF16
    assert O.max_rel_err(out.float().cpu().numpy(), rf + rb) <= tol
    assert O.max_rel_err(h.cpu().numpy(), hf + hb) <= tol


@pytest.mark.parametrize("S", [40, 700])
def test_many_segments_prefix(S):
    """Sequence split into many segments (more than one 512-segment round of the
    parallel prefix): equals the oracle."""
    inp = op_inputs(60 + S, 1, 16 * S + 5, 8, 16)
    for reverse in (False, True):
        got, hf = run_gpu(inp, window=16, reverse=reverse, return_last_state=True, seg_hint=S)
        ref, rhf = O.lbm_selective_scan(**inp, window=16, reverse=reverse, return_last_state=True)
        assert O.max_rel_err(got, ref) <= TOL_F32
        assert O.max_rel_err(hf, rhf) <= TOL_F32


@pytest.mark.parametrize("dtype,D", [(torch.float32, 192), (torch.bfloat16, 192), (torch.bfloat16, 384),
                                     (torch.float32, 64), (torch.bfloat16, 1024), (torch.float32, 6),
                                     (torch.bfloat16, 50), (torch.float32, 2048)])
@pytest.mark.parametrize("rows", [1, 3 * 37, 5000])
def test_rms_norm_bwd(dtype, D, rows):
    """lbs_rms_norm_bwd against torch autograd of the same formula in fp64 (on the same
    rounded inputs); dscale accumulated over rows by the fixed-order reduction."""
    from paper_2506_15976_b200.norm import rms_norm_bwd, rms_norm_train
    g = torch.Generator(device="cuda").manual_seed(rows + D)
    x = torch.randn(rows, D, device="cuda", generator=g).to(dtype)
    s = torch.randn(D, device="cuda", generator=g)
    dy = torch.randn(rows, D, device="cuda", generator=g).to(dtype)
    xd = x.double().requires_grad_(True)
    sd = s.double().requires_grad_(True)
    y = xd * torch.rsqrt((xd * xd).mean(-1, keepdim=True) + 1e-6) * sd
    y.backward(dy.double())
    dx, ds = rms_norm_bwd(x, s, dy)
    tol = 1e-5 if dtype == torch.float32 else 1e-2
    assert O.max_rel_err(dx.double().cpu().numpy(), xd.grad.cpu().numpy()) <= tol
    assert O.max_rel_err(ds.double().cpu().numpy(), sd.grad.cpu().numpy()) <= (1e-5 if dtype == torch.float32 else 1e-3)
    # deterministic, and the autograd Function routes through the same kernels
    dx2, ds2 = rms_norm_bwd(x, s, dy)
    assert torch.equal(dx, dx2) and torch.equal(ds, ds2)
    xr = x.clone().requires_grad_(True)
    sr = s.clone().requires_grad_(True)
    rms_norm_train(xr, sr).backward(dy)
    assert torch.equal(xr.grad, dx) and torch.equal(sr.grad, ds)


@pytest.mark.parametrize("D", [192, 384, 8, 1024])
@pytest.mark.parametrize("rows", [1, 3 * 37, 5000])
def test_rms_norm_f32_in_bf16_out(D, rows):
    """lbs_rms_norm_fwd with out_dtype bf16 for fp32 rows: bitwise the fp32 result rounded
    to bf16 (the training block's bf16 projection input, no separate cast)."""
    from paper_2506_15976_b200.norm import rms_norm
    g = torch.Generator(device="cuda").manual_seed(rows + D)
    x = torch.randn(rows, D, device="cuda", generator=g)
    s = torch.rand(D, device="cuda", generator=g) + 0.5
    got = rms_norm(x, s, out_dtype=torch.bfloat16)
    assert got.dtype == torch.bfloat16
    assert torch.equal(got, rms_norm(x, s).to(torch.bfloat16))


@pytest.mark.parametrize("dtype,D", [(torch.float32, 384), (torch.bfloat16, 192), (torch.float32, 6)])
def test_rms_norm_bwd_residual(dtype, D):
    """lbs_rms_norm_bwd with dres: dx + dres in one pass, equal to the separate add."""
    from paper_2506_15976_b200.norm import rms_norm_bwd
    g = torch.Generator(device="cuda").manual_seed(D)
    x = torch.randn(777, D, device="cuda", generator=g).to(dtype)
    s = torch.randn(D, device="cuda", generator=g)
    dy = torch.randn(777, D, device="cuda", generator=g).to(dtype)
    res = torch.randn(777, D, device="cuda", generator=g).to(dtype)
    dx, ds = rms_norm_bwd(x, s, dy)
    dxr, dsr = rms_norm_bwd(x, s, dy, dres=res)
    assert torch.equal(ds, dsr)
    ref = (dx.float() + res.float())
    tol = 1e-6 if dtype == torch.float32 else 1e-2
    assert ((dxr.float() - ref).abs().max() / ref.abs().max()).item() <= tol
