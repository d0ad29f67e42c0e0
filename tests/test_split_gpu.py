"""Parity of the sequence-split launch plans with the CPU oracle (-m gpu).

When few (batch row, channel block) pairs exist, both kernels cut the sequence
into segments so more CTAs run: the forward enters segment s with the state
folded from the earlier segments' affine aggregates h -> P h + H (core.py:48-55),
the backward enters it with the carry mu = a*lam of the global adjoint folded
from the later segments' maps mu -> P mu + M (autodiff.py:125-137).  The LB
record and its adjoint are tile-local and segments are whole chunks of whole
tiles, so nothing else crosses a segment boundary.  These tests force every
segment count the planner could pick (seg_hint) and check the automatic plan
on the shapes that take it (configs[0], an 8-way batch shard of configs[2])."""

import numpy as np
import pytest

from helpers import TOL_F32, TOL_GRAD, op_inputs
from oracle import lbscan_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2506_15976_b200.scan import lbm_selective_scan_bwd, lbm_selective_scan_fwd  # noqa: E402

SEQ = ("u", "delta", "z", "B", "C")
GRADS = ("du", "ddelta", "dA", "dB", "dC", "dD", "dz", "ddelta_bias")


def dev(x, dtype=torch.float32):
    return None if x is None else torch.as_tensor(np.ascontiguousarray(x), dtype=dtype, device="cuda")


def tens(inp, dtype=torch.float32):
    return {k: (dev(v, dtype) if k in SEQ else dev(v)) for k, v in inp.items()}


def np_grads(g):
    return {k: (None if v is None else v.float().cpu().numpy()) for k, v in g.items()}


def check(got, ref, tol, what):
    for k in GRADS:
        if ref[k] is None:
            assert got[k] is None, (what, k)
            continue
        err = O.max_rel_err(got[k], ref[k])
        assert err <= tol, f"{what} {k}: max rel err {err:.3e} > {tol}"


@pytest.mark.parametrize("L", [64, 197, 300])
@pytest.mark.parametrize("M", [1, 3, 8, 16])
@pytest.mark.parametrize("S", [1, 2, 3, 7])
def test_bwd_forced_segments(L, M, S):
    inp = op_inputs(500 + L + 7 * M + S, 2, L, 40, 16)
    dout = O.seeded_rng(L + M).standard_normal((2, L, 40))
    for reverse in (False, True):
        g = np_grads(lbm_selective_scan_bwd(dev(dout), **tens(inp), window=M, reverse=reverse, seg_hint=S))
        ref = O.lbm_selective_scan_bwd(dout, **inp, window=M, reverse=reverse)
        check(g, ref, TOL_GRAD, f"L={L} M={M} S={S} rev={reverse}")


@pytest.mark.parametrize("S", [2, 5, 32])
def test_bwd_segments_options(S):
    """linear discretisation, no gate, no bias, N=4 — through split plans."""
    inp = op_inputs(77 + S, 3, 150, 24, 4)
    dout = O.seeded_rng(S).standard_normal((3, 150, 24))
    for drop, mode in (("z", "exp"), ("delta_bias", "exp"), (None, "linear")):
        x = dict(inp)
        if drop:
            x[drop] = None
        if mode == "linear":
            x["A"] = -np.abs(inp["A"]) * 0.05  # contractive decay a = dl*A (block.py:94)
        g = np_grads(lbm_selective_scan_bwd(dev(dout), **tens(x), window=4, discretize_mode=mode, seg_hint=S))
        ref = O.lbm_selective_scan_bwd(dout, **x, window=4, mode=mode)
        check(g, ref, TOL_GRAD, f"S={S} drop={drop} mode={mode}")


def test_bwd_split_checkpoints_equal_recompute_and_deterministic():
    """Training-forward checkpoints vs the checkpoint-only recompute sweep under the
    automatic split plan: bitwise equal gradients, and bitwise repeatable."""
    inp = op_inputs(9, 2, 197, 96, 16)
    t = tens(inp)
    dout = dev(O.seeded_rng(3).standard_normal((2, 197, 96)))
    _, ck = lbm_selective_scan_fwd(**t, window=8, save_checkpoints=True)
    g1 = np_grads(lbm_selective_scan_bwd(dout, **t, window=8, checkpoints=ck))
    g2 = np_grads(lbm_selective_scan_bwd(dout, **t, window=8))
    g3 = np_grads(lbm_selective_scan_bwd(dout, **t, window=8))
    for k in GRADS:
        np.testing.assert_array_equal(g1[k], g2[k], err_msg=k)
        np.testing.assert_array_equal(g2[k], g3[k], err_msg=k)
    ref = O.lbm_selective_scan_bwd(O.seeded_rng(3).standard_normal((2, 197, 96)), **inp, window=8)
    check(g1, ref, TOL_GRAD, "auto split")


def test_auto_split_shard_shape():
    """A batch shard of configs[2] (few rows, L=197): the automatic plan splits the
    sequence in both directions; fp32 forward at 1e-5, gradients at 1e-4."""
    inp = op_inputs(31, 4, 197, 256, 16)
    t = tens(inp)
    dout = O.seeded_rng(5).standard_normal((4, 197, 256))
    for reverse in (False, True):
        y = lbm_selective_scan_fwd(**t, window=8, reverse=reverse).cpu().numpy()
        assert O.max_rel_err(y, O.lbm_selective_scan(**inp, window=8, reverse=reverse)) <= TOL_F32
        g = np_grads(lbm_selective_scan_bwd(dev(dout), **t, window=8, reverse=reverse))
        check(g, O.lbm_selective_scan_bwd(dout, **inp, window=8, reverse=reverse), TOL_GRAD, f"rev={reverse}")


@pytest.mark.parametrize("L,S", [(197, 1), (197, 4), (197, 25), (600, 38)])
def test_fwd_short_sequence_segments(L, S):
    """configs[0] shape with forced segment counts: <= 32 segments fold their
    aggregates inside the main pass, more go through the prefix kernel."""
    inp = op_inputs(0, 2, L, 192, 16)
    t = tens(inp)
    for reverse in (False, True):
        y, hf = lbm_selective_scan_fwd(**t, window=8, reverse=reverse, return_last_state=True, seg_hint=S)
        ref, rhf = O.lbm_selective_scan(**inp, window=8, reverse=reverse, return_last_state=True)
        assert O.max_rel_err(y.cpu().numpy(), ref) <= TOL_F32
        assert O.max_rel_err(hf.cpu().numpy(), rhf) <= TOL_F32


@pytest.mark.parametrize("dt", ["fp32"])  # the launch plan uses TMA staging for fp32 I/O
@pytest.mark.parametrize("E", [384, 200, 64])
def test_tma_staging_bitwise_equals_cp_async(dt, E):
    """The forward's TMA tensor-copy staging (3-D maps over (E, L, B), reverse direction
    read back from physically ordered rows, out-of-bounds columns of a partial channel
    block zero-filled) gives bitwise the results of the cp.async staging: outputs, last
    state and checkpoints, both directions, LB and forward-only, contiguous inputs and
    the LBVim block's strided views (delta, B, C column slices of one projection)."""
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    g = torch.Generator(device="cuda").manual_seed(E)
    # enough rows that the launch plan does not split the sequence (TMA staging is
    # used for unsplit launches; seg_hint=3 below checks a split launch as well)
    Bt, L, N = {384: 4, 200: 6, 64: 20}[E], 197, 16
    proj = torch.randn(Bt, L, E + 2 * N + 32, generator=g, device="cuda").to(tdt)
    xz = torch.randn(Bt, L, 2 * E, generator=g, device="cuda").to(tdt)
    base = dict(A=-torch.rand(E, N, generator=g, device="cuda") * N - 0.5, D=torch.ones(E, device="cuda"),
                delta_bias=torch.full((E,), -3.0, device="cuda"))
    cases = {"views": dict(u=xz[..., :E], delta=proj[..., :E], B=proj[..., E:E + N], C=proj[..., E + N:E + 2 * N],
                           z=xz[..., E:]),
             "contiguous": dict(u=xz[..., :E].contiguous(), delta=proj[..., :E].contiguous(),
                                B=proj[..., E:E + N].contiguous(), C=proj[..., E + N:E + 2 * N].contiguous(), z=None)}
    for name, x in cases.items():
        for reverse in (False, True):
            for lb in (True, False):
                for seg in (0, 3):
                    kw = dict(window=8, reverse=reverse, lb=lb, return_last_state=True, save_checkpoints=True,
                              seg_hint=seg)
                    y1, h1, c1 = lbm_selective_scan_fwd(**x, **base, **kw)
                    y0, h0, c0 = lbm_selective_scan_fwd(**x, **base, **kw, tma=False)
                    assert torch.equal(y1, y0) and torch.equal(h1, h0) and torch.equal(c1, c0), \
                        (name, reverse, lb, seg)


@pytest.mark.parametrize("S", [33, 120, 250])
def test_bwd_many_segments_prefix_path(S):
    """More than 32 backward segments: the adjoint-carry maps are stored right to left
    and folded by the parallel segment prefix (the long-bag training case)."""
    inp = op_inputs(900 + S, 1, 2000, 40, 16)
    dout = O.seeded_rng(S).standard_normal((1, 2000, 40))
    for reverse in (False, True):
        g = np_grads(lbm_selective_scan_bwd(dev(dout), **tens(inp), window=8, reverse=reverse, seg_hint=S))
        ref = O.lbm_selective_scan_bwd(dout, **inp, window=8, reverse=reverse)
        check(g, ref, TOL_GRAD, f"S={S} rev={reverse}")


def test_bwd_long_bag_shard_auto_plan():
    """One channel shard of the configs[4] bag shape at a reduced length (E=64, L=20k,
    window 16): the automatic plan splits the backward into hundreds of segments."""
    inp = op_inputs(77, 1, 20000, 64, 16)
    dout = O.seeded_rng(78).standard_normal((1, 20000, 64))
    g = np_grads(lbm_selective_scan_bwd(dev(dout), **tens(inp), window=16))
    check(g, O.lbm_selective_scan_bwd(dout, **inp, window=16), TOL_GRAD, "bag shard")
