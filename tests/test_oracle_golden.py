"""Pin the CPU oracle (test infrastructure) against golden vectors produced by
the unmodified reference (oracle/gen_golden.py).  CPU only."""

import os

import numpy as np
import pytest

from oracle import lbscan_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return np.load(os.path.join(GOLD, f"{name}.npz"))


GRID_L = (1, 5, 31, 128, 129, 197, 256, 257)
GRID_M = (1, 3, 4, 8, 16)


@pytest.fixture(scope="module")
def grid():
    return load("scan_grid")


def test_random_scan_params_reproduces_reference_draws(grid):
    for L in GRID_L:
        abar, bx, c, dx = O.random_scan_params(O.seeded_rng(L), 2, L, 3, 4)
        np.testing.assert_array_equal(abar, grid[f"L{L}_abar"])
        np.testing.assert_array_equal(bx, grid[f"L{L}_bx"])
        np.testing.assert_array_equal(c, grid[f"L{L}_c"])
        np.testing.assert_array_equal(dx, grid[f"L{L}_dx"])


@pytest.mark.parametrize("L", GRID_L)
def test_forward_and_lbm_match_reference_oracle(grid, L):
    p = [grid[f"L{L}_{k}"] for k in ("abar", "bx", "c", "dx")]
    y, h = O.forward_scan(*p)
    assert O.max_rel_err(y, grid[f"L{L}_fwd_y"]) <= 1e-13
    assert O.max_rel_err(h, grid[f"L{L}_fwd_h"]) <= 1e-13
    for M in GRID_M:
        y, h = O.lbm_scan(*p, M)
        assert O.max_rel_err(y, grid[f"L{L}_M{M}_lbm_y"]) <= 1e-13, M
        # the reference's fp32 engine agrees with its oracle within its own bar
        assert O.max_rel_err(grid[f"L{L}_M{M}_engine32_y"], y) <= 1e-5


@pytest.mark.parametrize("L", GRID_L)
def test_reverse_direction_matches_reference_engine(grid, L):
    """engine._run(reverse=True) == flip . lbm . flip (tiles aligned in scan order)."""
    p = [grid[f"L{L}_{k}"][:, ::-1] for k in ("abar", "bx", "c", "dx")]
    for M in GRID_M:
        y, h = O.lbm_scan(*p, M)
        assert O.max_rel_err(y[:, ::-1], grid[f"L{L}_M{M}_rev_y"]) <= 1e-12, M
        assert O.max_rel_err(h, grid[f"L{L}_M{M}_rev_h"]) <= 1e-12, M


def test_scan_grad_matches_reference_autodiff():
    g = load("scan_grads")
    for i in range(4):
        L, M, B, E, N, seed = g[f"c{i}_meta"]
        p = [g[f"c{i}_{k}"] for k in ("abar", "bx", "c")]
        gy = g[f"c{i}_gy"]
        ga, gb, gc, gdx = O.lbm_scan_grad(*p, gy, int(M))
        for name, got in (("abar", ga), ("bx", gb), ("c", gc), ("dx", gdx)):
            assert O.max_rel_err(got, g[f"c{i}_g_{name}"]) <= 1e-12, (i, name)
        ga, gb, gc, gdx = O.lbm_scan_grad(*p, gy, 1, local=False)
        for name, got in (("abar", ga), ("bx", gb), ("c", gc), ("dx", gdx)):
            assert O.max_rel_err(got, g[f"c{i}_gf_{name}"]) <= 1e-12, (i, name)


def _block(g, i):
    D, E, N, L, B, M, k, linear, rev, seed = [int(v) for v in g[f"b{i}_meta"]]
    w = {f: g[f"b{i}_w_{f}"] for f in O.BLOCK_FIELDS}
    return dict(D=D, E=E, N=N, L=L, B=B, M=M, k=k, mode="linear" if linear else "exp",
                rev=bool(rev)), w


@pytest.mark.parametrize("i", range(4))
def test_block_forward_matches_reference(i):
    g = load("block")
    meta, w = _block(g, i)
    out, inter = O.block_forward(g[f"b{i}_T"], w, meta["M"], reverse=meta["rev"],
                                 mode=meta["mode"], return_intermediates=True)
    assert O.max_rel_err(out, g[f"b{i}_out"]) <= 1e-12
    assert O.max_rel_err(inter["xs"], g[f"b{i}_cache_xs"]) <= 1e-13
    # fused-op oracle on the reference's own block intermediates
    xs, z = g[f"b{i}_cache_xs"], g[f"b{i}_cache_z"]
    yg = O.lbm_selective_scan(xs, xs @ w["w_delta"], -np.exp(w["a_log"]), xs @ w["w_b"],
                              xs @ w["w_c"], D=w["d_param"], z=z, delta_bias=w["delta_bias"],
                              window=meta["M"], mode=meta["mode"])
    assert O.max_rel_err(yg, g[f"b{i}_cache_yg"]) <= 1e-12


@pytest.mark.parametrize("i", range(4))
def test_fused_backward_matches_reference_block_backward(i):
    """The fused-op adjoint (du, ddelta, dA, dB, dC, dD, dz, ddelta_bias) mapped
    onto the block's weights reproduces block.block_backward exactly."""
    g = load("block")
    meta, w = _block(g, i)
    T = g[f"b{i}_T"]
    gout = g[f"b{i}_gout"]
    if meta["rev"]:
        gout = gout[:, ::-1]
    xs, z, x, xc = (g[f"b{i}_cache_{k}"] for k in ("xs", "z", "x", "xc"))
    A = -np.exp(w["a_log"])
    dout = gout @ w["w_out"].T
    r = O.lbm_selective_scan_bwd(dout, xs, xs @ w["w_delta"], A, xs @ w["w_b"], xs @ w["w_c"],
                                 D=w["d_param"], z=z, delta_bias=w["delta_bias"],
                                 window=meta["M"], mode=meta["mode"])
    xT = lambda a, b: np.tensordot(a, b, axes=((0, 1), (0, 1)))
    xn = O.rms_norm(T, w["norm_scale"])
    got = {
        "d_param": r["dD"], "delta_bias": r["ddelta_bias"], "a_log": r["dA"] * A,
        "w_b": xT(xs, r["dB"]), "w_c": xT(xs, r["dC"]), "w_delta": xT(xs, r["ddelta"]),
        "w_z": xT(xn, r["dz"]),
    }
    g_xs = r["du"] + r["ddelta"] @ w["w_delta"].T + r["dB"] @ w["w_b"].T + r["dC"] @ w["w_c"].T
    _, got["conv_kernel"] = O.causal_conv1d_grad(x, w["conv_kernel"], g_xs * O.silu_grad(xc))
    for name, v in got.items():
        assert O.max_rel_err(v, g[f"b{i}_g_{name}"]) <= 1e-10, name


def test_conv_matches_reference():
    g = load("conv")
    assert O.max_rel_err(O.causal_conv1d(g["x"], g["k"]), g["y"]) <= 1e-14
    gx, gk = O.causal_conv1d_grad(g["x"], g["k"], g["g"])
    assert O.max_rel_err(gx, g["gx"]) <= 1e-14
    assert O.max_rel_err(gk, g["gk"]) <= 1e-14


@pytest.mark.parametrize("i", range(3))
def test_model_forward_matches_reference(i):
    g = load("model")
    pre = f"m{i}_"
    cfg = {k[len(pre) + 4:]: g[k].item() for k in g.files if k.startswith(pre + "cfg_")}
    if cfg.get("tile_len") == "auto":
        cfg["tile_len"] = None
    cfg["tile_len"] = None if cfg["tile_len"] in (None, "auto") else int(cfg["tile_len"])
    params = {k[len(pre) + 2:]: g[k] for k in g.files if k.startswith(pre + "p_")}
    logits = O.model_forward(g[pre + "images"], cfg, params)
    assert O.max_rel_err(logits, g[pre + "logits"]) <= 1e-11


def test_bidir_matches_reference():
    g = load("bidir")
    pf = [g["f_" + k] for k in ("abar", "bx", "c", "dx")]
    pb = [g["b_" + k] for k in ("abar", "bx", "c", "dx")]
    y, h = O.global_bidir_scan(pf, pb)
    assert O.max_rel_err(y, g["y"]) <= 1e-13
    assert O.max_rel_err(h, g["h"]) <= 1e-13


# -- structural properties the reference's own oracle tests assert ----------

def test_tile_rule():
    """test_engine.py:11-19."""
    assert [O.select_tile_len(L) for L in (1024, 257, 256, 200, 129, 128, 64, 1)] == \
        [16, 16, 8, 8, 8, 4, 4, 4]


def test_m1_and_tile_end_identities():
    """test_oracle.py:154-168 (tile ends) and :169-175 (M=1 == forward)."""
    p = O.random_scan_params(O.seeded_rng(16), 2, 12, 3, 4)
    yf, _ = O.forward_scan(*p)
    for M in (1, 2, 3, 4, 5):
        y, _ = O.lbm_scan(*p, M)
        for i in range(12):
            if i == O.tile_end(i, 12, M):
                np.testing.assert_array_equal(y[:, i], yf[:, i])


def test_fused_bwd_matches_finite_differences():
    """Independent check of the fused adjoint chain (test_autodiff.py:8-47 style)."""
    rng = O.seeded_rng(3)
    Bt, L, E, N, M = 1, 7, 2, 3, 3
    u = rng.standard_normal((Bt, L, E))
    dl = 0.3 * rng.standard_normal((Bt, L, E))
    A = -rng.uniform(0.5, 2.0, (E, N))
    Bm = rng.standard_normal((Bt, L, N))
    C = rng.standard_normal((Bt, L, N))
    D = rng.standard_normal(E)
    z = rng.standard_normal((Bt, L, E))
    bias = rng.standard_normal(E) * 0.1
    dout = rng.standard_normal((Bt, L, E))
    for rev in (False, True):
        args = dict(u=u, delta=dl, A=A, B=Bm, C=C, D=D, z=z, delta_bias=bias)

        def f():
            return float(np.sum(dout * O.lbm_selective_scan(**args, window=M, reverse=rev)))

        r = O.lbm_selective_scan_bwd(dout, **args, window=M, reverse=rev)
        for key, gk in (("u", "du"), ("delta", "ddelta"), ("A", "dA"), ("B", "dB"), ("C", "dC"),
                        ("D", "dD"), ("z", "dz"), ("delta_bias", "ddelta_bias")):
            x = args[key]
            num = np.zeros_like(x)
            fl, nf = x.reshape(-1), num.reshape(-1)
            for j in range(fl.size):
                o = fl[j]
                fl[j] = o + 1e-6
                fp = f()
                fl[j] = o - 1e-6
                fm = f()
                fl[j] = o
                nf[j] = (fp - fm) / 2e-6
            assert O.max_rel_err(r[gk], num) <= 1e-6, (rev, key)
