"""Regression: the backward's dB/dC block sums must ignore threads past the last
channel (E % 128 != 0) even when the shared memory they read holds NaN from an
earlier kernel (found by running after kernels that leave NaN in shared memory)."""

import pytest
import torch


@pytest.mark.gpu
@pytest.mark.parametrize("E", [16, 100, 200])
def test_bwd_partial_cta_ignores_stale_shared_memory(E):
    from paper_2506_15976_b200.scan import lbm_selective_scan_bwd, lbm_selective_scan_fwd
    # leave NaN in shared memory: a forward over NaN inputs with full 128-channel CTAs
    n = torch.full((2, 64, 256), float("nan"), device="cuda")
    Bn = torch.full((2, 64, 16), float("nan"), device="cuda")
    lbm_selective_scan_fwd(n, n, -torch.ones(256, 16, device="cuda"), Bn, Bn, z=n, window=8)
    g = torch.Generator(device="cuda").manual_seed(E)
    B, L, N = 2, 37, 4
    r = lambda *s: torch.randn(*s, generator=g, device="cuda")  # noqa: E731
    x = dict(u=r(B, L, E), delta=0.5 * r(B, L, E), A=-torch.arange(1, N + 1, device="cuda").float().repeat(E, 1),
             B=r(B, L, N), C=r(B, L, N), D=torch.ones(E, device="cuda"), z=r(B, L, E),
             delta_bias=torch.full((E,), -3.0, device="cuda"))
    dy = r(B, L, E)
    for ck in (None, lbm_selective_scan_fwd(**x, window=8, save_checkpoints=True)[1]):
        lbm_selective_scan_fwd(n, n, -torch.ones(256, 16, device="cuda"), Bn, Bn, z=n, window=8)
        gr = lbm_selective_scan_bwd(dy, **x, window=8, checkpoints=ck)
        for k, v in gr.items():
            if v is not None:
                assert torch.isfinite(v).all(), k


def _poison():
    from paper_2506_15976_b200.scan import lbm_selective_scan_fwd
    n = torch.full((2, 64, 256), float("nan"), device="cuda")
    Bn = torch.full((2, 64, 16), float("nan"), device="cuda")
    lbm_selective_scan_fwd(n, n, -torch.ones(256, 16, device="cuda"), Bn, Bn, z=n, window=8)


@pytest.mark.gpu
@pytest.mark.parametrize("E", [16, 100, 200])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_partial_ctas_after_poison_fwd_and_conv(E, dtype):
    """Forward scan and conv1d+SiLU (fwd/bwd) on partial channel tiles right after a
    kernel left NaN in shared memory: every output finite and equal to a clean run."""
    from paper_2506_15976_b200.conv import causal_conv1d_silu_bwd, causal_conv1d_silu_fwd
    from paper_2506_15976_b200.scan import lbm_selective_scan_fwd
    g = torch.Generator(device="cuda").manual_seed(E + 1)
    B, L, N = 2, 53, 16
    r = lambda *s: torch.randn(*s, generator=g, device="cuda")  # noqa: E731
    x = dict(u=r(B, L, E).to(dtype), delta=(0.5 * r(B, L, E)).to(dtype),
             A=-torch.arange(1, N + 1, device="cuda").float().repeat(E, 1),
             B=r(B, L, N).to(dtype), C=r(B, L, N).to(dtype), D=torch.ones(E, device="cuda"),
             z=r(B, L, E).to(dtype), delta_bias=torch.full((E,), -3.0, device="cuda"))
    w = r(E, 4)
    dy = r(B, L, E).to(dtype)
    clean = (lbm_selective_scan_fwd(**x, window=8), causal_conv1d_silu_fwd(x["u"], w),
             causal_conv1d_silu_bwd(x["u"], w, None, dy)[:2])
    _poison()
    y = lbm_selective_scan_fwd(**x, window=8)
    _poison()
    c = causal_conv1d_silu_fwd(x["u"], w)
    _poison()
    dx, dw, _ = causal_conv1d_silu_bwd(x["u"], w, None, dy)
    assert torch.equal(y, clean[0]) and torch.equal(c, clean[1])
    assert torch.equal(dx, clean[2][0]) and torch.equal(dw, clean[2][1])
