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
