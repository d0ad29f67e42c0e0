"""torch.library registration of the fused scan (torch_ops.py): the op exists with
a fake implementation on CPU; on the GPU it equals the eager operator, its autograd
formula equals LbmSelectiveScanFn's gradients, and torch.library.opcheck passes."""

import pytest
import torch

from paper_2506_15976_b200 import torch_ops  # noqa: F401  (registers torch.ops.lbscan.*)


def _inputs(device, dtype=torch.float32, B=2, L=37, E=16, N=4, seed=0, grad=False):
    g = torch.Generator(device=device).manual_seed(seed)
    r = lambda *s: torch.randn(*s, generator=g, device=device, dtype=torch.float32)  # noqa: E731
    t = dict(u=r(B, L, E).to(dtype), delta=(0.5 * r(B, L, E)).to(dtype),
             A=-torch.arange(1, N + 1, device=device, dtype=torch.float32).repeat(E, 1),
             B=r(B, L, N).to(dtype), C=r(B, L, N).to(dtype), D=torch.ones(E, device=device),
             z=r(B, L, E).to(dtype), delta_bias=torch.full((E,), -3.0, device=device))
    if grad:
        for k in t:
            t[k] = t[k].detach().requires_grad_(True)
    return t


def test_op_registered_with_fake_impl():
    assert hasattr(torch.ops.lbscan, "lbm_selective_scan")
    from torch._subclasses.fake_tensor import FakeTensorMode
    with FakeTensorMode():
        x = _inputs("cpu")
        y = torch.ops.lbscan.lbm_selective_scan(x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"],
                                                x["delta_bias"], True, 8, False)
        assert y.shape == x["u"].shape and y.dtype == x["u"].dtype


@pytest.mark.gpu
@pytest.mark.parametrize("reverse", [False, True])
def test_op_matches_eager_and_autograd(reverse):
    from paper_2506_15976_b200.scan import lbm_selective_scan
    x = _inputs("cuda", grad=True)
    y = torch.ops.lbscan.lbm_selective_scan(x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"],
                                            x["delta_bias"], True, 8, reverse)
    x2 = {k: v.detach().clone().requires_grad_(True) for k, v in x.items()}
    y2 = lbm_selective_scan(**x2, window=8, reverse=reverse)
    assert torch.equal(y, y2)
    dy = torch.randn_like(y)
    y.backward(dy)
    y2.backward(dy)
    for k in x:
        ref = x2[k].grad
        err = ((x[k].grad - ref).abs().max() / ref.abs().max().clamp_min(1e-30)).item()
        assert err < 1e-5, (k, err)


@pytest.mark.gpu
def test_opcheck():
    x = _inputs("cuda", grad=True)
    args = (x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"], x["delta_bias"], True, 8, False)
    torch.library.opcheck(torch.ops.lbscan.lbm_selective_scan.default, args,
                          test_utils=("test_schema", "test_autograd_registration", "test_faketensor"))
