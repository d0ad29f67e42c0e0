"""MambaMIL-style bag pipeline (paper_2506_15976_b200/mil.py) on the channel-sharded
LB scan.  CPU: world-size 1 and 2 over gloo with the oracle scan as the per-shard
scan — both ranks must return the single-process logits (the all_reduce of the
x_proj partials and the all_gather of the pooled features are the only
exchanges).  GPU: the fused kernels (bf16 and fp32) against a plain torch
composition around the oracle scan."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import lbscan_oracle as O
from paper_2506_15976_b200.errors import ShapeError
from paper_2506_15976_b200.mil import MILBag, MILConfig, init_mil_params


def oracle_scan(u, delta, A, B, C, D, z, delta_bias, window, reverse, delta_softplus):
    n = lambda t: None if t is None else t.double().cpu().numpy()  # noqa: E731
    y = O.lbm_selective_scan(n(u), n(delta), n(A), n(B), n(C), D=n(D), z=n(z), delta_bias=n(delta_bias),
                             window=window, reverse=reverse, delta_softplus=delta_softplus)
    return torch.from_numpy(np.ascontiguousarray(y)).to(u.device)


def torch_conv(x, w, b):
    # reference tap order (nn.py:87-99): out[l] = b + sum_q w[e, q] x[l - q], then SiLU
    x = x.double()
    L, K = x.shape[1], w.shape[1]
    acc = b.double().expand_as(x).clone()
    for q in range(K):
        acc[:, q:] += w[:, q].double() * x[:, :L - q]
    return acc * torch.sigmoid(acc)


def torch_norm(x, scale):
    x = x.double()
    return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + 1e-6) * scale.double()


CPU_FNS = dict(scan_fn=oracle_scan, conv_fn=torch_conv, norm_fn=torch_norm)
CFG = MILConfig(d_in=24, dim=12, state_dim=4, dt_rank=3, num_classes=3)
L_BAG = 37


def _bag(cfg, L, seed=5):
    g = torch.Generator().manual_seed(seed)
    return torch.randn(L, cfg.d_in, generator=g, dtype=torch.float64)


def test_mil_single_process_cpu():
    p = init_mil_params(CFG, seed=1)
    X = _bag(CFG, L_BAG)
    out = MILBag(CFG, p, dtype=torch.float64, **CPU_FNS)(X)
    assert out.shape == (CFG.num_classes,) and torch.isfinite(out).all()
    # pooling before the out projection == projecting every instance then pooling (linearity)
    m = MILBag(CFG, p, dtype=torch.float64, **CPU_FNS)
    with pytest.raises(ShapeError):
        m(torch.zeros(2, L_BAG, CFG.d_in, dtype=torch.float64))
    with pytest.raises(ShapeError):
        m(torch.zeros(L_BAG, CFG.d_in + 1, dtype=torch.float64))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = init_mil_params(CFG, seed=1)
        out = MILBag(CFG, p, dtype=torch.float64, **CPU_FNS)(_bag(CFG, L_BAG))
        q.put((rank, out.numpy()))
    except Exception as exc:
        q.put(("error", repr(exc)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_mil_channel_sharded_gloo(world):
    want = MILBag(CFG, init_mil_params(CFG, seed=1), dtype=torch.float64, **CPU_FNS)(_bag(CFG, L_BAG)).numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = {}
    for _ in range(world):
        k, v = q.get(timeout=120)
        assert k != "error", v
        got[k] = v
    for pr in procs:
        pr.join(timeout=60)
    for r in range(world):
        np.testing.assert_allclose(got[r], want, rtol=1e-10, atol=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-4), (torch.bfloat16, 3e-2)])
def test_mil_gpu_matches_torch_oracle(dtype, tol):
    cfg = MILConfig(d_in=64, dim=128, state_dim=16, dt_rank=8, num_classes=2)
    p = init_mil_params(cfg, seed=2)
    X = _bag(cfg, 1000, seed=3).float()
    got = MILBag(cfg, {k: v.cuda() for k, v in p.items()}, dtype=dtype)(X.cuda()).cpu().double()
    # reference: same composition in fp64 on the CPU, oracle scan; bf16 run compared on
    # the bf16-rounded weights and bag
    pr = {k: (v.to(dtype).double() if dtype == torch.bfloat16 and k in ("w_fc", "w_in", "w_xproj", "w_dt")
              else v.double()) for k, v in p.items()}
    Xr = X.to(dtype).double()
    want = MILBag(cfg, pr, dtype=torch.float64, **CPU_FNS)(Xr)
    err = (got - want).abs().max() / want.abs().max()
    assert err < tol, (err, got, want)
