"""Multi-process partitioning logic on CPU: world size 2, gloo,
127.0.0.1 rendezvous.  The per-shard scan is the CPU oracle (test
infrastructure); on the GPU box the same code runs the CUDA op over NCCL."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import op_inputs
from oracle import lbscan_oracle as O
from paper_2506_15976_b200.sharding import batch_shard, channel_sharded_scan, shard_range


def oracle_scan(u, delta, A, B, C, D, z, delta_bias, window, reverse, delta_softplus):
    n = lambda t: None if t is None else t.double().numpy()  # noqa: E731
    y = O.lbm_selective_scan(n(u), n(delta), n(A), n(B), n(C), D=n(D), z=n(z), delta_bias=n(delta_bias),
                             window=window, reverse=reverse, delta_softplus=delta_softplus)
    return torch.from_numpy(np.ascontiguousarray(y))


def test_shard_range_covers_exactly():
    for n in (1, 5, 64, 512, 513):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def test_batch_shard():
    x = torch.arange(10).reshape(10, 1)
    got = torch.cat([batch_shard(x, 4, r) for r in range(4)])
    assert torch.equal(got, x)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, E, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _body(rank, world, E, q)
    except Exception as exc:  # surface worker failures instead of timing out
        q.put(("error", repr(exc)))
        raise
    finally:
        dist.destroy_process_group()


def _body(rank, world, E, q):
    if True:
        inp = op_inputs(5, 1, 300, E, 16)
        t = {k: torch.from_numpy(np.ascontiguousarray(v)) for k, v in inp.items()}
        full = channel_sharded_scan(**t, window=16, gather="full", scan_fn=oracle_scan)
        pooled = channel_sharded_scan(**t, window=16, gather="pooled", scan_fn=oracle_scan)
        lo, hi = shard_range(E, world, rank)
        loc = {k: (v[..., lo:hi] if k in ("u", "delta", "z") else v[lo:hi] if k in ("A", "D", "delta_bias") else v)
               for k, v in t.items()}
        local = channel_sharded_scan(**loc, window=16, gather="full", scan_fn=oracle_scan, inputs_are_local=True)
        if rank == 0:
            q.put((full.numpy(), pooled.numpy(), local.numpy()))


@pytest.mark.parametrize("E", [64, 37])
def test_channel_sharded_scan_gloo_world2(E):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, E, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    assert not (isinstance(res[0], str) and res[0] == "error"), res
    full, pooled, local = res
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    inp = op_inputs(5, 1, 300, E, 16)
    ref = O.lbm_selective_scan(**inp, window=16)
    assert O.max_rel_err(full, ref) <= 1e-12
    assert O.max_rel_err(local, ref) <= 1e-12
    assert O.max_rel_err(pooled, ref.mean(1)) <= 1e-12
