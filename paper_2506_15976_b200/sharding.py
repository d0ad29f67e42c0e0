"""Multi-GPU partitioning of the LB scan.

Lanes (b, e, n) of the scan are independent (engine.py:94-99: the reference
already partitions work over batch x channel blocks), so the scan itself never
needs a collective:

* ``batch_shard`` — LBVim configs: each rank owns ``B / world`` rows; weights
  replicated; no data-path collective at all.
* ``channel_sharded_scan`` — long MambaMIL bags (B = 1, L ~ 1e5): each rank
  scans a contiguous block of ``E / world`` channels with B and C replicated;
  the only exchange is ONE ``all_gather`` of the per-rank outputs (or of the
  per-rank pooled features, ``gather="pooled"``), over NCCL on the GPU box.

``scan_fn`` defaults to the fused CUDA operator; it is a parameter only so the
host-side partitioning logic can be exercised by world-size-2 gloo tests on a
CPU-only machine with the CPU oracle as the per-shard scan.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .errors import ShapeError


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of ``n`` items for ``rank`` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ShapeError(f"bad rank {rank} for world size {world}")
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def batch_shard(x: torch.Tensor, world: int, rank: int) -> torch.Tensor:
    """Rows of the global batch owned by ``rank`` (weak or strong scaling)."""
    lo, hi = shard_range(x.shape[0], world, rank)
    return x[lo:hi]


def _default_scan(**kw):
    from .scan import lbm_selective_scan
    return lbm_selective_scan(**kw)


def channel_sharded_scan(u, delta, A, B, C, D=None, z=None, delta_bias=None, *, window=None,
                         reverse=False, delta_softplus=True, gather="full", group=None,
                         scan_fn=None, inputs_are_local=False):
    """LB scan of a (B, L, E) problem partitioned over the ranks of ``group`` by channel.

    ``u, delta, z`` and the per-channel ``A, D, delta_bias`` are either the full
    tensors (each rank slices its block) or, with ``inputs_are_local=True``, this
    rank's channel block already.  ``B, C`` (B, L, N) are replicated.

    ``gather="full"``   -> (B, L, E) output on every rank (one all_gather of
                            (B, L, E/world) blocks);
    ``gather="pooled"`` -> (B, E) mean over L on every rank (all_gather of (B, E/world));
    ``gather="none"``   -> this rank's (B, L, E/world) block, no collective.
    """
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    scan_fn = scan_fn or _default_scan
    if gather not in ("full", "pooled", "none"):
        raise ShapeError(f"unknown gather mode {gather!r}")
    if inputs_are_local:
        E_loc = u.shape[-1]
        sizes = [None] * world
        if dist.is_initialized() and world > 1:
            t = torch.tensor([E_loc], device=u.device)
            got = [torch.zeros_like(t) for _ in range(world)]
            dist.all_gather(got, t, group=group)
            sizes = [int(g.item()) for g in got]
        else:
            sizes = [E_loc]
        sl = lambda x: x  # noqa: E731
    else:
        E = u.shape[-1]
        lo, hi = shard_range(E, world, rank)
        sizes = [shard_range(E, world, r)[1] - shard_range(E, world, r)[0] for r in range(world)]
        sl = lambda x: None if x is None else x[..., lo:hi]  # noqa: E731
        sl0 = lambda x: None if x is None else x[lo:hi]  # noqa: E731
        A, D, delta_bias = sl0(A), sl0(D), sl0(delta_bias)
    y = scan_fn(u=sl(u), delta=sl(delta), A=A, B=B, C=C, D=D, z=sl(z), delta_bias=delta_bias,
                window=window, reverse=reverse, delta_softplus=delta_softplus)
    if gather == "none" or world == 1:
        return y.mean(1) if gather == "pooled" else y
    if gather == "pooled":
        y = y.mean(1)
    # one all_gather of equal-size blocks (ragged channel counts are padded to the
    # largest block and trimmed after)
    smax = max(sizes)
    if y.shape[-1] < smax:
        y = torch.nn.functional.pad(y, (0, smax - y.shape[-1]))
    y = y.contiguous()
    out = torch.empty((world * y.shape[0],) + tuple(y.shape[1:]), dtype=y.dtype, device=y.device)
    dist.all_gather_into_tensor(out, y, group=group)
    parts = out.view((world,) + tuple(y.shape)).unbind(0)
    return torch.cat([p[..., :s] for p, s in zip(parts, sizes)], dim=-1)
