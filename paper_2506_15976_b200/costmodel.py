"""Analytic scan / model cost counters with the reference's conventions
(costmodel.py:1-227): the closed-form numbers its engine tallies and its
``bench`` CSV reports (cli/__init__.py:182-218), so a report from this package
lines up column for column with one from the reference.

Conventions (costmodel.py:1-17): a multiply or add is 1 flop, a multiply-add
2, exp / softplus / SiLU / GELU 4; HBM traffic is unique element loads and
stores of the reference's pre-discretised contract (abar, bx, c, dx in;
y, h_final out); a tile exchange is one serial carry hand-off between
consecutive tiles of one (b, e, n) lane.  The global bi-directional baseline
is exactly two forward sweeps.

These are the REFERENCE engine's counters (an emulated machine), kept for
like-for-like reports.  The fused B200 kernels never materialise abar/bx;
their own algorithmic bytes are ``fused_scan_bytes``.
"""

from __future__ import annotations

import io
from dataclasses import dataclass, field

from .errors import ShapeError

ELEMWISE_FLOPS = 4  # costmodel.py:23
VARIANTS = ("forward", "lbm", "global_bidir")
_COUNTERS = ("flops", "hbm_reads", "hbm_writes", "tile_exchanges", "register_ops")


@dataclass
class CostReport:
    """costmodel.py:26-66: counter bundle for one scan call or model forward."""

    variant: str
    flops: int = 0
    hbm_reads: int = 0
    hbm_writes: int = 0
    tile_exchanges: int = 0
    register_ops: int = 0
    breakdown: dict = field(default_factory=dict, repr=False)

    def __post_init__(self):
        bad = [k for k in _COUNTERS if getattr(self, k) < 0]
        if bad:
            raise ValueError(f"{bad[0]} must be >= 0")

    def __add__(self, other: "CostReport") -> "CostReport":
        name = self.variant if self.variant == other.variant else f"{self.variant}+{other.variant}"
        parts = dict(self.breakdown)
        for k, v in other.breakdown.items():
            parts[k] = parts.get(k, 0) + v
        return CostReport(name, *(getattr(self, k) + getattr(other, k) for k in _COUNTERS), breakdown=parts)

    def counters(self) -> dict:
        return {k: getattr(self, k) for k in _COUNTERS}


def _lb_record_flops_per_lane(L: int, M: int) -> int:
    """In-tile reverse record of one lane (costmodel.py:75-87): a tile of r >= 2
    steps costs 3r - 4 (r-1 decay multiplies, r-1 adds into the state, r-2
    injection adds); 1-step tiles cost nothing."""

    def tile(r: int) -> int:
        return 3 * r - 4 if r >= 2 else 0

    n_full, tail = divmod(L, M)
    return n_full * tile(M) + tile(tail)


def count_scan_cost(variant: str, B: int, L: int, E: int, N: int, M: int) -> CostReport:
    """costmodel.py:90-144: closed-form counters of one engine call.

    Per lane: in-tile pair scan 3 flops/step, serial carry over the T-1 tile
    hand-offs 3 flops each, carry application 3 flops/step; per (b, l, e) the
    output contraction 2N + 1.  "lbm" adds the in-register record; the
    bidirectional baseline doubles every forward counter.
    """
    if min(B, L, E, N, M) < 1:
        raise ShapeError("all dimensions and the tile length must be >= 1")
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r}")
    lanes = B * E * N
    hand_offs = -(-L // M) - 1
    phases = {
        "intile": 3 * L * lanes,
        "exchange": 3 * hand_offs * lanes,
        "apply": 3 * L * lanes,
        "output": (2 * N + 1) * B * L * E,
    }
    sweep_flops = sum(phases.values())
    reads = 2 * L * lanes + B * L * N + B * L * E  # abar, bx, c, dx
    writes = B * L * E + lanes  # y, h_final
    sweeps = 2 if variant == "global_bidir" else 1
    record = _lb_record_flops_per_lane(L, M) * lanes if variant == "lbm" else 0
    flops = sweeps * sweep_flops + record
    breakdown = {k: sweeps * v for k, v in phases.items()}
    breakdown["backward"] = record
    return CostReport(variant=variant, flops=flops, hbm_reads=sweeps * reads, hbm_writes=sweeps * writes,
                      tile_exchanges=sweeps * hand_offs * lanes,
                      register_ops=flops - breakdown["exchange"], breakdown=breakdown)


def _gemm(L: int, d_in: int, d_out: int) -> int:
    return 2 * L * d_in * d_out


def count_model_cost(config) -> CostReport:
    """costmodel.py:151-202: per-image flops of backbone + head (ModelConfig from
    this package or the reference); HBM / exchange counters are the scan's × depth."""
    D, E, N, depth = config.embed_dim, config.inner_dim, config.state_dim, config.depth
    L, M, k = config.seq_len, config.resolved_tile_len, config.conv_width
    patch_in = config.patch_size ** 2 * config.in_channels
    scan = count_scan_cost(config.scan_variant, 1, L, E, N, M)
    ew = ELEMWISE_FLOPS
    block = (L * (4 * D + 6)                      # RMSNorm
             + 2 * _gemm(L, D, E)                 # x / z projections
             + L * E * 2 * k + L * E * ew         # depthwise causal conv + SiLU
             + 2 * _gemm(L, E, N)                 # B / C projections
             + _gemm(L, E, E) + L * E             # delta projection + bias
             + L * E * ew                         # softplus
             + L * E * N * (1 + ew)               # abar = exp(delta A)
             + 2 * L * E * N + L * E              # bx, D skip
             + scan.flops
             + L * E * (ew + 1)                   # y * SiLU(z)
             + _gemm(L, E, D) + L * D)            # out projection + residual
    flops = _gemm(config.num_patches, patch_in, D) + L * D + depth * block
    if config.head == "gap":
        flops += L * D
    else:  # MAP head: K, V projections, scores, softmax, weighted pooling
        flops += 2 * _gemm(L, D, D) + 2 * L * D + L * config.map_heads * ew + 2 * L * D
    hidden = 4 * D
    flops += _gemm(1, D, hidden) + hidden * ew + _gemm(1, hidden, config.num_classes)
    return CostReport(variant=config.scan_variant, flops=flops, hbm_reads=depth * scan.hbm_reads,
                      hbm_writes=depth * scan.hbm_writes, tile_exchanges=depth * scan.tile_exchanges,
                      register_ops=flops - depth * scan.breakdown["exchange"],
                      breakdown={"per_block": block, "scan_per_block": scan.flops})


def reports_to_csv(reports) -> str:
    """costmodel.py:205-213."""
    buf = io.StringIO()
    buf.write(",".join(("variant",) + _COUNTERS) + "\n")
    for r in reports:
        buf.write(",".join([r.variant] + [str(getattr(r, k)) for k in _COUNTERS]) + "\n")
    return buf.getvalue()


def format_table(reports) -> str:
    """costmodel.py:216-227: fixed-width text table (header left-, cells right-aligned)."""
    head = ("variant",) + _COUNTERS
    rows = [[r.variant] + [str(getattr(r, k)) for k in _COUNTERS] for r in reports]
    w = [max([len(h)] + [len(row[i]) for row in rows]) for i, h in enumerate(head)]
    out = ["  ".join(h.ljust(w[i]) for i, h in enumerate(head))]
    out += ["  ".join(c.rjust(w[i]) for i, c in enumerate(row)) for row in rows]
    return "\n".join(out)


def fused_scan_bytes(B: int, L: int, E: int, N: int, s_io: int, s_bc: int, *, has_z: bool = True,
                     last_state: bool = False) -> int:
    """Algorithmic HBM bytes of one fused ``lbs_scan_fwd`` call:
    u, delta (+z) and out per (b, l, e), B and C per (b, l), A, D, bias once."""
    per_bl = s_io * E * (3 if has_z else 2) + s_bc * 2 * N + s_io * E
    return B * L * per_bl + 4 * (E * N + 2 * E) + (4 * B * E * N if last_state else 0)
