"""Tile (local window) rule and plan — mirror of engine.select_tile_len /
engine.TilePlan (engine.py:54-85)."""

from __future__ import annotations

from dataclasses import dataclass

from .errors import ShapeError


def select_tile_len(L: int) -> int:
    """engine.py:54-62: M = 16 if L > 256, 8 if 128 < L <= 256, else 4."""
    if L < 1:
        raise ShapeError(f"sequence length must be >= 1, got {L}")
    if L > 256:
        return 16
    if L > 128:
        return 8
    return 4


@dataclass(frozen=True)
class TilePlan:
    """engine.py:65-85."""

    tile_len: int
    num_tiles: int

    @classmethod
    def for_length(cls, L: int, tile_len: int | None = None) -> "TilePlan":
        if L < 1:
            raise ShapeError(f"sequence length must be >= 1, got {L}")
        m = select_tile_len(L) if tile_len in (None, "auto") else int(tile_len)
        if m < 1:
            raise ShapeError(f"tile length must be >= 1, got {m}")
        return cls(tile_len=m, num_tiles=-(-L // m))

    def check(self, L: int) -> None:
        if self.num_tiles != -(-L // self.tile_len):
            raise ShapeError(f"plan ({self.tile_len} x {self.num_tiles}) inconsistent with L={L}")
