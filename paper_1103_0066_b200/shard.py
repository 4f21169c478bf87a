"""Element-range sharding.

Elements are independent and the store is element-major, so a contiguous,
tile-aligned slot range per device/rank produces exactly the corresponding
contiguous slice of the store; concatenating shard outputs reproduces the
single-device store bitwise.  No collective is needed on the data path.

``shard_bounds`` is the split the C ABI uses for ``devices=[...]``
(csrc/fb_capi.cpp run_job); ``rank_elements`` is the weak-scaling slice
bench.py gives each torchrun rank.
"""
from __future__ import annotations

TILE = 288  # fbk::kTile: shard boundaries stay tile (and 16-byte) aligned


def shard_bounds(nslots: int, parts: int, tile: int = TILE):
    """[b_0=0, b_1, ..., b_P=nslots]: contiguous tile-aligned slot ranges."""
    if parts < 1:
        raise ValueError("parts must be >= 1")
    tiles = -(-nslots // tile)
    return [min(nslots, tiles * g // parts * tile) for g in range(parts + 1)]


def rank_elements(ne_per_rank: int, rank: int):
    """Weak scaling: rank r owns elements [r*ne, (r+1)*ne) of the global mesh."""
    return rank * ne_per_rank, (rank + 1) * ne_per_rank
