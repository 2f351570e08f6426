"""Host-side mirror of the packed Delta layout (csrc/jofc_layout.h).

Used by the sharding plan, bench.py's byte accounting and the CPU tests of
the multi-GPU partition.  Row blocks of 128 rows x column tiles of 64 columns,
block (B, J) stored for J >= 2B, stream order (modality, B, J); a shard owns
a balanced contiguous range of the stream.
"""
from __future__ import annotations

import math

ROWS, COLS = 128, 64


def geometry(n):
    nT = (n + COLS - 1) // COLS
    nB = (nT + 1) // 2
    return nT, nB, row_first(nT, nB)


def row_first(nT, B):
    return B * nT - B * (B - 1)


def block_coords(g, nT, bpm):
    l, r = divmod(g, bpm)
    b = nT + 1.0
    B = int((b - math.sqrt(max(b * b - 4.0 * r, 0.0))) * 0.5)
    nB = (nT + 1) // 2
    B = min(max(B, 0), nB - 1)
    while B > 0 and row_first(nT, B) > r:
        B -= 1
    while B + 1 < nB and row_first(nT, B + 1) <= r:
        B += 1
    return l, B, 2 * B + (r - row_first(nT, B))


def shard_range(m, n, rank, world):
    """[begin, end) stream indices owned by `rank` (balanced by block count)."""
    _, _, bpm = geometry(n)
    total = m * bpm
    return total * rank // world, total * (rank + 1) // world


def blocks(m, n, rank=0, world=1):
    """Yield (l, B, J) of this shard's blocks in stream order."""
    nT, _, bpm = geometry(n)
    lo, hi = shard_range(m, n, rank, world)
    for g in range(lo, hi):
        yield block_coords(g, nT, bpm)


def packed_bytes(m, n, rank=0, world=1):
    lo, hi = shard_range(m, n, rank, world)
    return (hi - lo) * ROWS * COLS * 8
