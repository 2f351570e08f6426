"""Host-side mirror of the packed Delta layout (csrc/jofc_layout.h).

Used by the sharding plan, bench.py's byte accounting and the CPU tests of
the multi-GPU partition.  Row blocks of 128 rows x column tiles of 64 columns,
block (B, J) stored for J >= 2B, stream order (modality, B, J); a shard owns
a contiguous range of the stream of equal estimated pass-kernel cost
(block_cost, the model of csrc/jofc_capi.cu: make_layout / pass_bounds).
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


BAND_COST = 1.0  # a row band entered: flush, X row-block staging, two CTA barriers
MASK_COST = 0.1  # diagonal-crossing or padded block (masked pairs)


def block_cost(n, B, J, enters_band):
    masked = J <= 2 * B + 1 or COLS * (J + 1) > n or ROWS * (B + 1) > n
    return 1.0 + (MASK_COST if masked else 0.0) + (BAND_COST if enters_band else 0.0)


def shard_range(m, n, rank, world):
    """[begin, end) stream indices owned by `rank`: equal estimated cost, the
    same cut (same summation order) as make_layout in csrc/jofc_capi.cu."""
    nT, nB, bpm = geometry(n)
    total = m * bpm
    if world == 1:
        return 0, total
    cost = [block_cost(n, B, J, J == 2 * B)
            for _ in range(m) for B in range(nB) for J in range(2 * B, nT)]
    s = 0.0
    for v in cost:
        s += v
    lo, hi, acc = 0, total, 0.0
    for g, v in enumerate(cost):
        acc += v
        if rank > 0 and lo == 0 and acc >= s * rank / world:
            lo = g + 1
        if acc >= s * (rank + 1) / world and rank + 1 < world:
            hi = g + 1
            break
    return lo, hi


def blocks(m, n, rank=0, world=1):
    """Yield (l, B, J) of this shard's blocks in stream order."""
    nT, _, bpm = geometry(n)
    lo, hi = shard_range(m, n, rank, world)
    for g in range(lo, hi):
        yield block_coords(g, nT, bpm)


def packed_bytes(m, n, rank=0, world=1):
    lo, hi = shard_range(m, n, rank, world)
    return (hi - lo) * ROWS * COLS * 8
