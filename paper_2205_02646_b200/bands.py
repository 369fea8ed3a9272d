"""Row-band partitioning for one-process-per-GPU runs.

The padded image's block rows [0, padM/B) are split into `world` contiguous bands of
floor/ceil(nbr/world) rows. A band needs the frame rows its (clamped, GLOBAL)
window origins touch -- a 14 px (7 frame row) halo at the defaults -- and writes a
disjoint slice of output rows, so no collective sits on the data path. Class
selection uses global origins (origin mod P), so every band reproduces exactly the
per-block arithmetic of the whole-frame run.
"""
from __future__ import annotations

import math


def padded_rows(frame_rows: int, block: int) -> int:
    step = math.lcm(block, 2)
    return -(-2 * frame_rows // step) * step


def band(frame_rows: int, block: int, rank: int, world: int) -> tuple[int, int]:
    """Block-row band [br0, br1) of `rank`."""
    nbr = padded_rows(frame_rows, block) // block
    return rank * nbr // world, (rank + 1) * nbr // world


def band_frame_rows(frame_rows: int, window: int, block: int, br0: int, br1: int) -> tuple[int, int]:
    """Frame rows [f0, f1) the band's windows read (halo included, clamped)."""
    padM = padded_rows(frame_rows, block)
    lead = (window - block) // 2
    if br1 <= br0:
        return 0, 0
    omin = min(max(br0 * block - lead, 0), padM - window)
    omax = min(max((br1 - 1) * block - lead, 0), padM - window)
    return min(omin // 2, frame_rows - 1), min(frame_rows, (omax + window - 1) // 2 + 1)


def band_output_rows(frame_rows: int, block: int, br0: int, br1: int) -> tuple[int, int]:
    return br0 * block, min(br1 * block, 2 * frame_rows)
