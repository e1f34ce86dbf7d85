"""Multi-GPU row-band sharding.

Every rank holds the full parameter replica, renders a band of tile rows,
produces partial gradients + partial loss sums into one float64 buffer, and a
single sum-allreduce (NCCL over NVLink/NVSwitch) makes every replica's Adam
step identical.  Bands are balanced by a per-tile-row cost computed
identically on every rank from replicated state (no communication).
"""

from __future__ import annotations

import numpy as np
import torch

from .compositor import Band


def row_bands(nty: int, world: int, row_cost: np.ndarray | None = None) -> list[Band]:
    """Split tile rows [0, nty) into `world` contiguous bands of ~equal cost.

    row_cost[ty] is the work of tile row ty (e.g. sum over its tiles of
    256 * list length); None = uniform.  Every band gets >= 1 row when
    nty >= world.
    """
    if world < 1:
        raise ValueError("world must be >= 1")
    if world == 1:
        return [Band(0, nty)]
    cost = np.ones(nty) if row_cost is None else np.asarray(row_cost, dtype=np.float64) + 1e-9
    csum = np.concatenate(([0.0], np.cumsum(cost)))
    total = csum[-1]
    cuts = [0]
    for r in range(1, world):
        c = int(np.searchsorted(csum, total * r / world, side="left"))
        lo = cuts[-1] + 1
        hi = nty - (world - r)
        cuts.append(int(min(max(c, lo), hi)))
    cuts.append(nty)
    return [Band(cuts[i], cuts[i + 1]) for i in range(world)]


def row_cost_from_bins(bin_off: np.ndarray, ntx: int, nty: int) -> np.ndarray:
    """Per tile-row cost = sum of list lengths of its tiles (full-canvas bins)."""
    lens = np.diff(np.asarray(bin_off, dtype=np.int64)).reshape(nty, ntx)
    return lens.sum(axis=1).astype(np.float64) + 1.0


def make_allreduce(group=None):
    """Sum-allreduce of the gradient + loss buffer (stream-ordered, capturable)."""
    import torch.distributed as dist

    def _ar(buf: torch.Tensor) -> None:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)

    return _ar
