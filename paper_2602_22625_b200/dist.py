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


def sum_bands(srcs: list[torch.Tensor], dsts: list[torch.Tensor] | None = None,
              begin: int = 0, end: int | None = None, stream=None) -> None:
    """Fixed-order sum of float64 band buffers into every destination
    (pf_sum_bands; in place when ``dsts`` is None).  Stream-ordered, capturable."""
    import ctypes as C

    from . import _native as nat
    from .compositor import _stream_handle

    dsts = srcs if dsts is None else dsts
    count = srcs[0].numel()
    if any(t.dtype != torch.float64 or t.numel() != count for t in list(srcs) + list(dsts)):
        raise ValueError("band buffers must be float64 of one size")
    end = count if end is None else end
    s_arr = (C.c_void_p * len(srcs))(*[t.data_ptr() for t in srcs])
    d_arr = (C.c_void_p * len(dsts))(*[t.data_ptr() for t in dsts])
    nat.check(nat.load().pf_sum_bands(s_arr, len(srcs), d_arr, len(dsts), int(begin), int(end),
                                      _stream_handle(stream)), "pf_sum_bands")


class LocalBandGroup:
    """Every row band of an N-way split on ONE device: the single-GPU stand-in
    for the N-rank step (tests, projections).  One step = each band's render
    (bin + fit step into its own gradient + loss buffer), the fixed-order band
    sum (pf_sum_bands, in place), then each band's Adam + next records --
    exactly the ranks' sequence with the allreduce replaced by a device kernel,
    so the whole group step can be captured in one CUDA graph."""

    def __init__(self, scene, cfg, loss_spec, total: int, world: int, *, row_cost=None,
                 use_graph: bool = True, device=None):
        from .fit import StepEngine

        nty = -(-scene.canvas_h // 16)
        self.bands = row_bands(nty, world, row_cost)
        self.engines = [StepEngine(scene, cfg, loss_spec, total, band=b, use_graph=False,
                                   device=device) for b in self.bands]
        self.use_graph = use_graph
        self.graph = None
        self.done = 0

    def launch_step(self) -> None:
        for e in self.engines:
            e.launch_render(reduced=True)
        sum_bands([e.gbuf for e in self.engines])
        for e in self.engines:
            e.launch_update()

    def step(self) -> None:
        if self.graph is not None:
            self.graph.replay()
        else:
            if self.done == 0:
                for e in self.engines:
                    e.refresh()
            self.launch_step()
            if self.use_graph:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    self.launch_step()
                self.graph = g
        self.done += 1
        for e in self.engines:
            e.done = self.done
