"""Backward API (drop-in for pkg/src/primfit/grad.py) on the CUDA path.

``backward`` (grad.py:134-187) keeps the reference's checks -- fingerprint
staleness, dL/dI and dL/dA shapes, background identity -- and then runs the
K4 kernel, which replaces backward_tiles + reduce_partials
(_kernels.py:258-363, grad.py:190-206).  The finite-difference and dense
reference backwards are oracles and live under ``oracle/``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .errors import LengthMismatch, ShapeMismatch, StaleSavedState
from .compositor import pixels4
from .raster import SavedForward, resolve_background
from .scene import FloatArray, scene_fingerprint


@dataclass(eq=False)
class Gradients:
    """Per-primitive gradients, columns = PARAM_GROUPS (reference grad.py:58-102)."""

    data: FloatArray  # (N, 8)

    @classmethod
    def zeros(cls, n: int) -> "Gradients":
        return cls(np.zeros((n, 8)))

    @property
    def n_primitives(self) -> int:
        return int(self.data.shape[0])

    @property
    def x(self):
        return self.data[:, 0]

    @property
    def y(self):
        return self.data[:, 1]

    @property
    def scale(self):
        return self.data[:, 2]

    @property
    def rotation(self):
        return self.data[:, 3]

    @property
    def opacity_logit(self):
        return self.data[:, 4]

    @property
    def color_logits(self):
        return self.data[:, 5:8]

    def to_vector(self) -> FloatArray:
        return self.data.reshape(-1).copy()


def reduce_partials(per_tile_partials: list[Gradients]) -> Gradients:
    """Elementwise sum in list order (reference grad.py:190-206; host utility)."""
    if not per_tile_partials:
        raise LengthMismatch("no partials to reduce")
    n = per_tile_partials[0].n_primitives
    acc = np.zeros((n, 8))
    for part in per_tile_partials:
        if part.n_primitives != n:
            raise LengthMismatch(f"partial has {part.n_primitives} primitives, expected {n}")
        acc += part.data
    return Gradients(acc)


def backward(scene, saved: SavedForward, dL_dI: FloatArray, dL_dA: FloatArray | None = None,
             background=None) -> Gradients:
    """Pixel-loss gradients -> per-primitive parameter gradients on the GPU."""
    if saved.fingerprint != scene_fingerprint(scene):
        raise StaleSavedState("saved forward state is for a different scene")
    H, W = scene.canvas_h, scene.canvas_w
    dL_dI = np.asarray(dL_dI, dtype=np.float64)
    if dL_dI.shape != (H, W, 3):
        raise ShapeMismatch(f"dL_dI shape {dL_dI.shape} != {(H, W, 3)}")
    if dL_dA is not None:
        dL_dA = np.asarray(dL_dA, dtype=np.float64)
        if dL_dA.shape != (H, W):
            raise ShapeMismatch(f"dL_dA shape {dL_dA.shape} != {(H, W)}")
    if background is not None:
        bg = resolve_background(scene, background)
        if not np.array_equal(bg, saved.background):
            raise StaleSavedState("background differs from the one composited in the forward")
    comp = saved.compositor
    dev = comp.device
    d4 = torch.from_numpy(pixels4(dL_dI, dL_dA)).to(dev)
    grads = torch.zeros(comp.n * 8 + 4, dtype=torch.float64, device=dev)
    rgb = saved.bg_rgb if saved.bg_rgb is not None else (0.0, 0.0, 0.0)
    comp.backward(d4, grads, bg_rgb=rgb, bg4=saved.bg4)
    return Gradients(grads[: comp.n * 8].view(comp.n, 8).cpu().numpy())
