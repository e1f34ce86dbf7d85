"""Forward renderer API (drop-in for pkg/src/primfit/raster.py) on the CUDA path.

Same entry points, argument meaning and errors as the reference:
``bin_tiles`` (raster.py:227-265), ``render_forward`` (raster.py:290-363),
``resolve_background`` (273-287), ``noisy_background`` (268-270),
``bbox_half_side`` (222-224) and the ``TileBins`` / ``SavedForward`` /
``RenderOutput`` result types.  All pixel work runs in the sm_100a kernels
behind the C ABI (include/primfit_b200.h); this module validates, uploads and
downloads.  ``render_naive`` is deliberately absent: it is the reference's
oracle, and the oracle lives under ``oracle/`` (test infrastructure only).

Differences by design: the GPU always renders on 16x16 tiles
(output is tile-size independent, reference SPEC.md:192), so a ``bins``
argument is validated for canvas shape and otherwise only documents intent;
``SavedForward`` keeps the per-pixel contribution lists in HBM instead of
host CSR arrays.
"""

from __future__ import annotations

import math
import weakref
from dataclasses import dataclass, field

import numpy as np
import torch

from .compositor import (POOL, RENDER_TILE, Compositor, DeviceAtlas, bin_capacity, cached_atlas,
                         pixels4)
from .errors import ShapeMismatch
from .scene import NOISE_BACKGROUND, FloatArray, param_matrix, scene_fingerprint, structure_arrays, validate_scene

DEFAULT_TILE_SIZE = 32
DEFAULT_TILE_PADDING = 2.0
DEFAULT_EPS_SKIP = 1.0 / 1024.0


@dataclass(eq=False)
class TileBins:
    """Per-tile front-to-back primitive lists in CSR form (reference raster.py:99-119)."""

    tile_size: int
    padding: float
    canvas_w: int
    canvas_h: int
    n_tiles_x: int
    n_tiles_y: int
    offsets: np.ndarray  # int64 (n_tiles + 1,)
    indices: np.ndarray  # int32 primitive indices, ascending z per tile

    @property
    def n_tiles(self) -> int:
        return self.n_tiles_x * self.n_tiles_y

    def tile_list(self, tx: int, ty: int) -> np.ndarray:
        t = ty * self.n_tiles_x + tx
        return self.indices[self.offsets[t] : self.offsets[t + 1]]


@dataclass(eq=False)
class RenderOutput:
    color: FloatArray  # (H, W, 3)
    alpha: FloatArray  # (H, W)


@dataclass(eq=False)
class SavedForward:
    """Forward state the backward replays (reference raster.py:122-148).

    The contribution lists live in HBM inside ``compositor`` (list position +
    incoming transmittance per contributing entry); ``t_final`` and
    ``background`` are host copies like the reference's.
    """

    canvas_w: int
    canvas_h: int
    compositor: Compositor
    t_final: FloatArray
    background: FloatArray
    bg_rgb: tuple | None
    bg4: torch.Tensor | None
    fingerprint: str
    eps_skip: float
    n_entries: int = field(default=0)


def bbox_half_side(scale: float, aspect: float = 1.0, padding: float = 0.0) -> float:
    """Conservative half side for any rotation (reference raster.py:222-224)."""
    return scale * math.hypot(1.0, max(1.0, aspect)) + padding


def noisy_background(w: int, h: int, rng: np.random.Generator) -> FloatArray:
    """Uniform noise canvas from the caller's PCG64 stream (reference raster.py:268-270)."""
    return rng.random((h, w, 3))


def resolve_background(scene, background=None) -> FloatArray:
    """Normalise a background argument to (H, W, 3) float64 (reference raster.py:273-287)."""
    if background is None:
        if isinstance(scene.background, str) and scene.background == NOISE_BACKGROUND:
            raise ValueError(
                "scene wants a noise background; sample one with noisy_background and pass it in"
            )
        background = scene.background
    bg = np.asarray(background, dtype=np.float64)
    if bg.shape == (3,):
        bg = np.broadcast_to(bg, (scene.canvas_h, scene.canvas_w, 3)).copy()
    if bg.shape != (scene.canvas_h, scene.canvas_w, 3):
        raise ShapeMismatch(f"background shape {bg.shape} does not fit the canvas")
    return np.ascontiguousarray(bg)


def _solid_rgb(scene, background):
    """(r, g, b) when the background is one colour, else None."""
    if background is None:
        bgv = scene.background
        if isinstance(bgv, str):
            return None
        return tuple(float(v) for v in np.asarray(bgv, dtype=np.float64))
    a = np.asarray(background, dtype=np.float64)
    if a.shape == (3,):
        return tuple(float(v) for v in a)
    return None


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2602_22625_b200 renders on a CUDA device; none is available")
    return torch.device("cuda")


def make_compositor(scene, *, padding: float, bin_tile: int = RENDER_TILE,
                    params: np.ndarray | None = None, device=None) -> tuple[Compositor, torch.Tensor]:
    """Upload a scene and size a compositor whose capacity bounds this scene's bins
    (a fresh one; the per-call API leases pooled ones through lease_compositor)."""
    comp, d_params, _ = lease_compositor(scene, padding=padding, bin_tile=bin_tile,
                                         params=params, device=device)
    return comp, d_params


def lease_compositor(scene, *, padding: float, bin_tile: int = RENDER_TILE,
                     params: np.ndarray | None = None, device=None):
    """(compositor, device params, release) for one call: the atlas is cached by
    template content and the compositor comes from the per-structure pool;
    ``release()`` returns it once its buffers are no longer needed."""
    dev = device or _device()
    pm = param_matrix(scene) if params is None else params
    tid, z = structure_arrays(scene)
    atlas = cached_atlas(scene.templates, bool(scene.preserve_aspect), dev)
    ntx = -(-scene.canvas_w // bin_tile)
    nty = -(-scene.canvas_h // bin_tile)
    cap = bin_capacity(pm[:, 2] if len(pm) else np.zeros(0), tid, atlas.hyp, padding,
                       bin_tile, ntx, nty)
    tid32 = np.ascontiguousarray(tid, dtype=np.int32)
    z64 = np.ascontiguousarray(z, dtype=np.int64)
    key = (id(atlas), tid32.tobytes(), z64.tobytes(), scene.canvas_w, scene.canvas_h,
           float(scene.alpha_max), float(scene.mu_blend), float(padding), int(bin_tile), str(dev))

    def factory(capacity):
        return Compositor(tid32, z64, atlas, scene.canvas_w, scene.canvas_h,
                          alpha_max=scene.alpha_max, mu_blend=scene.mu_blend, padding=padding,
                          capacity=capacity, bin_tile=bin_tile, device=dev)

    comp = POOL.acquire(key, cap, factory)
    d_params = torch.from_numpy(np.ascontiguousarray(pm, dtype=np.float64)).to(dev)
    return comp, d_params, (lambda: POOL.release(key, comp))


def bin_tiles(scene, tile_size: int = DEFAULT_TILE_SIZE,
              padding: float = DEFAULT_TILE_PADDING) -> TileBins:
    """GPU tile binning (K1 + K2), bit-identical to the reference's bin_tiles."""
    validate_scene(scene)
    comp, d_params, release = lease_compositor(scene, padding=padding, bin_tile=tile_size)
    try:
        comp.preprocess(d_params)
        comp.bin()
        k = comp.check_overflow()
        offsets = comp.bin_off.cpu().numpy().astype(np.int64)
        indices = comp.bin_idx[:k].cpu().numpy().astype(np.int32)
    finally:
        release()
    return TileBins(tile_size, padding, scene.canvas_w, scene.canvas_h, comp.ntx, comp.nty,
                    offsets, indices)


def render_forward(scene, bins: TileBins | None = None, background=None, save: bool = False,
                   eps_skip: float = DEFAULT_EPS_SKIP):
    """Tile-parallel GPU composite; returns (RenderOutput, SavedForward | None)."""
    validate_scene(scene)
    padding = DEFAULT_TILE_PADDING
    if bins is not None:
        if (bins.canvas_w, bins.canvas_h) != (scene.canvas_w, scene.canvas_h):
            raise ShapeMismatch("bins were built for a different canvas")
        padding = bins.padding
    bg = resolve_background(scene, background)
    rgb = _solid_rgb(scene, background)
    comp, d_params, release = lease_compositor(scene, padding=padding)
    dev = comp.device
    bg4 = None
    if rgb is None:
        bg4 = torch.from_numpy(pixels4(bg)).to(dev)
        rgb = (0.0, 0.0, 0.0)
    try:
        comp.preprocess(d_params)
        comp.bin()
        comp.forward(save=save, eps_skip=eps_skip, bg_rgb=rgb, bg4=bg4)
        comp.check_overflow()
        H, W = scene.canvas_h, scene.canvas_w
        color = comp.color().double().cpu().numpy()
        alpha = comp.alpha().double().cpu().numpy()
    except BaseException:
        release()
        raise
    out = RenderOutput(color, alpha)
    if not save:
        release()
        return out, None
    saved = SavedForward(
        canvas_w=W, canvas_h=H, compositor=comp, t_final=1.0 - alpha, background=bg,
        bg_rgb=None if bg4 is not None else rgb, bg4=bg4,
        fingerprint=scene_fingerprint(scene), eps_skip=eps_skip,
        n_entries=int(comp.ent_n.sum().item()))
    # the saved contribution lists live in the leased compositor's buffers: it
    # goes back to the pool only when this SavedForward is collected
    weakref.finalize(saved, release)
    return out, saved
