"""Layered export: every primitive rendered alone, on the GPU.

Mirrors the reference's exportio (pkg/src/primfit/exportio.py:272-410):
``scale_scene`` (272-288), ``layer_bbox`` (291-307), ``render_layer`` (310-346)
and ``export_layers`` (349-410).  The per-primitive layers come from one
primitive-parallel kernel launch (``pf_layer_bboxes`` + ``pf_render_layers``:
a block per primitive over its own box of the rho-times denser canvas, the
reference's float64 sampling chain); the composite is ``raster.render_forward``
with ``eps_skip = 0``.  There is no CPU path.
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from . import _native as nat
from .compositor import DeviceAtlas, _stream_handle
from .errors import PrimfitError
from .raster import _device, render_forward
from .scene import param_matrix, structure_arrays, validate_scene

EXPORT_SCALES = (1, 2, 4)   # exportio.py:77
LAYER_BBOX_PAD = 1.0        # exportio.py:78


class DegenerateBBox(PrimfitError):
    """The primitive lies fully off-canvas (no layer)."""


def scale_scene(scene, rho: int):
    """The scene on a canvas rho times denser (exportio.py:272-288)."""
    shift = (rho - 1) / 2.0
    prims = [dataclasses.replace(p, x=rho * p.x + shift, y=rho * p.y + shift, scale=rho * p.scale)
             for p in scene.primitives]
    return dataclasses.replace(scene, primitives=prims, canvas_w=rho * scene.canvas_w,
                               canvas_h=rho * scene.canvas_h)


@dataclass
class DeviceLayers:
    """All layers of one export: boxes (x0, y0, x1, y1; -1 rows = off-canvas),
    row offsets into ``rgba`` (float32 premultiplied [pixels][4] on the device)."""

    rho: int
    bbox: np.ndarray
    offsets: np.ndarray
    rgba: torch.Tensor

    def layer(self, i: int) -> tuple[tuple[int, int, int, int], np.ndarray]:
        x0, y0, x1, y1 = (int(v) for v in self.bbox[i])
        if x0 < 0:
            raise DegenerateBBox(f"primitive {i} lies fully off-canvas")
        a, b = int(self.offsets[i]), int(self.offsets[i + 1])
        img = self.rgba[a:b].double().cpu().numpy().reshape(y1 - y0 + 1, x1 - x0 + 1, 4)
        return (x0, y0, x1, y1), img


def render_layers(scene, rho: int = 1) -> DeviceLayers:
    """Every primitive's layer at export scale rho, one kernel launch (GPU)."""
    if rho < 1:
        raise ValueError(f"export scale {rho} must be >= 1")
    validate_scene(scene)
    dev = _device()
    lib = nat.load()
    n = len(scene.primitives)
    pm = torch.from_numpy(np.ascontiguousarray(param_matrix(scene), dtype=np.float64)).to(dev)
    tid, _ = structure_arrays(scene)
    d_tid = torch.from_numpy(np.ascontiguousarray(tid, dtype=np.int32)).to(dev)
    atlas = DeviceAtlas(scene.templates, bool(scene.preserve_aspect), dev)
    bbox = torch.empty(max(n, 1) * 4, dtype=torch.int32, device=dev)
    area = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    offs = torch.empty(n + 1, dtype=torch.int64, device=dev)
    s = _stream_handle()
    nat.check(lib.pf_layer_bboxes(pm.data_ptr(), d_tid.data_ptr(), atlas.d_hyp.data_ptr(), n,
                                  scene.canvas_w, scene.canvas_h, int(rho), bbox.data_ptr(),
                                  area.data_ptr(), offs.data_ptr(), s), "pf_layer_bboxes")
    offsets = offs.cpu().numpy()
    rgba = torch.empty((max(int(offsets[-1]), 1), 4), dtype=torch.float32, device=dev)
    nat.check(lib.pf_render_layers(pm.data_ptr(), d_tid.data_ptr(), atlas.tex.data_ptr(),
                                   atlas.texels, atlas.d_base.data_ptr(), atlas.d_w.data_ptr(),
                                   atlas.d_h.data_ptr(), atlas.d_q.data_ptr(), n,
                                   float(scene.alpha_max), float(scene.mu_blend), int(rho),
                                   bbox.data_ptr(), offs.data_ptr(), rgba.data_ptr(), s),
              "pf_render_layers")
    return DeviceLayers(int(rho), bbox[: n * 4].view(n, 4).cpu().numpy().astype(np.int64),
                        offsets, rgba[: int(offsets[-1])])


def layer_bbox(scene, i: int) -> tuple[int, int, int, int]:
    """Conservative pixel rect of primitive i, clipped (exportio.py:291-307)."""
    x0, y0, x1, y1 = (int(v) for v in render_layers(scene, 1).bbox[i])
    if x0 < 0:
        raise DegenerateBBox(f"primitive {i} lies fully off-canvas")
    return x0, y0, x1, y1


def render_layer(scene, i: int):
    """Primitive i alone, premultiplied RGBA over its bbox (exportio.py:310-346)."""
    return render_layers(scene, 1).layer(i)


def export_layers(scene, rho: int, outdir: str | Path):
    """Per-primitive 16-bit PNG layers in paint order, a composite and a text
    manifest (exportio.py:349-410); the rendering runs on the GPU."""
    import cv2  # image encoding only

    if rho not in EXPORT_SCALES:
        raise ValueError(f"export scale {rho} not in {EXPORT_SCALES}")
    outdir = Path(outdir)
    outdir.mkdir(parents=True, exist_ok=True)
    layers = render_layers(scene, rho)
    scaled = scale_scene(scene, rho)
    noise = isinstance(scene.background, str)
    bg = (1.0, 1.0, 1.0) if noise else tuple(float(v) for v in scene.background)
    z = np.asarray([p.z for p in scene.primitives], dtype=np.int64)
    paint = np.argsort(z, kind="stable")[::-1]  # ascending z composites front-to-back
    lines = [f"scale {rho}", f"canvas {scaled.canvas_w} {scaled.canvas_h}",
             "background " + " ".join(repr(v) for v in bg), "composite composite.png"]
    for k, i in enumerate(paint):
        try:
            bbox, rgba = layers.layer(int(i))
        except DegenerateBBox:
            lines.append(f"layer {k} {int(i)} none")
            continue
        name = f"layer_{k:04d}.png"
        a = np.clip(rgba[:, :, 3], 0.0, 1.0)
        c = np.where(a[..., None] > 0, rgba[:, :, :3] / np.maximum(a[..., None], 1e-300), 0.0)
        img = np.concatenate([c[:, :, ::-1], a[..., None]], axis=2)
        cv2.imwrite(str(outdir / name), np.round(np.clip(img, 0, 1) * 65535).astype(np.uint16))
        lines.append(f"layer {k} {int(i)} {' '.join(str(v) for v in bbox)} {name}")
    out, _ = render_forward(scaled, background=np.broadcast_to(np.asarray(bg),
                                                               (scaled.canvas_h, scaled.canvas_w, 3)),
                            eps_skip=0.0)
    cv2.imwrite(str(outdir / "composite.png"),
                np.round(np.clip(out.color[:, :, ::-1], 0, 1) * 255).astype(np.uint8))
    (outdir / "manifest.txt").write_text("\n".join(lines) + "\n")
    return layers
