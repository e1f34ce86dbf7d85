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


@dataclass
class LayerRecord:
    """One manifest entry; bbox and file are None for skipped layers
    (exportio.py:250-258)."""

    z: int
    prim: int
    params: tuple[float, ...]
    bbox: tuple[int, int, int, int] | None
    file: str | None


@dataclass
class LayerManifest:
    """Everything needed to re-composite an exported scene (exportio.py:261-269)."""

    scale: int
    canvas_w: int
    canvas_h: int
    background: tuple[float, float, float]
    composite: str
    layers: list[LayerRecord]


MANIFEST_FORMAT = "primfit-layers"  # exportio.py:75
MANIFEST_VERSION = 1                # exportio.py:76


def save_image(path: str | Path, rgb, alpha=None, bits: int = 8) -> None:
    """Float RGB(A) in [0, 1] -> 8- or 16-bit PNG, round-half-even quantisation
    (save_image, exportio.py:108-126)."""
    import cv2  # image encoding only

    if bits not in (8, 16):
        raise ValueError(f"bits must be 8 or 16, got {bits}")
    peak, dtype = (255, np.uint8) if bits == 8 else (65535, np.uint16)
    img = np.asarray(rgb, dtype=np.float64)[:, :, ::-1]  # RGB -> BGR (cv2 order)
    if alpha is not None:
        img = np.concatenate([img, np.asarray(alpha, dtype=np.float64)[:, :, None]], axis=2)
    if not cv2.imwrite(str(path), np.rint(np.clip(img, 0.0, 1.0) * peak).astype(dtype)):
        raise OSError(f"could not write image {path}")


def load_image(path: str | Path):
    """PNG -> float RGB in [0, 1] + optional alpha (load_image, exportio.py:83-106)."""
    import cv2

    raw = cv2.imread(str(path), cv2.IMREAD_UNCHANGED)
    if raw is None:
        raise OSError(f"could not decode {path}")
    img = raw.astype(np.float64) / (65535.0 if raw.dtype == np.uint16 else 255.0)
    if img.ndim == 2:
        return np.repeat(img[:, :, None], 3, axis=2), None
    if img.shape[2] == 3:
        return img[:, :, ::-1].copy(), None
    return img[:, :, 2::-1].copy(), np.ascontiguousarray(img[:, :, 3])


def write_manifest(path: str | Path, manifest: LayerManifest) -> None:
    """The reference's fixed-field manifest grammar (write_manifest,
    exportio.py:413-431; module docstring 18-33)."""
    lines = [
        f"format {MANIFEST_FORMAT}",
        f"version {MANIFEST_VERSION}",
        f"scale {manifest.scale}",
        f"canvas {manifest.canvas_w} {manifest.canvas_h}",
        "background " + " ".join(repr(float(v)) for v in manifest.background),
        f"composite {manifest.composite}",
        f"layers {len(manifest.layers)}",
    ]
    for rec in manifest.layers:
        if rec.bbox is None:
            mid = "skipped off-canvas"
        else:
            x0, y0, x1, y1 = rec.bbox
            mid = f"bbox {x0} {y0} {x1} {y1} file {rec.file}"
        params = " ".join(repr(float(v)) for v in rec.params)
        lines.append(f"layer {rec.z} prim {rec.prim} {mid} params {params}")
    Path(path).write_text("\n".join(lines) + "\n")


def parse_manifest(text: str) -> LayerManifest:
    """Inverse of write_manifest; ValueError on malformed text (exportio.py:435-478)."""
    lines = [ln for ln in text.splitlines() if ln.strip()]

    def field(k: int, key: str) -> list[str]:
        parts = lines[k].split()
        if parts[0] != key:
            raise ValueError(f"manifest line {k + 1}: expected {key!r}")
        return parts[1:]

    if field(0, "format") != [MANIFEST_FORMAT]:
        raise ValueError("not a layer manifest")
    if int(field(1, "version")[0]) != MANIFEST_VERSION:
        raise ValueError("unsupported manifest version")
    scale = int(field(2, "scale")[0])
    cw, ch = (int(v) for v in field(3, "canvas"))
    bg = tuple(float(v) for v in field(4, "background"))
    composite = field(5, "composite")[0]
    layers = []
    for k in range(int(field(6, "layers")[0])):
        parts = lines[7 + k].split()
        if parts[0] != "layer" or parts[2] != "prim":
            raise ValueError(f"manifest layer line {k} malformed")
        if parts[4] == "bbox" and parts[9] == "file":
            bbox, file, rest = tuple(int(v) for v in parts[5:9]), parts[10], parts[11:]
        elif parts[4] == "skipped":
            bbox, file, rest = None, None, parts[6:]
        else:
            raise ValueError(f"manifest layer line {k} malformed")
        if rest[0] != "params" or len(rest) != 9:
            raise ValueError(f"manifest layer line {k}: bad params")
        layers.append(LayerRecord(int(parts[1]), int(parts[3]),
                                  tuple(float(v) for v in rest[1:]), bbox, file))
    return LayerManifest(scale, cw, ch, bg, composite, layers)


def read_manifest(path: str | Path) -> LayerManifest:
    return parse_manifest(Path(path).read_text())


def compose_layers(manifest: LayerManifest, layer_dir: str | Path):
    """Back-to-front "over" of the stored premultiplied layers (compose_layers,
    exportio.py:482-512): the export's consistency check, host-side."""
    from .raster import RenderOutput

    layer_dir = Path(layer_dir)
    h, w = manifest.canvas_h, manifest.canvas_w
    rgb = np.broadcast_to(np.asarray(manifest.background, dtype=np.float64), (h, w, 3)).copy()
    cov = np.zeros((h, w))
    for rec in sorted(manifest.layers, key=lambda r: r.z):
        if rec.file is None:
            continue
        lrgb, la = load_image(layer_dir / rec.file)
        if la is None:
            raise OSError(f"layer {rec.file} lost its alpha channel")
        x0, y0, x1, y1 = rec.bbox
        view = rgb[y0 : y1 + 1, x0 : x1 + 1]
        view *= 1.0 - la[:, :, None]
        view += lrgb
        cov[y0 : y1 + 1, x0 : x1 + 1] = la + (1.0 - la) * cov[y0 : y1 + 1, x0 : x1 + 1]
    return RenderOutput(color=rgb, alpha=cov)


def write_export(scene, rho: int, outdir: str | Path, layer, composite) -> LayerManifest:
    """The export's file side (exportio.py:370-410): ``layer(i)`` gives primitive
    i's (bbox, premultiplied float RGBA) on the scaled canvas or raises
    DegenerateBBox; ``composite`` is the scaled render (H, W, 3).  Layers are
    written back to front (descending z), 16-bit premultiplied RGB + alpha."""
    outdir = Path(outdir)
    outdir.mkdir(parents=True, exist_ok=True)
    scaled_w, scaled_h = rho * scene.canvas_w, rho * scene.canvas_h
    noise = isinstance(scene.background, str)
    bg = (1.0, 1.0, 1.0) if noise else tuple(float(v) for v in scene.background)
    z = np.asarray([p.z for p in scene.primitives], dtype=np.int64)
    paint = np.argsort(z, kind="stable")[::-1]  # ascending z is front to back
    records = []
    for k, i in enumerate(int(v) for v in paint):
        p = scene.primitives[i]
        params = (p.x, p.y, p.scale, p.rotation, p.opacity_logit, *p.color_logits)
        params = tuple(float(v) for v in params)
        try:
            bbox, rgba = layer(i)
        except DegenerateBBox:
            records.append(LayerRecord(k, i, params, None, None))
            continue
        name = f"layer_{k:04d}.png"
        save_image(outdir / name, rgba[:, :, :3], rgba[:, :, 3], bits=16)
        records.append(LayerRecord(k, i, params, tuple(int(v) for v in bbox), name))
    save_image(outdir / "composite.png", composite)
    manifest = LayerManifest(rho, scaled_w, scaled_h, bg, "composite.png", records)
    write_manifest(outdir / "manifest.txt", manifest)
    return manifest


def export_layers(scene, rho: int, outdir: str | Path) -> LayerManifest:
    """Per-primitive layers, a composite and the manifest (exportio.py:349-410),
    rendered on the GPU: all layers in one primitive-parallel launch, the
    composite through render_forward with eps_skip = 0 and a noise background
    resolved to white.  Returns the LayerManifest, as the reference."""
    if rho not in EXPORT_SCALES:
        raise ValueError(f"export scale {rho} not in {EXPORT_SCALES}")
    layers = render_layers(scene, rho)
    scaled = scale_scene(scene, rho)
    noise = isinstance(scene.background, str)
    bg = (1.0, 1.0, 1.0) if noise else tuple(float(v) for v in scene.background)
    out, _ = render_forward(scaled, background=np.broadcast_to(
        np.asarray(bg), (scaled.canvas_h, scaled.canvas_w, 3)), eps_skip=0.0)
    return write_export(scene, rho, outdir, layers.layer, out.color)
