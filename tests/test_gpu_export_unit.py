"""The reference's export tests (tests/test_export.py:191-293) on the GPU
exporter (export.export_layers: primitive-parallel layer kernel + the composite
through the GPU forward), on the reference's own scenes (golden export_tests.npz
= conftest.random_scene with the same seeds and sizes)."""

from __future__ import annotations

from dataclasses import replace

import numpy as np
import pytest

from conftest import load_case, scene_from

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ex():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_22625_b200 import export, raster

    return export, raster


def _scene(tag: str):
    d = load_case("export_tests")
    return scene_from({k[len(tag) + 1:]: d[k] for k in d if k.startswith(tag + "_")})


def test_export_layers_and_compose(ex, tmp_path):
    export, raster = ex
    scene = _scene("x8")
    prims = list(scene.primitives)
    prims[2] = replace(prims[2], x=-200.0, y=-200.0)  # fully off canvas: skipped
    scene = replace(scene, primitives=prims)
    manifest = export.export_layers(scene, 1, tmp_path)
    assert manifest.scale == 1
    assert (tmp_path / "manifest.txt").is_file() and (tmp_path / "composite.png").is_file()
    assert [rec.z for rec in manifest.layers] == list(range(5))
    assert [rec.prim for rec in manifest.layers if rec.file is None] == [2]
    for rec in manifest.layers:
        p = scene.primitives[rec.prim]
        assert rec.params == (p.x, p.y, p.scale, p.rotation, p.opacity_logit, *p.color_logits)
        if rec.file is not None:
            assert (tmp_path / rec.file).is_file()
    front = min(range(5), key=lambda i: scene.primitives[i].z)
    assert manifest.layers[-1].prim == front  # the front-most paints last
    out, _ = raster.render_forward(scene, eps_skip=0.0)
    composed = export.compose_layers(manifest, tmp_path)
    assert np.abs(composed.color - np.asarray(out.color)).max() < 5e-4
    assert np.abs(composed.alpha - np.asarray(out.alpha)).max() < 5e-4
    comp_png, _ = export.load_image(tmp_path / "composite.png")
    assert np.abs(comp_png - np.asarray(out.color)).max() <= 0.5 / 255.0 + 1e-6


def test_export_rejects_bad_scale(ex, tmp_path):
    export, _ = ex
    with pytest.raises(ValueError):
        export.export_layers(_scene("x9"), 3, tmp_path)


def test_export_noise_background_composites_white(ex, tmp_path):
    export, _ = ex
    manifest = export.export_layers(replace(_scene("x10"), background="noise"), 1, tmp_path)
    assert manifest.background == (1.0, 1.0, 1.0)


def test_stacking_order_front_wins(ex, tmp_path):
    export, _ = ex
    from paper_2602_22625_b200.scene import PrimitiveParams, PrimitiveTemplate, Scene

    size = 13
    yy, xx = np.mgrid[0:size, 0:size].astype(np.float64)
    c = (size - 1) / 2
    disk = np.zeros((size, size, 4))
    disk[:, :, 0], disk[:, :, 1], disk[:, :, 2] = 0.9, 0.5, 0.3
    disk[:, :, 3] = np.clip(1.0 - (np.hypot(yy - c, xx - c) / c) ** 2, 0.0, 1.0) ** 2

    def mk(z, col):
        return PrimitiveParams(x=10.0, y=10.0, scale=6.0, rotation=0.0, opacity_logit=50.0,
                               color_logits=col, template_id=0, z=z)

    scene = Scene([mk(0, (50.0, -50.0, -50.0)), mk(1, (-50.0, 50.0, -50.0))],
                  [PrimitiveTemplate(disk)], 20, 20, background=(0.0, 0.0, 0.0))
    composed = export.compose_layers(export.export_layers(scene, 1, tmp_path), tmp_path)
    assert composed.color[10, 10, 0] > 0.99 and composed.color[10, 10, 1] < 0.01


def test_manifest_round_trip(ex, tmp_path):
    export, _ = ex
    manifest = export.export_layers(_scene("x11"), 2, tmp_path)
    assert export.read_manifest(tmp_path / "manifest.txt") == manifest


def _one_prim_scene(x=14.0, y=10.0, scale=5.0, mu_blend=0.0, w=32, h=24):
    # test_export.py:191-198
    from paper_2602_22625_b200.scene import PrimitiveParams, PrimitiveTemplate, Scene

    size = 13
    yy, xx = np.mgrid[0:size, 0:size].astype(np.float64)
    c = (size - 1) / 2
    disk = np.zeros((size, size, 4))
    disk[:, :, 0], disk[:, :, 1], disk[:, :, 2] = 0.9, 0.5, 0.3
    disk[:, :, 3] = np.clip(1.0 - (np.hypot(yy - c, xx - c) / c) ** 2, 0.0, 1.0) ** 2
    p = PrimitiveParams(x=x, y=y, scale=scale, rotation=0.7, opacity_logit=1.2,
                        color_logits=(0.4, -0.3, 0.8), template_id=0, z=0)
    return Scene([p], [PrimitiveTemplate(disk)], w, h, background=(0.25, 0.5, 0.75),
                 mu_blend=mu_blend)


def test_layer_bbox_matches_half_side(ex):
    # test_export.py:201-211
    import math

    export, _ = ex
    r = 5.0 * math.hypot(1.0, 1.0) + export.LAYER_BBOX_PAD
    assert export.layer_bbox(_one_prim_scene(), 0) == (
        max(math.floor(14.0 - r), 0), max(math.floor(10.0 - r), 0),
        min(math.ceil(14.0 + r), 31), min(math.ceil(10.0 + r), 23))
    with pytest.raises(export.DegenerateBBox):
        export.layer_bbox(_one_prim_scene(x=-50.0, y=-50.0), 0)


@pytest.mark.parametrize("mu_blend", [0.0, 0.35])
def test_render_layer_reproduces_contribution(ex, mu_blend):
    # test_export.py:214-223 (atol 1e-12 there on float64; the GPU layer is float32)
    export, raster = ex
    scene = _one_prim_scene(mu_blend=mu_blend)
    (x0, y0, x1, y1), rgba = export.render_layer(scene, 0)
    img = np.broadcast_to(np.asarray(scene.background), (24, 32, 3)).copy()
    view = img[y0:y1 + 1, x0:x1 + 1]
    view *= 1.0 - rgba[:, :, 3:4]
    view += rgba[:, :, :3]
    out, _ = raster.render_forward(scene, eps_skip=0.0)
    np.testing.assert_allclose(img, np.asarray(out.color), atol=1e-6)
