"""GPU parity of the SURVEY §8 f3 / f4 rows against the reference's own outputs
(golden vectors from tests/golden/make_golden.py --aux): layered export
(exportio.scale_scene / layer_bbox / render_layer at rho 1, 2, 4) and the video
heuristics (dyn.diff_mask / freeze_flags / remove_stuck)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_case, scene_from

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.parametrize("case", ["export_aspect_mu", "export_random"])
def test_export_layers_match_reference(torch_cuda, case):
    from paper_2602_22625_b200 import export

    d = load_case(case)
    sc = scene_from(d)
    for rho in (1, 2, 4):
        lay = export.render_layers(sc, rho)
        np.testing.assert_array_equal(lay.bbox, d[f"rho{rho}_bbox"])
        np.testing.assert_array_equal(lay.offsets, d[f"rho{rho}_off"])
        got = lay.rgba.double().cpu().numpy()
        # float32 output of float64 math (16-bit PNG export): absolute 1e-6
        np.testing.assert_allclose(got, d[f"rho{rho}_rgba"], rtol=0, atol=1e-6)
    # reference-shaped single-layer API on the scaled scene
    scaled = export.scale_scene(sc, 2)
    i = int(np.flatnonzero(d["rho2_bbox"][:, 0] >= 0)[0])
    bbox, rgba = export.render_layer(scaled, i)
    assert tuple(bbox) == tuple(int(v) for v in d["rho2_bbox"][i])
    a, b = d["rho2_off"][i], d["rho2_off"][i + 1]
    np.testing.assert_allclose(rgba.reshape(-1, 4), d["rho2_rgba"][a:b], rtol=0, atol=1e-6)


def test_export_degenerate_bbox(torch_cuda):
    from paper_2602_22625_b200 import export

    d = load_case("export_random")
    sc = scene_from(d)
    sc.primitives[0].x = -500.0  # fully off-canvas
    with pytest.raises(export.DegenerateBBox):
        export.layer_bbox(sc, 0)


def test_video_heuristics_match_reference(torch_cuda):
    from paper_2602_22625_b200 import video

    d = load_case("video_heuristics")
    sc = scene_from(d)
    for tau in (0.0, 2.0 / 255.0, 0.02):
        m = video.diff_mask(d["prev"], d["cur"], tau)
        np.testing.assert_array_equal(m.mask, d[f"mask_{tau!r}"])
    m = video.diff_mask(d["prev"], d["cur"], 2.0 / 255.0)
    for pad in (2.0, 5.0):
        np.testing.assert_array_equal(video.freeze_flags(sc, m, pad), d[f"frozen_p{int(pad)}"])
    pol = video.StuckPolicy(grid=(3, 4), k=2, tau_scale=0.02, tau_alpha=0.3, zeta=0.3, eta=0.5)
    new, dec = video.remove_stuck(sc, d["frozen_p2"], pol)
    assert dec == list(d["stuck_decayed"])
    nu = np.asarray([p.opacity_logit for p in new.primitives])
    np.testing.assert_allclose(nu, d["stuck_params"][:, 4], rtol=0, atol=1e-15)
    _, dec0 = video.remove_stuck(sc, None, pol)
    assert dec0 == list(d["stuck_decayed_nofrozen"])


def test_optimize_video_chain(torch_cuda):
    """optimize_video (dyn.py:180-238) on the GPU fit loop: frame 0 == run_loop
    alone; on frame 1 every primitive frozen by the diff mask keeps its
    parameters bit for bit, the others move; the stuck-decay hooks run."""
    import copy

    from paper_2602_22625_b200 import synth, video
    from paper_2602_22625_b200.fit import LossSpec, effective_padding, run_loop
    from paper_2602_22625_b200.scene import pack_params

    w = synth.make_workload("c1")
    cfg = copy.deepcopy(w.cfg)
    cfg.num_iterations, cfg.sequential_iterations = 10, 8
    cfg.freeze_static, cfg.remove_stuck, cfg.stuck_triggers = True, True, (3, 6)
    f0 = w.target
    f1 = f0.copy()
    f1[100:160, 60:120] = 1.0 - f1[100:160, 60:120]  # one changed region
    scenes, hists = video.optimize_video([f0, f1], copy.deepcopy(w.scene), cfg)
    assert [len(h) for h in hists] == [10, 8]
    # frame 0 is run_loop alone (same rng stream)
    s0, _, _ = run_loop(copy.deepcopy(w.scene), cfg, LossSpec(kind="mse", target=f0),
                        np.random.default_rng(cfg.seed), iterations=10)
    p0, p1 = pack_params(scenes[0])[0].reshape(-1, 8), pack_params(scenes[1])[0].reshape(-1, 8)
    np.testing.assert_array_equal(p0, pack_params(s0)[0].reshape(-1, 8))
    frozen = video.freeze_flags(scenes[0], video.diff_mask(f0, f1), effective_padding(cfg))
    assert 0 < frozen.sum() < len(frozen)
    np.testing.assert_array_equal(p1[frozen], p0[frozen])
    assert (p1[~frozen] != p0[~frozen]).any(axis=1).all()


@pytest.mark.parametrize("rho", [1, 2])
def test_export_layers_files_recompose(torch_cuda, tmp_path, rho):
    """export_layers end to end on the GPU: the reference's file format (premultiplied
    16-bit layers, write_manifest grammar), re-composited back to front within PNG
    quantisation of render_forward on the scaled canvas (exportio.py:482-512; the
    reference's bar, test_export.py:250-254)."""
    import dataclasses

    from paper_2602_22625_b200 import export, raster

    sc = scene_from(load_case("export_random"))
    prims = list(sc.primitives)
    prims[2] = dataclasses.replace(prims[2], x=-500.0, y=-500.0)
    sc = dataclasses.replace(sc, primitives=prims)
    man = export.export_layers(sc, rho, tmp_path)
    assert isinstance(man, export.LayerManifest)
    assert export.read_manifest(tmp_path / "manifest.txt") == man
    assert [r.prim for r in man.layers if r.file is None] == [2]
    scaled = export.scale_scene(sc, rho)
    bg = np.broadcast_to(np.asarray(man.background), (scaled.canvas_h, scaled.canvas_w, 3))
    ref, _ = raster.render_forward(scaled, background=bg, eps_skip=0.0)
    composed = export.compose_layers(man, tmp_path)
    assert np.abs(composed.color - ref.color).max() < 5e-4
    assert np.abs(composed.alpha - ref.alpha).max() < 5e-4
