"""The reference's acceptance criteria that cover this path, on the CUDA path.

test_acceptance.py (reference):
  01  run_gradcheck(20): analytic gradients vs central finite differences on the
      20 gradcheck scenes, a scalar passing when rel <= 1e-2 (relative to the
      finite difference) or abs <= 1e-5 (grad.py:378-420).  Here: the GPU
      backward against the reference's own finite differences (golden).
  02  tiled forward vs the sequential reference on 50 random scenes (n = 4..200,
      128x128), worst |diff| <= 1e-6 at eps_skip = 0.  Here: the GPU forward
      against the pinned oracle (itself within 1e-13 of the reference).
  04  compositing invariants: coverage identity (alpha + prod(1 - a_i) = 1),
      an opaque front primitive occludes everything behind it exactly, and
      raising any opacity never lowers coverage.
  06, 07, 08a, 08b  behaviour of the fit loop, the spatial loss and the video
      heuristics, through fit.optimize / video.optimize_video / run_loop hooks.
Scenes: tests/golden/acceptance.npz (make_golden.py --acceptance).
"""

from __future__ import annotations

import math
from dataclasses import replace

import numpy as np
import pytest

from conftest import load_case, scene_from

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pf():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_22625_b200 import grad, raster

    return raster, grad


@pytest.fixture(scope="module")
def acc():
    return load_case("acceptance")


def _sub(d, prefix: str) -> dict:
    return {k[len(prefix):]: d[k] for k in d if k.startswith(prefix)}


def test_criterion_01_gradcheck_20_scenes(pf, acc):
    raster, grad = pf
    n_checked = n_fail = 0
    worst = 0.0
    for seed in range(20):
        d = _sub(acc, f"g{seed}_")
        sc = scene_from(d)
        target = d["target"]
        out, saved = raster.render_forward(sc, save=True, eps_skip=0.0)
        dL = 2.0 * (np.asarray(out.color, dtype=np.float64) - target) / target.size
        g = grad.backward(sc, saved, dL).data
        fd = d["fd"]
        adiff = np.abs(g - fd)
        rel = adiff / np.maximum(np.abs(fd), 1e-300)
        ok = (rel <= 1e-2) | (adiff <= 1e-5)
        n_checked += ok.size
        n_fail += int((~ok).sum())
        over = rel[adiff > 1e-5]
        if over.size:
            worst = max(worst, float(over.max()))
    assert n_checked > 0 and n_fail == 0, f"{n_fail}/{n_checked} failures, worst rel {worst:.2e}"


def test_criterion_02_forward_50_scenes(pf, acc, oracle):
    raster, _ = pf
    worst = 0.0
    for seed in range(50):
        sc = scene_from(_sub(acc, f"r{seed}_"))
        assert sc.n == 4 + (196 * seed) // 49
        pk = oracle.Packed(sc)
        off, idx = oracle.bin_tiles(pk, 32, 2.0)
        img, alpha, _ = oracle.render_forward(pk, off, idx, 32, oracle.background(sc), False,
                                              0.0)
        out, _ = raster.render_forward(sc, eps_skip=0.0)
        worst = max(worst, float(np.abs(np.asarray(out.color) - img).max()),
                    float(np.abs(np.asarray(out.alpha) - alpha).max()))
    assert worst <= 1e-6, f"worst |diff| {worst:.2e}"


def _soft_disk(size: int = 15) -> np.ndarray:
    # the reference test fixture (tests/conftest.py:25-36)
    yy, xx = np.mgrid[0:size, 0:size].astype(np.float64)
    c = (size - 1) / 2
    r = np.hypot(yy - c, xx - c) / c
    rgba = np.zeros((size, size, 4))
    rgba[:, :, 0], rgba[:, :, 1], rgba[:, :, 2] = 0.9, 0.5, 0.3
    rgba[:, :, 3] = np.clip(1.0 - r**2, 0.0, 1.0) ** 2
    return rgba


def _alpha_plane(sc, i: int, W: int, H: int) -> np.ndarray:
    """a_i at every pixel centre: raster.py canvas_to_prim / prim_to_texel /
    sample_bilinear / primitive_alpha in numpy float64 (no eps skip)."""
    p = sc.primitives[i]
    rgba = np.asarray(sc.templates[p.template_id].rgba)
    ht, wt = rgba.shape[:2]
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)
    dx, dy = xx - p.x, yy - p.y
    c, s = math.cos(p.rotation), math.sin(p.rotation)
    u = (c * dx + s * dy) / p.scale
    v = (-s * dx + c * dy) / p.scale
    U = (u + 1.0) * 0.5 * (wt - 1)
    V = (v + 1.0) * 0.5 * (ht - 1)
    inside = (U >= 0) & (U <= wt - 1) & (V >= 0) & (V <= ht - 1)
    pad = np.zeros((ht + 1, wt + 1))
    pad[:ht, :wt] = rgba[:, :, 3]
    u0 = np.clip(np.floor(U), 0, wt - 1).astype(int)
    v0 = np.clip(np.floor(V), 0, ht - 1).astype(int)
    wu, wv = U - u0, V - v0
    m = ((1 - wu) * (1 - wv) * pad[v0, u0] + wu * (1 - wv) * pad[v0, u0 + 1]
         + (1 - wu) * wv * pad[v0 + 1, u0] + wu * wv * pad[v0 + 1, u0 + 1])
    sig = 1.0 / (1.0 + math.exp(-p.opacity_logit))
    return np.where(inside, sc.alpha_max * sig * m, 0.0)


def test_criterion_04_compositing_invariants(pf):
    raster, _ = pf
    from paper_2602_22625_b200.scene import PrimitiveParams, PrimitiveTemplate, Scene

    tpl_soft = PrimitiveTemplate(_soft_disk(15))
    ones = np.ones((9, 9, 4))
    ones[:, :, 0], ones[:, :, 1], ones[:, :, 2] = 0.8, 0.2, 0.1
    tpl_hard = PrimitiveTemplate(ones)

    def prim(x, y, s, nu, z, tid=0):
        return PrimitiveParams(x=x, y=y, scale=s, rotation=0.4 * z, opacity_logit=nu,
                               color_logits=(0.5, -0.2, 0.1), template_id=tid, z=z)

    # coverage identity: alpha and the residual transmittance sum to 1 (the GPU
    # stores float32: 1e-6 instead of the reference's float64 1e-12)
    sc = Scene([prim(9.0, 11.0, 5.0, 0.8, 0), prim(14.0, 12.0, 6.0, -0.5, 1),
                prim(20.0, 9.0, 4.0, 2.0, 2)], [tpl_soft], 28, 24,
               background=(0.3, 0.6, 0.9), alpha_max=0.9)
    out, _ = raster.render_forward(sc, eps_skip=0.0)
    T = np.ones((24, 28))
    for i in range(sc.n):
        T *= 1.0 - _alpha_plane(sc, i, 28, 24)
    assert float(np.abs(np.asarray(out.alpha) + T - 1.0).max()) <= 1e-6
    # opaque front: the pixels it saturates are untouched by anything behind
    front, back = prim(10.0, 10.0, 4.0, 50.0, 0), prim(11.0, 10.0, 5.0, 1.0, 1)
    pair = Scene([front, back], [tpl_hard], 24, 20, background=(0.1, 0.1, 0.1))
    alone = replace(pair, primitives=[front])
    out_pair, _ = raster.render_forward(pair, eps_skip=0.0)
    out_alone, _ = raster.render_forward(alone, eps_skip=0.0)
    sat = _alpha_plane(pair, 0, 24, 20) == 1.0
    assert sat.sum() > 20
    assert np.array_equal(np.asarray(out_pair.color)[sat], np.asarray(out_alone.color)[sat])
    assert np.all(np.asarray(out_pair.alpha)[sat] == 1.0)
    # coverage only rises as any opacity rises
    a0 = np.asarray(out.alpha)
    for k in range(sc.n):
        prims = list(sc.primitives)
        prims[k] = replace(prims[k], opacity_logit=prims[k].opacity_logit + 2.0)
        bumped, _ = raster.render_forward(replace(sc, primitives=prims), eps_skip=0.0)
        b = np.asarray(bumped.alpha)
        assert np.all(b >= a0 - 1e-7)
        assert b.max() > a0.max() - 1e-7


def _hard_disk(size: int = 25) -> np.ndarray:
    # the acceptance suite's template (scripts/make_assets.py:70-79)
    yy, xx = np.mgrid[0:size, 0:size].astype(np.float64)
    c = (size - 1) / 2
    rgba = np.zeros((size, size, 4))
    rgba[:, :, :3] = 1.0
    rgba[:, :, 3] = (np.hypot(yy - c, xx - c) <= c - 1.0).astype(np.float64)
    return rgba


def test_optimize_matches_reference(pf):
    """fit.optimize (fit.py:524-555) against the reference's own run: seeded
    template preparation, init_scene, the config's spatial loss and reinit
    boundaries, then the GPU run_loop (make_golden.py --hooks)."""
    from paper_2602_22625_b200 import fit
    from paper_2602_22625_b200.scene import PrimitiveTemplate, pack_params

    d = load_case("optimize_small")
    assert np.array_equal(d["disk"], _hard_disk())
    cfg = fit.FitConfig(num_primitives=40, num_iterations=8, seed=2, loss="spatial",
                        alpha_loss_weight=0.3, do_reinit=True, reinit_period=3, reinit_warmup=2)
    sc, hist = fit.optimize(d["target"], [PrimitiveTemplate(_hard_disk())], cfg,
                            target_alpha=d["target_alpha"])
    assert [h.reinit_count for h in hist] == list(d["hist_reinit"])
    np.testing.assert_allclose([h.loss for h in hist], d["hist_loss"], rtol=1e-5)
    np.testing.assert_allclose([h.psnr for h in hist], d["hist_psnr"], rtol=1e-6)
    np.testing.assert_array_equal([p.template_id for p in sc.primitives], d["tid"])
    np.testing.assert_allclose(pack_params(sc)[0].reshape(-1, 8), d["final_params"],
                               rtol=1e-4, atol=1e-5)


def _gaussian_smooth(rng_seed: int, sigma: float, size: int = 128) -> np.ndarray:
    from scipy.ndimage import gaussian_filter

    tex = gaussian_filter(np.random.default_rng(rng_seed).random((size, size, 3)),
                          sigma=(sigma, sigma, 0))
    return (tex - tex.min()) / (tex.max() - tex.min())


def test_criterion_06_noisy_background_forces_coverage(pf):
    """test_acceptance.py:229-252 through fit.optimize on the GPU: fitting
    against a noise background raises the coverage of a white target region by
    >= 0.2 over fitting against white."""
    raster, _ = pf
    from paper_2602_22625_b200 import fit
    from paper_2602_22625_b200.scene import PrimitiveTemplate

    target = np.clip(0.2 + 0.6 * _gaussian_smooth(77, 3.0), 0.0, 1.0)
    target[36:92, 36:92] = 1.0
    region = np.zeros((128, 128), dtype=bool)
    region[36:92, 36:92] = True

    def coverage(bg):
        cfg = fit.FitConfig(num_primitives=250, num_iterations=100, bg_color=bg, seed=0,
                            compute_psnr=False)
        scene, _ = fit.optimize(target, [PrimitiveTemplate(_hard_disk())], cfg)
        out, _ = raster.render_forward(scene, raster.bin_tiles(scene),
                                       background=(1.0, 1.0, 1.0))
        return float(np.asarray(out.alpha)[region].mean())

    solid, noisy = coverage("white"), coverage("noise")
    assert noisy - solid >= 0.2, (solid, noisy)


def test_criterion_07_spatial_constraint_confines_opacity(pf):
    """test_acceptance.py:255-313 through fit.optimize on the GPU: with the
    spatial loss, primitives entirely outside the mask end at mean opacity < 0.1
    and the in-mask PSNR stays within 1 dB of the plain MSE fit."""
    raster, _ = pf
    from paper_2602_22625_b200 import fit
    from paper_2602_22625_b200.scene import PrimitiveTemplate

    target = np.clip(0.15 + 0.8 * _gaussian_smooth(55, 2.5), 0.0, 1.0)
    yy, xx = np.mgrid[0:128, 0:128]
    mask = (((yy - 64.0) ** 2 + (xx - 64.0) ** 2) <= 48.0**2).astype(np.float64)
    inside = mask > 0

    def run(kind):
        cfg = fit.FitConfig(num_primitives=250, num_iterations=150, loss=kind,
                            alpha_loss_weight=0.3, do_reinit=True, reinit_period=30,
                            reinit_warmup=59, seed=0, compute_psnr=False)
        scene, _ = fit.optimize(target, [PrimitiveTemplate(_hard_disk())], cfg,
                                target_alpha=mask if kind == "spatial" else None)
        out, _ = raster.render_forward(scene, raster.bin_tiles(scene),
                                       background=(1.0, 1.0, 1.0))
        return scene, np.asarray(out.color, dtype=np.float64)

    sc_sp, col_sp = run("spatial")
    _, col_ms = run("mse")
    outside = []
    for p in sc_sp.primitives:
        r = p.scale * math.hypot(1.0, 1.0)  # bbox_half_side(scale) (raster.py:222-224)
        x0, x1 = max(math.ceil(p.x - r), 0), min(math.floor(p.x + r), 127)
        y0, y1 = max(math.ceil(p.y - r), 0), min(math.floor(p.y + r), 127)
        if x0 > x1 or y0 > y1 or not inside[y0:y1 + 1, x0:x1 + 1].any():
            outside.append(1.0 / (1.0 + math.exp(-p.opacity_logit)))
    mean_outside = float(np.mean(outside)) if outside else 0.0
    psnr_sp = 10 * math.log10(1.0 / float(np.mean((col_sp[inside] - target[inside]) ** 2)))
    psnr_ms = 10 * math.log10(1.0 / float(np.mean((col_ms[inside] - target[inside]) ** 2)))
    assert mean_outside < 0.1, (len(outside), mean_outside)
    assert psnr_sp >= psnr_ms - 1.0, (psnr_sp, psnr_ms)


def _square_video():
    # test_acceptance.py:_square_video: a red square sliding over a static backdrop
    from scipy.ndimage import gaussian_filter

    rng = np.random.default_rng(99)
    backdrop = np.full((64, 64, 3), 0.55)
    band = gaussian_filter(rng.random((24, 64, 3)), sigma=(2, 2, 0))
    backdrop[40:64] = 0.15 + 0.7 * (band - band.min()) / (band.max() - band.min())
    frames = []
    for t in range(8):
        f = backdrop.copy()
        x0 = 6 + 6 * t
        f[8:18, x0:x0 + 10] = (0.95, 0.3, 0.2)
        frames.append(np.clip(f, 0.0, 1.0))
    return frames


def test_criterion_08a_freezing_keeps_static_primitives_bit_identical(pf):
    """test_acceptance.py:316-350 through video.optimize_video on the GPU: every
    primitive frozen for a transition is bit-identical across it, unfrozen ones
    move, and some primitives stay frozen (and identical) end to end."""
    from paper_2602_22625_b200 import fit, video
    from paper_2602_22625_b200.scene import PrimitiveTemplate

    frames = _square_video()
    cfg = fit.FitConfig(num_primitives=120, num_iterations=80, sequential_iterations=40,
                        scale_min=1.5, scale_max=4.0, freeze_static=True, seed=3,
                        compute_psnr=False)
    scenes, _ = video.optimize_video(frames, [PrimitiveTemplate(_hard_disk())], cfg)
    pad = fit.effective_padding(cfg)
    min_frozen, changed_counts, always = cfg.num_primitives, [], None
    for t in range(1, 8):
        mask = video.diff_mask(frames[t - 1], frames[t], cfg.diff_threshold)
        flags = video.freeze_flags(scenes[t - 1], mask, pad)
        min_frozen = min(min_frozen, int(flags.sum()))
        changed = 0
        for i, flag in enumerate(flags):
            same = scenes[t].primitives[i] == scenes[t - 1].primitives[i]
            if flag:
                assert same, (t, i)
            elif not same:
                changed += 1
        changed_counts.append(changed)
        held = set(np.nonzero(flags)[0].tolist())
        always = held if always is None else (always & held)
    assert min_frozen > 0 and min(changed_counts) > 0 and len(always) > 0
    assert all(scenes[7].primitives[i] == scenes[0].primitives[i] for i in always)


def test_criterion_08b_stuck_decay_lowers_video_error(pf):
    """test_acceptance.py:353-406 on the GPU run_loop with video.remove_stuck as
    hooks: decaying the dominant (stuck) primitive strictly lowers the error."""
    raster, _ = pf
    from paper_2602_22625_b200 import fit, video
    from paper_2602_22625_b200.scene import (PrimitiveParams, PrimitiveTemplate, Scene,
                                             pack_params)

    c1, c2 = (0.95, 0.90, 0.10), (0.05, 0.10, 0.20)
    mean = tuple((a + b) / 2 for a, b in zip(c1, c2))

    def logit(c):
        return tuple(float(math.log(v / (1 - v))) for v in c)

    target = np.ones((64, 64, 3))
    for cy in range(4):
        for cx in range(4):
            target[32 + cy * 4:36 + cy * 4, 32 + cx * 4:36 + cx * 4] = \
                c1 if (cy + cx) % 2 == 0 else c2

    def build():
        prims = [PrimitiveParams(x=39.5, y=39.5, scale=13.0, rotation=0.0, opacity_logit=2.5,
                                 color_logits=logit(mean), template_id=0, z=0)]
        z = 1
        for cy in range(4):
            for cx in range(4):
                prims.append(PrimitiveParams(
                    x=32 + cx * 4 + 1.5, y=32 + cy * 4 + 1.5, scale=2.8, rotation=0.0,
                    opacity_logit=-4.0, color_logits=logit(c1 if (cy + cx) % 2 == 0 else c2),
                    template_id=0, z=z))
                z += 1
        return Scene(prims, [PrimitiveTemplate(_hard_disk())], 64, 64,
                     background=(1.0, 1.0, 1.0))

    triggers = (10, 25, 40)
    policy = video.StuckPolicy(triggers=triggers)

    def final_mse(with_decay):
        scene = build()
        cfg = fit.FitConfig(num_iterations=80, eps_skip=0.0, compute_psnr=False)
        spec = fit.LossSpec(kind="mse", target=target)
        state = fit.OptimState.fresh(pack_params(scene)[1])
        hooks = ({t: (lambda s, st: video.remove_stuck(s, st.frozen, policy)[0])
                  for t in triggers} if with_decay else None)
        out_scene, _, _ = fit.run_loop(scene, cfg, spec, np.random.default_rng(0),
                                       iterations=80, state=state, hooks=hooks)
        out, _ = raster.render_forward(out_scene, raster.bin_tiles(out_scene))
        return float(np.mean((np.asarray(out.color, dtype=np.float64) - target) ** 2))

    off, on = final_mse(False), final_mse(True)
    assert on < off, (off, on)


# -- compositing algebra known-answer tests (test_raster.py:118-190) on the GPU --------

def _one_prim_scene(opacity_logit=2.0, alpha_max=1.0):
    from paper_2602_22625_b200.scene import PrimitiveParams, PrimitiveTemplate, Scene

    t = np.zeros((5, 5, 4))
    t[:, :, 3] = 1.0
    t[:, :, :3] = 0.5
    prim = PrimitiveParams(x=8.0, y=8.0, scale=3.0, rotation=0.0, opacity_logit=opacity_logit,
                           color_logits=(4.0, -4.0, 0.0))
    return Scene([prim], [PrimitiveTemplate(t)], 16, 16, background=(0.0, 0.0, 1.0),
                 alpha_max=alpha_max)


def test_single_primitive_center_pixel_algebra(pf):
    # test_raster.py:130-137 (atol 1e-12 on float64; the GPU image is float32)
    raster, _ = pf
    out, _ = raster.render_forward(_one_prim_scene(), eps_skip=0.0)
    a = 1.0 / (1.0 + np.exp(-2.0))
    c = np.array([1 / (1 + np.exp(-4.0)), 1 / (1 + np.exp(4.0)), 0.5])
    expect = a * c + (1 - a) * np.array([0.0, 0.0, 1.0])
    np.testing.assert_allclose(np.asarray(out.color)[8, 8], expect, atol=1e-7)
    assert float(np.asarray(out.alpha)[8, 8]) == pytest.approx(a, abs=1e-7)


def test_two_primitive_over_order_front_wins(pf):
    # test_raster.py:140-153: the z-front opaque layer hides the one behind it
    raster, _ = pf
    from paper_2602_22625_b200.scene import PrimitiveParams, PrimitiveTemplate, Scene

    t = np.zeros((5, 5, 4))
    t[:, :, 3] = 1.0
    t[:, :, :3] = 0.5
    front = PrimitiveParams(x=8, y=8, scale=4, opacity_logit=50.0,
                            color_logits=(9.0, -9.0, -9.0), z=0)
    back = PrimitiveParams(x=8, y=8, scale=4, opacity_logit=50.0,
                           color_logits=(-9.0, 9.0, -9.0), z=1)
    sc = Scene([back, front], [PrimitiveTemplate(t)], 16, 16, background=(0, 0, 0))
    out, _ = raster.render_forward(sc, eps_skip=0.0)
    np.testing.assert_allclose(np.asarray(out.color)[8, 8], [1, 0, 0], atol=1e-3)


def test_eps_skip_zero_vs_default_differ_only_slightly(pf):
    # test_raster.py:165-170 (there on random_scene(3, n=15); here the golden random_s3 =
    # random_scene(3, n=12, 40x36))
    raster, _ = pf
    sc = scene_from(load_case("random_s3"))
    exact, _ = raster.render_forward(sc, eps_skip=0.0)
    fast, _ = raster.render_forward(sc)
    d = np.abs(np.asarray(exact.color) - np.asarray(fast.color)).max()
    assert 0.0 < d < 5e-2


def test_optimize_reduces_loss_logs_and_dumps(pf, tmp_path):
    """test_fit.py:283-301 through fit.optimize on the GPU (default templates,
    the reference's smoke config), plus the dump_dir / dump_every images
    (fit.py:509-518: the pre-update render of every dump_every-th iteration)."""
    import csv

    from scipy.ndimage import gaussian_filter

    from paper_2602_22625_b200 import fit

    img = gaussian_filter(np.random.default_rng(0).random((32, 32, 3)), (6, 6, 0))
    target = (img - img.min()) / (img.max() - img.min())
    log = tmp_path / "fit_log.csv"
    cfg = fit.FitConfig(num_primitives=20, num_iterations=80, seed=0, tile_size=16,
                        scale_min=2.0, scale_max=8.0, do_reinit=False, compute_psnr=True,
                        bg_color="black", dump_every=40)
    scene, history = fit.optimize(target, None, cfg, log_path=log, dump_dir=tmp_path / "dump")
    assert scene.n == 20 and len(history) == 80
    first, last = history[0], history[-1]
    assert last.loss < first.loss * 0.5
    assert last.psnr > first.psnr
    assert history[0].lr == pytest.approx(cfg.learning_rate)
    assert history[-1].lr == pytest.approx(cfg.learning_rate * cfg.decay_final_fraction)
    with open(log, newline="") as f:
        rows = list(csv.reader(f))
    assert rows[0] == ["iter", "loss", "psnr", "lr", "reinit_count"]
    assert len(rows) == 81
    assert float(rows[1][1]) == pytest.approx(first.loss)
    assert int(rows[-1][0]) == 79
    dumps = sorted(p.name for p in (tmp_path / "dump").iterdir())
    assert dumps == ["iter_00000.png", "iter_00040.png"]


def test_bin_tiles_culls_far_primitives(pf):
    # test_raster.py:217-226 on the GPU binning
    raster, _ = pf
    from paper_2602_22625_b200.scene import PrimitiveParams, PrimitiveTemplate, Scene

    near = PrimitiveParams(x=8.0, y=8.0, scale=3.0, z=0)
    far = PrimitiveParams(x=100.0, y=100.0, scale=3.0, z=1)
    sc = Scene([near, far], [PrimitiveTemplate(_soft_disk(15))], 128, 128)
    bins = raster.bin_tiles(sc, tile_size=32, padding=2.0)
    first = list(bins.tile_list(0, 0))
    assert 0 in first and 1 not in first


def test_render_ignores_fully_offcanvas_primitive(pf):
    # test_raster.py:229-238: bit-identical image with and without an off-canvas primitive
    raster, _ = pf
    from paper_2602_22625_b200.scene import PrimitiveParams, PrimitiveTemplate, Scene

    tpl = PrimitiveTemplate(_soft_disk(15))
    both = Scene([PrimitiveParams(x=10.0, y=10.0, scale=4.0, z=0),
                  PrimitiveParams(x=-50.0, y=-50.0, scale=4.0, z=1)], [tpl], 24, 24)
    only = Scene([PrimitiveParams(x=10.0, y=10.0, scale=4.0, z=0)], [tpl], 24, 24)
    a, _ = raster.render_forward(both, raster.bin_tiles(both), eps_skip=0.0)
    b, _ = raster.render_forward(only, raster.bin_tiles(only), eps_skip=0.0)
    np.testing.assert_array_equal(np.asarray(a.color), np.asarray(b.color))
