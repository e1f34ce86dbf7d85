"""GPU parity: the CUDA path (through the C ABI) against reference golden vectors.

Bar (north_star): binning bit-exact; forward |d| <= 1e-5 * max(|ref|, 1e-3);
gradients |d| <= 1e-3 * max(|ref|, 1e-2 * column max); Adam to float64
rounding.  The achieved errors are far tighter (float64 decision chain), and
the tests also assert those tighter observed levels so regressions show up.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import RENDER_CASES, fwd_close, grad_close, load_case, scene_from

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pf():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_22625_b200 import fit, grad, raster

    return raster, grad, fit


@pytest.mark.parametrize("case", RENDER_CASES)
def test_gpu_bins_bit_exact(pf, case):
    raster, _, _ = pf
    d = load_case(case)
    sc = scene_from(d)
    for tile, pad in ((16, 2), (32, 2), (16, 5)):
        b = raster.bin_tiles(sc, tile, float(pad))
        np.testing.assert_array_equal(b.offsets, d[f"bin{tile}_p{pad}_off"])
        np.testing.assert_array_equal(b.indices, d[f"bin{tile}_p{pad}_idx"])


@pytest.mark.parametrize("case", RENDER_CASES)
def test_gpu_forward_matches_reference(pf, case):
    raster, _, _ = pf
    d = load_case(case)
    sc = scene_from(d)
    bg = d.get("bg_image")
    out0, _ = raster.render_forward(sc, background=bg, eps_skip=0.0)
    ok, err = fwd_close(out0.color, d["img_eps0"])
    assert ok, f"eps0 color rel err {err}"
    ok, err = fwd_close(out0.alpha, d["alpha_eps0"])
    assert ok, f"eps0 alpha rel err {err}"
    out, saved = raster.render_forward(sc, background=bg, save=True)
    ok, err = fwd_close(out.color, d["img"])
    assert ok, f"color rel err {err}"
    ok, err = fwd_close(out.alpha, d["alpha"])
    assert ok, f"alpha rel err {err}"
    # float64 chain + float32 store: observed error is float32 rounding only
    assert np.abs(out.color - d["img"]).max() < 1e-6
    assert saved.n_entries == int(d["n_entries"])


@pytest.mark.parametrize("case", RENDER_CASES)
def test_gpu_backward_matches_reference(pf, case):
    raster, grad, _ = pf
    d = load_case(case)
    sc = scene_from(d)
    bg = d.get("bg_image")
    out, saved = raster.render_forward(sc, background=bg, save=True)
    g = grad.backward(sc, saved, d["dI"])
    assert np.all(np.isfinite(g.data))
    ok, err = grad_close(g.data, d["grads"])
    assert ok, f"grad rel err {err}"
    assert err < 5e-4  # observed <= 2.4e-4 with fp32 per-pixel math (bar 1e-3)
    out0, saved0 = raster.render_forward(sc, background=bg, save=True, eps_skip=0.0)
    g0 = grad.backward(sc, saved0, d["dI_eps0"])
    ok, err = grad_close(g0.data, d["grads_eps0"])
    assert ok, f"eps0 grad rel err {err}"
    if "grads_alpha_obj" in d:
        g2 = grad.backward(sc, saved, np.zeros_like(d["dI"]), dL_dA=d["dA"])
        ok, err = grad_close(g2.data, d["grads_alpha_obj"])
        assert ok, f"alpha-objective grad rel err {err}"
        assert np.abs(g2.data[:, 4]).max() > 0.0


@pytest.mark.parametrize("case", ["gradcheck_s1", "gradcheck_s7"])
def test_gpu_backward_matches_finite_differences(pf, case):
    """The reference's finite-difference check (test_grad.py:33-46, steps of
    grad.py:48-55, central differences, its tolerance 1e-5 abs or 1e-2 rel), run
    entirely on the CUDA path: the backward's gradient of the MSE against central
    differences of the GPU forward (eps_skip 0) on the reference's gradcheck
    scenes (smooth templates)."""
    raster, grad, _ = pf
    from paper_2602_22625_b200.scene import pack_params, unpack_params

    d = load_case(case)
    sc = scene_from(d)
    target = d["target"]
    out, saved = raster.render_forward(sc, save=True, eps_skip=0.0)
    dL = 2.0 * (np.asarray(out.color) - target) / target.size
    g = grad.backward(sc, saved, dL).data
    steps = (1e-2, 1e-2, 1e-2, 1e-3, 1e-3, 1e-3, 1e-3, 1e-3)
    vec, layout = pack_params(sc)
    fd = np.empty_like(vec)
    for i in range(vec.size):
        h = steps[i % 8]
        lo = []
        for sgn in (1.0, -1.0):
            probe = vec.copy()
            probe[i] = vec[i] + sgn * h
            o, _ = raster.render_forward(unpack_params(probe, layout, sc), eps_skip=0.0)
            lo.append(float(np.mean((np.asarray(o.color, dtype=np.float64) - target) ** 2)))
        fd[i] = (lo[0] - lo[1]) / (2.0 * h)
    fd = fd.reshape(-1, 8)
    for i in range(sc.n):
        for j in range(8):
            a, n = g[i, j], fd[i, j]
            assert abs(a - n) <= 1e-5 or abs(a - n) / max(abs(a), abs(n)) <= 1e-2, (i, j, a, n)


def test_gpu_saturated_alpha_exact(pf):
    # test_grad.py:73-115: alpha == 1 exactly; no division by (1 - alpha)
    raster, grad, _ = pf
    d = load_case("saturated")
    sc = scene_from(d)
    out, saved = raster.render_forward(sc, save=True, eps_skip=0.0)
    assert out.alpha.max() == 1.0
    g = grad.backward(sc, saved, d["dI_eps0"])
    assert np.all(np.isfinite(g.data))
    ok, err = grad_close(g.data, d["grads_eps0"])
    assert ok, err


def test_gpu_stale_and_shape_errors(pf):
    from paper_2602_22625_b200.errors import ShapeMismatch, StaleSavedState

    raster, grad, _ = pf
    sc = scene_from(load_case("small_scene"))
    out, saved = raster.render_forward(sc, save=True)
    with pytest.raises(ShapeMismatch):
        grad.backward(sc, saved, np.zeros((3, 3, 3)))
    sc.primitives[0].x += 1.0
    with pytest.raises(StaleSavedState):
        grad.backward(sc, saved, np.zeros((sc.canvas_h, sc.canvas_w, 3)))


def test_gpu_invisible_primitive_zero_grad(pf):
    # test_grad.py:118-132
    from paper_2602_22625_b200.scene import PrimitiveParams, PrimitiveTemplate, Scene

    raster, grad, _ = pf
    t = np.zeros((7, 7, 4))
    t[1:-1, 1:-1, 3] = 1.0
    t[:, :, :3] = 0.5
    prims = [PrimitiveParams(x=10.0, y=10.0, scale=3.0, opacity_logit=1.0, z=0),
             PrimitiveParams(x=200.0, y=200.0, scale=3.0, opacity_logit=1.0, z=1)]
    sc = Scene(prims, [PrimitiveTemplate(t)], 24, 24)
    out, saved = raster.render_forward(sc, save=True, eps_skip=0.0)
    dL = 2.0 * out.color / out.color.size
    g = grad.backward(sc, saved, dL)
    np.testing.assert_array_equal(g.data[1], np.zeros(8))
    assert np.abs(g.data[0]).max() > 0.0


def test_gpu_adam_rollout(pf):
    _, _, fit = pf
    from paper_2602_22625_b200.scene import ParamLayout

    d = load_case("adam_rollout")
    layout = ParamLayout(d["p0"].size // 8)
    st = fit.OptimState.fresh(layout)
    st.frozen[:] = d["frozen"]
    cur = d["p0"].copy()
    for t in range(4):
        cur = fit.adam_step(cur, d["grads"][t], st, float(d["lrs"][t]), d["gains"],
                            s_min=4.0, s_max=6.0, layout=layout)
        np.testing.assert_allclose(cur, d["outs"][t], rtol=0, atol=1e-14)
    assert st.step == 4
    np.testing.assert_allclose(st.m, d["m"], rtol=0, atol=1e-15)


def test_gpu_run_loop_rollout(pf):
    _, _, fit = pf
    d = load_case("run_loop_small")
    sc = scene_from(d)
    cfg = fit.FitConfig(num_iterations=int(d["iters"]), scale_min=float(d["scale_min"]),
                        scale_max=float(d["scale_max"]))
    spec = fit.LossSpec(kind="mse", target=d["target"])
    end, hist, st = fit.run_loop(sc, cfg, spec, np.random.default_rng(3))
    hl = np.asarray([h.loss for h in hist])
    hp = np.asarray([h.psnr for h in hist])
    np.testing.assert_allclose(hl, d["hist_loss"], rtol=1e-5)
    np.testing.assert_allclose(hp, d["hist_psnr"], rtol=1e-6)
    np.testing.assert_allclose([h.lr for h in hist], d["hist_lr"], rtol=0, atol=0)
    from paper_2602_22625_b200.scene import pack_params

    got = pack_params(end)[0].reshape(-1, 8)
    np.testing.assert_allclose(got, d["final_params"], rtol=1e-4, atol=1e-5)
    assert st.step == int(d["iters"])


@pytest.mark.parametrize("case", ["run_loop_reinit", "run_loop_reinit_noise"])
def test_gpu_run_loop_reinit(pf, case):
    """run_loop with low-opacity reinit at period boundaries (fit.py:454-475):
    the reinit draws come from the caller's rng before the iteration's noise
    background, exactly as the reference; reinit counts, loss history and final
    parameters against the reference's own run."""
    _, _, fit = pf
    from paper_2602_22625_b200.scene import pack_params

    d = load_case(case)
    sc = scene_from(d)
    cfg = fit.FitConfig(num_iterations=int(d["iters"]), num_primitives=sc.n, seed=3,
                        scale_min=float(d["scale_min"]), scale_max=float(d["scale_max"]),
                        do_reinit=True, reinit_period=3, reinit_warmup=1)
    spec = fit.LossSpec(kind="mse", target=d["target"])
    end, hist, st = fit.run_loop(sc, cfg, spec, np.random.default_rng(4))
    assert [h.reinit_count for h in hist] == list(d["hist_reinit"])
    np.testing.assert_allclose([h.loss for h in hist], d["hist_loss"], rtol=1e-5)
    np.testing.assert_allclose([h.psnr for h in hist], d["hist_psnr"], rtol=1e-6)
    got = pack_params(end)[0].reshape(-1, 8)
    np.testing.assert_allclose(got, d["final_params"], rtol=1e-4, atol=1e-5)
    assert st.step == int(d["iters"])


def test_gpu_run_loop_hooks_and_resume(pf):
    """run_loop's contract against the reference's own run (make_golden.py
    --hooks): scene-rewriting hooks before iterations 2 and 4 (fit.py:436-439),
    frozen rows in the passed OptimState, lr gains and the decaying schedule,
    the combined loss; then a resumed run_loop on the same state with
    iterations=4 and the spatial loss (test_fit.py:304-336 as goldens)."""
    from dataclasses import replace as _rep

    _, _, fit = pf
    from paper_2602_22625_b200.scene import pack_params

    d = load_case("run_loop_hook_resume")
    sc = scene_from(d)
    cfg = fit.FitConfig(num_iterations=6, num_primitives=sc.n, seed=6,
                        scale_min=float(d["scale_min"]), scale_max=float(d["scale_max"]),
                        do_decay=True, decay_final_fraction=0.2, lr_gain_x=2.0, lr_gain_y=0.5,
                        lr_gain_scale=3.0, lr_gain_rotation=0.7, lr_gain_opacity=1.3,
                        lr_gain_color=0.8)
    st0 = fit.OptimState.fresh(pack_params(sc)[1])
    st0.frozen[:] = d["frozen"]
    seen = []

    def fade(s, state):
        seen.append(state.step)
        return _rep(s, primitives=[_rep(p, opacity_logit=-6.0) if i % 3 == 0 else p
                                   for i, p in enumerate(s.primitives)])

    def shift(s, state):
        seen.append(state.step)
        return _rep(s, primitives=[_rep(p, x=p.x + 3.0) if i % 2 == 0 else p
                                   for i, p in enumerate(s.primitives)])

    spec1 = fit.LossSpec(kind="combined", target=d["target"], mse_w=0.7, gray_l1_w=0.4)
    s1, h1, st = fit.run_loop(sc, cfg, spec1, np.random.default_rng(7), state=st0,
                              hooks={2: fade, 4: shift})
    assert seen == list(d["hook_steps"])
    np.testing.assert_allclose([h.loss for h in h1], d["h1_loss"], rtol=1e-5)
    np.testing.assert_allclose([h.psnr for h in h1], d["h1_psnr"], rtol=1e-6)
    np.testing.assert_allclose([h.lr for h in h1], d["h1_lr"], rtol=0, atol=0)
    p1 = pack_params(s1)[0].reshape(-1, 8)
    np.testing.assert_allclose(p1, d["params1"], rtol=1e-4, atol=1e-5)
    frozen = np.asarray(d["frozen"])
    # frozen rows: Adam leaves them alone, only the hooks' edits apply (bit for bit)
    assert np.array_equal(p1[frozen], np.asarray(d["params1"])[frozen])
    spec2 = fit.LossSpec(kind="spatial_constrained", target=d["target"],
                         target_alpha=d["target_alpha"], alpha_w=0.5)
    s2, h2, st = fit.run_loop(s1, cfg, spec2, np.random.default_rng(8), iterations=4, state=st)
    np.testing.assert_allclose([h.loss for h in h2], d["h2_loss"], rtol=1e-5)
    np.testing.assert_allclose([h.lr for h in h2], d["h2_lr"], rtol=0, atol=0)
    np.testing.assert_allclose(pack_params(s2)[0].reshape(-1, 8), d["final_params"],
                               rtol=1e-4, atol=1e-5)
    assert st.step == int(d["final_step"])
    np.testing.assert_allclose(st.m, d["m"], rtol=1e-3, atol=1e-7)
    np.testing.assert_allclose(st.v, d["v"], rtol=1e-3, atol=1e-9)


def test_gpu_optimize_video_dropin(pf):
    """video.optimize_video(frames, None, cfg) against dyn.optimize_video: default
    templates through prepare_templates, init_scene from the config, frame 1
    with freezing and stuck decay at the trigger iterations."""
    _, _, fit = pf
    from paper_2602_22625_b200 import video
    from paper_2602_22625_b200.scene import pack_params

    d = load_case("video_dropin")
    cfg = fit.FitConfig(num_iterations=5, sequential_iterations=4, num_primitives=30, seed=5,
                        scale_min=2.0, scale_max=8.0, freeze_static=True, remove_stuck=True,
                        stuck_triggers=(1, 3), stuck_tau_scale=0.5, stuck_tau_alpha=0.5)
    scenes, hists = video.optimize_video([d["f0"], d["f1"]], None, cfg)
    np.testing.assert_array_equal(np.asarray(scenes[0].templates[0].rgba), d["tpl0"])
    assert [p.template_id for p in scenes[0].primitives] == list(d["tid"])
    np.testing.assert_allclose([h.loss for h in hists[0]], d["loss0"], rtol=1e-5)
    np.testing.assert_allclose([h.loss for h in hists[1]], d["loss1"], rtol=1e-5)
    # The default template is a radially symmetric blob: its rotation gradient is
    # round-off (the sampling grid's residual asymmetry), which Adam normalises into
    # +-lr steps of random sign on both sides; those rotations then perturb x / y
    # slightly.  Bar: rotations within the Adam step bound, the other columns
    # mostly equal and all within the bound (test_step_engine_matches_oracle_loop).
    gains = np.asarray([10, 10, 10, 1, 1.5, 1, 1, 1.0])
    for k, steps in ((0, 5), (1, 9)):
        got = pack_params(scenes[k])[0].reshape(-1, 8)
        ref = d[f"params{k}"]
        assert np.all(np.abs(got - ref) <= 2 * 0.1 * gains[None, :] * steps)
        app = [2, 4, 5, 6, 7]  # scale, opacity, colours
        close = np.isclose(got[:, app], ref[:, app], rtol=1e-4, atol=1e-4)
        assert close.mean() > 0.9, close.mean()
        assert (np.abs(got[:, :2] - ref[:, :2]) < 0.25).mean() > 0.95  # positions, px
