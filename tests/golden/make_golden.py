"""Generate golden vectors by running the REFERENCE package (primfit) itself.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Writes tests/golden/*.npz.  Each case stores the inputs (packed params,
template ids, z, templates, canvas, background, flags) and the reference's
outputs: bin_tiles at tile 16 and 32 (padding 2 and 5), render_forward
image/alpha at eps 0 and default eps, the saved-entry count, backward
gradients for an MSE pull-back (and an alpha objective where noted), and
Adam / run_loop rollouts.  Scenes come from the reference's own test
fixtures (conftest.random_scene, small_scene, grad.gradcheck_scene,
test_grad's saturated-alpha scene) plus aspect / mu_blend / noise-background
/ spatial-loss variants and a structure-aware init check for the synthetic
workload generator.  These files are committed; the GPU box never reads
/root/reference.
"""

from __future__ import annotations

import hashlib
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ.setdefault("NUMBA_NUM_THREADS", "4")
REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(OUT.parent.parent))

import numpy as np  # noqa: E402
from conftest import random_scene, soft_disk  # noqa: E402  (reference test fixtures)
from primfit import config as rconfig  # noqa: E402
from primfit import fit as rfit  # noqa: E402
from primfit import grad as rgrad  # noqa: E402
from primfit import prep as rprep  # noqa: E402
from primfit import raster as rr  # noqa: E402
from primfit.scene import PrimitiveParams, PrimitiveTemplate, Scene, pack_params  # noqa: E402


def scene_arrays(scene) -> dict:
    vec, _ = pack_params(scene)
    d = {
        "params": vec.reshape(-1, 8),
        "tid": np.asarray([p.template_id for p in scene.primitives], dtype=np.int32),
        "z": np.asarray([p.z for p in scene.primitives], dtype=np.int64),
        "canvas": np.asarray([scene.canvas_w, scene.canvas_h]),
        "alpha_max": np.float64(scene.alpha_max),
        "mu_blend": np.float64(scene.mu_blend),
        "preserve_aspect": np.bool_(scene.preserve_aspect),
        "n_templates": np.int64(len(scene.templates)),
    }
    if isinstance(scene.background, str):
        d["background_noise"] = np.bool_(True)
    else:
        d["background"] = np.asarray(scene.background, dtype=np.float64)
    for k, t in enumerate(scene.templates):
        d[f"tpl{k}"] = t.rgba
    return d


def render_case(name: str, scene, target=None, *, bg=None, dA_target=None, extra=None):
    d = scene_arrays(scene)
    for tile, pad in ((16, 2.0), (32, 2.0), (16, 5.0)):
        b = rr.bin_tiles(scene, tile, pad)
        d[f"bin{tile}_p{int(pad)}_off"] = b.offsets
        d[f"bin{tile}_p{int(pad)}_idx"] = b.indices
    if bg is not None:
        d["bg_image"] = bg
    bins = rr.bin_tiles(scene)
    out0, _ = rr.render_forward(scene, bins, background=bg, eps_skip=0.0)
    d["img_eps0"], d["alpha_eps0"] = out0.color, out0.alpha
    out, saved = rr.render_forward(scene, bins, background=bg, save=True)
    d["img"], d["alpha"] = out.color, out.alpha
    d["n_entries"] = np.int64(saved.n_entries)
    if target is None:
        target = np.random.default_rng(1234).random((scene.canvas_h, scene.canvas_w, 3))
    d["target"] = target
    value, dI = rfit.loss_mse(out.color, target)
    d["loss"] = np.float64(value)
    d["dI"] = dI
    d["grads"] = rgrad.backward(scene, saved, dI).data
    # eps 0 saved pass + grads, for the tight fast-vs-dense style checks
    out0s, saved0 = rr.render_forward(scene, bins, background=bg, save=True, eps_skip=0.0)
    _, dI0 = rfit.loss_mse(out0s.color, target)
    d["dI_eps0"] = dI0
    d["grads_eps0"] = rgrad.backward(scene, saved0, dI0).data
    if dA_target is not None:
        dA = 2.0 * (out.alpha - dA_target) / dA_target.size
        dIz = np.zeros_like(out.color)
        d["dA"] = dA
        d["grads_alpha_obj"] = rgrad.backward(scene, saved, dIz, dL_dA=dA).data
    if extra:
        d.update(extra)
    np.savez_compressed(OUT / f"{name}.npz", **d)
    print(name, "n", scene.n, "K16", len(d["bin16_p2_idx"]), "E", saved.n_entries)


def small_scene():
    prims = [
        PrimitiveParams(x=10.0, y=12.0, scale=5.0, rotation=0.3, opacity_logit=1.0,
                        color_logits=(0.2, -0.4, 0.8), z=0),
        PrimitiveParams(x=20.0, y=18.0, scale=7.0, rotation=-1.1, opacity_logit=0.0,
                        color_logits=(-0.5, 0.5, 0.0), z=1),
        PrimitiveParams(x=16.0, y=8.0, scale=4.0, rotation=2.0, opacity_logit=-1.0,
                        color_logits=(1.0, 0.0, -1.0), z=2),
    ]
    return Scene(primitives=prims, templates=[PrimitiveTemplate(soft_disk())], canvas_w=32,
                 canvas_h=28, background=(0.1, 0.2, 0.3))


def saturated_scene():
    t = np.zeros((35, 35, 4))
    t[9:-9, 9:-9, 3] = 1.0
    t[:, :, :3] = 0.3
    tpl = rprep.gaussian_blur_template(
        rprep.gaussian_blur_template(PrimitiveTemplate(t), 1.2), 1.0)
    prims = [
        PrimitiveParams(x=12.0, y=12.0, scale=8.0, opacity_logit=40.0,
                        color_logits=(1.0, 0.0, -1.0), z=0),
        PrimitiveParams(x=13.0, y=12.0, scale=8.0, opacity_logit=0.5,
                        color_logits=(-1.0, 0.5, 0.2), z=1),
    ]
    return Scene(primitives=prims, templates=[tpl], canvas_w=24, canvas_h=24,
                 background=(0.2, 0.2, 0.2))


def aspect_scene(seed: int):
    rng = np.random.default_rng(seed)
    tpls = []
    for (h, w) in ((12, 30), (26, 10)):
        raw = np.zeros((h, w, 4))
        raw[2:-2, 2:-2, 3] = 0.3 + 0.7 * rng.random((h - 4, w - 4))
        raw[:, :, :3] = rng.random((h, w, 3))
        tpls.append(rprep.gaussian_blur_template(PrimitiveTemplate(raw), 1.0))
    n = 14
    zp = rng.permutation(n)
    prims = [PrimitiveParams(x=float(rng.uniform(-5, 60)), y=float(rng.uniform(-5, 50)),
                             scale=float(rng.uniform(2.0, 12.0)),
                             rotation=float(rng.uniform(-7, 7)),
                             opacity_logit=float(rng.uniform(-2, 3)),
                             color_logits=tuple(float(v) for v in rng.uniform(-2, 2, 3)),
                             template_id=int(rng.integers(0, 2)), z=int(zp[i])) for i in range(n)]
    return Scene(prims, tpls, 56, 44, background=(0.9, 0.5, 0.1), alpha_max=0.8, mu_blend=0.35,
                 preserve_aspect=True)


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    render_case("small_scene", small_scene())
    for seed in range(6):
        sc = random_scene(seed, n=12, w=40, h=36)
        render_case(f"random_s{seed}", sc,
                    np.random.default_rng(seed + 100).random((36, 40, 3)))
    # alpha objective (test_grad.py:59-70)
    sc = random_scene(5, n=6)
    ta = np.zeros((sc.canvas_h, sc.canvas_w))
    ta[8:30, 8:30] = 1.0
    render_case("alpha_obj_s5", sc, dA_target=ta)
    for seed in (1, 7):
        sc, tgt = rgrad.gradcheck_scene(seed)
        render_case(f"gradcheck_s{seed}", sc, tgt)
    render_case("saturated", saturated_scene(), np.full((24, 24, 3), 0.6))
    for seed in (0, 1):
        render_case(f"aspect_mu_s{seed}", aspect_scene(seed))
    # per-pixel (noise) background
    sc = random_scene(9, n=15, w=48, h=40)
    sc.background = "noise"
    bg = rr.noisy_background(48, 40, np.random.default_rng(77))
    render_case("noise_bg", sc, bg=bg)
    # medium scene: many prims, several tiles, long lists
    sc = random_scene(21, n=300, w=160, h=120, n_templates=3)
    render_case("medium_n300", sc, np.random.default_rng(5).random((120, 160, 3)))

    # Adam rollout with frozen rows, gains and clamp (fit.py:195-238)
    rng = np.random.default_rng(4)
    from primfit.scene import ParamLayout
    n = 5
    layout = ParamLayout(n)
    p0 = rng.normal(size=layout.size) + 5.0
    state = rfit.OptimState.fresh(layout)
    state.frozen[2] = True
    gains = rfit.gains_vector(layout, {"x": 10.0, "y": 10.0, "scale": 10.0, "opacity": 1.5})
    cur = p0.copy()
    gs, outs = [], []
    for t in range(1, 5):
        g = rng.normal(size=layout.size)
        cur = rfit.adam_step(cur, g, state, 0.05 * t, gains, s_min=4.0, s_max=6.0, layout=layout)
        gs.append(g)
        outs.append(cur.copy())
    np.savez_compressed(OUT / "adam_rollout.npz", p0=p0, grads=np.stack(gs), outs=np.stack(outs),
                        m=state.m, v=state.v, frozen=state.frozen, gains=gains,
                        lrs=np.asarray([0.05 * t for t in range(1, 5)]))

    # run_loop rollout (the hot path's caller, fit.py:403-521)
    from paper_2602_22625_b200 import synth
    tpls = [PrimitiveTemplate(t.rgba) for t in synth.prepare([synth.disc(32)])]
    target = synth.smooth_target(64, 48, seed=3)
    cfg = rconfig.FitConfig(num_iterations=6, num_primitives=40, seed=3, scale_min=2.0,
                            scale_max=9.0)
    scene = rfit.init_scene(target, tpls, cfg, np.random.default_rng(3))
    spec = rfit.LossSpec(kind="mse", target=target)
    scene_end, hist, st = rfit.run_loop(scene, cfg, spec, np.random.default_rng(3))
    d = scene_arrays(scene)
    d.update(target=target, final_params=pack_params(scene_end)[0].reshape(-1, 8),
             hist_loss=np.asarray([h.loss for h in hist]),
             hist_psnr=np.asarray([h.psnr for h in hist]),
             hist_lr=np.asarray([h.lr for h in hist]), m=st.m, v=st.v,
             iters=np.int64(6), scale_min=2.0, scale_max=9.0,
             padding=np.float64(rfit.effective_padding(cfg)))
    np.savez_compressed(OUT / "run_loop_small.npz", **d)
    print("run_loop", hist[0].loss, hist[-1].loss)

    # structure-aware init of the synthetic workloads (c1, and a c3 crop count)
    w1 = synth.make_workload("c1")
    cfg1 = rconfig.FitConfig(num_primitives=200, seed=0, scale_min=2.0, scale_max=16.0)
    ref1 = rfit.init_scene(w1.target, [PrimitiveTemplate(t.rgba) for t in w1.scene.templates],
                           cfg1, np.random.default_rng(0))
    np.savez_compressed(OUT / "synth_c1_init.npz", params=pack_params(ref1)[0].reshape(-1, 8),
                        tid=np.asarray([p.template_id for p in ref1.primitives]),
                        z=np.asarray([p.z for p in ref1.primitives]),
                        tpl0=ref1.templates[0].rgba,
                        target_sha=hashlib.sha256(w1.target.tobytes()).hexdigest())
    print("synth c1 ok")


def aux_cases():
    """f3 / f4 rows of SURVEY §8: layered export (exportio.scale_scene / layer_bbox /
    render_layer, exportio.py:272-346) and the video heuristics (dyn.diff_mask /
    freeze_flags / remove_stuck, dyn.py:86-177), straight from the reference."""
    from primfit import dyn as rdyn
    from primfit import exportio as rex
    from primfit.errors import DegenerateBBox

    # export: mixed scenes (aspect + mu_blend > 0, plain), every layer at rho 1, 2, 4
    for name, sc in (("export_aspect_mu", aspect_scene(1)), ("export_random", random_scene(3, n=10, w=40, h=36))):
        d = scene_arrays(sc)
        for rho in (1, 2, 4):
            scaled = rex.scale_scene(sc, rho)
            boxes, chunks, offs = [], [], [0]
            for i in range(sc.n):
                try:
                    bbox, rgba = rex.render_layer(scaled, i)
                except DegenerateBBox:
                    bbox, rgba = (-1, -1, -1, -1), np.zeros((0, 0, 4))
                boxes.append(bbox)
                chunks.append(rgba.reshape(-1, 4))
                offs.append(offs[-1] + rgba.shape[0] * rgba.shape[1])
            d[f"rho{rho}_bbox"] = np.asarray(boxes, dtype=np.int64)
            d[f"rho{rho}_off"] = np.asarray(offs, dtype=np.int64)
            d[f"rho{rho}_rgba"] = np.concatenate(chunks, axis=0)
        np.savez_compressed(OUT / f"{name}.npz", **d)

    # video heuristics on a medium scene with a partly changed frame pair
    sc = random_scene(4, n=60, w=96, h=80)
    rng = np.random.default_rng(21)
    prev = rng.random((80, 96, 3))
    cur = prev.copy()
    cur[10:40, 20:70] += rng.uniform(-0.05, 0.05, (30, 50, 3))
    d = scene_arrays(sc)
    d["prev"], d["cur"] = prev, cur
    for tau in (0.0, 2.0 / 255.0, 0.02):
        m = rdyn.diff_mask(prev, cur, tau).mask
        d[f"mask_{tau!r}"] = m
    m = rdyn.diff_mask(prev, cur, 2.0 / 255.0)
    for pad in (2.0, 5.0):
        d[f"frozen_p{int(pad)}"] = rdyn.freeze_flags(sc, m, pad)
    frozen = d["frozen_p2"]
    # a policy loose enough that several primitives qualify
    pol = rdyn.StuckPolicy(grid=(3, 4), k=2, tau_scale=0.02, tau_alpha=0.3, zeta=0.3, eta=0.5)
    new, decayed = rdyn.remove_stuck(sc, frozen, pol)
    d["stuck_decayed"] = np.asarray(decayed, dtype=np.int64)
    d["stuck_params"] = pack_params(new)[0].reshape(-1, 8)
    d["stuck_policy"] = np.asarray([3, 4, 2, 0.02, 0.3, 0.3, 0.5])
    new0, dec0 = rdyn.remove_stuck(sc, None, pol)
    d["stuck_decayed_nofrozen"] = np.asarray(dec0, dtype=np.int64)
    np.savez_compressed(OUT / "video_heuristics.npz", **d)


def loop_cases():
    """f1 / f3 callers of the fit loop, straight from the reference: low-opacity
    reinit (fit.reinit_low_opacity, fit.py:261-335, unit + inside run_loop at
    period boundaries, also with a noise background so the rng draw order is
    pinned) and the video driver (dyn.optimize_video, dyn.py:180-238, default
    templates)."""
    from primfit import dyn as rdyn
    from paper_2602_22625_b200 import synth

    # unit: reinit on a scene with mixed opacities, some frozen, non-zero moments
    sc = random_scene(5, n=30, w=48, h=40)
    rng = np.random.default_rng(17)
    prims = list(sc.primitives)
    for i in range(len(prims)):
        prims[i].opacity_logit = float(-3.0 if i % 3 else 1.5)
    target = synth.smooth_target(48, 40, seed=5)
    vec, layout = pack_params(sc)
    st = rfit.OptimState.fresh(layout)
    st.m[:] = rng.normal(size=st.m.shape)
    st.v[:] = rng.random(st.v.shape)
    frozen = np.zeros(sc.n, dtype=bool)
    frozen[[1, 4, 7]] = True
    d = scene_arrays(sc)
    d.update(target=target, m0=st.m.copy(), v0=st.v.copy(), frozen=frozen)
    new, count = rfit.reinit_low_opacity(sc, target, 0.3, np.random.default_rng(23), st,
                                         s_min=2.0, s_max=9.0, v_init_bias=-4.0, sigma_c=0.02,
                                         density_cap=100, base_prob=0.1, window=7, frozen=frozen)
    d.update(new_params=pack_params(new)[0].reshape(-1, 8), count=np.int64(count), m1=st.m,
             v1=st.v)
    np.savez_compressed(OUT / "reinit_unit.npz", **d)
    print("reinit unit", count)

    # run_loop with reinit every 3 iterations past warmup 1 (boundaries 3 and 6)
    tpls = [PrimitiveTemplate(t.rgba) for t in synth.prepare([synth.disc(32)])]
    for name, bg in (("run_loop_reinit", "white"), ("run_loop_reinit_noise", "noise")):
        target = synth.smooth_target(64, 48, seed=3)
        cfg = rconfig.FitConfig(num_iterations=9, num_primitives=40, seed=3, scale_min=2.0,
                                scale_max=9.0, do_reinit=True, reinit_period=3,
                                reinit_warmup=1, bg_color=bg)
        scene = rfit.init_scene(target, tpls, cfg, np.random.default_rng(3))
        for i, p in enumerate(scene.primitives):
            if i % 2 == 0:
                p.opacity_logit = 1.0  # well above the threshold: never re-seeded
        spec = rfit.LossSpec(kind="mse", target=target)
        scene_end, hist, st = rfit.run_loop(scene, cfg, spec, np.random.default_rng(4))
        d = scene_arrays(scene)
        d.update(target=target, final_params=pack_params(scene_end)[0].reshape(-1, 8),
                 hist_loss=np.asarray([h.loss for h in hist]),
                 hist_psnr=np.asarray([h.psnr for h in hist]),
                 hist_lr=np.asarray([h.lr for h in hist]),
                 hist_reinit=np.asarray([h.reinit_count for h in hist]), m=st.m, v=st.v,
                 iters=np.int64(9), scale_min=2.0, scale_max=9.0,
                 padding=np.float64(rfit.effective_padding(cfg)))
        np.savez_compressed(OUT / f"{name}.npz", **d)
        print(name, [h.reinit_count for h in hist], hist[0].loss, hist[-1].loss)

    # the video driver: default templates, init_scene from the config, 2 frames
    f0 = synth.smooth_target(48, 40, seed=8)
    f1 = f0.copy()
    f1[10:25, 12:30] = 1.0 - f1[10:25, 12:30]
    cfg = rconfig.FitConfig(num_iterations=5, sequential_iterations=4, num_primitives=30,
                            seed=5, scale_min=2.0, scale_max=8.0, freeze_static=True,
                            remove_stuck=True, stuck_triggers=(1, 3), stuck_tau_scale=0.5,
                            stuck_tau_alpha=0.5)
    scenes, hists = rdyn.optimize_video([f0, f1], None, cfg)
    np.savez_compressed(
        OUT / "video_dropin.npz", f0=f0, f1=f1,
        params0=pack_params(scenes[0])[0].reshape(-1, 8),
        params1=pack_params(scenes[1])[0].reshape(-1, 8),
        loss0=np.asarray([h.loss for h in hists[0]]), loss1=np.asarray([h.loss for h in hists[1]]),
        tid=np.asarray([p.template_id for p in scenes[0].primitives]),
        z=np.asarray([p.z for p in scenes[0].primitives]), tpl0=scenes[0].templates[0].rgba)
    print("video", hists[0][-1].loss, hists[1][-1].loss)


def hook_cases():
    """run_loop's remaining contract, from the reference's own run: hooks that
    rewrite the scene before an iteration's render (fit.py:436-439; test_fit.py's
    test_run_loop_hook_rewrites_scene), frozen rows in the optimizer state, lr
    gains and the decaying schedule, the combined loss (fit.py:163-170), then a
    resumed run_loop on the same OptimState with an explicit iteration count and
    the spatial loss (fit.py:128-151; test_run_loop_reuses_optimizer_state)."""
    from dataclasses import replace as _rep

    from paper_2602_22625_b200 import synth

    tpls = [PrimitiveTemplate(t.rgba) for t in synth.prepare([synth.disc(32)])]
    target = synth.smooth_target(64, 48, seed=11)
    cfg = rconfig.FitConfig(num_iterations=6, num_primitives=40, seed=6, scale_min=2.0,
                            scale_max=9.0, do_decay=True, decay_final_fraction=0.2,
                            lr_gain_x=2.0, lr_gain_y=0.5, lr_gain_scale=3.0,
                            lr_gain_rotation=0.7, lr_gain_opacity=1.3, lr_gain_color=0.8)
    scene = rfit.init_scene(target, tpls, cfg, np.random.default_rng(6))
    vec, layout = pack_params(scene)
    st0 = rfit.OptimState.fresh(layout)
    st0.frozen[[0, 5, 9]] = True
    seen = []

    def fade(s, state):  # iteration 2: every third primitive nearly transparent
        seen.append(("fade", state.step))
        return _rep(s, primitives=[_rep(p, opacity_logit=-6.0) if i % 3 == 0 else p
                                   for i, p in enumerate(s.primitives)])

    def shift(s, state):  # iteration 4: even primitives move right by 3 px
        seen.append(("shift", state.step))
        return _rep(s, primitives=[_rep(p, x=p.x + 3.0) if i % 2 == 0 else p
                                   for i, p in enumerate(s.primitives)])

    spec1 = rfit.LossSpec(kind="combined", target=target, mse_w=0.7, gray_l1_w=0.4)
    s1, h1, st = rfit.run_loop(scene, cfg, spec1, np.random.default_rng(7), state=st0,
                               hooks={2: fade, 4: shift})
    p1 = pack_params(s1)[0].reshape(-1, 8)
    ta = np.zeros((48, 64))
    ta[6:40, 10:50] = 0.8
    spec2 = rfit.LossSpec(kind="spatial_constrained", target=target, target_alpha=ta,
                          alpha_w=0.5)
    s2, h2, st = rfit.run_loop(s1, cfg, spec2, np.random.default_rng(8), iterations=4,
                               state=st)
    d = scene_arrays(scene)
    d.update(target=target, target_alpha=ta, frozen=st0.frozen.copy(), params1=p1,
             final_params=pack_params(s2)[0].reshape(-1, 8),
             h1_loss=np.asarray([h.loss for h in h1]), h1_psnr=np.asarray([h.psnr for h in h1]),
             h1_lr=np.asarray([h.lr for h in h1]),
             h2_loss=np.asarray([h.loss for h in h2]), h2_lr=np.asarray([h.lr for h in h2]),
             hook_steps=np.asarray([s for _, s in seen]), final_step=np.int64(st.step),
             m=st.m, v=st.v, scale_min=2.0, scale_max=9.0)
    np.savez_compressed(OUT / "run_loop_hook_resume.npz", **d)
    print("hook/resume", seen, h1[-1].loss, h2[-1].loss, st.step)

    # optimize (fit.py:524-555): seed -> prepare_templates -> init_scene -> config
    # loss -> run_loop, on the acceptance suite's hard disk (make_assets.py:70-79)
    size = 25
    yy, xx = np.mgrid[0:size, 0:size].astype(np.float64)
    c = (size - 1) / 2
    disk = np.zeros((size, size, 4))
    disk[:, :, :3] = 1.0
    disk[:, :, 3] = (np.hypot(yy - c, xx - c) <= c - 1.0).astype(np.float64)
    target = synth.smooth_target(64, 48, seed=12)
    ta = np.zeros((48, 64))
    ta[8:40, 12:52] = 1.0
    cfg = rconfig.FitConfig(num_primitives=40, num_iterations=8, seed=2, loss="spatial",
                            alpha_loss_weight=0.3, do_reinit=True, reinit_period=3,
                            reinit_warmup=2)
    sc, hist = rfit.optimize(target, [PrimitiveTemplate(disk)], cfg, target_alpha=ta)
    np.savez_compressed(OUT / "optimize_small.npz", target=target, target_alpha=ta, disk=disk,
                        final_params=pack_params(sc)[0].reshape(-1, 8),
                        tid=np.asarray([p.template_id for p in sc.primitives]),
                        z=np.asarray([p.z for p in sc.primitives]),
                        hist_loss=np.asarray([h.loss for h in hist]),
                        hist_psnr=np.asarray([h.psnr for h in hist]),
                        hist_reinit=np.asarray([h.reinit_count for h in hist]))
    print("optimize", hist[0].loss, hist[-1].loss, [h.reinit_count for h in hist])


def acceptance_cases():
    """The reference's acceptance criteria on this path (test_acceptance.py):
    01 -- run_gradcheck(20) (grad.py:378-420): the 20 gradcheck scenes with the
    reference's central finite differences through render_naive; 02 -- the 50
    random scenes (n = 4..200 on 128x128) of the tiled-vs-naive forward check
    (scenes only: the GPU test checks them against the pinned oracle)."""
    d = {}
    for seed in range(20):
        scene, target = rgrad.gradcheck_scene(seed)

        def loss_fn(o, target=target):
            return float(np.mean((o.color - target) ** 2))

        fd = rgrad.finite_diff_grad(scene, loss_fn)
        for k, v in scene_arrays(scene).items():
            d[f"g{seed}_{k}"] = v
        d[f"g{seed}_target"] = target
        d[f"g{seed}_fd"] = fd.data
    for seed in range(50):
        n = 4 + (196 * seed) // 49
        scene = random_scene(seed, n=n, w=128, h=128)
        for k, v in scene_arrays(scene).items():
            d[f"r{seed}_{k}"] = v
    np.savez_compressed(OUT / "acceptance.npz", **d)
    print("acceptance", len(d))
    # the scenes of the reference's export tests (test_export.py:226-293)
    e = {}
    for tag, (seed, n, w, h) in {"x8": (8, 5, 36, 28), "x9": (9, 2, 48, 48),
                                 "x10": (10, 3, 20, 20), "x11": (11, 4, 24, 24)}.items():
        for k, v in scene_arrays(random_scene(seed, n=n, w=w, h=h)).items():
            e[f"{tag}_{k}"] = v
    np.savez_compressed(OUT / "export_tests.npz", **e)


if __name__ == "__main__":
    if "--acceptance" in sys.argv:
        acceptance_cases()
        raise SystemExit(0)
    if "--hooks" in sys.argv:
        hook_cases()
        raise SystemExit(0)
    if "--loops" in sys.argv:
        loop_cases()
        raise SystemExit(0)
    if "--aux" in sys.argv:
        aux_cases()
        raise SystemExit(0)
    main()
