"""GPU parity at BASELINE.json sizes against the CPU oracle (same seeded inputs).

c1 (256^2) and c3 (1024x809, the metric config) are rendered on both sides;
bins must be bit-identical, the forward within 1e-5, gradients within 1e-3.
Size-independent properties checked at full size: alpha == 1 - T_final
identity via the saved count, image in [0, 1], step-engine loss history equal
to an independent host loss evaluation.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import fwd_close, grad_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_workload_bins_forward_backward_vs_oracle(torch_cuda, oracle, name):
    from paper_2602_22625_b200 import grad, raster, synth
    from paper_2602_22625_b200.fit import effective_padding

    w = synth.make_workload(name)
    sc = w.scene
    pad = effective_padding(w.cfg)
    pk = oracle.Packed(sc)
    # bins: bit-exact at the GPU render tile (16) and the reference default (32)
    for tile in (16, 32):
        off, idx = oracle.bin_tiles(pk, tile, pad)
        b = raster.bin_tiles(sc, tile, pad)
        np.testing.assert_array_equal(b.offsets, off)
        np.testing.assert_array_equal(b.indices, idx)
    # perturb to a mid-optimisation state: jitter centres, raise opacity
    rng = np.random.default_rng(123)
    for p in sc.primitives:
        p.x += float(rng.uniform(-0.5, 0.5))
        p.y += float(rng.uniform(-0.5, 0.5))
        p.opacity_logit = float(rng.uniform(-2.0, 3.0))
    pk = oracle.Packed(sc)
    off, idx = oracle.bin_tiles(pk, 32, pad)
    bg = oracle.background(sc)
    img, alpha, sv = oracle.render_forward(pk, off, idx, 32, bg, True, 1 / 1024)
    out, saved = raster.render_forward(sc, raster.bin_tiles(sc, 16, pad), save=True)
    ok, err = fwd_close(out.color, img)
    assert ok, f"{name} forward rel err {err}"
    ok, err = fwd_close(out.alpha, alpha)
    assert ok, f"{name} alpha rel err {err}"
    assert saved.n_entries == sv["n_entries"]
    _, dI = oracle.loss_mse(img, w.target)
    g_ref = oracle.backward(pk, sv, dI, None)
    g = grad.backward(sc, saved, dI)
    ok, err = grad_close(g.data, g_ref)
    assert ok, f"{name} grad rel err {err}"


@pytest.mark.parametrize("name,total", [("c1", 8), ("c3", 5)])
def test_step_engine_matches_oracle_loop(torch_cuda, oracle, name, total):
    from paper_2602_22625_b200 import synth
    from paper_2602_22625_b200.fit import StepEngine, effective_padding

    w = synth.make_workload(name)
    w.cfg.num_iterations = total
    eng = StepEngine(w.scene, w.cfg, w.loss, total)
    loop = oracle.Loop(w.scene, w.target, w.cfg, effective_padding(w.cfg), tile=32)
    for it in range(total):
        eng.step()
        loop.step(it, total)
    eng.check()
    hist = eng.history()
    np.testing.assert_allclose([h.loss for h in hist], [h[1] for h in loop.history], rtol=1e-5)
    p_gpu = eng.params_host().reshape(-1, 8)
    p_ref = loop.vec.reshape(-1, 8)
    # Adam normalises each gradient by its own RMS, so a gradient that is zero up
    # to round-off (e.g. a symmetric primitive's rotation) takes a +-lr*gain step
    # whose sign is noise on both sides.  Bar: almost all parameters agree to
    # 1e-4, and every parameter stays within the Adam step bound lr*gain*steps.
    close = np.isclose(p_gpu, p_ref, rtol=1e-4, atol=1e-4)
    assert close.mean() > 0.99, close.mean()
    gains = np.asarray([10, 10, 10, 1, 1.5, 1, 1, 1.0])
    bound = 2 * w.cfg.learning_rate * gains * total
    assert np.all(np.abs(p_gpu - p_ref) <= bound[None, :])


@pytest.fixture
def diag_reload():
    """Re-read the PF_* switches after the test's monkeypatch is undone (list this
    fixture before monkeypatch so its teardown runs after the env is restored)."""
    yield
    from paper_2602_22625_b200 import _native

    _native.load().pf_diag_reload()


@pytest.mark.parametrize("name,two", [("c3", "1"), ("c5", "auto"), ("c5", "0")])
def test_bins_two_level_bit_exact(diag_reload, torch_cuda, oracle, monkeypatch, name, two):
    """Both binning paths (one-level row scan; two-level row counts + stable
    scatter, the default for c5) against the oracle's bin_tiles, full canvas and
    every band of an 8-way row split (the multi-GPU bands)."""
    from paper_2602_22625_b200 import raster, synth
    from paper_2602_22625_b200.dist import row_bands
    from paper_2602_22625_b200.fit import effective_padding

    from paper_2602_22625_b200 import _native

    if two != "auto":
        monkeypatch.setenv("PF_BIN_TWO_LEVEL", two)
    else:
        monkeypatch.delenv("PF_BIN_TWO_LEVEL", raising=False)
    _native.load().pf_diag_reload()  # the switches are read once per process
    w = synth.make_workload(name)
    sc = w.scene
    pad = effective_padding(w.cfg)
    pk = oracle.Packed(sc)
    off, idx = oracle.bin_tiles(pk, 16, pad)
    b = raster.bin_tiles(sc, 16, pad)
    np.testing.assert_array_equal(b.offsets, off)
    np.testing.assert_array_equal(b.indices, idx)
    if name == "c5":
        from paper_2602_22625_b200 import _native as nat

        lib = nat.load()
        H, W = sc.canvas_h, sc.canvas_w
        nty, ntx = -(-H // 16), -(-W // 16)
        launches = lib.pf_bin_launches(sc.n, W, H, 16, 0, nty)
        assert launches == (1 if two == "0" else 4)
        from paper_2602_22625_b200.fit import StepEngine

        monkeypatch.setenv("PF_CSR_STEP", "1")  # the engines' pf_bin (CSR) path
        for band in row_bands(nty, 8):
            eng = StepEngine(sc, w.cfg, w.loss, 1, band=band, use_graph=False)
            eng.refresh()
            eng.comp.bin()
            k = eng.comp.check_overflow()
            t0, t1 = band.ty_begin * ntx, band.ty_end * ntx
            np.testing.assert_array_equal(eng.comp.bin_off.cpu().numpy()[: t1 - t0 + 1],
                                          off[t0 : t1 + 1] - off[t0])
            np.testing.assert_array_equal(eng.comp.bin_idx[:k].cpu().numpy(), idx[off[t0] : off[t1]])


def test_graph_replay_equals_eager(torch_cuda):
    from paper_2602_22625_b200 import synth
    from paper_2602_22625_b200.fit import StepEngine

    w = synth.make_workload("c1")
    w.cfg.num_iterations = 5
    a = StepEngine(w.scene, w.cfg, w.loss, 5, use_graph=True)
    b = StepEngine(w.scene, w.cfg, w.loss, 5, use_graph=False)
    a.run(5)
    b.run(5)
    ha = [h.loss for h in a.history()]
    hb = [h.loss for h in b.history()]
    np.testing.assert_allclose(ha, hb, rtol=1e-12)
    np.testing.assert_allclose(a.params_host(), b.params_host(), rtol=1e-9, atol=1e-12)


def test_chunked_run_equals_steps(torch_cuda):
    """run() with multi-step graphs (CHUNK steps per replay) == single-step replays."""
    from paper_2602_22625_b200 import synth
    from paper_2602_22625_b200.fit import StepEngine

    w = synth.make_workload("c1")
    w.cfg.num_iterations = 21
    a = StepEngine(w.scene, w.cfg, w.loss, 21, use_graph=True)
    b = StepEngine(w.scene, w.cfg, w.loss, 21, use_graph=True)
    a.run(21)  # 1 eager + 2 chunks of 8 + 4 single replays
    for _ in range(21):
        b.step()
    np.testing.assert_array_equal(a.params_host(), b.params_host())
    assert [h.loss for h in a.history()] == [h.loss for h in b.history()]
    assert [h.lr for h in a.history()] == [h.lr for h in b.history()]


def test_host_io_zero_copy_matches_device(torch_cuda):
    """host_io engine (parameters + loss partials in pinned host memory, read and
    written by the kernels directly) == device-resident engine, including a host
    edit of the parameters between two host-driven steps."""
    torch = torch_cuda
    from paper_2602_22625_b200 import synth
    from paper_2602_22625_b200.fit import StepEngine

    w = synth.make_workload("c1")
    w.cfg.num_iterations = 9
    a = StepEngine(w.scene, w.cfg, w.loss, 9, use_graph=True)
    b = StepEngine(w.scene, w.cfg, w.loss, 9, use_graph=True, host_io=True)
    a.run(2)
    b.run(2)
    b.capture_host_io_step()
    n = b.n
    for k in range(5):
        if k == 2:  # host edit: move every primitive by +0.75 px in x
            edited = b.host_vector().reshape(n, 8)
            edited[:, 0] += 0.75
            a.params[:, 0] += 0.75
        if k == 3:  # sparse edit: three primitives jump by 40 px (other tiles)
            edited = b.host_vector().reshape(n, 8)
            for i in (0, 17, n - 1):
                edited[i, 1] += 40.0
                a.params[i, 1] += 40.0
        a.refresh()
        a.step()
        b.host_step()
        torch.cuda.synchronize()
    np.testing.assert_array_equal(a.params_host(), b.io.numpy()[: n * 8])
    np.testing.assert_array_equal(a.last_part.cpu().numpy().reshape(-1, 3), b.host_loss_part())
    np.testing.assert_array_equal(a.hist_part.cpu().numpy().reshape(9, -1, 3)[5],
                                  b.host_loss_part(-2))
    assert [h.loss for h in a.history()] == [h.loss for h in b.history()]


def test_autograd_function_matches_api(torch_cuda):
    torch = torch_cuda
    from paper_2602_22625_b200 import grad, raster
    from paper_2602_22625_b200.autograd import Renderer
    from paper_2602_22625_b200.scene import param_matrix, structure_arrays
    from conftest import load_case, scene_from

    d = load_case("medium_n300")
    sc = scene_from(d)
    tid, z = structure_arrays(sc)
    r = Renderer(sc.templates, tid, z, sc.canvas_w, sc.canvas_h, background=sc.background,
                 alpha_max=sc.alpha_max, mu_blend=sc.mu_blend)
    params = torch.tensor(param_matrix(sc), device="cuda", requires_grad=True)
    img, alpha = r(params)
    target = torch.tensor(d["target"], device="cuda", dtype=torch.float32)
    loss = ((img - target) ** 2).mean()
    loss.backward()
    out, saved = raster.render_forward(sc, save=True)
    # (the forward runs the fit-step kernel in render mode: fp32 compositing,
    # ~1e-7 relative; the north_star bar is 1e-5)
    ok, err = fwd_close(img.detach().cpu().numpy(), out.color)
    assert ok, err
    ok, err = fwd_close(alpha.detach().cpu().numpy(), out.alpha)
    assert ok, err
    dI = 2.0 * (out.color - d["target"]) / out.color.size
    g = grad.backward(sc, saved, dI)
    ok, err = grad_close(params.grad.cpu().numpy(), g.data)
    assert ok, err


@pytest.mark.parametrize("case,bg", [("medium_n300", False), ("saturated", False),
                                     ("random_s3", False), ("random_s3", True)])
def test_autograd_render_mode_matches_k3(torch_cuda, monkeypatch, case, bg):
    """The Renderer's forward through the fit-step kernel (PF_LOSS_RENDER) against
    the K3 forward (PF_RENDER_K3=1): image within the forward bar, gradients of the
    following backward (which reuses the same lists) within the gradient bar of each other."""
    torch = torch_cuda
    from paper_2602_22625_b200.autograd import Renderer
    from paper_2602_22625_b200.scene import param_matrix, structure_arrays
    from conftest import load_case, scene_from

    d = load_case(case)
    sc = scene_from(d)
    tid, z = structure_arrays(sc)
    target = torch.tensor(d["target"], device="cuda", dtype=torch.float32)
    g = torch.Generator(device="cuda").manual_seed(5)
    bg_img = (torch.rand(sc.canvas_h, sc.canvas_w, 3, device="cuda", generator=g)
              if bg else None)
    out = []
    for k3 in ("0", "1"):
        monkeypatch.setenv("PF_RENDER_K3", k3)
        r = Renderer(sc.templates, tid, z, sc.canvas_w, sc.canvas_h, background=sc.background,
                     alpha_max=sc.alpha_max, mu_blend=sc.mu_blend)
        assert r.render_k34 == (k3 == "0")
        p = torch.tensor(param_matrix(sc), device="cuda", requires_grad=True)
        with torch.no_grad():  # forwards without a backward pass (classes left clean)
            r(p, bg_img)
            r(p, bg_img)
        for _ in range(2):  # twice: the pooled compositor's second use
            p.grad = None
            img, alpha = r(p, bg_img)
            (((img - target) ** 2).mean() + 0.5 * (alpha ** 2).mean()).backward()
        out.append((img.detach().cpu().numpy(), alpha.detach().cpu().numpy(),
                    p.grad.cpu().numpy()))
    (i0, a0, g0), (i1, a1, g1) = out
    ok, err = fwd_close(i0, i1)
    assert ok, err
    ok, err = fwd_close(a0, a1)
    assert ok, err
    ok, err = grad_close(g0, g1)
    assert ok, err


def test_autograd_loss_mse_matches_reference_and_torch(torch_cuda, monkeypatch):
    """autograd.loss_mse (the reference's loss_mse, fit.py:110-115, as a fused op):
    loss value against the reference's float64 loss_mse on the same image,
    gradients against the reference backward and the torch-loss path, and the
    renderer's backward takes loss_mse's rows without the repacking kernel."""
    torch = torch_cuda
    from paper_2602_22625_b200 import _native as nat, autograd, grad, raster
    from paper_2602_22625_b200.autograd import Renderer, loss_mse
    from paper_2602_22625_b200.errors import ShapeMismatch
    from paper_2602_22625_b200.scene import param_matrix, structure_arrays
    from conftest import load_case, scene_from

    d = load_case("medium_n300")
    sc = scene_from(d)
    tid, z = structure_arrays(sc)
    r = Renderer(sc.templates, tid, z, sc.canvas_w, sc.canvas_h, background=sc.background,
                 alpha_max=sc.alpha_max, mu_blend=sc.mu_blend)
    target = torch.tensor(d["target"], device="cuda", dtype=torch.float32)
    packs = []
    real = nat.load()

    class Lib:  # counts pf_pack_grad4 calls, forwards everything
        def __getattr__(self, k):
            if k == "pf_pack_grad4":
                packs.append(1)
            return getattr(real, k)

    monkeypatch.setattr(autograd.nat, "load", lambda: Lib())
    p1 = torch.tensor(param_matrix(sc), device="cuda", requires_grad=True)
    img, _ = r(p1)
    loss = loss_mse(img, target)
    loss.backward()
    assert not packs  # loss_mse's rows went to the fit step as they are
    p2 = torch.tensor(param_matrix(sc), device="cuda", requires_grad=True)
    img2, _ = r(p2)
    ((img2 - target) ** 2).mean().backward()
    assert packs
    out, saved = raster.render_forward(sc, save=True)
    ref = float(np.mean((out.color - d["target"]) ** 2))
    assert abs(float(loss.detach()) - ref) <= 1e-6 * ref
    dI = 2.0 * (out.color - d["target"]) / out.color.size
    ok, err = grad_close(p1.grad.cpu().numpy(), grad.backward(sc, saved, dI).data)
    assert ok, err
    ok, err = grad_close(p1.grad.cpu().numpy(), p2.grad.cpu().numpy(), rel=1e-4)
    assert ok, err
    # deterministic: the same image gives the same bits
    assert float(loss_mse(img.detach(), target)) == float(loss.detach())
    with pytest.raises(ShapeMismatch):
        loss_mse(img, target[:-1])
    with pytest.raises(ValueError):
        loss_mse(img.contiguous(), target)


def _fused_grads(eng, image=True):
    """One K2 + K34 launch on the engine's current parameters (no Adam)."""
    eng.refresh()
    c = eng.comp
    c.bin()
    eng.gbuf.zero_()
    c.fit_step(eng.gbuf, eng.sums, eps_skip=eng.eps_skip, bg_rgb=eng.bg_rgb, bg4=eng.bg4,
               loss_kind=eng.loss_kind, tgt4=eng.tgt4, alpha_w=eng.alpha_w, w_mse=eng.w_mse,
               w_gray=eng.w_gray, P_total=eng.P,
               image=image)
    c.check_overflow()
    return (eng.grads.view(-1, 8).cpu().numpy(), eng.sums.cpu().numpy(),
            c.color().double().cpu().numpy(), c.alpha().double().cpu().numpy())


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_fused_combined_loss_matches_oracle(torch_cuda, oracle, name):
    """K34 with the combined loss (mse_w * MSE + gray_l1_w * grayscale L1,
    reference fit.py:119-125, 162-168): loss sums and gradients against the
    oracle's forward + backward driven by the reference formula's dL/dI."""
    from paper_2602_22625_b200 import synth
    from paper_2602_22625_b200.fit import LossSpec, StepEngine, effective_padding, evaluate_loss

    w = synth.make_workload(name)
    sc = w.scene
    rng = np.random.default_rng(11)
    for p in sc.primitives:
        p.x += float(rng.uniform(-0.5, 0.5))
        p.opacity_logit = float(rng.uniform(-2.0, 3.0))
    spec = LossSpec(kind="combined", target=w.target, mse_w=0.7, gray_l1_w=0.4)
    eng = StepEngine(sc, w.cfg, spec, 1, use_graph=False)
    assert eng.fused
    g, sums, color, alpha = _fused_grads(eng)
    pk = oracle.Packed(sc)
    off, idx = oracle.bin_tiles(pk, 32, effective_padding(w.cfg))
    img, a_ref, sv = oracle.render_forward(pk, off, idx, 32, oracle.background(sc), True,
                                           w.cfg.eps_skip)
    ok, err = fwd_close(color, img)
    assert ok, f"{name} combined colour rel err {err}"
    value, dI, dA = evaluate_loss(spec, img, a_ref)
    assert dA is None
    P = img.shape[0] * img.shape[1]
    loss_dev = 0.7 * sums[0] / (3 * P) + 0.4 * sums[1] / P
    np.testing.assert_allclose(loss_dev, value, rtol=1e-5)
    g_ref = oracle.backward(pk, sv, dI, None)
    ok, err = grad_close(g, g_ref)
    assert ok, f"{name} combined grad rel err {err}"


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_fused_step_matches_oracle(torch_cuda, oracle, name):
    """K34 (render -> loss -> backward in one kernel) against the oracle's
    render_forward + loss + backward on the same perturbed mid-fit state."""
    from paper_2602_22625_b200 import synth
    from paper_2602_22625_b200.fit import StepEngine, effective_padding

    w = synth.make_workload(name)
    sc = w.scene
    rng = np.random.default_rng(7)
    for p in sc.primitives:
        p.x += float(rng.uniform(-0.5, 0.5))
        p.y += float(rng.uniform(-0.5, 0.5))
        p.opacity_logit = float(rng.uniform(-2.0, 3.0))
    eng = StepEngine(sc, w.cfg, w.loss, 1, use_graph=False)
    assert eng.fused
    g, sums, color, alpha = _fused_grads(eng)
    pk = oracle.Packed(sc)
    off, idx = oracle.bin_tiles(pk, 32, effective_padding(w.cfg))
    img, a_ref, sv = oracle.render_forward(pk, off, idx, 32, oracle.background(sc), True,
                                           w.cfg.eps_skip)
    ok, err = fwd_close(color, img)
    assert ok, f"{name} fused colour rel err {err}"
    ok, err = fwd_close(alpha, a_ref)
    assert ok, f"{name} fused alpha rel err {err}"
    P = img.shape[0] * img.shape[1]
    diff = img - w.target
    if w.loss.kind == "mse":
        dI, dA = 2.0 * diff / diff.size, None
        np.testing.assert_allclose(sums[0] / (3 * P), np.mean(diff**2), rtol=1e-5)
    else:
        ta = np.asarray(w.loss.target_alpha, dtype=np.float64)
        mk = (ta > 0).astype(np.float64)
        dI = 2.0 * diff * mk[..., None] / diff.size
        dA = w.loss.alpha_w * 2.0 * (a_ref - ta) / P
        np.testing.assert_allclose(sums[1], np.sum((diff * mk[..., None]) ** 2), rtol=1e-5)
        np.testing.assert_allclose(sums[2], np.sum((a_ref - ta) ** 2), rtol=1e-5, atol=1e-9)
    g_ref = oracle.backward(pk, sv, dI, dA)
    ok, err = grad_close(g, g_ref)
    assert ok, f"{name} fused grad rel err {err}"


def test_fused_step_equals_two_kernel_path(torch_cuda, monkeypatch):
    """K34 vs K3 + K4 over a graph-replayed rollout: same loss history and
    parameters (both backwards are fp32 with the same operation order)."""
    from paper_2602_22625_b200 import synth
    from paper_2602_22625_b200.fit import StepEngine

    w = synth.make_workload("c1")
    w.cfg.num_iterations = 6
    a = StepEngine(w.scene, w.cfg, w.loss, 6)
    monkeypatch.setenv("PF_TWO_KERNEL", "1")
    b = StepEngine(w.scene, w.cfg, w.loss, 6)
    assert a.fused and not b.fused
    a.run(6)
    b.run(6)
    np.testing.assert_allclose([h.loss for h in a.history()], [h.loss for h in b.history()],
                               rtol=1e-6)
    # Adam amplifies round-off-level gradient differences (atomic order) into
    # +-lr steps on near-zero components: bar as in the oracle rollout test
    close = np.isclose(a.params_host(), b.params_host(), rtol=1e-4, atol=1e-6)
    assert close.mean() > 0.99, close.mean()


def test_fused_step_deep_stack_spill(torch_cuda, oracle):
    """Pixels with more than 4 contributions exercise the HBM spill of K34's
    shared-memory stack: many overlapping primitives on a small canvas."""
    from paper_2602_22625_b200 import synth
    from paper_2602_22625_b200.fit import StepEngine, effective_padding

    w = synth.make_workload("c1")
    sc = w.scene
    rng = np.random.default_rng(3)
    for p in sc.primitives:  # pile everything into the centre
        p.x = 128.0 + float(rng.uniform(-20, 20))
        p.y = 128.0 + float(rng.uniform(-20, 20))
        p.opacity_logit = -3.0  # low alpha: long lists before T runs out
    eng = StepEngine(sc, w.cfg, w.loss, 1, use_graph=False)
    g, sums, color, alpha = _fused_grads(eng)
    pk = oracle.Packed(sc)
    off, idx = oracle.bin_tiles(pk, 32, effective_padding(w.cfg))
    img, a_ref, sv = oracle.render_forward(pk, off, idx, 32, oracle.background(sc), True,
                                           w.cfg.eps_skip)
    assert np.diff(sv["offsets"]).max() > 8  # the spill path is taken
    ok, err = fwd_close(color, img)
    assert ok, err
    dI = 2.0 * (img - w.target) / img.size
    g_ref = oracle.backward(pk, sv, dI, None)
    ok, err = grad_close(g, g_ref)
    assert ok, f"spill grad rel err {err}"


def _edge_scene(kind: str):
    """Edge scenes for the fused step: primitives off the canvas and one covering
    all of it; a canvas smaller than one tile; a single primitive."""
    from paper_2602_22625_b200 import synth
    from paper_2602_22625_b200.fit import LossSpec
    from paper_2602_22625_b200.scene import PrimitiveParams, Scene

    w = synth.make_workload("c1")
    rng = np.random.default_rng(19)
    if kind == "offcanvas":
        sc = w.scene
        for i, p in enumerate(sc.primitives):
            if i % 3 == 0:
                p.x = -400.0 - 10.0 * i  # far outside (empty rect)
            elif i % 3 == 1:
                p.y = 256.0 + p.scale * 0.5  # straddling the bottom edge
        sc.primitives[5].scale = 200.0  # covers the whole canvas
        sc.primitives[5].opacity_logit = -1.0
        return sc, w.cfg, w.loss
    W, H, n = {"tiny": (13, 9, 6), "single": (40, 36, 1), "empty": (40, 36, 0)}[kind]
    prims = [PrimitiveParams(x=float(rng.uniform(0, W)), y=float(rng.uniform(0, H)),
                             scale=float(rng.uniform(3, 9)), rotation=float(rng.uniform(-3, 3)),
                             opacity_logit=float(rng.uniform(-1, 2)),
                             color_logits=tuple(float(v) for v in rng.uniform(-2, 2, 3)), z=i)
             for i in range(n)]
    sc = Scene(prims, w.scene.templates, W, H, background=(0.3, 0.6, 0.9))
    target = rng.random((H, W, 3))
    return sc, w.cfg, LossSpec(kind="mse", target=target)


@pytest.mark.parametrize("kind", ["offcanvas", "tiny", "single", "empty"])
def test_fused_step_edge_scenes(torch_cuda, oracle, kind):
    from paper_2602_22625_b200.fit import StepEngine, effective_padding

    sc, cfg, loss = _edge_scene(kind)
    eng = StepEngine(sc, cfg, loss, 1, use_graph=False)
    g, sums, color, alpha = _fused_grads(eng)
    pk = oracle.Packed(sc)
    off, idx = oracle.bin_tiles(pk, 32, effective_padding(cfg))
    img, a_ref, sv = oracle.render_forward(pk, off, idx, 32, oracle.background(sc), True,
                                           cfg.eps_skip)
    ok, err = fwd_close(color, img)
    assert ok, f"{kind} colour rel err {err}"
    ok, err = fwd_close(alpha, a_ref)
    assert ok, f"{kind} alpha rel err {err}"
    diff = img - loss.target
    np.testing.assert_allclose(sums[0], np.sum(diff**2), rtol=1e-5)
    if kind == "empty":  # no primitive: the background alone, no gradient
        assert g.size == 0
        return
    g_ref = oracle.backward(pk, sv, 2.0 * diff / diff.size, None)
    ok, err = grad_close(g, g_ref)
    assert ok, f"{kind} grad rel err {err}"
    if kind == "offcanvas":
        assert not g[::3].any()  # empty rects: exactly zero gradient


def test_bins_large_scene_4k(torch_cuda, oracle):
    """60k primitives on a 4K canvas (two-level binning, 470 row chunks): bins
    bit-exact against the oracle, then one fused step runs clean."""
    from paper_2602_22625_b200 import raster, synth
    from paper_2602_22625_b200.fit import LossSpec, StepEngine, effective_padding
    from paper_2602_22625_b200.scene import PrimitiveParams, Scene

    w = synth.make_workload("c1")
    rng = np.random.default_rng(5)
    W, H, n = 3840, 2160, 60000
    xs, ys = rng.uniform(-20, W + 20, n), rng.uniform(-20, H + 20, n)
    ss, rs = rng.uniform(2, 16, n), rng.uniform(-3, 3, n)
    prims = [PrimitiveParams(x=float(xs[i]), y=float(ys[i]), scale=float(ss[i]),
                             rotation=float(rs[i]), opacity_logit=0.5,
                             color_logits=(0.1, -0.2, 0.3), z=i) for i in range(n)]
    sc = Scene(prims, w.scene.templates, W, H)
    pad = effective_padding(w.cfg)
    pk = oracle.Packed(sc)
    off, idx = oracle.bin_tiles(pk, 16, pad)
    b = raster.bin_tiles(sc, 16, pad)
    np.testing.assert_array_equal(b.offsets, off)
    np.testing.assert_array_equal(b.indices, idx)
    target = np.full((H, W, 3), 0.5)
    eng = StepEngine(sc, w.cfg, LossSpec(kind="mse", target=target), 2, use_graph=False)
    eng.run(2)
    eng.check()
    h = eng.history()
    assert len(h) == 2 and all(np.isfinite(x.loss) for x in h)


@pytest.mark.parametrize("kind", ["noise_bg", "noise_bg_c2", "aspect_alpha_max"])
def test_fused_step_bg_and_aspect(torch_cuda, oracle, kind):
    """K34 with a per-pixel (noise) background (the BG kernel variant, staged
    background rows) and with preserve_aspect + alpha_max < 1 templates."""
    import dataclasses

    from conftest import load_case, scene_from
    from paper_2602_22625_b200 import synth
    from paper_2602_22625_b200.compositor import pixels4
    from paper_2602_22625_b200.fit import LossSpec, StepEngine, effective_padding

    torch = torch_cuda
    rng = np.random.default_rng(31)
    w = synth.make_workload("c2" if kind.endswith("c2") else "c1")  # c2: 64-entry stage
    if kind.startswith("noise_bg"):
        sc = dataclasses.replace(w.scene, background="noise")
        bg = rng.random((sc.canvas_h, sc.canvas_w, 3)).astype(np.float32).astype(np.float64)
        target = w.target
    else:
        sc = dataclasses.replace(scene_from(load_case("aspect_mu_s0")), mu_blend=0.0)
        bg = None
        target = rng.random((sc.canvas_h, sc.canvas_w, 3))
    eng = StepEngine(sc, w.cfg, LossSpec(kind="mse", target=target), 1, use_graph=False)
    assert eng.fused
    if bg is not None:
        eng.bg4.copy_(torch.from_numpy(pixels4(bg)))
    g, sums, color, alpha = _fused_grads(eng)
    pk = oracle.Packed(sc)
    off, idx = oracle.bin_tiles(pk, 32, effective_padding(w.cfg))
    img, a_ref, sv = oracle.render_forward(pk, off, idx, 32, oracle.background(sc, bg), True,
                                           w.cfg.eps_skip)
    ok, err = fwd_close(color, img)
    assert ok, f"{kind} colour rel err {err}"
    ok, err = fwd_close(alpha, a_ref)
    assert ok, f"{kind} alpha rel err {err}"
    diff = img - target
    np.testing.assert_allclose(sums[0], np.sum(diff**2), rtol=1e-5)
    g_ref = oracle.backward(pk, sv, 2.0 * diff / diff.size, None)  # (bg saved in sv)
    ok, err = grad_close(g, g_ref)
    assert ok, f"{kind} grad rel err {err}"


@pytest.mark.parametrize("world", [2, 4])
def test_row_band_gradients_sum_to_full_canvas(torch_cuda, world):
    """The multi-GPU decomposition on one GPU: the K34 gradients and loss sums of
    the row bands of an N-way split (each band binned and rendered alone, as a
    rank does) add up to the full-canvas step's (fp64 atomics: round-off only)."""
    from paper_2602_22625_b200 import synth
    from paper_2602_22625_b200.dist import row_bands
    from paper_2602_22625_b200.fit import StepEngine

    w = synth.make_workload("c3")
    full = StepEngine(w.scene, w.cfg, w.loss, 1, use_graph=False)
    g_full, s_full, _, _ = _fused_grads(full)
    nty = -(-w.scene.canvas_h // 16)
    g_sum, s_sum = np.zeros_like(g_full), np.zeros_like(s_full)
    for band in row_bands(nty, world):
        eng = StepEngine(w.scene, w.cfg, w.loss, 1, band=band, use_graph=False)
        g, s, _, _ = _fused_grads(eng)
        g_sum += g
        s_sum += s
    np.testing.assert_allclose(s_sum[:3], s_full[:3], rtol=1e-12)
    ok, err = grad_close(g_sum, g_full, rel=1e-9)
    assert ok, f"band-sum grad rel err {err}"


def test_adam_only_then_preprocess_equals_fused_records(torch_cuda):
    """pf_adam_preprocess with rec = NULL (Adam only) followed by pf_preprocess
    gives the same next step as the fused Adam + records launch."""
    torch = torch_cuda
    from paper_2602_22625_b200 import synth
    from paper_2602_22625_b200.fit import StepEngine

    w = synth.make_workload("c1")
    w.cfg.num_iterations = 6
    a = StepEngine(w.scene, w.cfg, w.loss, 6, use_graph=False)
    b = StepEngine(w.scene, w.cfg, w.loss, 6, use_graph=False)
    a.refresh()
    b.refresh()
    for _ in range(3):
        a.launch_step()
        a.done += 1
        b.launch_step(records=False)
        b.refresh()
        b.done += 1
    torch.cuda.synchronize()
    np.testing.assert_array_equal(a.params_host(), b.params_host())
    assert [h.loss for h in a.history()] == [h.loss for h in b.history()]


def test_long_run_c3(torch_cuda):
    """300 graph-replayed steps of the metric config through run_loop: finite
    history, the loss falls, no bin overflow, parameters finite."""
    from paper_2602_22625_b200 import synth
    from paper_2602_22625_b200.fit import run_loop

    w = synth.make_workload("c3")
    w.cfg.num_iterations = 300
    sc, hist, state = run_loop(w.scene, w.cfg, w.loss, np.random.default_rng(0))
    losses = np.array([h.loss for h in hist])
    assert len(losses) == 300 and np.isfinite(losses).all()
    assert losses[-1] < 0.5 * losses[0]
    assert np.all(np.diff(losses[:50]) < 0.05 * losses[0])  # no blow-up early on
    assert state.step == 300
    from paper_2602_22625_b200.scene import pack_params

    assert np.isfinite(pack_params(sc)[0]).all()


def test_host_io_noise_background_matches_step(torch_cuda):
    """Host-driven steps of a noise-background scene draw the background from the
    caller's rng every step, like step(): same parameters as the device engine."""
    import dataclasses

    torch = torch_cuda
    from paper_2602_22625_b200 import synth
    from paper_2602_22625_b200.fit import StepEngine

    w = synth.make_workload("c1")
    sc = dataclasses.replace(w.scene, background="noise")
    w.cfg.num_iterations = 7
    a = StepEngine(sc, w.cfg, w.loss, 7, use_graph=True)
    b = StepEngine(sc, w.cfg, w.loss, 7, use_graph=True, host_io=True)
    ra, rb = np.random.default_rng(9), np.random.default_rng(9)
    a.run(2, ra)
    b.run(2, rb)
    b.capture_host_io_step()
    for _ in range(4):
        a.step(ra)
        b.host_step(rb)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(a.params_host(), b.io.numpy()[: b.n * 8])
    with pytest.raises(ValueError, match="rng"):
        b.host_step()


@pytest.mark.parametrize("name,total,loss", [("c1", 8, "mse"), ("c1", 8, "combined"),
                                             ("c3", 5, "mse")])
def test_two_kernel_step_engine_matches_oracle_loop(torch_cuda, oracle, name, total, loss):
    """The two-kernel StepEngine path (mu_blend > 0: K3 forward with the loss fused
    and saved 16-byte entries, K4 backward, K5+K1) against the oracle's run_loop
    body over a graph-replayed rollout, for MSE and the combined loss on K3."""
    import dataclasses

    from paper_2602_22625_b200 import synth
    from paper_2602_22625_b200.fit import LossSpec, StepEngine, effective_padding

    w = synth.make_workload(name)
    sc = dataclasses.replace(w.scene, mu_blend=0.3)
    w.cfg.num_iterations = total
    spec = w.loss if loss == "mse" else LossSpec(kind="combined", target=w.target, mse_w=0.7,
                                                 gray_l1_w=0.4)
    eng = StepEngine(sc, w.cfg, spec, total)
    assert not eng.fused
    loop = oracle.Loop(sc, w.target, w.cfg, effective_padding(w.cfg), tile=32,
                       loss=None if loss == "mse" else ("combined", 0.7, 0.4))
    for it in range(total):
        eng.step()
        loop.step(it, total)
    eng.check()
    np.testing.assert_allclose([h.loss for h in eng.history()], [h[1] for h in loop.history],
                               rtol=1e-5)
    p_gpu = eng.params_host().reshape(-1, 8)
    p_ref = loop.vec.reshape(-1, 8)
    close = np.isclose(p_gpu, p_ref, rtol=1e-4, atol=1e-4)
    # (the combined loss's L1 term has a sign() subgradient: pixels with d ~ 0
    # flip with round-off, so a few more components carry Adam noise)
    assert close.mean() > (0.99 if loss == "mse" else 0.98), close.mean()
    gains = np.asarray([10, 10, 10, 1, 1.5, 1, 1, 1.0])
    assert np.all(np.abs(p_gpu - p_ref) <= 2 * w.cfg.learning_rate * gains[None, :] * total)


def test_autograd_step_graph_capture_matches_eager(torch_cuda):
    """A training step through the autograd Function (forward, torch MSE,
    backward, a device-side update) captured in one CUDA graph replays the
    eager step exactly (no host sync, no allocation inside the Function)."""
    torch = torch_cuda
    from paper_2602_22625_b200 import synth
    from paper_2602_22625_b200.autograd import Renderer
    from paper_2602_22625_b200.fit import effective_padding
    from paper_2602_22625_b200.scene import param_matrix, structure_arrays

    w = synth.make_workload("c1")
    sc = w.scene
    tid, z = structure_arrays(sc)

    def run(graphed: bool, steps: int = 4):
        r = Renderer(sc.templates, tid, z, sc.canvas_w, sc.canvas_h,
                     background=tuple(sc.background), alpha_max=sc.alpha_max,
                     padding=effective_padding(w.cfg), s_max=w.cfg.scale_max)
        params = torch.tensor(param_matrix(sc), device="cuda", requires_grad=True)
        target = torch.tensor(w.target, device="cuda", dtype=torch.float32)
        losses = []

        def step():
            img, _ = r(params)
            loss = ((img - target) ** 2).mean()
            loss.backward()
            with torch.no_grad():
                params.sub_(1e-3 * params.grad)
                params.grad.zero_()
            return loss.detach()

        if not graphed:
            for _ in range(steps + 2):
                losses.append(float(step()))
            return params.detach().cpu().numpy(), losses[2:]
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(2):
                step()
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            out = step()
        for _ in range(steps):
            g.replay()
            losses.append(float(out))
        r.check()
        return params.detach().cpu().numpy(), losses

    p_e, l_e = run(False)
    p_g, l_g = run(True)
    np.testing.assert_allclose(l_g, l_e, rtol=1e-6)
    np.testing.assert_allclose(p_g, p_e, rtol=1e-9, atol=1e-9)
