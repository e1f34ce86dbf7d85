"""Pin the CPU oracle against golden vectors produced by the reference itself.

The oracle (oracle/primfit_oracle.c) is the checker for every GPU parity
test, so it is pinned first: binning bit-exact, forward / backward / Adam to
float64 rounding, run_loop rollout to 1e-12.  CPU only.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import RENDER_CASES, load_case, scene_from


@pytest.mark.parametrize("case", RENDER_CASES)
def test_oracle_bins_bit_exact(oracle, case):
    d = load_case(case)
    pk = oracle.Packed(scene_from(d))
    for tile, pad in ((16, 2), (32, 2), (16, 5)):
        off, idx = oracle.bin_tiles(pk, tile, float(pad))
        np.testing.assert_array_equal(off, d[f"bin{tile}_p{pad}_off"])
        np.testing.assert_array_equal(idx, d[f"bin{tile}_p{pad}_idx"])


@pytest.mark.parametrize("case", RENDER_CASES)
def test_oracle_forward_backward_match_reference(oracle, case):
    d = load_case(case)
    sc = scene_from(d)
    pk = oracle.Packed(sc)
    bg = d["bg_image"] if "bg_image" in d else oracle.background(sc)
    off, idx = oracle.bin_tiles(pk, 32, 2.0)
    img0, a0, _ = oracle.render_forward(pk, off, idx, 32, bg, False, 0.0)
    np.testing.assert_allclose(img0, d["img_eps0"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(a0, d["alpha_eps0"], rtol=0, atol=1e-13)
    img, a, sv = oracle.render_forward(pk, off, idx, 32, bg, True, 1.0 / 1024.0)
    np.testing.assert_allclose(img, d["img"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(a, d["alpha"], rtol=0, atol=1e-13)
    assert sv["n_entries"] == int(d["n_entries"])
    g = oracle.backward(pk, sv, d["dI"], None)
    np.testing.assert_allclose(g, d["grads"], rtol=1e-11, atol=1e-15)
    if "grads_alpha_obj" in d:
        g2 = oracle.backward(pk, sv, np.zeros_like(d["dI"]), d["dA"])
        np.testing.assert_allclose(g2, d["grads_alpha_obj"], rtol=1e-11, atol=1e-15)


def test_oracle_tile_size_independent(oracle):
    # reference SPEC.md:192 -- conservative bins make the image tile-size independent
    d = load_case("medium_n300")
    sc = scene_from(d)
    pk = oracle.Packed(sc)
    bg = oracle.background(sc)
    o16, i16 = oracle.bin_tiles(pk, 16, 5.0)
    o32, i32 = oracle.bin_tiles(pk, 32, 2.0)
    a, _, _ = oracle.render_forward(pk, o16, i16, 16, bg, False, 1 / 1024)
    b, _, _ = oracle.render_forward(pk, o32, i32, 32, bg, False, 1 / 1024)
    np.testing.assert_array_equal(a, b)


def test_oracle_thread_count_determinism(oracle):
    # reference acceptance criterion 03: bytewise identical across thread counts
    d = load_case("medium_n300")
    pk = oracle.Packed(scene_from(d))
    bg = oracle.background(scene_from(d))
    off, idx = oracle.bin_tiles(pk, 32, 2.0)
    outs = []
    n0 = oracle.threads()
    for t in (1, 2, 4):
        oracle.set_threads(t)
        img, _, sv = oracle.render_forward(pk, off, idx, 32, bg, True, 1 / 1024)
        outs.append((img, oracle.backward(pk, sv, d["dI"], None)))
    oracle.set_threads(n0)
    for img, g in outs[1:]:
        assert img.tobytes() == outs[0][0].tobytes()
        assert g.tobytes() == outs[0][1].tobytes()


def test_oracle_adam_rollout(oracle):
    d = load_case("adam_rollout")
    p = d["p0"].copy()
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    frozen = d["frozen"].astype(np.uint8)
    gains8 = d["gains"][:8]
    for t in range(4):
        oracle.adam(p, d["grads"][t].copy(), m, v, t + 1, float(d["lrs"][t]), frozen=frozen,
                    gains8=gains8, s_min=4.0, s_max=6.0)
        np.testing.assert_allclose(p, d["outs"][t], rtol=0, atol=1e-14)
    np.testing.assert_allclose(m, d["m"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(v, d["v"], rtol=0, atol=1e-15)


def test_oracle_run_loop_rollout(oracle):
    from paper_2602_22625_b200.fit import FitConfig

    d = load_case("run_loop_small")
    sc = scene_from(d)
    cfg = FitConfig(num_iterations=int(d["iters"]), scale_min=float(d["scale_min"]),
                    scale_max=float(d["scale_max"]))
    loop = oracle.Loop(sc, d["target"], cfg, float(d["padding"]), tile=32)
    total = int(d["iters"])
    for it in range(total):
        loop.step(it, total)
    hl = np.asarray([h[1] for h in loop.history])
    hp = np.asarray([h[2] for h in loop.history])
    np.testing.assert_allclose(hl, d["hist_loss"], rtol=1e-12)
    np.testing.assert_allclose(hp, d["hist_psnr"], rtol=1e-12)
    np.testing.assert_allclose(loop.vec.reshape(-1, 8), d["final_params"], rtol=1e-11, atol=1e-12)


@pytest.mark.parametrize("case", ["export_aspect_mu", "export_random"])
def test_oracle_export_layers_match_reference(oracle, case):
    """f4: scale_scene + layer_bbox + render_layer (exportio.py:272-346) at rho 1, 2, 4."""
    d = load_case(case)
    pk = oracle.Packed(scene_from(d))
    for rho in (1, 2, 4):
        box, off, rgba = oracle.export_layers_arrays(pk, rho)
        np.testing.assert_array_equal(box, d[f"rho{rho}_bbox"])
        np.testing.assert_array_equal(off, d[f"rho{rho}_off"])
        np.testing.assert_allclose(rgba, d[f"rho{rho}_rgba"], rtol=0, atol=1e-14)


def test_oracle_video_heuristics_match_reference(oracle):
    """f3: diff_mask, freeze_flags, remove_stuck (dyn.py:86-177)."""
    d = load_case("video_heuristics")
    pk = oracle.Packed(scene_from(d))
    for tau in (0.0, 2.0 / 255.0, 0.02):
        np.testing.assert_array_equal(oracle.diff_mask(d["prev"], d["cur"], tau),
                                      d[f"mask_{tau!r}"])
    m = d["mask_" + repr(2.0 / 255.0)]
    for pad in (2.0, 5.0):
        np.testing.assert_array_equal(oracle.freeze_flags(pk, m, pad), d[f"frozen_p{int(pad)}"])
    nu, dec = oracle.remove_stuck(pk, d["z"], d["frozen_p2"], (3, 4), 2, 0.02, 0.3, 0.3, 0.5)
    assert dec == list(d["stuck_decayed"])
    np.testing.assert_allclose(nu, d["stuck_params"][:, 4], rtol=0, atol=1e-15)
    _, dec0 = oracle.remove_stuck(pk, d["z"], None, (3, 4), 2, 0.02, 0.3, 0.3, 0.5)
    assert dec0 == list(d["stuck_decayed_nofrozen"])


def test_oracle_gradcheck_criterion_01(oracle):
    """Acceptance criterion 01 (test_acceptance.py:63-72, grad.py:378-420) for the
    checker itself: the oracle's backward against the reference's own central
    finite differences on the 20 gradcheck scenes, its gate (rel 1e-2 or abs 1e-5)."""
    acc = load_case("acceptance")
    fails = checked = 0
    for seed in range(20):
        d = {k[len(f"g{seed}_"):]: acc[k] for k in acc if k.startswith(f"g{seed}_")}
        sc = scene_from(d)
        pk = oracle.Packed(sc)
        off, idx = oracle.bin_tiles(pk, 32, 2.0)
        img, _, sv = oracle.render_forward(pk, off, idx, 32, oracle.background(sc), True, 0.0)
        g = oracle.backward(pk, sv, 2.0 * (img - d["target"]) / d["target"].size, None)
        adiff = np.abs(g - d["fd"])
        ok = (adiff / np.maximum(np.abs(d["fd"]), 1e-300) <= 1e-2) | (adiff <= 1e-5)
        checked += ok.size
        fails += int((~ok).sum())
    assert checked > 0 and fails == 0, f"{fails}/{checked}"
