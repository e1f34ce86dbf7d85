"""CPU-side checks: the C-ABI library loads and exports every declared symbol,
host-side validation/packing mirrors the reference, capacity bounds hold,
and the synthetic workload generator reproduces the reference's init."""

from __future__ import annotations

import ctypes
import hashlib
import math
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN, RENDER_CASES, ROOT, load_case, scene_from


def _declared_symbols() -> list[str]:
    text = (ROOT / "include" / "primfit_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|long long)\s+(pf_\w+)\(", text, re.M)))


def test_header_declares_entry_points():
    syms = _declared_symbols()
    for s in ("pf_preprocess", "pf_bin", "pf_forward", "pf_backward", "pf_adam",
              "pf_bin_scratch_bytes", "pf_record_bytes", "pf_abi_version"):
        assert s in syms


def test_native_library_exports_every_declared_symbol():
    from paper_2602_22625_b200 import _native, build

    build.build()
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    for s in _declared_symbols():
        assert hasattr(lib, s), s
    assert set(_declared_symbols()) == set(_native.SIGNATURES)
    typed = _native.load()
    assert typed.pf_abi_version() == 8
    assert typed.pf_record_bytes() == 480
    assert typed.pf_render_tile() == 16
    assert typed.pf_saved_capacity(10) == 2560


def test_library_is_sm100a():
    import subprocess

    from paper_2602_22625_b200 import _native

    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_validate_scene_errors():
    from paper_2602_22625_b200.errors import (BadChannelRange, BadTemplateRef, InvalidScale,
                                              NonPermutationZ, ShapeMismatch)
    from paper_2602_22625_b200.scene import validate_scene

    base = scene_from(load_case("small_scene"))
    validate_scene(base)
    sc = scene_from(load_case("small_scene"))
    sc.primitives[1].scale = -1.0
    with pytest.raises(InvalidScale):
        validate_scene(sc)
    sc = scene_from(load_case("small_scene"))
    sc.primitives[1].template_id = 5
    with pytest.raises(BadTemplateRef):
        validate_scene(sc)
    sc = scene_from(load_case("small_scene"))
    sc.primitives[1].z = 0
    with pytest.raises(NonPermutationZ):
        validate_scene(sc)
    sc = scene_from(load_case("small_scene"))
    sc.templates[0].rgba[0, 0, 0] = 2.0
    with pytest.raises(BadChannelRange):
        validate_scene(sc)
    sc = scene_from(load_case("small_scene"))
    sc.canvas_w = 0
    with pytest.raises(ShapeMismatch):
        validate_scene(sc)


def test_pack_unpack_roundtrip_and_fingerprint():
    from paper_2602_22625_b200.scene import pack_params, scene_fingerprint, unpack_params

    sc = scene_from(load_case("random_s3"))
    vec, layout = pack_params(sc)
    sc2 = unpack_params(vec, layout, sc)
    assert scene_fingerprint(sc) == scene_fingerprint(sc2)
    np.testing.assert_array_equal(pack_params(sc2)[0], vec)
    v2 = vec.copy()
    v2[3] += 1e-9
    assert scene_fingerprint(unpack_params(v2, layout, sc)) != scene_fingerprint(sc)


@pytest.mark.parametrize("case", RENDER_CASES)
def test_capacity_bound_holds(oracle, case):
    from paper_2602_22625_b200.compositor import bin_capacity

    d = load_case(case)
    sc = scene_from(d)
    pk = oracle.Packed(sc)
    hyp_t = np.zeros(len(sc.templates))
    for i, t in enumerate(pk.tid):
        hyp_t[t] = pk.hyp[i]
    W, H = sc.canvas_w, sc.canvas_h
    for tile, pad in ((16, 2.0), (32, 2.0), (16, 5.0)):
        off, _ = oracle.bin_tiles(pk, tile, pad)
        cap = bin_capacity(pk.s, pk.tid, hyp_t, pad, tile, -(-W // tile), -(-H // tile))
        assert cap >= off[-1]


def test_lr_schedule_and_gains_match_reference_semantics():
    from paper_2602_22625_b200.fit import gains_vector, lr_schedule
    from paper_2602_22625_b200.scene import ParamLayout

    assert lr_schedule(0, 100, 0.02) == pytest.approx(0.02)
    assert lr_schedule(99, 100, 0.02) == pytest.approx(0.002)
    assert lr_schedule(50, 101, 0.02) == pytest.approx(0.02 * math.sqrt(0.1))
    assert lr_schedule(0, 1, 0.02) == 0.02
    with pytest.raises(ValueError):
        lr_schedule(100, 100, 0.02)
    g = gains_vector(ParamLayout(2), {"x": 2.0, "color": 3.0})
    np.testing.assert_array_equal(g[:8], [2, 1, 1, 1, 1, 3, 3, 3])
    d = load_case("run_loop_small")
    n = len(d["hist_lr"])
    np.testing.assert_array_equal([lr_schedule(i, n, 0.1) for i in range(n)], d["hist_lr"])


def test_host_losses_match_reference_formulas():
    from paper_2602_22625_b200.fit import LossSpec, loss_mse, loss_spatial, psnr

    rng = np.random.default_rng(0)
    I = rng.random((5, 6, 3))
    t = rng.random((5, 6, 3))
    v, g = loss_mse(I, t)
    assert v == pytest.approx(np.mean((I - t) ** 2))
    np.testing.assert_allclose(g, 2 * (I - t) / I.size)
    ta = (rng.random((5, 6)) > 0.5).astype(float)
    Ia = rng.random((5, 6))
    val, dI, dA = loss_spatial(I, Ia, LossSpec("spatial_constrained", t, ta, alpha_w=0.3))
    assert val == pytest.approx(np.sum(((I - t) * ta[..., None]) ** 2) / I.size
                                + 0.3 * np.mean((Ia - ta) ** 2))
    assert psnr(I, I) == math.inf


def test_synth_reproduces_reference_structure_aware_init():
    from paper_2602_22625_b200 import synth

    d = load_case("synth_c1_init")
    w = synth.make_workload("c1")
    assert hashlib.sha256(w.target.tobytes()).hexdigest() == str(d["target_sha"])
    np.testing.assert_array_equal(w.scene.templates[0].rgba, d["tpl0"])
    pm = np.asarray([[p.x, p.y, p.scale, p.rotation, p.opacity_logit, *p.color_logits]
                     for p in w.scene.primitives])
    np.testing.assert_array_equal(pm, d["params"])
    np.testing.assert_array_equal([p.template_id for p in w.scene.primitives], d["tid"])
    np.testing.assert_array_equal([p.z for p in w.scene.primitives], d["z"])


def test_golden_files_present():
    assert len(RENDER_CASES) >= 15
    assert (GOLDEN / "make_golden.py").exists()


def test_video_host_logic_matches_reference_semantics():
    """Host side of the f3 row (no GPU): StuckPolicy validation (dyn.py:44-72),
    policy_from_config over a config without video fields (reference defaults),
    and optimize_video's argument checks (dyn.py:190-199)."""
    import types

    from paper_2602_22625_b200 import video
    from paper_2602_22625_b200.errors import ShapeMismatch

    for bad in ({"grid": (0, 4)}, {"k": -1}, {"eta": 1.0}, {"zeta": 0.0}):
        with pytest.raises(ValueError):
            video.StuckPolicy(**bad)
    cfg = types.SimpleNamespace(loss="mse", seed=0)
    pol = video.policy_from_config(cfg)
    assert (pol.grid, pol.k, pol.triggers) == ((4, 4), 4, (20, 45, 70))
    cfg2 = types.SimpleNamespace(stuck_grid_x=3, stuck_grid_y=2, stuck_top_k=1,
                                 stuck_triggers=(5,))
    pol2 = video.policy_from_config(cfg2)
    assert (pol2.grid, pol2.k, pol2.triggers) == ((2, 3), 1, (5,))
    with pytest.raises(ValueError):
        video.optimize_video([], None, cfg)
    with pytest.raises(ShapeMismatch):
        video.optimize_video([np.zeros((4, 4, 3)), np.zeros((5, 4, 3))], None, cfg)
    with pytest.raises(ValueError):
        video.optimize_video([np.zeros((4, 4, 3))], None,
                             types.SimpleNamespace(loss="spatial", seed=0))


def test_synth_template_preparation_matches_reference():
    """Non-circular check of the bench inputs' template pipeline: synth.prepare
    (blur) and synth.radial_falloff against the reference's own
    prepare_templates / radial_falloff (prep.py:76-89, 260-275), imported from
    /root/reference when it is present (the GPU box does not have it)."""
    import sys
    from pathlib import Path

    ref_src = Path("/root/reference/pkg/src")
    if not (ref_src / "primfit").is_dir():
        pytest.skip("reference package not present")
    sys.path.insert(0, str(ref_src))
    try:
        from primfit import prep as rprep
        from primfit.scene import PrimitiveTemplate as RT
    finally:
        sys.path.remove(str(ref_src))
    from paper_2602_22625_b200 import synth

    for raw in (synth.disc(32), synth.logo(48), synth.fingerprint(40), synth.autograph(24, 48),
                synth.flower(32)):
        ours = synth.prepare([raw])[0].rgba
        ref = rprep.prepare_templates([RT(raw.copy())], blur_sigma=1.0, do_blur=True)[0].rgba
        np.testing.assert_allclose(ours, ref, rtol=0, atol=1e-15)
        np.testing.assert_allclose(synth.radial_falloff(raw), rprep.radial_falloff(RT(raw.copy())).rgba,
                                   rtol=0, atol=1e-15)
