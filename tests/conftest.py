"""Shared fixtures: golden-vector loaders and the oracle import path.

Golden vectors (tests/golden/*.npz) were produced by the reference package
itself (tests/golden/make_golden.py); the GPU box never reads /root/reference.
"""

from __future__ import annotations

import glob
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
GOLDEN = Path(__file__).resolve().parent / "golden"

from paper_2602_22625_b200.scene import PrimitiveParams, PrimitiveTemplate, Scene  # noqa: E402

RENDER_CASES = sorted(
    Path(p).stem for p in glob.glob(str(GOLDEN / "*.npz"))
    if Path(p).stem not in ("adam_rollout", "run_loop_small", "synth_c1_init", "video_heuristics",
                            "reinit_unit", "run_loop_reinit", "run_loop_reinit_noise",
                            "video_dropin", "run_loop_hook_resume", "acceptance", "optimize_small", "export_tests")
    and not Path(p).stem.startswith("export_")
)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running")


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def load_case(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def scene_from(d: dict) -> Scene:
    pm = d["params"]
    prims = [
        PrimitiveParams(x=float(r[0]), y=float(r[1]), scale=float(r[2]), rotation=float(r[3]),
                        opacity_logit=float(r[4]),
                        color_logits=(float(r[5]), float(r[6]), float(r[7])),
                        template_id=int(t), z=int(z))
        for r, t, z in zip(pm, d["tid"], d["z"])
    ]
    tpls = [PrimitiveTemplate(d[f"tpl{k}"]) for k in range(int(d["n_templates"]))]
    bg = "noise" if "background_noise" in d else tuple(float(v) for v in d["background"])
    W, H = (int(v) for v in d["canvas"])
    return Scene(prims, tpls, W, H, background=bg, alpha_max=float(d["alpha_max"]),
                 mu_blend=float(d["mu_blend"]), preserve_aspect=bool(d["preserve_aspect"]))


def fwd_close(got, ref, rel=1e-5):
    """north_star forward tolerance: |d| <= rel * max(|ref|, 1e-3), elementwise."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    bound = rel * np.maximum(np.abs(ref), 1e-3)
    bad = np.abs(got - ref) > bound
    return (not bad.any()), float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-3)))


def grad_close(got, ref, rel=1e-3):
    """north_star gradient tolerance: |d| <= rel * max(|ref|, 1e-2 * max_col|ref|, 1e-4 * max|ref|)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    colmax = np.abs(ref).max(axis=0, keepdims=True)
    # columns that vanish by symmetry hold pure round-off (~1e-19 next to 1e-3
    # entries); any summation order leaves eps * sum|terms| there (~1e-8 of the
    # largest gradient with fp32 per-pixel math), so components are floored at
    # 1e-4 of the scene's largest gradient: |d| <= 1e-7 * max|ref| for them
    floor = np.maximum(np.maximum(1e-2 * colmax, 1e-4 * np.abs(ref).max()), 1e-300)
    scale = np.maximum(np.abs(ref), floor)
    err = np.abs(got - ref) / scale
    return bool((err <= rel).all()), float(err.max()) if err.size else 0.0


@pytest.fixture(scope="session")
def oracle():
    import cpu_oracle as orc

    orc.build()
    return orc
