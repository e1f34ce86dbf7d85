"""Synthetic workloads c1..c5 (BASELINE.json configs).

Procedural templates, smooth random targets and the structure-aware
initialiser, restated so that the bench can build its inputs on a box where
the reference package is absent.  The initialiser consumes the numpy PCG64
stream in the reference's documented order (prep.py:10-14: positions, then
rotations, then colour noise, then template choices) so a given seed yields
the reference's own initial scene (checked in tests/test_abi_host.py::test_synth_reproduces_reference_structure_aware_init against a
golden fingerprint made with the reference).

Sources restated: gaussian_blur_template (prep.py:51-73), radial_falloff
(prep.py:76-89), local_variance_map (prep.py:92-132), structure_aware_init
(prep.py:147-219), init_scene (fit.py:358-400), effective_padding
(fit.py:338-341).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
from scipy.ndimage import correlate1d, gaussian_filter

from .fit import FitConfig, LossSpec
from .scene import PrimitiveParams, PrimitiveTemplate, Scene


# -- template preparation ----------------------------------------------------

def _gauss_taps(sigma: float) -> np.ndarray:
    rad = int(math.ceil(3.0 * sigma))
    x = np.arange(-rad, rad + 1, dtype=np.float64)
    k = np.exp(-(x * x) / (2.0 * sigma * sigma))
    return k / k.sum()


def blur_rgba(rgba: np.ndarray, sigma: float) -> np.ndarray:
    """Separable truncated Gaussian, renormalised over the clipped window, clipped to [0,1]."""
    if sigma == 0:
        return rgba.copy()
    k = _gauss_taps(sigma)

    def sep(a):
        return correlate1d(correlate1d(a, k, axis=0, mode="constant", cval=0.0), k, axis=1,
                           mode="constant", cval=0.0)

    norm = sep(np.ones(rgba.shape[:2]))
    out = np.stack([sep(rgba[:, :, c]) / norm for c in range(4)], axis=-1)
    return np.clip(out, 0.0, 1.0)


def radial_falloff(rgba: np.ndarray) -> np.ndarray:
    """Cosine alpha falloff from the centre, zero past the smaller half extent."""
    h, w = rgba.shape[:2]
    cy, cx = (h - 1) / 2.0, (w - 1) / 2.0
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    r = np.minimum(np.hypot(yy - cy, xx - cx) / min(cy, cx), 1.0)
    out = rgba.copy()
    out[:, :, 3] *= 0.5 * (1.0 + np.cos(np.pi * r))
    return out


# -- procedural bitmaps ------------------------------------

def disc(size: int = 64) -> np.ndarray:
    c = (size - 1) / 2.0
    yy, xx = np.mgrid[0:size, 0:size].astype(np.float64)
    out = np.ones((size, size, 4))
    out[:, :, 3] = (np.hypot(yy - c, xx - c) <= c - 1).astype(np.float64)
    return out


def logo(size: int = 128) -> np.ndarray:
    yy, xx = np.mgrid[0:size, 0:size]
    inner = (yy >= size // 8) & (yy < size - size // 8) & (xx >= size // 8) & (xx < size - size // 8)
    checker = ((yy // 16 + xx // 16) % 2).astype(np.float64)
    out = np.zeros((size, size, 4))
    out[:, :, :3] = np.random.default_rng(0).random(3)
    out[:, :, 3] = inner * (0.6 + 0.4 * checker)
    return out


def fingerprint(size: int = 64) -> np.ndarray:
    c = (size - 1) / 2.0
    yy, xx = np.mgrid[0:size, 0:size].astype(np.float64)
    r = np.hypot(yy - c, xx - c)
    out = np.ones((size, size, 4))
    ridge = 0.5 + 0.5 * np.cos(0.9 * r + 0.15 * xx)
    out[:, :, 0] = out[:, :, 1] = out[:, :, 2] = ridge
    return radial_falloff(out)


def autograph(h: int = 48, w: int = 96) -> np.ndarray:
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    curve = h / 2.0 + 0.3 * h * np.sin(4.0 * np.pi * xx / w)
    out = np.zeros((h, w, 4))
    out[:, :, :3] = 0.1
    out[:, :, 3] = np.clip(1.0 - np.abs(yy - curve) / 3.0, 0.0, 1.0)
    out[0, :, 3] = out[-1, :, 3] = out[:, 0, 3] = out[:, -1, 3] = 0.0
    return out


def flower(size: int = 32, petals: int = 5) -> np.ndarray:
    c = (size - 1) / 2.0
    yy, xx = np.mgrid[0:size, 0:size].astype(np.float64)
    r = np.hypot(yy - c, xx - c) / c
    th = np.arctan2(yy - c, xx - c)
    out = np.zeros((size, size, 4))
    out[:, :, 0], out[:, :, 1], out[:, :, 2] = 0.9, 0.4, 0.6
    out[:, :, 3] = (r <= 0.55 + 0.4 * np.cos(petals * th)).astype(np.float64)
    out[0, :, 3] = out[-1, :, 3] = out[:, 0, 3] = out[:, -1, 3] = 0.0
    return out


def prepare(rgbas, blur_sigma: float = 1.0) -> list[PrimitiveTemplate]:
    return [PrimitiveTemplate(blur_rgba(a, blur_sigma)) for a in rgbas]


def smooth_target(w: int, h: int, seed: int = 0) -> np.ndarray:
    t = gaussian_filter(np.random.default_rng(seed).random((h, w, 3)), (4, 4, 0))
    return (t - t.min()) / (t.max() - t.min())


# -- structure-aware initialisation -------------------------------------------

def _window_mean(a: np.ndarray, window: int) -> np.ndarray:
    h, w = a.shape
    r = window // 2
    ii = np.zeros((h + 1, w + 1))
    ii[1:, 1:] = a.cumsum(0).cumsum(1)
    ys = np.arange(h)
    xs = np.arange(w)
    y0, y1 = np.maximum(ys - r, 0), np.minimum(ys + r + 1, h)
    x0, x1 = np.maximum(xs - r, 0), np.minimum(xs + r + 1, w)
    s = ii[y1][:, x1] - ii[y0][:, x1] - ii[y1][:, x0] + ii[y0][:, x0]
    return s / ((y1 - y0)[:, None] * (x1 - x0)[None, :])


def variance_map(target: np.ndarray, window: int = 7) -> np.ndarray:
    var = np.zeros(target.shape[:2])
    for c in range(3):
        m = _window_mean(target[:, :, c], window)
        var += np.maximum(_window_mean(target[:, :, c] ** 2, window) - m * m, 0.0)
    var /= 3.0
    lo, hi = float(var.min()), float(var.max())
    return np.zeros_like(var) if hi - lo <= 0.0 else (var - lo) / (hi - lo)


def structure_aware_scene(target: np.ndarray, templates, n: int, s_min: float, s_max: float,
                          rng: np.random.Generator, *, v_init: float = -4.0,
                          sigma_c: float = 0.02, density_cap: int = 100,
                          base_prob: float = 0.1, window: int = 7,
                          background=(1.0, 1.0, 1.0)) -> Scene:
    h, w = target.shape[:2]
    nlv = variance_map(target, window)
    wgt = base_prob + (1.0 - base_prob) * nlv
    prob = (wgt / wgt.sum()).reshape(-1)
    picked: list[int] = []
    used = np.zeros(h * w, dtype=np.int64)
    while len(picked) < n:
        for cell in rng.choice(h * w, size=n - len(picked), p=prob):
            if used[cell] < density_cap:
                used[cell] += 1
                picked.append(int(cell))
    cells = np.asarray(picked, dtype=np.int64)
    scales = s_max - (s_max - s_min) * nlv.reshape(-1)[cells]
    thetas = rng.uniform(0.0, 2.0 * np.pi, n)
    cols = target[cells // w, cells % w, :] + rng.normal(0.0, sigma_c, (n, 3))
    cols = np.clip(cols, 1e-4, 1.0 - 1e-4)
    logits = np.log(cols) - np.log1p(-cols)
    tids = rng.integers(0, len(templates), n)
    prims = [
        PrimitiveParams(x=float(cells[i] % w), y=float(cells[i] // w), scale=float(scales[i]),
                        rotation=float(thetas[i]), opacity_logit=v_init,
                        color_logits=(float(logits[i, 0]), float(logits[i, 1]), float(logits[i, 2])),
                        template_id=int(tids[i]), z=i)
        for i in range(n)
    ]
    return Scene(prims, list(templates), canvas_w=w, canvas_h=h, background=background)


# -- BASELINE.json configurations ---------------------------------------------

@dataclass
class Workload:
    name: str
    scene: Scene
    target: np.ndarray
    cfg: FitConfig
    loss: LossSpec
    steps: int


def make_workload(name: str, seed: int = 0) -> Workload:
    """c1..c5 of BASELINE.json (c4 = one 512x512 frame of the video config)."""
    if name == "c1":
        W = H = 256
        tpls, n, smin, smax, steps = prepare([disc(64)]), 200, 2.0, 16.0, 100
    elif name == "c2":
        W = H = 512
        tpls, n, smin, smax, steps = prepare([logo(128)]), 2000, 4.0, 20.0, 500
    elif name == "c3":
        W, H = 1024, 809
        tpls, n, smin, smax, steps = prepare([fingerprint(64), autograph()]), 5000, 2.0, 10.0, 1000
    elif name == "c4":
        W = H = 512
        tpls = prepare([flower(32, 5), flower(32, 6)])
        n, smin, smax, steps = 2000, 2.0, 20.0, 100
    elif name == "c5":
        W, H = 3840, 2160
        tpls = prepare([disc(64), logo(128), fingerprint(64), autograph()])
        n, smin, smax, steps = 20000, 2.0, 16.0, 100
    else:
        raise ValueError(f"unknown workload {name!r}")
    target = smooth_target(W, H, seed)
    cfg = FitConfig(num_iterations=steps, num_primitives=n, seed=seed, scale_min=smin,
                    scale_max=smax)
    scene = structure_aware_scene(target, tpls, n, smin, smax, np.random.default_rng(seed))
    if name == "c3":
        for i, p in enumerate(scene.primitives):
            p.template_id = 0 if i < 3000 else 1
    loss = LossSpec(kind="mse", target=target)
    if name == "c4":
        yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)
        ta = (np.hypot(yy - (H - 1) / 2.0, xx - (W - 1) / 2.0) <= 200.0).astype(np.float64)
        cfg.loss = "spatial"
        loss = LossSpec(kind="spatial_constrained", target=target, target_alpha=ta, alpha_w=0.3)
    return Workload(name, scene, target, cfg, loss, steps)
