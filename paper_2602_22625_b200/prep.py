"""One-time host setup around the fit loop: template preparation and scene init.

Not on the per-step hot path (SURVEY §2 marks prep / init out of scope); it is
restated here because two callers of the GPU fit loop need it with the
reference's exact random-stream semantics:
  * ``video.optimize_video`` (dyn.py:180-238) builds frame 0's scene with
    prepare_templates -> init_scene from the caller's config and rng;
  * ``fit.run_loop`` with ``do_reinit`` re-seeds low-opacity primitives with the
    structure-aware law (fit.py:261-335), drawing from the caller's rng.
All randomness flows through the caller's numpy Generator in the reference's
documented order (prep.py:10-14): positions, then rotations, then colour
noise, then template choices.

Sources restated (pkg/src/primfit): gaussian_blur_template (prep.py:51-73),
radial_falloff (76-89), _clipped_window_mean / local_variance_map (92-132),
_color_logits_near (139-144), structure_aware_init (147-219), random_init
(222-257), prepare_templates (260-274), default_templates (277-292),
init_scene (fit.py:358-400), background_from_config (config.py:197-212).
"""

from __future__ import annotations

import dataclasses
import math
from dataclasses import dataclass

import numpy as np
from scipy.ndimage import correlate1d

from .errors import PrimfitError, ShapeMismatch
from .scene import NOISE_BACKGROUND, PrimitiveParams, PrimitiveTemplate, Scene

COLOR_CLAMP_EPS = 1e-4        # prep.py:34
DEFAULT_OPACITY_LOGIT = -4.0  # scene.py:42


class InfeasibleDensity(PrimfitError):
    """The density cap cannot hold the requested primitive count."""


@dataclass(eq=False)
class VarianceMap:
    """Normalised local variance of a target image, in [0, 1] (prep.py:38-41)."""

    nlv: np.ndarray


def _gauss_taps(sigma: float) -> np.ndarray:
    rad = math.ceil(3.0 * sigma)
    xs = np.arange(-rad, rad + 1, dtype=np.float64)
    k = np.exp(-(xs**2) / (2.0 * sigma * sigma))
    return k / k.sum()


def gaussian_blur_template(t: PrimitiveTemplate, sigma: float) -> PrimitiveTemplate:
    """Separable truncated Gaussian on all four channels, renormalised over the
    clipped window, clipped to [0, 1]."""
    if sigma < 0:
        raise ValueError(f"sigma {sigma} must be nonnegative")
    rgba = np.asarray(t.rgba, dtype=np.float64)
    if sigma == 0:
        return PrimitiveTemplate(rgba.copy())
    k = _gauss_taps(sigma)

    def sep(plane):
        return correlate1d(correlate1d(plane, k, axis=0, mode="constant", cval=0.0), k, axis=1,
                           mode="constant", cval=0.0)

    norm = sep(np.ones(rgba.shape[:2]))
    out = np.empty_like(rgba)
    for ch in range(4):
        out[:, :, ch] = sep(rgba[:, :, ch]) / norm
    return PrimitiveTemplate(np.clip(out, 0.0, 1.0))


def radial_falloff(t: PrimitiveTemplate) -> PrimitiveTemplate:
    """Cosine alpha falloff from the centre, 0 past the smaller half extent."""
    rgba = np.asarray(t.rgba, dtype=np.float64)
    h, w = rgba.shape[:2]
    cy, cx = (h - 1) / 2.0, (w - 1) / 2.0
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    r = np.hypot(yy - cy, xx - cx) / min(cy, cx)
    out = rgba.copy()
    out[:, :, 3] *= 0.5 * (1.0 + np.cos(np.pi * np.minimum(r, 1.0)))
    return PrimitiveTemplate(out)


def prepare_templates(templates, blur_sigma: float = 1.0, do_blur: bool = True,
                      falloff: bool = False) -> list[PrimitiveTemplate]:
    """Optional falloff, then optional blur, per template."""
    out = []
    for t in templates:
        if falloff:
            t = radial_falloff(t)
        if do_blur and blur_sigma > 0:
            t = gaussian_blur_template(t, blur_sigma)
        out.append(t)
    return out


def default_templates(size: int = 31) -> list[PrimitiveTemplate]:
    """The built-in soft brush blob: white, alpha (1 - r^2)^2, zero border."""
    yy, xx = np.mgrid[0:size, 0:size].astype(np.float64)
    c = (size - 1) / 2.0
    r = np.hypot(yy - c, xx - c) / (c - 1.0)
    rgba = np.empty((size, size, 4))
    rgba[:, :, :3] = 1.0
    rgba[:, :, 3] = np.clip(1.0 - r * r, 0.0, 1.0) ** 2
    rgba[0, :, 3] = rgba[-1, :, 3] = rgba[:, 0, 3] = rgba[:, -1, 3] = 0.0
    return [PrimitiveTemplate(rgba)]


def _window_mean(a: np.ndarray, window: int) -> np.ndarray:
    h, w = a.shape
    r = window // 2
    ii = np.zeros((h + 1, w + 1))
    ii[1:, 1:] = np.cumsum(np.cumsum(a, axis=0), axis=1)
    y0, y1 = np.clip(np.arange(h) - r, 0, None), np.clip(np.arange(h) + r + 1, None, h)
    x0, x1 = np.clip(np.arange(w) - r, 0, None), np.clip(np.arange(w) + r + 1, None, w)
    s = ii[np.ix_(y1, x1)] - ii[np.ix_(y0, x1)] - ii[np.ix_(y1, x0)] + ii[np.ix_(y0, x0)]
    return s / ((y1 - y0)[:, None] * (x1 - x0)[None, :])


def local_variance_map(target: np.ndarray, window: int = 7) -> VarianceMap:
    """Min-max normalised local variance averaged over RGB (clipped windows)."""
    if window < 3 or window % 2 == 0:
        raise ValueError(f"window {window} must be odd and >= 3")
    target = np.asarray(target, dtype=np.float64)
    if target.ndim != 3 or target.shape[2] != 3:
        raise ShapeMismatch(f"target shape {target.shape} is not (H, W, 3)")
    var = np.zeros(target.shape[:2])
    for ch in range(3):
        m = _window_mean(target[:, :, ch], window)
        var += np.maximum(_window_mean(target[:, :, ch] ** 2, window) - m * m, 0.0)
    var /= 3.0
    lo, hi = float(var.min()), float(var.max())
    if hi - lo <= 0.0:
        return VarianceMap(np.zeros_like(var))
    return VarianceMap((var - lo) / (hi - lo))


def color_logits_near(colors: np.ndarray, sigma_c: float, rng: np.random.Generator) -> np.ndarray:
    """Logits whose sigmoid scatters normally around ``colors``."""
    noisy = np.clip(colors + rng.normal(0.0, sigma_c, colors.shape), COLOR_CLAMP_EPS,
                    1.0 - COLOR_CLAMP_EPS)
    return np.log(noisy) - np.log1p(-noisy)


def sample_cells(nlv: np.ndarray, k: int, base_prob: float, density_cap: int,
                 rng: np.random.Generator, stall_limit: int | None = None) -> np.ndarray:
    """k pixel cells drawn with probability ~ base + (1 - base) * nlv, rejecting
    draws past ``density_cap`` per cell (batches of the missing count)."""
    h, w = nlv.shape
    weights = base_prob + (1.0 - base_prob) * nlv
    p = (weights / weights.sum()).reshape(-1)
    chosen = np.empty(k, dtype=np.int64)
    counts = np.zeros(h * w, dtype=np.int64)
    got = attempts = 0
    while got < k:
        attempts += 1
        if stall_limit is not None and attempts > stall_limit:
            raise InfeasibleDensity("rejection sampling stalled against the density cap")
        for cell in rng.choice(h * w, size=k - got, p=p):
            if counts[cell] < density_cap:
                counts[cell] += 1
                chosen[got] = cell
                got += 1
    return chosen


def structure_aware_init(target, n: int, s_min: float, s_max: float,
                         v_init_bias: float = DEFAULT_OPACITY_LOGIT, sigma_c: float = 0.02,
                         rng: np.random.Generator | None = None, density_cap: int = 100,
                         templates=None, base_prob: float = 0.1, window: int = 7) -> Scene:
    """Primitives where the target has detail; depth = draw order (0 in front)."""
    if n < 1:
        raise ValueError("need at least one primitive")
    target = np.asarray(target, dtype=np.float64)
    h, w = target.shape[:2]
    if n > density_cap * h * w:
        raise InfeasibleDensity(f"{n} primitives cannot fit {density_cap} per pixel on {w}x{h}")
    rng = rng or np.random.default_rng()
    templates = templates or default_templates()
    nlv = local_variance_map(target, window).nlv
    chosen = sample_cells(nlv, n, base_prob, density_cap, rng, stall_limit=100 + 20 * n)
    scales = s_max - (s_max - s_min) * nlv.reshape(-1)[chosen]
    thetas = rng.uniform(0.0, 2.0 * np.pi, n)
    cl = color_logits_near(target[chosen // w, chosen % w, :], sigma_c, rng)
    tids = rng.integers(0, len(templates), n)
    prims = [PrimitiveParams(x=float(chosen[i] % w), y=float(chosen[i] // w),
                             scale=float(scales[i]), rotation=float(thetas[i]),
                             opacity_logit=v_init_bias,
                             color_logits=(float(cl[i, 0]), float(cl[i, 1]), float(cl[i, 2])),
                             template_id=int(tids[i]), z=i) for i in range(n)]
    return Scene(prims, list(templates), canvas_w=w, canvas_h=h)


def random_init(canvas_w: int, canvas_h: int, n: int, s_min: float, s_max: float,
                v_init_bias: float = DEFAULT_OPACITY_LOGIT, sigma_c: float = 0.02,
                rng: np.random.Generator | None = None, templates=None) -> Scene:
    """Everything uniform, blind to the target."""
    if n < 1:
        raise ValueError("need at least one primitive")
    rng = rng or np.random.default_rng()
    templates = templates or default_templates()
    xs = rng.uniform(0.0, canvas_w - 1.0, n)
    ys = rng.uniform(0.0, canvas_h - 1.0, n)
    scales = rng.uniform(s_min, s_max, n)
    thetas = rng.uniform(0.0, 2.0 * np.pi, n)
    cl = rng.normal(0.0, 1.0, (n, 3)) * sigma_c
    tids = rng.integers(0, len(templates), n)
    prims = [PrimitiveParams(x=float(xs[i]), y=float(ys[i]), scale=float(scales[i]),
                             rotation=float(thetas[i]), opacity_logit=v_init_bias,
                             color_logits=(float(cl[i, 0]), float(cl[i, 1]), float(cl[i, 2])),
                             template_id=int(tids[i]), z=i) for i in range(n)]
    return Scene(prims, list(templates), canvas_w=canvas_w, canvas_h=canvas_h)


def background_from_config(cfg):
    """bg_color -> a scene background (white | black | noise | r,g,b)."""
    name = str(getattr(cfg, "bg_color", "white")).strip().lower()
    if name == "white":
        return (1.0, 1.0, 1.0)
    if name == "black":
        return (0.0, 0.0, 0.0)
    if name in ("noise", "random"):
        return NOISE_BACKGROUND
    parts = [p for p in name.replace(",", " ").split() if p]
    if len(parts) != 3:
        raise ValueError(f"bg_color {cfg.bg_color!r} not understood")
    rgb = tuple(float(p) for p in parts)
    if any(not 0.0 <= v <= 1.0 for v in rgb):
        raise ValueError("bg_color components must lie in [0, 1]")
    return rgb


def init_scene(target, templates, cfg, rng: np.random.Generator) -> Scene:
    """The starting scene a config describes, templates as given (fit.py:358-400)."""
    g = lambda k, d: getattr(cfg, k, d)  # noqa: E731  (duck-typed FitConfig)
    h, w = np.asarray(target).shape[:2]
    kind = g("initializer", "structure_aware")
    common = dict(v_init_bias=g("opacity_logit_init", DEFAULT_OPACITY_LOGIT),
                  sigma_c=g("color_init_noise", 0.02), rng=rng, templates=templates)
    if kind == "structure_aware":
        scene = structure_aware_init(target, cfg.num_primitives, cfg.scale_min, cfg.scale_max,
                                     density_cap=g("max_prims_per_pixel", 100),
                                     base_prob=g("variance_base_prob", 0.1),
                                     window=g("variance_window_size", 7), **common)
    elif kind == "random":
        scene = random_init(w, h, cfg.num_primitives, cfg.scale_min, cfg.scale_max, **common)
    else:
        raise ValueError(f"unknown initializer {kind!r}")
    return dataclasses.replace(scene, background=background_from_config(cfg),
                               alpha_max=g("alpha_max", 1.0), mu_blend=g("mu_blend", 0.0),
                               preserve_aspect=g("preserve_aspect", False))
