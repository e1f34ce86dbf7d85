"""torch.autograd.Function front end of the compositor.

The reference's renderer entry point is the pair render_forward(save=True) /
backward (raster.py:290-363, grad.py:134-187); here it is one autograd
Function whose forward runs K1+K2+K3 and whose backward runs K4, so the
compositor composes with any torch loss:

    r = Renderer(templates, template_id, z, W, H, background=(1, 1, 1))
    img, alpha = r(params)            # params: (N, 8) float64 CUDA, requires_grad
    ((img - target) ** 2).mean().backward()   # params.grad = dL/dparams

The saved contribution lists live in the per-call Compositor held by ctx
(the reference keeps them in SavedForward + a fingerprint; autograd's graph
ownership replaces the fingerprint check).
"""

from __future__ import annotations

import numpy as np
import torch

from .compositor import Compositor, DeviceAtlas, bin_capacity
from .raster import DEFAULT_EPS_SKIP


class _Composite(torch.autograd.Function):
    @staticmethod
    def forward(ctx, params, renderer: "Renderer", bg4):
        comp = renderer._new_compositor(params)
        comp.preprocess(params)
        comp.bin()
        comp.forward(save=True, eps_skip=renderer.eps_skip, bg_rgb=renderer.bg_rgb, bg4=bg4)
        ctx.comp = comp
        ctx.renderer = renderer
        ctx.bg4 = bg4
        return comp.color().clone(), comp.alpha().clone()

    @staticmethod
    def backward(ctx, d_img, d_alpha):
        comp: Compositor = ctx.comp
        r = ctx.renderer
        n = comp.n
        grads = torch.zeros(n * 8 + 4, dtype=torch.float64, device=comp.device)
        d4 = torch.zeros(r.H, r.W, 4, dtype=torch.float32, device=comp.device)
        if d_img is not None:
            d4[:, :, :3] = d_img
        if d_alpha is not None:
            d4[:, :, 3] = d_alpha
        comp.backward(d4.view(-1), grads, bg_rgb=r.bg_rgb, bg4=ctx.bg4)
        return grads[: n * 8].view(n, 8), None, None


class Renderer:
    """Scene structure bound to a device; call with (N, 8) float64 params."""

    def __init__(self, templates, template_id, z, canvas_w: int, canvas_h: int, *,
                 background=(1.0, 1.0, 1.0), alpha_max: float = 1.0, mu_blend: float = 0.0,
                 preserve_aspect: bool = False, eps_skip: float = DEFAULT_EPS_SKIP,
                 padding: float = 2.0, s_max: float | None = None, device="cuda"):
        self.dev = torch.device(device)
        self.W, self.H = int(canvas_w), int(canvas_h)
        self.alpha_max, self.mu_blend = float(alpha_max), float(mu_blend)
        self.eps_skip, self.padding, self.s_max = float(eps_skip), float(padding), s_max
        self.tid = np.ascontiguousarray(template_id, dtype=np.int32)
        self.z = np.asarray(z, dtype=np.int64)
        self.atlas = DeviceAtlas(templates, preserve_aspect, self.dev)
        self.d_tid = torch.from_numpy(self.tid).to(self.dev)
        order = np.argsort(self.z, kind="stable").astype(np.int32)
        self.d_zorder = torch.from_numpy(order).to(self.dev)
        self.bg_rgb = tuple(float(c) for c in background)

    def _new_compositor(self, params: torch.Tensor) -> Compositor:
        n = len(self.tid)
        if self.s_max is not None:
            scales = np.full(n, float(self.s_max))
        else:
            scales = params[:, 2].detach().double().cpu().numpy() if n else np.zeros(0)
        cap = bin_capacity(scales, self.tid, self.atlas.hyp, self.padding, 16,
                           -(-self.W // 16), -(-self.H // 16))
        return Compositor(self.tid, self.z, self.atlas, self.W, self.H, alpha_max=self.alpha_max,
                          mu_blend=self.mu_blend, padding=self.padding, capacity=cap,
                          device=self.dev, d_tid=self.d_tid, d_zorder=self.d_zorder)

    def __call__(self, params: torch.Tensor, bg_img: torch.Tensor | None = None):
        """Render; ``bg_img`` (H, W, 3) is an optional per-pixel background."""
        if params.dtype != torch.float64 or params.shape != (len(self.tid), 8):
            raise ValueError(f"params must be float64 ({len(self.tid)}, 8)")
        bg4 = None
        if bg_img is not None:
            bg4 = torch.zeros(self.H, self.W, 4, dtype=torch.float32, device=self.dev)
            bg4[:, :, :3] = bg_img.to(device=self.dev, dtype=torch.float32)
            bg4 = bg4.view(-1)
        return _Composite.apply(params.contiguous(), self, bg4)
