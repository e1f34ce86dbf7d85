"""torch.autograd.Function front end of the compositor.

The reference's renderer entry point is the pair render_forward(save=True) /
backward (raster.py:290-363, grad.py:134-187); here it is one autograd
Function whose forward runs K1+K2+K3 and whose backward runs the fit-step
kernel on the upstream gradients (K4 on saved lists when mu_blend > 0), so the
compositor composes with any torch loss:

    r = Renderer(templates, template_id, z, W, H, background=(1, 1, 1))
    img, alpha = r(params)            # params: (N, 8) float64 CUDA, requires_grad
    ((img - target) ** 2).mean().backward()   # params.grad = dL/dparams

``loss_mse(img, target)`` is the reference's loss_mse (fit.py:110-115) as a
fused autograd op on the renderer's output: one reduction kernel forward, one
kernel backward that writes the gradient straight into the rows the fit-step
kernel reads (the renderer's backward then skips its repacking pass).

The saved contribution lists live in a pooled Compositor held by ctx until
the backward (the reference keeps them in SavedForward + a fingerprint;
autograd's graph ownership replaces the fingerprint check).
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _native as nat
from .compositor import Compositor, _stream_handle, bin_capacity, cached_atlas
from .errors import BinOverflow
from .raster import DEFAULT_EPS_SKIP


def _current_stream() -> torch.cuda.Stream:
    # torch.cuda.current_stream() without its device-index resolution (~15 us of
    # Python per call on the eager path)
    sid, dev, dtype = torch._C._cuda_getCurrentStream(torch._C._cuda_getDevice())
    return torch.cuda.Stream(stream_id=sid, device_index=dev, device_type=dtype)


class _Composite(torch.autograd.Function):
    # mu_blend == 0 (colour from the primitive): the forward renders without saving
    # the contribution lists and the backward re-runs the forward on chip inside
    # the fit-step kernel with the upstream dL/dI, dL/dA per pixel (PF_LOSS_EXTERN)
    # -- no 16-byte saved entry per contribution written and read back through
    # HBM; mu_blend > 0 keeps K3(save) + K4.
    @staticmethod
    def forward(ctx, params, renderer: "Renderer", bg4):
        comp = renderer._lease(params)
        comp.preprocess(params)
        comp.bin()
        recompute = renderer.mu_blend == 0.0
        # a fresh (r, g, b, alpha) buffer per call: the outputs are views of it, no
        # copies (the caching allocator makes this free)
        comp.img4 = torch.empty(renderer.H * renderer.W * 4, dtype=torch.float32,
                                device=renderer.dev)
        if recompute and renderer.render_k34:
            # the fit-step kernel as a forward: the lists and their tile classes
            # stay for the backward's pass
            comp.render(eps_skip=renderer.eps_skip, bg_rgb=renderer.bg_rgb, bg4=bg4)
        else:
            comp.forward(save=not recompute, eps_skip=renderer.eps_skip, bg_rgb=renderer.bg_rgb,
                         bg4=bg4)
        if not torch.cuda.is_current_stream_capturing():
            renderer._watch(comp)
        img, alpha = comp.color(), comp.alpha()
        if ctx.needs_input_grad[0]:
            ctx.comp = comp  # the saved contribution lists: held until backward
        else:
            if comp.tile_classes is not None:
                comp.tile_classes[:16].zero_()  # (no backward pass to consume them)
            renderer._give_back(comp)
        ctx.renderer = renderer
        ctx.bg4 = bg4
        # an unused output's gradient arrives as None, not as a zero tensor
        ctx.set_materialize_grads(False)
        return img, alpha

    @staticmethod
    def backward(ctx, d_img, d_alpha):
        comp: Compositor = ctx.comp
        r = ctx.renderer
        if not torch.cuda.is_current_stream_capturing():
            r._raise_pending()
        n = comp.n
        grads = r._grads(n)
        d4 = r._d4()
        base = d_img._base if d_img is not None else None
        if (d_alpha is None and base is not None and getattr(base, "_pf_grad4", False)
                and d_img.stride() == (4 * r.W, 4, 1) and d_img.shape == (r.H, r.W, 3)
                and d_img.data_ptr() == base.data_ptr()):
            d4 = base  # loss_mse's (r, g, b, 0) rows: already the fit step's layout
        else:
            if d_img is None:
                d_img = torch.zeros(r.H, r.W, 3, dtype=torch.float32, device=r.dev)
            nat.check(nat.load().pf_pack_grad4(
                d_img.to(torch.float32).contiguous().data_ptr(),
                nat.ptr(d_alpha.to(torch.float32).contiguous() if d_alpha is not None else None),
                r.H * r.W, d4.data_ptr(), _stream_handle()),
                "pf_pack_grad4")
        if r.mu_blend == 0.0:
            comp.fit_step(grads, None, eps_skip=r.eps_skip, bg_rgb=r.bg_rgb, bg4=ctx.bg4,
                          loss_kind=nat.PF_LOSS_EXTERN, tgt4=d4.view(-1))
        else:
            comp.backward(d4.view(-1), grads, bg_rgb=r.bg_rgb, bg4=ctx.bg4)
        out = grads[: n * 8].view(n, 8)  # (a fresh buffer per call: no copy)
        ctx.comp = None
        r._give_back(comp)
        return out, None, None


def _rows4(img: torch.Tensor) -> bool:
    """img is the (H, W, 3) colour view of (r, g, b, alpha) float32 rows."""
    return (img.is_cuda and img.dtype == torch.float32 and img.dim() == 3
            and img.shape[2] == 3 and img.stride() == (4 * img.shape[1], 4, 1)
            and img.data_ptr() % 16 == 0)


_MSE_SCRATCH: dict = {}  # device -> zeroed PF_MSE4_SCRATCH doubles (self-resetting)


class _LossMSE(torch.autograd.Function):
    @staticmethod
    def forward(ctx, img, target):
        P = img.shape[0] * img.shape[1]
        sc = _MSE_SCRATCH.get(img.device)
        if sc is None:
            sc = _MSE_SCRATCH[img.device] = torch.zeros(2048, dtype=torch.float64,
                                                        device=img.device)
        loss = torch.empty((), dtype=torch.float32, device=img.device)
        st = _stream_handle()
        nat.check(nat.load().pf_mse4(img.data_ptr(), target.data_ptr(), P, sc.data_ptr(),
                                     loss.data_ptr(), st), "pf_mse4")
        ctx.save_for_backward(img, target)
        return loss

    @staticmethod
    def backward(ctx, g):
        img, target = ctx.saved_tensors
        H, W = img.shape[0], img.shape[1]
        out4 = torch.empty(H, W, 4, dtype=torch.float32, device=img.device)
        out4._pf_grad4 = True  # (r, g, b, 0) rows: _Composite.backward takes them as is
        g = g.to(torch.float32).contiguous()
        nat.check(nat.load().pf_mse4_grad(img.data_ptr(), target.data_ptr(), H * W, g.data_ptr(),
                                          out4.data_ptr(), _stream_handle()),
                  "pf_mse4_grad")
        return out4[:, :, :3], None


def loss_mse(img: torch.Tensor, target: torch.Tensor) -> torch.Tensor:
    """mean((img - target)^2) over all pixels and channels (fit.py:110-115) as an
    autograd op.  ``img`` is a Renderer's colour output (the (H, W, 3) view of its
    (r, g, b, alpha) rows); ``target`` (H, W, 3).  Returns a float32 scalar.
    Raises ShapeMismatch like the reference; any other image layout is rejected
    (ValueError) rather than copied."""
    from .errors import ShapeMismatch
    if tuple(img.shape) != tuple(target.shape):
        raise ShapeMismatch(f"shape {tuple(img.shape)} vs {tuple(target.shape)}")
    if not _rows4(img):
        raise ValueError("loss_mse: img must be a Renderer colour output ((H, W, 3) view of "
                         "float32 (r, g, b, alpha) rows on the GPU)")
    target = target.to(device=img.device, dtype=torch.float32).contiguous()
    return _LossMSE.apply(img, target)


class Renderer:
    """Scene structure bound to a device; call with (N, 8) float64 params.

    Per call there is no allocation and -- with ``s_max`` -- no host sync: the
    compositors (HBM buffers sized by the bin capacity) come from a small pool
    owned by the renderer, a forward's compositor being held by its autograd ctx
    until the backward ran.  ``s_max`` must bound every scale the renderer sees
    (an Adam loop with the reference's clamp guarantees it); the kernels flag a
    capacity overflow on the device and the flag is checked asynchronously:
    ``BinOverflow`` is raised at the next backward / call once the flagged
    forward has completed, or at ``check()``.  Without ``s_max`` every call sizes
    the capacity from the current scales (one device-to-host read).

    A whole training step through the Function (forward, torch loss, backward,
    an optimizer that keeps its state on the device) can be captured in a CUDA
    graph once ``s_max`` is set (the usual torch.cuda.graph recipe: eager
    warm-up on a side stream, then capture); inside a capture the asynchronous
    overflow watch is skipped -- the capacity bound makes it unnecessary.
    """

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
        self.atlas = cached_atlas(templates, preserve_aspect, self.dev)
        self.d_tid = torch.from_numpy(self.tid).to(self.dev)
        order = np.argsort(self.z, kind="stable").astype(np.int32)
        self.d_zorder = torch.from_numpy(order).to(self.dev)
        self.bg_rgb = tuple(float(c) for c in background)
        self._free: list[Compositor] = []
        self._pending: list[tuple] = []  # (event, pinned status copy, capacity)
        self._d4buf = None
        # forward through the fit-step kernel (PF_LOSS_RENDER) rather than K3 (A/B
        # switch PF_RENDER_K3=1)
        self.render_k34 = os.environ.get("PF_RENDER_K3", "0") != "1"
        self.lpt = os.environ.get("PF_RENDER_LPT", "1") == "1"

    # -- pooled per-call state
    def _capacity(self, params: torch.Tensor) -> int:
        n = len(self.tid)
        if self.s_max is not None:
            if getattr(self, "_cap_smax", None) is None:  # constant: computed once
                self._cap_smax = bin_capacity(np.full(n, float(self.s_max)), self.tid,
                                              self.atlas.hyp, self.padding, 16,
                                              -(-self.W // 16), -(-self.H // 16))
            return self._cap_smax
        else:
            scales = params[:, 2].detach().double().cpu().numpy() if n else np.zeros(0)
        return bin_capacity(scales, self.tid, self.atlas.hyp, self.padding, 16,
                            -(-self.W // 16), -(-self.H // 16))

    def _lease(self, params: torch.Tensor) -> Compositor:
        if not torch.cuda.is_current_stream_capturing():
            self._raise_pending()
        cap = self._capacity(params)
        for i, c in enumerate(self._free):
            if c.capacity >= cap:
                return self._free.pop(i)
        comp = Compositor(self.tid, self.z, self.atlas, self.W, self.H, alpha_max=self.alpha_max,
                          mu_blend=self.mu_blend, padding=self.padding, capacity=cap,
                          device=self.dev, d_tid=self.d_tid, d_zorder=self.d_zorder)
        if self.render_k34 and self.mu_blend == 0.0 and self.lpt:
            comp.enable_step_schedule()  # longest-first tile classes for both passes
        return comp

    def _give_back(self, comp: Compositor) -> None:
        if len(self._free) < 2:
            self._free.append(comp)

    def _grads(self, n: int) -> torch.Tensor:
        # per call (the caching allocator makes it a memset): handed to autograd
        # as the parameter gradient without a copy -- with params.grad None (the
        # usual zero_grad(set_to_none=True)) it becomes params.grad as is
        return torch.zeros(n * 8 + 4, dtype=torch.float64, device=self.dev)

    def _d4(self) -> torch.Tensor:
        if self._d4buf is None:
            self._d4buf = torch.zeros(self.H, self.W, 4, dtype=torch.float32, device=self.dev)
        return self._d4buf

    # -- asynchronous overflow check
    def _watch(self, comp: Compositor) -> None:
        # (pinned status copy + event pairs are recycled once checked)
        pool = self.__dict__.setdefault("_wpool", [])
        if pool:
            ev, st = pool.pop()
        else:
            ev, st = torch.cuda.Event(), torch.empty(2, dtype=torch.int32, pin_memory=True)
        st.copy_(comp.status[:2], non_blocking=True)
        ev.record(_current_stream())
        self._pending.append((ev, st, comp.capacity))

    def _raise_pending(self, wait: bool = False) -> None:
        keep = []
        pool = self.__dict__.setdefault("_wpool", [])
        for ev, st, cap in self._pending:
            if wait:
                ev.synchronize()
            elif not ev.query():
                keep.append((ev, st, cap))
                continue
            pool.append((ev, st))
            if int(st[1]):
                self._pending = []
                raise BinOverflow(f"{int(st[0])} bin entries exceed capacity {cap}: a scale "
                                  f"exceeded s_max={self.s_max}")
        self._pending = keep

    def check(self) -> None:
        """Wait for every issued forward and raise BinOverflow if one overflowed."""
        self._raise_pending(wait=True)

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
