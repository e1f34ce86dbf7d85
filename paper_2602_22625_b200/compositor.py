"""Device-resident compositor: owns the HBM buffers and launches the C-ABI stages.

One ``Compositor`` is bound to a scene *structure* (template ids, z order,
template atlas, canvas, row band) and a bin capacity; parameters change every
step and are passed as a float64 (N, 8) CUDA tensor.  The stages map to the
reference's per-iteration calls in fit.run_loop (pkg/src/primfit/fit.py:486-501):

    preprocess()+bin()  ->  bin_tiles        (raster.py:227-265)
    forward()           ->  render_forward   (raster.py:290-363) [+ loss, fit.py:112-151]
    backward()          ->  backward         (grad.py:134-206)
    adam()              ->  adam_step        (fit.py:195-238)

HBM layout: params/grads/moments float64 [N][8]; primitive
records 192 B/prim; atlas float64 planar [4][texels]; bins int32 CSR; saved
forward = float64 transmittance + texel coords U, V and uint16 list position
per contributing (pixel, primitive) at slot 256*bin_off[t] + k*256 + pixel;
pixel buffers float32.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .errors import BinOverflow

RENDER_TILE = 16


def _stream_handle(stream: torch.cuda.Stream | None = None) -> int:
    if stream is not None:
        return stream.cuda_stream
    # the current stream's raw handle without building a Stream object (that
    # costs ~20 us of Python per call: 7 launches per eager autograd step)
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


class DeviceAtlas:
    """Template atlas in HBM: planar float64 RGBA + per-template metadata.

    Replaces PackedScene.tex/toff/tw/th (raster.py:79-87); ``q`` is the v-axis
    aspect (th/tw when preserve_aspect, else 1, raster.py:88-91) and ``hyp`` the
    bbox factor hypot(1, max(1, q)) computed with Python's math.hypot so the
    binning bbox is bit-identical to bbox_half_side (raster.py:222-224).
    """

    def __init__(self, templates, preserve_aspect: bool, device="cuda"):
        rgbas = [np.asarray(t.rgba, dtype=np.float64) for t in templates]
        self.n_templates = len(rgbas)
        self.tw = np.asarray([a.shape[1] for a in rgbas], dtype=np.int32)
        self.th = np.asarray([a.shape[0] for a in rgbas], dtype=np.int32)
        sizes = self.tw.astype(np.int64) * self.th.astype(np.int64)
        self.base = np.concatenate(([0], np.cumsum(sizes)))[:-1].astype(np.int32)
        self.texels = int(sizes.sum())
        planar = np.zeros((4, max(self.texels, 1)), dtype=np.float64)
        for a, b, sz in zip(rgbas, self.base, sizes):
            planar[:, b : b + sz] = a.reshape(-1, 4).T
        if preserve_aspect:
            self.q = self.th.astype(np.float64) / self.tw.astype(np.float64)
        else:
            self.q = np.ones(self.n_templates, dtype=np.float64)
        self.hyp = np.asarray([math.hypot(1.0, max(1.0, float(q))) for q in self.q])
        dev = torch.device(device)
        self.tex = torch.from_numpy(planar).to(dev)
        self.d_base = torch.from_numpy(self.base).to(dev)
        self.d_w = torch.from_numpy(self.tw).to(dev)
        self.d_h = torch.from_numpy(self.th).to(dev)
        self.d_q = torch.from_numpy(self.q).to(dev)
        self.d_hyp = torch.from_numpy(self.hyp).to(dev)
        # alpha quad atlas (four bilinear taps per texel, zero padded), built on device
        self.quad = torch.zeros(max(self.texels, 1) * 4, dtype=torch.float32, device=dev)
        # zero-padded fp32 alpha plane ((w+1) x (h+1) per template) for pf_fit_step
        psz = (self.tw.astype(np.int64) + 1) * (self.th.astype(np.int64) + 1)
        self.pbase = np.concatenate(([0], np.cumsum(psz)))[:-1].astype(np.int32)
        self.pad_texels = int(-(-max(int(psz.sum()), 1) // 4) * 4)
        self.d_pbase = torch.from_numpy(self.pbase).to(dev)
        self.apad = torch.zeros(self.pad_texels, dtype=torch.float32, device=dev)
        self.apad64 = torch.zeros(self.pad_texels, dtype=torch.float64, device=dev)
        if self.texels:
            lib = nat.load()
            nat.check(lib.pf_atlas_quad(self.tex.data_ptr(), self.texels, self.d_base.data_ptr(),
                                        self.d_w.data_ptr(), self.d_h.data_ptr(),
                                        self.n_templates, self.quad.data_ptr(),
                                        _stream_handle()), "pf_atlas_quad")
            nat.check(lib.pf_atlas_pad(self.tex.data_ptr(), self.texels, self.d_base.data_ptr(),
                                       self.d_pbase.data_ptr(), self.d_w.data_ptr(),
                                       self.d_h.data_ptr(), self.n_templates, self.pad_texels,
                                       self.apad.data_ptr(), _stream_handle()), "pf_atlas_pad")
            # float64 copy of the padded plane (exact: built from the float64 atlas)
            pad64 = np.zeros(self.pad_texels, dtype=np.float64)
            for a_, pb, w_, h_ in zip(rgbas, self.pbase, self.tw, self.th):
                blk = np.zeros((h_ + 1, w_ + 1), dtype=np.float64)
                blk[:h_, :w_] = a_[:, :, 3]
                pad64[pb : pb + blk.size] = blk.reshape(-1)
            self.apad64.copy_(torch.from_numpy(pad64))


def bin_capacity(scales: np.ndarray, tids: np.ndarray, hyp: np.ndarray, padding: float,
                 tile: int, ntx: int, nty_band: int) -> int:
    """Upper bound on (tile, primitive) entries for the given per-primitive scales.

    A bbox of half side r covers at most floor(2r/tile)+2 tiles per axis.  The
    Adam step clamps scale to s_max, so bounding with s_max makes the bound
    hold for the whole fit (no device->host sync, no overflow).
    """
    if len(scales) == 0:
        return 0
    r = np.asarray(scales, dtype=np.float64) * hyp[tids] + padding
    span = np.floor(2.0 * r / tile) + 2.0
    per = np.minimum(span, ntx) * np.minimum(span, max(nty_band, 1))
    return int(min(per.sum(), float(2**31 - 1)))


@dataclass
class Band:
    ty_begin: int
    ty_end: int


class Compositor:
    """HBM buffers + stage launchers for one scene structure on one device."""

    def __init__(self, template_id: np.ndarray, z: np.ndarray, atlas: DeviceAtlas, W: int,
                 H: int, *, alpha_max: float, mu_blend: float, padding: float,
                 capacity: int, band: Band | None = None, bin_tile: int = RENDER_TILE,
                 device="cuda", d_tid: torch.Tensor | None = None,
                 d_zorder: torch.Tensor | None = None):
        self.lib = nat.load()
        self.device = torch.device(device)
        self.n = int(len(template_id))
        self.atlas = atlas
        self.W, self.H = int(W), int(H)
        self.alpha_max, self.mu_blend, self.padding = float(alpha_max), float(mu_blend), float(padding)
        self.tile = int(bin_tile)
        self.ntx = -(-self.W // self.tile)
        self.nty = -(-self.H // self.tile)
        self.band = band or Band(0, self.nty)
        self.n_tiles = (self.band.ty_end - self.band.ty_begin) * self.ntx
        self.capacity = int(capacity)
        # K34 stage depth: 64 staged list entries per tile when the capacity bound
        # says lists run long (c2 / c4: ~70 entries per tile bound), else 32
        self.stage_hint = 64 if self.capacity > 48 * max(self.n_tiles, 1) else 32
        dev = self.device
        if d_tid is None:
            d_tid = torch.from_numpy(np.ascontiguousarray(template_id, dtype=np.int32)).to(dev)
        if d_zorder is None:
            order = np.argsort(np.asarray(z, dtype=np.int64), kind="stable").astype(np.int32)
            d_zorder = torch.from_numpy(order).to(dev)
        self.d_tid, self.d_zorder = d_tid, d_zorder
        rb = int(self.lib.pf_record_bytes())
        self.rec = torch.empty(max(self.n, 1) * rb, dtype=torch.uint8, device=dev)
        self.scratch_bytes = int(self.lib.pf_bin_scratch_bytes(self.n, self.n_tiles, self.capacity))
        self.scratch = torch.zeros(self.scratch_bytes, dtype=torch.uint8, device=dev)
        a = atlas
        nat.check(self.lib.pf_scratch_init(self.scratch.data_ptr(), self.scratch_bytes,
                                           self.d_tid.data_ptr(), self.d_zorder.data_ptr(), self.n,
                                           a.d_base.data_ptr(), a.d_pbase.data_ptr(),
                                           a.d_w.data_ptr(), a.d_h.data_ptr(), a.d_q.data_ptr(),
                                           a.d_hyp.data_ptr(), a.n_templates, self.capacity,
                                           _stream_handle()), "pf_scratch_init")
        self.bin_off = torch.zeros(self.n_tiles + 1, dtype=torch.int32, device=dev)
        self.bin_idx = torch.zeros(max(self.capacity, 1), dtype=torch.int32, device=dev)
        # tile cost classes for pf_fit_step's longest-first schedule (fused path only)
        self.tile_classes = None
        # slot binning (fit step; enable_step_schedule(slot_m)): None = CSR lists
        self.slots = None
        self.slot_m = 0
        self.status = torch.zeros(4, dtype=torch.int32, device=dev)
        self._saved_alloc = False
        self.launches = 0  # kernels launched through this object (one per stage call)

    def enable_step_schedule(self, slot_m: int = 0) -> None:
        """Tile cost classes for pf_fit_step's longest-first schedule (call before
        the first preprocess / bin() of a fused fit loop).  ``slot_m > 0``: slot
        binning -- K1 scatters the tile lists itself (``slot_m`` slots per tile,
        overflow list beyond), pf_fit_step sorts them, bin() is a no-op."""
        if self.tile_classes is None:
            # counts, per-class tile lists, measured tile costs
            nt = max(self.n_tiles, 1)
            self.tile_classes = torch.zeros(16 + 16 * 4 * nt + nt, dtype=torch.int32,
                                            device=self.device)
        if slot_m > 0 and self.slots is None:
            if self.tile != RENDER_TILE:
                raise ValueError(f"slot binning needs bin tile {RENDER_TILE}, got {self.tile}")
            self.slot_m = int(slot_m)
            nbytes = int(self.lib.pf_slot_bytes(self.n_tiles, self.slot_m, self.capacity))
            self.slots = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)

    def _slot_args(self, classes: bool = True):
        if self.slots is None:
            return (None, 0, None)
        return (self.slots.data_ptr(), self.slot_m, self.tile_classes.data_ptr())

    def slot_lists(self) -> tuple[np.ndarray, np.ndarray]:
        """Diagnostics / tests (synchronising): the current slot lists (after a K1,
        before the fit step consumes them) as CSR (offsets, primitive indices),
        each tile's list sorted by z rank -- what pf_fit_step stages."""
        nt, m = self.n_tiles, self.slot_m
        raw = self.slots.cpu().numpy()
        ctl = raw[:256].view(np.uint32)
        off = 256
        cnt = raw[off : off + 4 * nt].view(np.int32).copy()
        off = -(-(off + 4 * max(nt, 1)) // 256) * 256
        slot = raw[off : off + 4 * nt * m].view(np.uint32).reshape(nt, m)
        # (the slot array is followed by the general-path pool, capacity + 64 entries)
        off = -(-(off + 4 * (nt * m + self.capacity + 64)) // 256) * 256
        novf = int(ctl[0])
        ovf = raw[off : off + 8 * novf].view(np.int32).reshape(-1, 2)
        zorder = self.d_zorder.cpu().numpy()
        lists = [list(slot[t, : min(int(cnt[t]), m)]) for t in range(nt)]
        for t, z in ovf:
            lists[int(t)].append(int(z))
        offs = np.zeros(nt + 1, dtype=np.int64)
        idx = []
        for t in range(nt):
            zs = sorted(int(z) for z in lists[t])
            idx.extend(int(zorder[z]) for z in zs)
            offs[t + 1] = offs[t] + len(zs)
        return offs, np.asarray(idx, dtype=np.int32)

    # -- buffers for rendering (allocated lazily; binning-only users skip them)
    def alloc_render(self, save: bool, loss: bool = False):
        if self.tile != RENDER_TILE:
            raise ValueError(f"render kernels need bin tile {RENDER_TILE}, got {self.tile}")
        dev, P = self.device, self.W * self.H
        if not hasattr(self, "img4"):
            # (r, g, b, alpha) per pixel: one 16-byte store
            self.img4 = torch.zeros(P * 4, dtype=torch.float32, device=dev)
        if save and not self._saved_alloc:
            self.saved_entries = int(self.lib.pf_saved_capacity(max(self.capacity, 1)))
            nbytes = int(self.lib.pf_saved_bytes(max(self.capacity, 1)))
            self.saved = torch.empty(nbytes, dtype=torch.uint8, device=dev)
            self.ent_n = torch.zeros(P, dtype=torch.int32, device=dev)
            self._saved_alloc = True
        if loss and not hasattr(self, "d4"):
            # (dL/dI r, g, b, dL/dA) per pixel
            self.d4 = torch.zeros(P * 4, dtype=torch.float32, device=dev)
            # per-warp loss partials (8 warps per tile, 3 sums each)
            self.part = torch.zeros(max(self.n_tiles, 1) * 8 * 3, dtype=torch.float64, device=dev)

    def color(self) -> torch.Tensor:
        return self.img4.view(self.H, self.W, 4)[:, :, :3]

    def alpha(self) -> torch.Tensor:
        return self.img4.view(self.H, self.W, 4)[:, :, 3]

    # -- K1 + K2
    def preprocess(self, params: torch.Tensor, stream=None) -> None:
        if self.slots is not None:
            # a full K1 re-scatters every primitive: empty the lists (and classes) first
            nat.check(self.lib.pf_slot_reset(self.slots.data_ptr(), self.n_tiles, self.slot_m,
                                             self.capacity, self.tile_classes.data_ptr(),
                                             _stream_handle(stream)), "pf_slot_reset")
        key = (nat.ptr(self.slots), nat.ptr(self.tile_classes))
        tail = self.__dict__.get("_pre_tail")
        if tail is None or tail[0] != key:
            # (everything after the parameter pointer except the stream: constant)
            tail = self._pre_tail = (key, [
                self.n, self.alpha_max, self.mu_blend, self.padding, self.W, self.H, self.tile,
                self.band.ty_begin, self.band.ty_end, self.capacity, self.rec.data_ptr(),
                self.scratch.data_ptr(), self.scratch_bytes, *self._slot_args()])
        nat.check(self.lib.pf_preprocess(params.data_ptr(), *tail[1], _stream_handle(stream)),
                  "pf_preprocess")
        self.launches += 1

    def preprocess_sync(self, params: torch.Tensor, src: torch.Tensor, stream=None) -> None:
        """K1 from ``src`` (e.g. a pinned host vector), recomputing only the
        primitives whose parameters differ from the device copy ``params``."""
        nat.check(
            self.lib.pf_preprocess_sync(
                params.data_ptr(), src.data_ptr(), self.n, self.alpha_max, self.mu_blend,
                self.padding, self.W, self.H, self.tile, self.band.ty_begin, self.band.ty_end,
                self.capacity, self.rec.data_ptr(), self.scratch.data_ptr(), self.scratch_bytes,
                *self._slot_args(), _stream_handle(stream)),
            "pf_preprocess_sync")
        self.launches += 1

    def adam_preprocess(self, params, grads, m, v, *, frozen, gains, lr_table, bc1_table,
                        bc2_table, s_min, s_max, sums=None, part=None, hist_part=None,
                        last_part=None, records: bool = True, mirror=None,
                        stream=None) -> None:
        """K5+K1 fused: Adam on every parameter, then the next step's records + rects
        (``records=False``: Adam only -- the caller re-runs preprocess() first).
        ``part``: pf_fit_step's loss partials (folded per block into ``hist_part``);
        ``sums``: already reduced loss sums (multi-rank path)."""
        g8 = (C.c_double * 8)(*[float(g) for g in gains])
        nat.check(
            self.lib.pf_adam_preprocess(
                params.data_ptr(), grads.data_ptr(), m.data_ptr(), v.data_ptr(), nat.ptr(frozen),
                C.addressof(g8), lr_table.data_ptr(), bc1_table.data_ptr(), bc2_table.data_ptr(),
                1, float(s_min), float(s_max), nat.ptr(sums), nat.ptr(part),
                self.n_part if part is not None else 0, nat.ptr(hist_part), nat.ptr(last_part),
                self.n,
                self.alpha_max, self.mu_blend, self.padding, self.W, self.H, self.tile,
                self.band.ty_begin, self.band.ty_end, self.capacity,
                self.rec.data_ptr() if records else None,
                self.scratch.data_ptr(), self.scratch_bytes, nat.ptr(mirror),
                *self._slot_args(), _stream_handle(stream)),
            "pf_adam_preprocess")
        self.launches += 1

    @property
    def adam_blocks(self) -> int:
        return int(self.lib.pf_adam_blocks(self.n))

    def bin(self, stream=None) -> None:
        """K2: CSR tile bins (z-ascending lists) from the rects of the last K1
        (slot mode: nothing to do -- K1 scattered the lists)."""
        if self.slots is not None:
            return
        key = nat.ptr(self.tile_classes)
        cached = self.__dict__.get("_bin_args")
        if cached is None or cached[0] != key:
            # (constant per compositor but for the tile classes, attached later)
            cached = self._bin_args = (key, [
                self.n, self.W, self.H, self.tile, self.band.ty_begin, self.band.ty_end,
                self.capacity, self.scratch.data_ptr(), self.scratch_bytes,
                self.bin_off.data_ptr(), self.bin_idx.data_ptr(), self.status.data_ptr(), key],
                int(self.lib.pf_bin_launches(self.n, self.W, self.H, self.tile,
                                             self.band.ty_begin, self.band.ty_end)))
        nat.check(self.lib.pf_bin(*cached[1], _stream_handle(stream)), "pf_bin")
        self.launches += cached[2]

    def check_overflow(self) -> int:
        """Synchronising read of K; raises BinOverflow when capacity was exceeded."""
        k, ovf = (int(v) for v in self.status[:2].cpu())
        if ovf:
            raise BinOverflow(f"{k} bin entries exceed capacity {self.capacity}")
        return k

    # -- K3
    def forward(self, *, save: bool, eps_skip: float, bg_rgb=(1.0, 1.0, 1.0),
                bg4: torch.Tensor | None = None, loss_kind: int = nat.PF_LOSS_NONE,
                tgt4: torch.Tensor | None = None, alpha_w: float = 0.0,
                w_mse: float = 1.0, w_gray: float = 0.0,
                P_total: int | None = None, stream=None) -> None:
        lossy = loss_kind != nat.PF_LOSS_NONE
        self.alloc_render(save, lossy)
        P = float(P_total if P_total is not None else self.W * self.H)
        p = nat.ptr
        nat.check(
            self.lib.pf_forward(
                self.rec.data_ptr(), self.n, self.atlas.tex.data_ptr(),
                self.atlas.quad.data_ptr(), self.atlas.texels,
                self.bin_off.data_ptr(), self.bin_idx.data_ptr(), self.status.data_ptr(),
                self.W, self.H, self.band.ty_begin, self.band.ty_end,
                float(eps_skip), self.mu_blend, float(bg_rgb[0]), float(bg_rgb[1]),
                float(bg_rgb[2]), p(bg4), p(self.saved) if save else None,
                self.saved_entries if save else 0, p(self.ent_n) if save else None,
                self.img4.data_ptr(), int(loss_kind), p(tgt4), float(alpha_w), float(w_mse),
                float(w_gray),
                1.0 / (3.0 * P), 1.0 / P, p(self.d4) if lossy else None,
                p(self.part) if lossy else None, _stream_handle(stream)),
            "pf_forward")
        self.launches += 1

    # -- K34 (fit step: forward + loss + backward in one kernel)
    def fit_step(self, grads: torch.Tensor | None, sums: torch.Tensor | None, *, eps_skip: float,
                 bg_rgb=(1.0, 1.0, 1.0), bg4: torch.Tensor | None = None,
                 loss_kind: int = nat.PF_LOSS_MSE, tgt4: torch.Tensor | None, alpha_w: float = 0.0,
                 w_mse: float = 1.0, w_gray: float = 0.0,
                 P_total: int | None = None, image: bool = False, stream=None) -> None:
        if self.mu_blend > 0.0:
            raise ValueError("pf_fit_step needs mu_blend == 0; use forward + backward")
        if self.tile != RENDER_TILE:
            raise ValueError(f"render kernels need bin tile {RENDER_TILE}, got {self.tile}")
        dev, P = self.device, self.W * self.H
        if not hasattr(self, "spill"):
            nbytes = int(self.lib.pf_step_spill_bytes(max(self.capacity, 1)))
            self.spill = torch.empty(nbytes, dtype=torch.uint8, device=dev)
            self.step_ctr = torch.zeros(4, dtype=torch.int32, device=dev)
            if not hasattr(self, "part"):
                self.part = torch.zeros(max(self.n_tiles, 1) * 8 * 3, dtype=torch.float64,
                                        device=dev)
        if image and not hasattr(self, "img4"):
            self.img4 = torch.zeros(P * 4, dtype=torch.float32, device=dev)
        Pt = float(P_total if P_total is not None else P)
        p = nat.ptr
        # the argument list minus the per-call pointers, built once per (mode,
        # scalars, the buffers that may be (re)attached) and reused (the eager
        # autograd step calls this twice per iteration)
        key = (int(loss_kind), float(eps_skip), tuple(float(c) for c in bg_rgb), float(alpha_w),
               float(w_mse), float(w_gray), Pt, self.part.data_ptr(), self.stage_hint,
               p(self.tile_classes), p(self.slots))
        cache = self.__dict__.setdefault("_fit_args", {})
        args = cache.get(key)
        if args is None:
            args = cache[key] = [
                self.rec.data_ptr(), self.n, self.atlas.tex.data_ptr(),
                self.atlas.apad.data_ptr(), self.atlas.apad64.data_ptr(), self.atlas.pad_texels,
                self.atlas.texels,
                self.bin_off.data_ptr(), self.bin_idx.data_ptr(), self.status.data_ptr(),
                self.W, self.H, self.band.ty_begin, self.band.ty_end, float(eps_skip),
                float(bg_rgb[0]), float(bg_rgb[1]), float(bg_rgb[2]), None, int(loss_kind),
                None, float(alpha_w), float(w_mse), float(w_gray), 1.0 / (3.0 * Pt), 1.0 / Pt,
                self.spill.data_ptr(), None, self.part.data_ptr(),
                None, self.step_ctr.data_ptr(), nat.ptr(self.tile_classes),
                self.stage_hint, self.scratch.data_ptr(), self.scratch_bytes, self.capacity,
                nat.ptr(self.slots), self.slot_m, None]
        args = list(args)
        args[18], args[20] = p(bg4), p(tgt4)
        args[27] = p(self.img4) if image else None
        args[29] = p(grads)
        args[38] = _stream_handle(stream)
        nat.check(self.lib.pf_fit_step(*args), "pf_fit_step")
        self.launches += 1
        if sums is not None:
            self.fold_loss(sums, stream)

    def render(self, *, eps_skip: float, bg_rgb=(1.0, 1.0, 1.0), bg4: torch.Tensor | None = None,
               stream=None) -> None:
        """The fit-step kernel as a forward only (PF_LOSS_RENDER): img4 from the
        pf_bin lists, which stay valid (with their tile classes) for a following
        fit_step(PF_LOSS_EXTERN) -- the autograd Function's forward."""
        self.fit_step(None, None, eps_skip=eps_skip, bg_rgb=bg_rgb, bg4=bg4,
                      loss_kind=nat.PF_LOSS_RENDER, tgt4=None, image=True, stream=stream)

    @property
    def n_part(self) -> int:
        """Loss partial triples per pf_fit_step launch (one per warp: 8 per band tile)."""
        return self.n_tiles * 8

    def fold_loss(self, sums: torch.Tensor, stream=None) -> None:
        if getattr(self, "fold_scratch", None) is None:
            self.fold_scratch = torch.zeros(int(self.lib.pf_fold_scratch_bytes(self.n_part)),
                                            dtype=torch.uint8, device=self.device)
        nat.check(self.lib.pf_fold_loss(self.part.data_ptr(), self.n_part, sums.data_ptr(),
                                        self.fold_scratch.data_ptr(), _stream_handle(stream)),
                  "pf_fold_loss")
        self.launches += 1

    # -- K4
    def backward(self, d4: torch.Tensor, grads: torch.Tensor, *, bg_rgb=(1.0, 1.0, 1.0),
                 bg4: torch.Tensor | None = None, sums: torch.Tensor | None = None,
                 stream=None) -> None:
        """K4 on d4 = (dL/dI, dL/dA) per pixel; with ``sums`` it also folds the fused
        loss partials of the last forward."""
        p = nat.ptr
        nat.check(
            self.lib.pf_backward(
                self.rec.data_ptr(), self.n, self.atlas.tex.data_ptr(),
                self.atlas.quad.data_ptr(), self.atlas.texels,
                self.bin_off.data_ptr(), self.bin_idx.data_ptr(), self.status.data_ptr(),
                self.saved.data_ptr(), self.saved_entries, self.ent_n.data_ptr(),
                d4.data_ptr(), float(bg_rgb[0]), float(bg_rgb[1]), float(bg_rgb[2]), p(bg4),
                self.mu_blend, self.W, self.H, self.band.ty_begin, self.band.ty_end,
                grads.data_ptr(), p(self.part) if sums is not None else None, p(sums),
                _stream_handle(stream)),
            "pf_backward")
        self.launches += 1


def pixels4(rgb: np.ndarray, w: np.ndarray | float | None = None) -> np.ndarray:
    """(H, W, 3) (+ optional (H, W) fourth channel) -> float32 (H*W*4) for the kernels."""
    rgb = np.asarray(rgb, dtype=np.float32)
    out = np.zeros(rgb.shape[:2] + (4,), dtype=np.float32)
    out[..., :3] = rgb
    if w is not None:
        out[..., 3] = np.asarray(w, dtype=np.float32)
    return out.reshape(-1)


_GAINS8: dict[tuple, object] = {}  # gains -> ctypes double[8] (adam_launch)


def adam_launch(params, grads, m, v, *, frozen=None, gains=None, n: int,
                lr_table=None, bc1_table=None, bc2_table=None, iter_counter=None,
                lr=0.0, bc1=1.0, bc2=1.0, clamp=False, s_min=0.0, s_max=0.0,
                zero_grads=True, sums=None, loss_kind=nat.PF_LOSS_MSE, alpha_w=0.0,
                P_total=1, hist_loss=None, hist_psnr=None, counter=None, stream=None):
    """K5 launcher (both modes of pf_adam)."""
    lib = nat.load()
    p = nat.ptr
    g8 = None
    if gains is not None:
        gk = tuple(float(g) for g in gains)
        g8 = _GAINS8.get(gk)
        if g8 is None:  # (kept alive here: the launch reads it by address)
            g8 = _GAINS8[gk] = (C.c_double * 8)(*gk)
    P = float(P_total)
    nat.check(
        lib.pf_adam(
            params.data_ptr(), grads.data_ptr(), m.data_ptr(), v.data_ptr(), p(frozen),
            C.addressof(g8) if g8 is not None else None, int(n), p(lr_table), p(bc1_table),
            p(bc2_table), p(iter_counter), float(lr), float(bc1), float(bc2), int(bool(clamp)),
            float(s_min), float(s_max), int(bool(zero_grads)), p(sums), int(loss_kind),
            float(alpha_w), 1.0 / (3.0 * P), 1.0 / P, p(hist_loss), p(hist_psnr), p(counter),
            _stream_handle(stream)),
        "pf_adam")


# -- per-structure caches for the per-call API (raster.render_forward, grad.backward,
#    bin_tiles, autograd.Renderer): the atlas upload and the compositor's HBM
#    buffers are built once per scene structure, not once per call.
_ATLASES: dict[tuple, DeviceAtlas] = {}


def cached_atlas(templates, preserve_aspect: bool, device) -> DeviceAtlas:
    """DeviceAtlas keyed by template content (sha256 of shape + texels)."""
    key = (tuple(t.content_hash() if hasattr(t, "content_hash") else
                 _rgba_hash(np.asarray(t.rgba)) for t in templates),
           bool(preserve_aspect), str(torch.device(device)))
    atlas = _ATLASES.get(key)
    if atlas is None:
        if len(_ATLASES) >= 16:
            _ATLASES.pop(next(iter(_ATLASES)))
        atlas = _ATLASES[key] = DeviceAtlas(templates, preserve_aspect, device)
    return atlas


def _rgba_hash(a: np.ndarray) -> str:
    import hashlib

    h = hashlib.sha256()
    h.update(np.asarray(a.shape, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


class CompositorPool:
    """Free compositors per structure key.  ``acquire`` returns one whose capacity
    covers the request (or builds one); ``release`` hands it back once its
    buffers are no longer referenced (the caller's saved forward state is gone).
    A leased compositor is never handed out twice, so saved contribution lists
    stay valid while their SavedForward / autograd ctx lives."""

    def __init__(self, max_keys: int = 8, per_key: int = 2):
        self.free: dict[tuple, list[Compositor]] = {}
        self.max_keys, self.per_key = max_keys, per_key

    def acquire(self, key: tuple, capacity: int, factory) -> Compositor:
        lst = self.free.get(key, [])
        for i, c in enumerate(lst):
            if c.capacity >= capacity:
                return lst.pop(i)
        return factory(capacity)

    def release(self, key: tuple, comp: Compositor) -> None:
        lst = self.free.setdefault(key, [])
        if len(lst) < self.per_key:
            lst.append(comp)
        while len(self.free) > self.max_keys:
            self.free.pop(next(iter(self.free)))


POOL = CompositorPool()
