"""Losses, Adam and the fit loop (drop-in for pkg/src/primfit/fit.py) on the CUDA path.

The hot path is ``run_loop`` (reference fit.py:403-521): every iteration is
bin -> forward(save) -> loss -> backward -> Adam -> psnr.  Here one iteration
is five stream-ordered native stages (K1..K5, include/primfit_b200.h) with no
host synchronisation: the lr schedule and Adam bias corrections are device
tables, the iteration counter and the loss/psnr history live in HBM, and the
whole step is captured once into a CUDA graph and replayed.

The small host helpers (``loss_mse``, ``psnr``, ``lr_schedule``,
``gains_vector``) keep the reference's numpy signatures for API users; inside
``run_loop`` their work is fused into the kernels (loss in K3, psnr and the
schedule lookup in K5).
"""

from __future__ import annotations

import os

import csv
import math
from collections.abc import Callable
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from . import _native as nat
from .compositor import Band, Compositor, DeviceAtlas, adam_launch, bin_capacity, pixels4
from .errors import LayoutMismatch, MissingAlphaTarget, ShapeMismatch
from .raster import DEFAULT_EPS_SKIP, _device, noisy_background
from .scene import (NOISE_BACKGROUND, FloatArray, ParamLayout, pack_params, structure_arrays,
                    unpack_params, validate_scene)

ADAM_BETA1 = 0.9
ADAM_BETA2 = 0.999
ADAM_EPS = 1e-8
GRAY_WEIGHTS = np.asarray([0.299, 0.587, 0.114])
_GAIN_GROUPS = ("x", "y", "scale", "rotation", "opacity", "color", "color", "color")


@dataclass
class FitConfig:
    """The reference FitConfig (config.py:20-99): same fields, same defaults.

    run_loop / optimize_video accept any object with these attributes,
    including the reference's own FitConfig.
    """

    num_iterations: int = 100
    sequential_iterations: int = 100
    num_primitives: int = 500
    learning_rate: float = 0.1
    lr_gain_x: float = 10.0
    lr_gain_y: float = 10.0
    lr_gain_scale: float = 10.0
    lr_gain_rotation: float = 1.0
    lr_gain_opacity: float = 1.5
    lr_gain_color: float = 1.0
    do_decay: bool = True
    decay_final_fraction: float = 0.1
    loss: str = "mse"
    mse_weight: float = 1.0
    gray_l1_weight: float = 0.0
    alpha_loss_weight: float = 0.3
    do_gaussian_blur: bool = True
    blur_sigma: float = 1.0
    radial_falloff: bool = False
    initializer: str = "structure_aware"
    variance_window_size: int = 7
    variance_base_prob: float = 0.1
    max_prims_per_pixel: int = 100
    opacity_logit_init: float = -4.0
    color_init_noise: float = 0.02
    scale_min: float = 2.0
    scale_max: float = 16.0
    alpha_max: float = 1.0
    mu_blend: float = 0.0
    bg_color: str = "white"
    preserve_aspect: bool = False
    do_reinit: bool = False
    reinit_threshold: float = 0.3
    reinit_period: int = 50
    reinit_warmup: int = 199
    tile_size: int = 32
    tile_padding: float = 2.0
    eps_skip: float = DEFAULT_EPS_SKIP
    freeze_static: bool = True
    diff_threshold: float = 2.0 / 255.0
    remove_stuck: bool = False
    stuck_grid_x: int = 4
    stuck_grid_y: int = 4
    stuck_top_k: int = 4
    stuck_tau_scale: float = 0.1
    stuck_tau_alpha: float = 0.7
    stuck_zeta: float = 0.7
    stuck_eta: float = 0.3
    stuck_triggers: tuple[int, ...] = (20, 45, 70)
    seed: int = 0
    compute_psnr: bool = True
    dump_every: int = 0
    threads: int = 0


@dataclass
class LossSpec:
    """Which loss to evaluate and against what (reference fit.py:61-76)."""

    kind: str = "mse"  # mse | spatial_constrained | combined
    target: FloatArray | None = None
    target_alpha: FloatArray | None = None
    mse_w: float = 1.0
    gray_l1_w: float = 0.0
    alpha_w: float = 0.3

    def __post_init__(self) -> None:
        if min(self.mse_w, self.gray_l1_w, self.alpha_w) < 0:
            raise ValueError("loss weights must be nonnegative")
        if self.kind == "spatial_constrained" and self.target_alpha is None:
            raise MissingAlphaTarget("spatial_constrained needs target_alpha")


@dataclass(eq=False)
class OptimState:
    """Adam moments + freeze flags (reference fit.py:79-95)."""

    m: FloatArray
    v: FloatArray
    step: int
    frozen: np.ndarray

    @classmethod
    def fresh(cls, layout: ParamLayout) -> "OptimState":
        return cls(np.zeros(layout.size), np.zeros(layout.size), 0,
                   np.zeros(layout.n_primitives, dtype=bool))


@dataclass
class HistoryEntry:
    iteration: int
    loss: float
    psnr: float
    lr: float
    reinit_count: int


def _check_image_pair(a, b) -> None:
    if a.shape != b.shape:
        raise ShapeMismatch(f"shape {a.shape} vs {b.shape}")


def loss_mse(I: FloatArray, target: FloatArray):
    """mean((I-t)^2) and its gradient 2(I-t)/size (reference fit.py:112-116)."""
    _check_image_pair(I, target)
    diff = I - target
    return float(np.mean(diff**2)), 2.0 * diff / diff.size


def loss_grayscale_l1(I: FloatArray, target: FloatArray):
    """mean |luma(I - t)| and its subgradient (reference fit.py:119-125); the device
    fit step fuses the same formula (PF_LOSS_COMBINED)."""
    _check_image_pair(I, target)
    d = (I - target) @ GRAY_WEIGHTS
    n = d.size
    grad = (np.sign(d)[:, :, None] * GRAY_WEIGHTS[None, None, :]) / n
    return float(np.mean(np.abs(d))), grad


def loss_spatial(I: FloatArray, I_alpha: FloatArray, spec: LossSpec):
    """Masked colour MSE + alpha_w * coverage MSE (reference fit.py:128-151)."""
    if spec.target_alpha is None:
        raise MissingAlphaTarget("spatial loss needs target_alpha")
    _check_image_pair(I, spec.target)
    ta = spec.target_alpha
    if ta.shape != I_alpha.shape:
        raise ShapeMismatch(f"alpha shape {ta.shape} vs {I_alpha.shape}")
    mask = (ta > 0).astype(np.float64)
    diff = (I - spec.target) * mask[:, :, None]
    color = float(np.sum(diff**2) / diff.size)
    adiff = I_alpha - ta
    alpha = float(np.mean(adiff**2))
    return color + spec.alpha_w * alpha, 2.0 * diff / diff.size, spec.alpha_w * 2.0 * adiff / adiff.size


def evaluate_loss(spec: LossSpec, I: FloatArray, I_alpha: FloatArray):
    """Dispatch on spec.kind -> (value, dL/dI, dL/dA or None) (reference fit.py:154-171)."""
    if spec.kind == "mse":
        value, dI = loss_mse(I, spec.target)
        return value, dI, None
    if spec.kind == "spatial_constrained":
        return loss_spatial(I, I_alpha, spec)
    if spec.kind == "combined":
        value_m, dI_m = loss_mse(I, spec.target)
        value_g, dI_g = loss_grayscale_l1(I, spec.target)
        return (spec.mse_w * value_m + spec.gray_l1_w * value_g,
                spec.mse_w * dI_m + spec.gray_l1_w * dI_g, None)
    raise ValueError(f"unknown loss kind {spec.kind!r}")


def lr_schedule(iteration: int, total: int, base_lr: float, decay_enabled: bool = True,
                final_fraction: float = 0.1) -> float:
    """base * final^(it/(total-1)) (reference fit.py:174-186)."""
    if not 0 <= iteration < total:
        raise ValueError(f"iteration {iteration} outside [0, {total})")
    if not decay_enabled or total <= 1:
        return base_lr
    return base_lr * final_fraction ** (iteration / (total - 1))


def gains_vector(layout: ParamLayout, gains: dict[str, float]) -> FloatArray:
    """Per-group gains expanded to one multiplier per packed scalar (fit.py:189-192)."""
    per_col = np.asarray([gains.get(g, 1.0) for g in _GAIN_GROUPS])
    return np.tile(per_col, layout.n_primitives)


def psnr(I: FloatArray, target: FloatArray) -> float:
    """10 log10(1/mse), inf when identical (reference fit.py:241-247)."""
    _check_image_pair(I, target)
    mse = float(np.mean((I - target) ** 2))
    if mse == 0.0:
        return math.inf
    return 10.0 * math.log10(1.0 / mse)


def effective_padding(cfg) -> float:
    """tile_padding + 3*blur_sigma (reference fit.py:338-341)."""
    blur = cfg.blur_sigma if cfg.do_gaussian_blur else 0.0
    return cfg.tile_padding + 3.0 * blur


def _gains8(gains) -> list[float] | None:
    if gains is None:
        return None
    g = np.asarray(gains, dtype=np.float64)
    if g.size % 8 or g.size == 0:
        raise LayoutMismatch(f"gains of size {g.size} are not 8 per primitive")
    rows = g.reshape(-1, 8)
    if not np.all(rows == rows[0]):
        raise ValueError("the fused Adam kernel takes per-column gains (as gains_vector builds)")
    return rows[0].tolist()


def adam_step(params: FloatArray, grads: FloatArray, state: OptimState, lr: float,
              gains: FloatArray | None = None, frozen: np.ndarray | None = None,
              s_min: float | None = None, s_max: float | None = None,
              layout: ParamLayout | None = None) -> FloatArray:
    """One Adam update on the GPU (K5, scalar mode); mutates state like fit.py:195-238."""
    params = np.asarray(params, dtype=np.float64)
    grads = np.asarray(grads, dtype=np.float64)
    if params.shape != grads.shape or params.shape != state.m.shape:
        raise LayoutMismatch(
            f"params {params.shape}, grads {grads.shape}, moments {state.m.shape} must agree")
    if layout is None:
        layout = ParamLayout(params.size // 8)
    if frozen is None:
        frozen = state.frozen
    dev = _device()
    n = layout.n_primitives
    state.step += 1
    t = state.step
    d_p = torch.from_numpy(params.copy()).to(dev)
    d_g = torch.from_numpy(grads.copy()).to(dev)
    d_m = torch.from_numpy(np.ascontiguousarray(state.m, dtype=np.float64)).to(dev)
    d_v = torch.from_numpy(np.ascontiguousarray(state.v, dtype=np.float64)).to(dev)
    d_f = torch.from_numpy(np.asarray(frozen, dtype=bool).astype(np.uint8)).to(dev)
    clamp = s_min is not None and s_max is not None
    adam_launch(d_p, d_g, d_m, d_v, frozen=d_f, gains=_gains8(gains), n=n, lr=lr,
                bc1=1 - ADAM_BETA1**t, bc2=1 - ADAM_BETA2**t, clamp=clamp,
                s_min=s_min if clamp else 0.0, s_max=s_max if clamp else 0.0, zero_grads=False)
    state.m[:] = d_m.cpu().numpy()
    state.v[:] = d_v.cpu().numpy()
    return d_p.cpu().numpy()


def _cfg_gains(cfg) -> list[float]:
    g = {"x": cfg.lr_gain_x, "y": cfg.lr_gain_y, "scale": cfg.lr_gain_scale,
         "rotation": cfg.lr_gain_rotation, "opacity": cfg.lr_gain_opacity,
         "color": cfg.lr_gain_color}
    return [float(g[k]) for k in _GAIN_GROUPS]


class StepEngine:
    """Device-resident optimisation loop: K1..K5 per step, CUDA-graph replayed.

    ``band`` restricts the render to a row band of tiles (multi-GPU); then
    ``allreduce`` (a callable on the float64 gradient+loss buffer) runs between
    the backward and the Adam step.
    """

    def __init__(self, scene, cfg, loss_spec: LossSpec, total: int, state: OptimState | None = None,
                 *, band: Band | None = None, allreduce: Callable | None = None,
                 use_graph: bool = True, device=None, host_io: bool = False):
        if loss_spec.kind not in ("mse", "spatial_constrained", "combined"):
            raise ValueError(f"unknown loss kind {loss_spec.kind!r}")
        validate_scene(scene)
        self.dev = device or _device()
        self.scene = scene
        self.cfg = cfg
        self.total = int(total)
        H, W = scene.canvas_h, scene.canvas_w
        self.H, self.W, self.P = H, W, H * W
        target = np.asarray(loss_spec.target, dtype=np.float64)
        if target.shape != (H, W, 3):
            raise ShapeMismatch(f"target shape {target.shape} != {(H, W, 3)}")
        self.loss_kind = {"mse": nat.PF_LOSS_MSE, "spatial_constrained": nat.PF_LOSS_SPATIAL,
                          "combined": nat.PF_LOSS_COMBINED}[loss_spec.kind]
        self.alpha_w = float(loss_spec.alpha_w)
        self.w_mse = float(getattr(loss_spec, "mse_w", 1.0))
        self.w_gray = float(getattr(loss_spec, "gray_l1_w", 0.0))
        vec, layout = pack_params(scene)
        self.layout = layout
        self.n = n = layout.n_primitives
        self.state = state if state is not None else OptimState.fresh(layout)
        self.step0 = int(self.state.step)
        dev = self.dev
        # parameters and the latest step's loss sums share one buffer, so a
        # host-driven step reads both back with a single copy
        self.adam_blocks = int(nat.load().pf_adam_blocks(n))
        # host_io: the buffer lives in pinned host memory and the kernels read the
        # parameters / write the updated ones and the loss partials through it
        # directly (zero-copy over the host link): a host-driven step needs no
        # copy nodes (see capture_host_io_step)
        # (host_io: two loss-partial slots, alternating between host steps, so a
        # step's loss can be read while the next step runs; the parameters stay
        # on the device and io[:8n] is their host mirror, written by every Adam
        # launch and read back -- changed primitives only -- by the next step)
        self.host_io = bool(host_io)
        nb3 = self.adam_blocks * 3
        if self.host_io:
            self.io = torch.zeros(n * 8 + 2 * nb3, dtype=torch.float64).pin_memory()
            self.io[: n * 8].copy_(torch.from_numpy(vec))
            self.params = torch.from_numpy(vec.reshape(n, 8).copy()).to(dev)
            self.host_params = self.io[: n * 8]
        else:
            self.io = torch.zeros(n * 8 + nb3, dtype=torch.float64, device=dev)
            self.params = self.io[: n * 8].view(n, 8)
            self.params.copy_(torch.from_numpy(vec.reshape(n, 8).copy()))
            self.host_params = None
        self.last_part = self.io[n * 8 : n * 8 + nb3]
        self.loss_slots = [self.last_part] + ([self.io[n * 8 + nb3 :]] if self.host_io else [])
        self.m = torch.from_numpy(np.asarray(self.state.m, dtype=np.float64).copy()).to(dev)
        self.v = torch.from_numpy(np.asarray(self.state.v, dtype=np.float64).copy()).to(dev)
        self.frozen = torch.from_numpy(np.asarray(self.state.frozen, dtype=bool).astype(np.uint8)).to(dev)
        self.gains = _cfg_gains(cfg)
        its = range(self.total)
        self.lr_host = [lr_schedule(i, self.total, cfg.learning_rate, cfg.do_decay,
                                    cfg.decay_final_fraction) for i in its]
        bc1 = [1 - ADAM_BETA1 ** (self.step0 + i + 1) for i in its]
        bc2 = [1 - ADAM_BETA2 ** (self.step0 + i + 1) for i in its]
        self.lr_table = torch.tensor(self.lr_host, dtype=torch.float64, device=dev)
        self.bc1_table = torch.tensor(bc1, dtype=torch.float64, device=dev)
        self.bc2_table = torch.tensor(bc2, dtype=torch.float64, device=dev)
        self.gbuf = torch.zeros(n * 8 + 4, dtype=torch.float64, device=dev)
        self.grads = self.gbuf[: n * 8]
        self.sums = self.gbuf[n * 8 :]
        ta = loss_spec.target_alpha if self.loss_kind == nat.PF_LOSS_SPATIAL else None
        # (target rgb, target alpha) per pixel, one 16-byte load in K3
        self.tgt4 = torch.from_numpy(pixels4(target, ta)).to(dev)
        self.noise_bg = isinstance(scene.background, str) and scene.background == NOISE_BACKGROUND
        self.bg_rgb = (0.0, 0.0, 0.0) if self.noise_bg else tuple(
            float(c) for c in np.asarray(scene.background, dtype=np.float64))
        self.bg4 = torch.zeros(self.P * 4, dtype=torch.float32, device=dev) if self.noise_bg else None
        tid, z = structure_arrays(scene)
        self.padding = effective_padding(cfg)
        self.atlas = DeviceAtlas(scene.templates, bool(scene.preserve_aspect), dev)
        band = band or Band(0, -(-H // 16))
        scales = np.maximum(vec.reshape(n, 8)[:, 2], float(cfg.scale_max)) if n else np.zeros(0)
        cap = bin_capacity(scales, tid, self.atlas.hyp, self.padding, 16, -(-W // 16),
                           band.ty_end - band.ty_begin)
        self.comp = Compositor(tid, z, self.atlas, W, H, alpha_max=scene.alpha_max,
                               mu_blend=scene.mu_blend, padding=self.padding, capacity=cap,
                               band=band, device=dev)
        # K34 stage depth from the FULL canvas's capacity bound, so every row band
        # of a multi-GPU split runs the same kernel configuration (same numerics)
        nty_full = -(-H // 16)
        full_cap = cap if (band.ty_begin, band.ty_end) == (0, nty_full) else bin_capacity(
            scales, tid, self.atlas.hyp, self.padding, 16, -(-W // 16), nty_full)
        self.comp.stage_hint = 64 if full_cap > 48 * (-(-W // 16)) * nty_full else 32
        # K34 (one kernel for render -> loss -> backward) whenever colour does not
        # come from the texture; PF_TWO_KERNEL=1 forces K3 + K4 (A/B checks)
        self.fused = scene.mu_blend == 0.0 and os.environ.get("PF_TWO_KERNEL", "0") != "1"
        if self.fused:
            # slot binning: K1 scatters the tile lists, K34 sorts them (no K2);
            # PF_CSR_STEP=1 keeps pf_bin's CSR lists (A/B), PF_SLOT_M overrides the
            # slots per tile (tests force the overflow path with a small value)
            slot_m = 0
            if os.environ.get("PF_CSR_STEP", "0") != "1":
                slot_m = int(os.environ.get("PF_SLOT_M", "0")) or slot_count(
                    vec.reshape(n, 8), tid, self.atlas.hyp, self.padding, W, H, band)
            self.comp.enable_step_schedule(slot_m)
        else:
            self.comp.alloc_render(save=True, loss=True)
        # per-iteration loss sums per Adam block (history; folded in order on the host)
        assert self.adam_blocks == self.comp.adam_blocks
        self.hist_part = torch.zeros(max(self.total, 1) * self.adam_blocks * 3, dtype=torch.float64,
                                     device=dev)
        self.allreduce = allreduce
        self.use_graph = use_graph
        self.graph: torch.cuda.CUDAGraph | None = None
        self.eps_skip = float(cfg.eps_skip)
        self.done = 0
        self.kernels_per_step: int | None = None

    # one full optimisation step, stream-ordered, no host sync:
    #   [K2 bin] -> [K3 forward + loss] -> [K4 backward]
    #   -> (allreduce) -> [K5+K1 Adam + next step's records/offsets]
    # (the very first step is preceded by a stand-alone K1, see step()).
    def launch_step(self, mark: Callable[[str], None] | None = None,
                    records: bool = True) -> None:
        mark = mark or (lambda name: None)
        self.launch_render(mark)
        if self.allreduce is not None:
            self.allreduce(self.gbuf)
            mark("allreduce")
        self.launch_update(mark, records)

    # The step's two halves around the cross-rank exchange: launch_render fills
    # gbuf (this band's gradients + loss sums), launch_update applies Adam and
    # builds the next records.  A caller that drives several band engines with
    # its own reduction between the halves (tests/test_gpu_multirank.py) calls
    # them directly; ``reduced`` says the gradients will be summed across bands
    # before launch_update (the loss partials are then folded into gbuf's sums).
    def launch_render(self, mark: Callable[[str], None] | None = None,
                      reduced: bool | None = None) -> None:
        c = self.comp
        mark = mark or (lambda name: None)
        if reduced is None:
            reduced = self.allreduce is not None
        self._reduced = bool(reduced)
        c.bin()
        mark("bin")
        fold_in_adam = self.fused and not reduced
        if self.fused:
            # one rank: the loss partials are folded inside the Adam launch; with an
            # allreduce they are folded first so the sums travel with the grads
            c.fit_step(self.gbuf, None if fold_in_adam else self.sums, eps_skip=self.eps_skip,
                       bg_rgb=self.bg_rgb, bg4=self.bg4, loss_kind=self.loss_kind,
                       tgt4=self.tgt4, alpha_w=self.alpha_w, w_mse=self.w_mse,
                       w_gray=self.w_gray, P_total=self.P)
            mark("step")
        else:
            c.forward(save=True, eps_skip=self.eps_skip, bg_rgb=self.bg_rgb, bg4=self.bg4,
                      loss_kind=self.loss_kind, tgt4=self.tgt4, alpha_w=self.alpha_w,
                      w_mse=self.w_mse, w_gray=self.w_gray, P_total=self.P)
            mark("forward")
            c.backward(c.d4, self.gbuf, bg_rgb=self.bg_rgb, bg4=self.bg4, sums=self.sums)
            mark("backward")

    def launch_update(self, mark: Callable[[str], None] | None = None,
                      records: bool = True) -> None:
        c = self.comp
        mark = mark or (lambda name: None)
        fold_in_adam = self.fused and not getattr(self, "_reduced", self.allreduce is not None)
        c.adam_preprocess(self.params, self.grads, self.m, self.v, frozen=self.frozen,
                          gains=self.gains, lr_table=self.lr_table, bc1_table=self.bc1_table,
                          bc2_table=self.bc2_table, s_min=self.cfg.scale_min,
                          s_max=self.cfg.scale_max, sums=None if fold_in_adam else self.sums,
                          part=c.part if fold_in_adam else None, hist_part=self.hist_part,
                          last_part=self.last_part, records=records,
                          mirror=self.host_params)
        mark("adam_preprocess")

    def refresh(self) -> None:
        """Rebuild records / offsets from the current params (after host edits)."""
        self.comp.preprocess(self.params)

    def capture(self) -> None:
        g = torch.cuda.CUDAGraph()
        before = self.comp.launches
        with torch.cuda.graph(g):
            self.launch_step()
        self.kernels_per_step = self.comp.launches - before  # this package's kernels only
        self.graph = g

    def capture_host_step(self, h_in: torch.Tensor, h_out: torch.Tensor) -> None:
        """One CUDA graph for a step driven through HOST buffers: H2D of the packed
        parameter vector (pinned ``h_in``, 8n doubles), preprocess, bin, fit step,
        Adam, and ONE D2H of the updated vector followed by the step's loss sums
        (pinned ``h_out``, 8n + 3 * adam_blocks doubles).  Replay with host_step()."""
        if self.graph is None and self.done == 0:
            raise RuntimeError("run one step() first (eager warm-up + capture)")
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.params.view(-1).copy_(h_in, non_blocking=True)
            self.refresh()
            self.launch_step()
            h_out.copy_(self.io, non_blocking=True)
        self.host_graph = g

    def capture_host_io_step(self) -> None:
        """host_io engines: one CUDA graph = preprocess from the host parameter
        vector (incremental: changed primitives only), bin, fit step, Adam (+ the
        next records) writing the updated vector and the loss partials back to
        host memory.  The caller reads / edits the parameters between host_step()
        replays through host_vector() (which first waits for the step in flight:
        the kernels write and read that memory)."""
        if not self.host_io:
            raise RuntimeError("capture_host_io_step needs StepEngine(host_io=True)")
        if self.graph is None and self.done == 0:
            raise RuntimeError("run one step() first (eager warm-up + capture)")
        graphs = []
        keep = self.last_part
        for slot in self.loss_slots:  # one graph per loss slot
            self.last_part = slot
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                # H2D: the host vector, read in place; primitives the host edited
                # since the last Adam launch get new records (pf_preprocess_sync)
                self.comp.preprocess_sync(self.params, self.host_params)
                self.launch_step()
            graphs.append(g)
        self.last_part = keep
        self.host_graphs = graphs
        self.host_graph = graphs[0]
        self.host_events = [torch.cuda.Event() for _ in graphs]
        self.host_issued = []  # (iteration, slot) of the host steps in flight / done

    def host_step(self, rng: np.random.Generator | None = None) -> None:
        """Enqueue one host-driven step (asynchronous).  host_io engines alternate
        two graphs / loss slots; read a step's loss with host_loss_part(), at most
        one step behind the newest.  A noise-background scene draws this step's
        background from ``rng`` (stream-ordered upload, as step())."""
        if self.done >= self.total:
            raise ValueError(f"iteration {self.done} outside [0, {self.total})")
        if self.noise_bg:
            if rng is None:
                raise ValueError("noise background needs the caller's rng")
            bg = pixels4(noisy_background(self.W, self.H, rng))
            self.bg4.copy_(torch.from_numpy(bg), non_blocking=False)
        if self.host_io and getattr(self, "host_graphs", None):
            slot = len(self.host_issued) % len(self.host_graphs)
            self.host_graphs[slot].replay()
            self.host_events[slot].record()
            self.host_issued.append((self.done, slot))
        else:
            self.host_graph.replay()
        self.done += 1

    def host_vector(self) -> np.ndarray:
        """The pinned host parameter vector (8n doubles, primitive-major) for
        reading or editing between host steps.  Every Adam launch writes it (the
        mirror) and the next step reads it in place, so it may only be touched
        while no host step is in flight: this waits for the newest one first.
        Edits are picked up by the next host_step (changed primitives only)."""
        if not self.host_io:
            raise RuntimeError("host_vector needs StepEngine(host_io=True)")
        if getattr(self, "host_issued", None):
            self.host_events[self.host_issued[-1][1]].synchronize()
        return self.io.numpy()[: self.n * 8]

    def host_loss_part(self, k: int = -1) -> np.ndarray:
        """Loss partials [adam_blocks][3] of host step k (default: the newest),
        after waiting for that step; valid for the two newest host steps."""
        it, slot = self.host_issued[k]
        if len(self.host_issued) - (k % len(self.host_issued)) > len(self.host_graphs):
            raise ValueError(f"host step {k} has been overwritten")
        self.host_events[slot].synchronize()
        return self.loss_slots[slot].numpy().reshape(-1, 3)

    def step(self, rng: np.random.Generator | None = None,
             background: np.ndarray | None = None) -> None:
        """One step; a noise-background scene draws this step's background from
        ``rng`` (or takes the already drawn ``background``, (H, W, 3))."""
        if self.done >= self.total:
            raise ValueError(f"iteration {self.done} outside [0, {self.total})")
        if self.noise_bg:
            if background is None:
                if rng is None:
                    raise ValueError("noise background needs the caller's rng")
                background = noisy_background(self.W, self.H, rng)
            self.bg4.copy_(torch.from_numpy(pixels4(background)), non_blocking=False)
        if self.graph is not None:
            self.graph.replay()
        else:
            if self.done == 0:
                self.refresh()
            self.launch_step()
            if self.use_graph:
                self.capture()  # step 0 ran eagerly (warm-up); later steps replay
        self.done += 1

    # steps per multi-step graph (run()): consecutive steps chained by
    # programmatic (PDL) edges instead of one graph launch per step
    CHUNK = 8

    def capture_chunk(self) -> None:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(self.CHUNK):
                self.launch_step()
        self.chunk_graph = g

    def run(self, k: int, rng=None) -> None:
        """k steps.  Without a per-step host input (noise background) the steps go
        out as CHUNK-step graph replays once the single-step graph exists; the
        device iteration counter indexes the lr / bias-correction tables, so the
        result is identical to k single steps (test_chunked_run_equals_steps)."""
        # (with an allreduce every step of the chunk graph carries its own captured
        # collective: ranks replay the same chunks in lockstep)
        chunked = self.use_graph and not self.noise_bg
        while k > 0:
            if chunked and self.graph is not None and k >= self.CHUNK and \
                    self.done + self.CHUNK <= self.total:
                if getattr(self, "chunk_graph", None) is None:
                    self.capture_chunk()
                self.chunk_graph.replay()
                self.done += self.CHUNK
                k -= self.CHUNK
            else:
                self.step(rng)
                k -= 1

    # host views (synchronising)
    def check(self) -> None:
        self.comp.check_overflow()

    def params_host(self) -> np.ndarray:
        return self.params.cpu().numpy().reshape(-1)

    def sync_state(self) -> OptimState:
        self.state.m[:] = self.m.cpu().numpy()
        self.state.v[:] = self.v.cpu().numpy()
        self.state.step = self.step0 + self.done
        return self.state

    def push_host(self, vec: np.ndarray, state: OptimState) -> None:
        """Re-upload params/moments/frozen in place (graph pointers stay valid)."""
        self.params.copy_(torch.from_numpy(np.asarray(vec, dtype=np.float64).reshape(self.n, 8)))
        if self.host_params is not None:
            self.host_params.copy_(self.params.view(-1).cpu())
        self.m.copy_(torch.from_numpy(np.asarray(state.m, dtype=np.float64)))
        self.v.copy_(torch.from_numpy(np.asarray(state.v, dtype=np.float64)))
        self.frozen.copy_(torch.from_numpy(np.asarray(state.frozen, dtype=bool).astype(np.uint8)))
        self.refresh()

    def loss_psnr(self, sums: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
        """History values from per-iteration loss sums [k][3] (fit.py:112-151, 241-247)."""
        inv_3P, inv_P = 1.0 / (3.0 * self.P), 1.0 / self.P
        mse = sums[:, 0] * inv_3P
        if self.loss_kind == nat.PF_LOSS_SPATIAL:
            loss = sums[:, 1] * inv_3P + self.alpha_w * (sums[:, 2] * inv_P)
        elif self.loss_kind == nat.PF_LOSS_COMBINED:
            loss = self.w_mse * mse + self.w_gray * (sums[:, 1] * inv_P)
        else:
            loss = mse
        with np.errstate(divide="ignore"):
            ps = np.where(mse == 0.0, np.inf, 10.0 * np.log10(1.0 / np.where(mse == 0.0, 1.0, mse)))
        return loss, ps

    def iteration_sums(self, part: np.ndarray) -> np.ndarray:
        """Fixed-order fold of hist_part blocks: [k][blocks][3] -> [k][3]."""
        part = part.reshape(-1, self.adam_blocks, 3)
        out = np.zeros((part.shape[0], 3), dtype=np.float64)
        for b in range(self.adam_blocks):
            out += part[:, b, :]
        return out

    def history(self, compute_psnr: bool = True) -> list[HistoryEntry]:
        k = self.done
        part = self.hist_part[: k * self.adam_blocks * 3].cpu().numpy()
        loss, ps = self.loss_psnr(self.iteration_sums(part))
        return [HistoryEntry(i, float(loss[i]), float(ps[i]) if compute_psnr else math.nan,
                             self.lr_host[i], 0) for i in range(k)]


def slot_count(params: np.ndarray, tids: np.ndarray, hyp: np.ndarray, padding: float, W: int,
               H: int, band: Band) -> int:
    """Slots per tile for slot binning: twice the longest tile list of the
    initial state (bbox as bin_tiles, raster.py:246-257), a power of two in
    [64, 1024].  Only a size: longer lists later take the overflow path."""
    n = len(params)
    if n == 0:
        return 64
    ntx, nty = -(-W // 16), -(-H // 16)
    x, y, s = params[:, 0], params[:, 1], params[:, 2]
    r = s * hyp[tids] + padding
    with np.errstate(invalid="ignore"):
        lo_x = np.maximum(np.ceil(x - r), 0.0)
        hi_x = np.minimum(np.floor(x + r), W - 1.0)
        lo_y = np.maximum(np.ceil(y - r), 0.0)
        hi_y = np.minimum(np.floor(y + r), H - 1.0)
        ok = (lo_x <= hi_x) & (lo_y <= hi_y)
    tx0, tx1 = (lo_x[ok] // 16).astype(np.int64), (hi_x[ok] // 16).astype(np.int64)
    ty0 = np.maximum((lo_y[ok] // 16).astype(np.int64), band.ty_begin)
    ty1 = np.minimum((hi_y[ok] // 16).astype(np.int64), band.ty_end - 1)
    keep = ty0 <= ty1
    diff = np.zeros((nty + 1, ntx + 1), dtype=np.int64)
    np.add.at(diff, (ty0[keep], tx0[keep]), 1)
    np.add.at(diff, (ty0[keep], tx1[keep] + 1), -1)
    np.add.at(diff, (ty1[keep] + 1, tx0[keep]), -1)
    np.add.at(diff, (ty1[keep] + 1, tx1[keep] + 1), 1)
    cnt = diff.cumsum(0).cumsum(1)[:nty, :ntx]
    mx = int(cnt.max()) if cnt.size else 0
    return int(min(1024, max(64, 1 << max(0, 2 * mx - 1).bit_length())))


def should_reinit(iteration: int, total: int, period: int, warmup: int) -> bool:
    """Period boundary, past warmup, a full period still to run (fit.py:250-258)."""
    return iteration % period == 0 and iteration > warmup and iteration + period <= total


def reinit_low_opacity(scene, target, threshold: float = 0.3,
                       rng: np.random.Generator | None = None, state: OptimState | None = None,
                       *, s_min: float = 2.0, s_max: float = 16.0, v_init_bias: float = -4.0,
                       sigma_c: float = 0.02, density_cap: int = 100, base_prob: float = 0.1,
                       window: int = 7, nlv=None, frozen: np.ndarray | None = None):
    """Re-seed every non-frozen primitive whose opacity fell below ``threshold``
    with the structure-aware law, keeping depth and template; zero their Adam
    moments (fit.py:261-335).  Host-side: a few draws from the caller's rng at a
    period boundary of the fit loop, in the reference's draw order."""
    import dataclasses

    from scipy.special import expit

    from .prep import color_logits_near, local_variance_map, sample_cells

    if not 0.0 < threshold < 1.0:
        raise ValueError(f"threshold {threshold} outside (0, 1)")
    rng = rng or np.random.default_rng()
    idx = [i for i, p in enumerate(scene.primitives)
           if expit(p.opacity_logit) < threshold and (frozen is None or not frozen[i])]
    if not idx:
        return scene, 0
    target = np.asarray(target, dtype=np.float64)
    h, w = target.shape[:2]
    if nlv is None:
        nlv = local_variance_map(target, window)
    k = len(idx)
    chosen = sample_cells(nlv.nlv, k, base_prob, density_cap, rng)
    scales = s_max - (s_max - s_min) * nlv.nlv.reshape(-1)[chosen]
    thetas = rng.uniform(0.0, 2.0 * np.pi, k)
    cl = color_logits_near(target[chosen // w, chosen % w, :], sigma_c, rng)
    prims = list(scene.primitives)
    for j, i in enumerate(idx):
        prims[i] = dataclasses.replace(
            prims[i], x=float(chosen[j] % w), y=float(chosen[j] // w), scale=float(scales[j]),
            rotation=float(thetas[j]), opacity_logit=v_init_bias,
            color_logits=(float(cl[j, 0]), float(cl[j, 1]), float(cl[j, 2])))
    if state is not None:
        for i in idx:
            state.m[8 * i : 8 * i + 8] = 0.0
            state.v[8 * i : 8 * i + 8] = 0.0
    return dataclasses.replace(scene, primitives=prims), k


def run_loop(scene, cfg, loss_spec: LossSpec, rng: np.random.Generator,
             iterations: int | None = None, state: OptimState | None = None, nlv=None,
             log_path: str | Path | None = None, dump_dir: str | Path | None = None,
             hooks: dict[int, Callable] | None = None):
    """GPU fit loop with the reference's contract (fit.py:403-521).

    The steps between host events run as CUDA-graph replays with no host sync.
    Host events are the iterations where the reference touches the scene on the
    host: a hook (before that iteration's render), a low-opacity reinit
    (``cfg.do_reinit`` at should_reinit boundaries, drawing from ``rng`` before
    the iteration's noise background, as the reference), and an image dump
    (``dump_dir`` with ``cfg.dump_every``: the iteration's pre-update render).
    Returns (scene after the last update, history, state); history entries
    describe the render before each update and carry the reinit counts.
    """
    total = cfg.num_iterations if iterations is None else iterations
    vec, layout = pack_params(scene)
    if state is None:
        state = OptimState.fresh(layout)
    eng = StepEngine(scene, cfg, loss_spec, total, state)
    g = lambda k, d: getattr(cfg, k, d)  # noqa: E731  (duck-typed FitConfig)
    reinit = bool(g("do_reinit", False))
    period, warmup = int(g("reinit_period", 50)), int(g("reinit_warmup", 199))
    dump_every = int(g("dump_every", 0)) if dump_dir is not None else 0
    if dump_every > 0:
        Path(dump_dir).mkdir(parents=True, exist_ok=True)
    events = set(hooks or ())
    if reinit:
        events |= {it for it in range(total) if should_reinit(it, total, period, warmup)}
    if dump_every > 0:
        events |= set(range(0, total, dump_every))
    reinit_counts = [0] * total
    it = 0
    while it < total:
        if it in events:
            if hooks and it in hooks:
                cur = unpack_params(eng.params_host(), layout, scene)
                st = eng.sync_state()
                cur = hooks[it](cur, st)
                vec2, layout2 = pack_params(cur)
                if layout2 != layout:
                    raise LayoutMismatch("hooks must keep the primitive count")
                scene = cur
                eng.push_host(vec2, st)
            if reinit and should_reinit(it, total, period, warmup):
                if nlv is None:
                    from .prep import local_variance_map

                    nlv = local_variance_map(loss_spec.target, int(g("variance_window_size", 7)))
                cur = unpack_params(eng.params_host(), layout, scene)
                st = eng.sync_state()
                cur, count = reinit_low_opacity(
                    cur, loss_spec.target, float(g("reinit_threshold", 0.3)), rng, st,
                    s_min=cfg.scale_min, s_max=cfg.scale_max,
                    v_init_bias=float(g("opacity_logit_init", -4.0)),
                    sigma_c=float(g("color_init_noise", 0.02)),
                    density_cap=int(g("max_prims_per_pixel", 100)),
                    base_prob=float(g("variance_base_prob", 0.1)),
                    window=int(g("variance_window_size", 7)), nlv=nlv, frozen=st.frozen)
                reinit_counts[it] = count
                if count:
                    scene = cur
                    eng.push_host(pack_params(cur)[0], st)
            bg = None
            if dump_every > 0 and it % dump_every == 0:
                from .export import save_image
                from .raster import render_forward

                cur = unpack_params(eng.params_host(), layout, scene)
                if eng.noise_bg:
                    bg = noisy_background(eng.W, eng.H, rng)
                out, _ = render_forward(cur, background=bg, eps_skip=eng.eps_skip)
                save_image(Path(dump_dir) / f"iter_{it:05d}.png", out.color)
            eng.step(rng, background=bg)
            it += 1
            continue
        later = [k for k in events if k > it]
        nxt = min(later) if later else total
        eng.run(nxt - it, rng)
        it = nxt
    eng.check()
    state = eng.sync_state()
    history = eng.history(getattr(cfg, "compute_psnr", True))
    for h in history:
        h.reinit_count = reinit_counts[h.iteration]
    if log_path is not None:
        with open(log_path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["iter", "loss", "psnr", "lr", "reinit_count"])
            for h in history:
                w.writerow([h.iteration, repr(h.loss), str(h.psnr), repr(h.lr), h.reinit_count])
    return unpack_params(eng.params_host(), layout, scene), history, state


def loss_spec_from_config(cfg, target: FloatArray, target_alpha: FloatArray | None) -> LossSpec:
    """The config's loss (fit.py:344-355): ``loss`` "spatial" is the spatial
    constraint, weights from mse_weight / gray_l1_weight / alpha_loss_weight."""
    kind = {"spatial": "spatial_constrained"}.get(cfg.loss, cfg.loss)
    return LossSpec(kind=kind, target=target, target_alpha=target_alpha, mse_w=cfg.mse_weight,
                    gray_l1_w=cfg.gray_l1_weight, alpha_w=cfg.alpha_loss_weight)


def optimize(target, templates, cfg, target_alpha=None, log_path=None, dump_dir=None):
    """Fit a fresh scene to one image (fit.py:524-555): the config's rng seed,
    prepare_templates (blur / falloff) on the given or default templates,
    init_scene, the config's loss, the target's local variance map for reinit,
    then the GPU run_loop.  Returns (scene, history)."""
    from .prep import default_templates, init_scene, local_variance_map, prepare_templates

    target = np.asarray(target, dtype=np.float64)
    if target.ndim != 3 or target.shape[2] != 3:
        raise ShapeMismatch(f"target shape {target.shape} is not (H, W, 3)")
    rng = np.random.default_rng(cfg.seed)
    tpls = prepare_templates(list(templates) if templates else default_templates(),
                             blur_sigma=cfg.blur_sigma, do_blur=cfg.do_gaussian_blur,
                             falloff=cfg.radial_falloff)
    scene = init_scene(target, tpls, cfg, rng)
    spec = loss_spec_from_config(cfg, target, target_alpha)
    nlv = local_variance_map(target, cfg.variance_window_size)
    scene, history, _ = run_loop(scene, cfg, spec, rng, nlv=nlv, log_path=log_path,
                                 dump_dir=dump_dir)
    return scene, history
