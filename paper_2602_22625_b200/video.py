"""Video-fit heuristics on the GPU.

Mirrors the reference's dyn (pkg/src/primfit/dyn.py:86-177): ``diff_mask``
(changed pixels between two frames), ``freeze_flags`` (primitives whose binning
box misses every change; their parameters and moments stay put in the device
Adam) and ``remove_stuck`` (per grid region, decay the opacity logit of the
top-k large, opaque, front-most primitives).  Kernels: ``pf_diff_mask``,
``pf_freeze_flags``, ``pf_remove_stuck``.  There is no CPU path.
"""

from __future__ import annotations

import dataclasses
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .compositor import _stream_handle
from .errors import ShapeMismatch
from .raster import _device
from .scene import param_matrix, structure_arrays

DEFAULT_DIFF_THRESHOLD = 2.0 / 255.0  # dyn.py:34


@dataclass
class DiffMask:
    """Boolean canvas: true where two frames disagree (dyn.py:37-41)."""

    mask: np.ndarray  # (H, W) bool


@dataclass
class StuckPolicy:
    """Knobs of remove_stuck (dyn.py:44-72), same validation."""

    grid: tuple[int, int] = (4, 4)
    k: int = 4
    tau_scale: float = 0.1
    tau_alpha: float = 0.7
    zeta: float = 0.7
    eta: float = 0.3
    triggers: tuple[int, ...] = (20, 45, 70)

    def __post_init__(self) -> None:
        if self.grid[0] < 1 or self.grid[1] < 1:
            raise ValueError(f"grid {self.grid} must be at least 1x1")
        if self.k < 0:
            raise ValueError(f"k {self.k} must be nonnegative")
        if not 0.0 < self.eta < 1.0:
            raise ValueError(f"eta {self.eta} outside (0, 1)")
        if not 0.0 < self.zeta < 1.0:
            raise ValueError(f"zeta {self.zeta} outside (0, 1)")


def _hyp_table(scene) -> np.ndarray:
    """hypot(1, max(1, aspect)) per template, as bbox_half_side (raster.py:222-224)."""
    out = []
    for t in scene.templates:
        h, w = np.asarray(t.rgba).shape[:2]
        q = h / w if scene.preserve_aspect else 1.0
        out.append(math.hypot(1.0, max(1.0, float(q))))
    return np.asarray(out, dtype=np.float64)


def diff_mask(prev, cur, tau_d: float = DEFAULT_DIFF_THRESHOLD) -> DiffMask:
    """True wherever any channel moved by more than tau_d (dyn.py:86-97)."""
    prev = np.asarray(prev, dtype=np.float64)
    cur = np.asarray(cur, dtype=np.float64)
    if prev.shape != cur.shape:
        raise ShapeMismatch(f"frame shapes {prev.shape} vs {cur.shape}")
    H, W = prev.shape[:2]
    dev = _device()
    a = torch.from_numpy(np.ascontiguousarray(prev)).to(dev)
    b = torch.from_numpy(np.ascontiguousarray(cur)).to(dev)
    m = torch.empty(H * W, dtype=torch.uint8, device=dev)
    nat.check(nat.load().pf_diff_mask(a.data_ptr(), b.data_ptr(), W, H, float(tau_d),
                                      m.data_ptr(), _stream_handle()), "pf_diff_mask")
    return DiffMask(m.cpu().numpy().reshape(H, W).astype(bool))


def freeze_flags(scene, mask: DiffMask, padding: float = 2.0) -> np.ndarray:
    """Per-primitive: frozen iff the binning box misses every change (dyn.py:100-130)."""
    m = np.asarray(mask.mask)
    if m.shape != (scene.canvas_h, scene.canvas_w):
        raise ShapeMismatch(f"mask {m.shape} vs canvas ({scene.canvas_h}, {scene.canvas_w})")
    n = len(scene.primitives)
    if n == 0:
        return np.zeros(0, dtype=bool)
    dev = _device()
    pm = torch.from_numpy(np.ascontiguousarray(param_matrix(scene), dtype=np.float64)).to(dev)
    tid, _ = structure_arrays(scene)
    d_tid = torch.from_numpy(np.ascontiguousarray(tid, dtype=np.int32)).to(dev)
    hyp = torch.from_numpy(_hyp_table(scene)).to(dev)
    d_m = torch.from_numpy(np.ascontiguousarray(m, dtype=np.uint8).reshape(-1)).to(dev)
    out = torch.empty(n, dtype=torch.uint8, device=dev)
    nat.check(nat.load().pf_freeze_flags(pm.data_ptr(), d_tid.data_ptr(), hyp.data_ptr(), n,
                                         scene.canvas_w, scene.canvas_h, float(padding),
                                         d_m.data_ptr(), out.data_ptr(), _stream_handle()),
              "pf_freeze_flags")
    return out.cpu().numpy().astype(bool)


def remove_stuck(scene, frozen: np.ndarray | None, policy: StuckPolicy):
    """Decay the opacity logit of dominant primitives per grid region (dyn.py:133-177).
    Returns (scene with decayed logits, sorted decayed indices)."""
    n = len(scene.primitives)
    if n == 0:
        return scene, []
    dev = _device()
    lib = nat.load()
    pm = torch.from_numpy(np.ascontiguousarray(param_matrix(scene), dtype=np.float64)).to(dev)
    z = torch.from_numpy(np.asarray([p.z for p in scene.primitives], dtype=np.int32)).to(dev)
    fr = None
    if frozen is not None:
        fr = torch.from_numpy(np.asarray(frozen, dtype=bool).astype(np.uint8)).to(dev)
    rows, cols = policy.grid
    nbytes = int(lib.pf_stuck_scratch_bytes(n, rows * cols))
    scratch = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    dec = torch.empty(n, dtype=torch.uint8, device=dev)
    nat.check(lib.pf_remove_stuck(pm.data_ptr(), z.data_ptr(), nat.ptr(fr), n, scene.canvas_w,
                                  scene.canvas_h, int(rows), int(cols), int(policy.k),
                                  float(policy.tau_scale), float(policy.tau_alpha),
                                  float(policy.zeta), float(policy.eta), float(scene.alpha_max),
                                  dec.data_ptr(), scratch.data_ptr(), nbytes, _stream_handle()),
              "pf_remove_stuck")
    decayed = sorted(int(i) for i in np.flatnonzero(dec.cpu().numpy()))
    if not decayed:
        return scene, []
    nu = pm[:, 4].cpu().numpy()
    prims = list(scene.primitives)
    for i in decayed:
        prims[i] = dataclasses.replace(prims[i], opacity_logit=float(nu[i]))
    return dataclasses.replace(scene, primitives=prims), decayed


def policy_from_config(cfg) -> StuckPolicy:
    """StuckPolicy from a FitConfig's video fields (dyn.py:74-83); missing fields
    take the reference defaults."""
    g = lambda k, d: getattr(cfg, k, d)  # noqa: E731
    return StuckPolicy(grid=(int(g("stuck_grid_y", 4)), int(g("stuck_grid_x", 4))),
                       k=int(g("stuck_top_k", 4)), tau_scale=float(g("stuck_tau_scale", 0.1)),
                       tau_alpha=float(g("stuck_tau_alpha", 0.7)), zeta=float(g("stuck_zeta", 0.7)),
                       eta=float(g("stuck_eta", 0.3)),
                       triggers=tuple(g("stuck_triggers", (20, 45, 70))))


def optimize_video(frames, templates, cfg, rng: np.random.Generator | None = None):
    """Fit one scene per frame, warm-starting each from the previous
    (dyn.py:180-238), every step in the GPU fit loop (fit.run_loop).

    As the reference: ``templates`` (a template list, or None for the built-in
    default) go through prepare_templates with the config's blur / falloff, and
    frame 0's scene comes from init_scene (initializer, opacity / colour init,
    density cap, variance window, background, alpha_max, mu_blend,
    preserve_aspect) drawing from ``default_rng(cfg.seed)``; frame 0 runs
    ``cfg.num_iterations`` steps; every later frame runs
    ``cfg.sequential_iterations`` from fresh Adam moments, with the primitives
    whose binning box misses every changed pixel frozen (``freeze_static``;
    diff_mask + freeze_flags on the GPU) and the stuck-primitive decay at the
    policy's trigger iterations (``remove_stuck``).  Extension: a prepared
    ``Scene`` in place of ``templates`` is used as frame 0's scene directly, and
    ``rng`` (default ``default_rng(cfg.seed)``) can be supplied (frame sharding).
    Returns (scenes, histories), one per frame.
    """
    from .fit import LossSpec, OptimState, effective_padding, run_loop
    from .prep import default_templates, init_scene, prepare_templates
    from .scene import Scene, pack_params

    if not frames:
        raise ValueError("need at least one frame")
    frames = [np.asarray(f, dtype=np.float64) for f in frames]
    for f in frames:
        if f.shape != frames[0].shape:
            raise ShapeMismatch("all frames must share one shape")
    if cfg.loss in ("spatial", "spatial_constrained"):
        raise ValueError("spatial loss is single-image only")
    rng = np.random.default_rng(cfg.seed) if rng is None else rng
    g = lambda k, d: getattr(cfg, k, d)  # noqa: E731  (duck-typed FitConfig)
    if isinstance(templates, Scene):
        scene = templates
    else:
        tpls = prepare_templates(list(templates) if templates else default_templates(),
                                 blur_sigma=g("blur_sigma", 1.0),
                                 do_blur=g("do_gaussian_blur", True),
                                 falloff=g("radial_falloff", False))
        scene = init_scene(frames[0], tpls, cfg, rng)
    padding = effective_padding(cfg)
    policy = policy_from_config(cfg)

    def spec(frame):  # dyn.py:241-247
        return LossSpec(kind=cfg.loss, target=frame, mse_w=g("mse_weight", 1.0),
                        gray_l1_w=g("gray_l1_weight", 0.0))

    scene, hist, _ = run_loop(scene, cfg, spec(frames[0]), rng, iterations=cfg.num_iterations)
    scenes, histories = [scene], [hist]
    for f in range(1, len(frames)):
        _, layout = pack_params(scene)
        state = OptimState.fresh(layout)
        if g("freeze_static", True):
            mask = diff_mask(frames[f - 1], frames[f],
                             float(g("diff_threshold", DEFAULT_DIFF_THRESHOLD)))
            state.frozen = freeze_flags(scene, mask, padding)
        hooks = None
        if g("remove_stuck", False):
            hooks = {t: (lambda s, st: remove_stuck(s, st.frozen, policy)[0])
                     for t in policy.triggers}
        scene, hist, state = run_loop(scene, cfg, spec(frames[f]), rng,
                                      iterations=int(g("sequential_iterations", 100)),
                                      state=state, hooks=hooks)
        scenes.append(scene)
        histories.append(hist)
    return scenes, histories


def frame_chunks(n_frames: int, world: int) -> list[range]:
    """Contiguous, balanced frame ranges, one per rank (earlier ranks take the
    remainder)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    base, extra = divmod(n_frames, world)
    out, start = [], 0
    for r in range(world):
        k = base + (1 if r < extra else 0)
        out.append(range(start, start + k))
        start += k
    return out


def chunk_rng(seed: int, chunk: int) -> np.random.Generator:
    """The rng of a frame chunk: chunk 0 draws from ``default_rng(seed)`` exactly
    as the sequential reference does; later chunks from ``default_rng([seed, c])``."""
    return np.random.default_rng(seed) if chunk == 0 else np.random.default_rng([seed, chunk])


def optimize_video_sharded(frames, templates, cfg, *, rank: int | None = None,
                           world: int | None = None, group=None):
    """BASELINE.json c4 ("frames sharded across 8 GPUs"): the frames are split into
    ``world`` contiguous chunks and rank r runs optimize_video's warm-start chain
    on chunk r on its own device -- no collective inside the fit; the per-frame
    scenes and histories are gathered to every rank at the end
    (``torch.distributed.all_gather_object``; without an initialised process
    group, or world == 1, this is optimize_video on the whole list).

    Difference from the sequential reference (dyn.py:180-238), by construction:
    the chain restarts at every chunk boundary -- the chunk's first frame is
    initialised with init_scene and runs the frame-0 budget ``num_iterations``
    -- so frames after the first chunk differ from a single sequential chain;
    chunk 0 (frames 0..k-1, ``default_rng(cfg.seed)``) is bit for bit the
    sequential run of those frames.  Returns (scenes, histories) for all frames.
    """
    import torch.distributed as dist

    if not frames:
        raise ValueError("need at least one frame")
    if world is None:
        world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    if rank is None:
        rank = dist.get_rank(group) if world > 1 else 0
    if world == 1:
        return optimize_video(frames, templates, cfg)
    chunks = frame_chunks(len(frames), world)
    mine = chunks[rank]
    local = ([], [])
    if len(mine):
        local = optimize_video([frames[i] for i in mine], templates, cfg,
                               rng=chunk_rng(int(getattr(cfg, "seed", 0)), rank))
    parts = [None] * world
    dist.all_gather_object(parts, local, group=group)
    scenes, histories = [], []
    for sc, hi in parts:
        scenes.extend(sc)
        histories.extend(hi)
    return scenes, histories
