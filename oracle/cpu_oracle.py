"""CPU ORACLE wrapper (test infrastructure only -- never on the product path).

numpy-level restatement of the reference's L2 API on top of the C oracle
(oracle/primfit_oracle.c).  Used by tests/ as the parity checker, by
__graft_entry__.smoke() as the checker, and by bench.py's ``cpu_baseline`` /
``--impl reference`` leg as the host-CPU timing arm.

Reference call sites restated (paths under /root/reference/pkg/src/primfit):
  pack            raster.py:63-96 (pack_scene)
  bin_tiles       raster.py:227-265
  render_forward  raster.py:290-363 (count -> cumsum -> fill)
  backward        grad.py:134-187
  loss_mse / psnr / adam_step / lr_schedule   fit.py:112-116, 241-247, 195-238, 174-186
  step            the body of fit.run_loop, fit.py:476-505
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "libprimfit_oracle.so"

_lib = None


def build() -> Path:
    subprocess.run(["make", "-C", str(HERE), "-s"], check=True)
    return LIB


def load() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        _lib = C.CDLL(str(LIB))
        _lib.orc_bin_tiles.restype = C.c_int64
        _lib.orc_max_threads.restype = C.c_int
    return _lib


def threads() -> int:
    return int(load().orc_max_threads())


def set_threads(n: int) -> None:
    load().orc_set_threads(int(n))


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Packed:
    """SoA arrays the oracle kernels take (the reference's PackedScene)."""

    def __init__(self, scene):
        prims = scene.primitives
        n = len(prims)
        self.n = n
        pm = np.empty((n, 8))
        for i, p in enumerate(prims):
            c = p.color_logits
            pm[i] = (p.x, p.y, p.scale, p.rotation, p.opacity_logit, c[0], c[1], c[2])
        self.params = pm
        self.tid = np.ascontiguousarray([p.template_id for p in prims], dtype=np.int32)
        z = np.asarray([p.z for p in prims], dtype=np.int64)
        self.order = np.argsort(z, kind="stable").astype(np.int32)
        tpls = [np.asarray(t.rgba, dtype=np.float64) for t in scene.templates]
        self.tw = np.asarray([a.shape[1] for a in tpls], dtype=np.int32)
        self.th = np.asarray([a.shape[0] for a in tpls], dtype=np.int32)
        sizes = self.tw.astype(np.int64) * self.th.astype(np.int64)
        self.toff = np.concatenate(([0], np.cumsum(sizes)))[:-1].astype(np.int64)
        self.tex = (np.ascontiguousarray(np.concatenate([a.reshape(-1, 4) for a in tpls]))
                    if tpls else np.zeros((0, 4)))
        if scene.preserve_aspect and n:
            self.q = self.th[self.tid].astype(np.float64) / self.tw[self.tid].astype(np.float64)
        else:
            self.q = np.ones(n)
        self.hyp = np.asarray([math.hypot(1.0, max(1.0, float(q))) for q in self.q])
        self.W, self.H = int(scene.canvas_w), int(scene.canvas_h)
        self.alpha_max, self.mu = float(scene.alpha_max), float(scene.mu_blend)
        self.set_params(pm)

    def set_params(self, pm: np.ndarray) -> None:
        pm = np.ascontiguousarray(pm, dtype=np.float64).reshape(self.n, 8)
        self.params = pm
        self.x = np.ascontiguousarray(pm[:, 0])
        self.y = np.ascontiguousarray(pm[:, 1])
        self.s = np.ascontiguousarray(pm[:, 2])
        self.r = np.ascontiguousarray(pm[:, 3])
        self.nu = np.ascontiguousarray(pm[:, 4])
        self.cv = np.ascontiguousarray(pm[:, 5:8])


def bin_tiles(pk: Packed, tile: int, padding: float):
    lib = load()
    ntx, nty = -(-pk.W // tile), -(-pk.H // tile)
    off = np.zeros(ntx * nty + 1, dtype=np.int64)
    args = (_p(pk.x), _p(pk.y), _p(pk.s), _p(pk.hyp), _p(pk.order), pk.n, pk.W, pk.H, tile,
            C.c_double(padding), _p(off))
    K = lib.orc_bin_tiles(*args, None, C.c_int64(0))
    idx = np.zeros(max(K, 1), dtype=np.int32)
    lib.orc_bin_tiles(*args, _p(idx), C.c_int64(K))
    return off, idx[:K]


def background(scene, bg=None) -> np.ndarray:
    if bg is None:
        bg = scene.background
    bg = np.asarray(bg, dtype=np.float64)
    if bg.shape == (3,):
        bg = np.broadcast_to(bg, (scene.canvas_h, scene.canvas_w, 3))
    return np.ascontiguousarray(bg)


def render_forward(pk: Packed, off, idx, tile: int, bg: np.ndarray, save: bool, eps: float):
    lib = load()
    W, H = pk.W, pk.H
    ntx, nty = -(-W // tile), -(-H // tile)
    img = np.empty((H, W, 3))
    alpha = np.empty((H, W))
    geo = (C.c_double(eps), tile, ntx, nty, W, H)
    if not save:
        lib.orc_fill_entries(_p(pk.x), _p(pk.y), _p(pk.s), _p(pk.r), _p(pk.nu), _p(pk.cv),
                             _p(pk.tid), _p(pk.q), _p(pk.tex), _p(pk.toff), _p(pk.tw), _p(pk.th),
                             _p(off), _p(idx), _p(bg), C.c_double(pk.alpha_max),
                             C.c_double(pk.mu), *geo, None, None, None, None, None, None, None,
                             _p(img), _p(alpha))
        return img, alpha, None
    counts = np.zeros(H * W, dtype=np.int64)
    lib.orc_count_entries(_p(pk.x), _p(pk.y), _p(pk.s), _p(pk.r), _p(pk.tid), _p(pk.q),
                          _p(pk.tex), _p(pk.toff), _p(pk.tw), _p(pk.th), _p(off), _p(idx),
                          *geo, _p(counts))
    ent_off = np.concatenate(([0], np.cumsum(counts))).astype(np.int64)
    M = int(ent_off[-1])
    sv = {
        "offsets": ent_off,
        "prim": np.empty(max(M, 1), dtype=np.int32),
        "alpha": np.empty(max(M, 1)),
        "color": np.empty((max(M, 1), 3)),
        "mask": np.empty(max(M, 1)),
        "U": np.empty(max(M, 1)),
        "V": np.empty(max(M, 1)),
        "bg": bg,
        "n_entries": M,
    }
    lib.orc_fill_entries(_p(pk.x), _p(pk.y), _p(pk.s), _p(pk.r), _p(pk.nu), _p(pk.cv),
                         _p(pk.tid), _p(pk.q), _p(pk.tex), _p(pk.toff), _p(pk.tw), _p(pk.th),
                         _p(off), _p(idx), _p(bg), C.c_double(pk.alpha_max), C.c_double(pk.mu),
                         *geo, _p(ent_off), _p(sv["prim"]), _p(sv["alpha"]), _p(sv["color"]),
                         _p(sv["mask"]), _p(sv["U"]), _p(sv["V"]), _p(img), _p(alpha))
    return img, alpha, sv


def backward(pk: Packed, sv: dict, dI: np.ndarray, dA: np.ndarray | None) -> np.ndarray:
    lib = load()
    grads = np.zeros((pk.n, 8))
    dI = np.ascontiguousarray(dI, dtype=np.float64)
    dA = None if dA is None else np.ascontiguousarray(dA, dtype=np.float64)
    lib.orc_backward(_p(pk.s), _p(pk.r), _p(pk.nu), _p(pk.cv), _p(pk.tid), _p(pk.q), _p(pk.tex),
                     _p(pk.toff), _p(pk.tw), _p(pk.th), _p(sv["offsets"]), _p(sv["prim"]),
                     _p(sv["alpha"]), _p(sv["color"]), _p(sv["mask"]), _p(sv["U"]), _p(sv["V"]),
                     _p(sv["bg"]), _p(dI), _p(dA), C.c_double(pk.alpha_max), C.c_double(pk.mu),
                     pk.n, pk.W, pk.H, _p(grads))
    return grads


def adam(params, grads, m, v, step_t: int, lr: float, frozen=None, gains8=None,
         s_min=None, s_max=None):
    """In-place Adam on float64 arrays (n*8); gains8: per-column gains or None."""
    lib = load()
    n = params.size // 8
    gains = None if gains8 is None else np.ascontiguousarray(np.tile(np.asarray(gains8, float), n))
    fz = None if frozen is None else np.ascontiguousarray(frozen, dtype=np.uint8)
    clamp = s_min is not None and s_max is not None
    lib.orc_adam(_p(params), _p(grads), _p(m), _p(v), _p(fz), _p(gains), n, int(step_t),
                 C.c_double(lr), int(clamp), C.c_double(s_min or 0.0), C.c_double(s_max or 0.0))


def loss_mse(I, t):
    diff = I - t
    return float(np.mean(diff**2)), 2.0 * diff / diff.size


def psnr(I, t) -> float:
    mse = float(np.mean((I - t) ** 2))
    return math.inf if mse == 0.0 else 10.0 * math.log10(1.0 / mse)


def lr_schedule(it: int, total: int, base: float, decay: bool = True, final: float = 0.1) -> float:
    if not decay or total <= 1:
        return base
    return base * final ** (it / (total - 1))


GRAY = np.asarray([0.299, 0.587, 0.114])


def loss_gray_l1(I, t):
    """loss_grayscale_l1 (fit.py:119-125): mean |luma(I - t)| and its subgradient."""
    d = (I - t) @ GRAY
    return float(np.mean(np.abs(d))), (np.sign(d)[:, :, None] * GRAY[None, None, :]) / d.size


def loss_combined(I, t, mse_w: float, gray_w: float):
    """evaluate_loss kind "combined" (fit.py:162-168)."""
    vm, gm = loss_mse(I, t)
    vg, gg = loss_gray_l1(I, t)
    return mse_w * vm + gray_w * vg, mse_w * gm + gray_w * gg


class Loop:
    """The body of fit.run_loop (solid background; mse, or the combined loss with
    ``loss=("combined", mse_w, gray_w)``) on the oracle."""

    def __init__(self, scene, target, cfg, padding: float, tile: int = 32, loss=None):
        self.loss = loss
        self.pk = Packed(scene)
        self.target = np.asarray(target, dtype=np.float64)
        self.cfg = cfg
        self.padding = padding
        self.tile = tile
        self.bg = background(scene)
        self.vec = self.pk.params.reshape(-1).copy()
        self.m = np.zeros_like(self.vec)
        self.v = np.zeros_like(self.vec)
        self.t = 0
        c = cfg
        self.gains8 = [c.lr_gain_x, c.lr_gain_y, c.lr_gain_scale, c.lr_gain_rotation,
                       c.lr_gain_opacity, c.lr_gain_color, c.lr_gain_color, c.lr_gain_color]
        self.history = []

    def step(self, it: int, total: int):
        c = self.cfg
        lr = lr_schedule(it, total, c.learning_rate, c.do_decay, c.decay_final_fraction)
        self.pk.set_params(self.vec)
        off, idx = bin_tiles(self.pk, self.tile, self.padding)
        img, alpha, sv = render_forward(self.pk, off, idx, self.tile, self.bg, True, c.eps_skip)
        if self.loss is None:
            value, dI = loss_mse(img, self.target)
        else:
            value, dI = loss_combined(img, self.target, self.loss[1], self.loss[2])
        g = backward(self.pk, sv, dI, None).reshape(-1)
        self.t += 1
        adam(self.vec, g, self.m, self.v, self.t, lr, gains8=self.gains8, s_min=c.scale_min,
             s_max=c.scale_max)
        q = psnr(img, self.target)
        self.history.append((it, value, q, lr))
        return value, q


# ---------------------------------------------------------------------------
# f4 layered export and f3 video heuristics, numpy restatements.
# Paths under /root/reference/pkg/src/primfit.

def _expit(x):
    x = np.asarray(x, dtype=np.float64)
    return np.where(x >= 0, 1.0 / (1.0 + np.exp(-np.abs(x))), np.exp(-np.abs(x)) / (1.0 + np.exp(-np.abs(x))))


LAYER_BBOX_PAD = 1.0  # exportio.py:78


def export_layers_arrays(pk: Packed, rho: int):
    """scale_scene (exportio.py:272-288) + layer_bbox (291-307) + render_layer (310-346)
    for every primitive: (bbox int64 [n][4] (-1 rows: DegenerateBBox), offsets
    int64 [n+1], premultiplied rgba float64 [sum of areas][4])."""
    shift = (rho - 1) / 2.0
    W, H = rho * pk.W, rho * pk.H
    boxes, chunks, offs = [], [], [0]
    for i in range(pk.n):
        x = rho * pk.x[i] + shift
        y = rho * pk.y[i] + shift
        s = rho * pk.s[i]
        q = float(pk.q[i])
        r = s * math.hypot(1.0, max(1.0, q)) + LAYER_BBOX_PAD
        x0, x1 = max(math.floor(x - r), 0), min(math.ceil(x + r), W - 1)
        y0, y1 = max(math.floor(y - r), 0), min(math.ceil(y + r), H - 1)
        if x0 > x1 or y0 > y1:
            boxes.append((-1, -1, -1, -1))
            offs.append(offs[-1])
            continue
        xx, yy = np.meshgrid(np.arange(x0, x1 + 1, dtype=np.float64),
                             np.arange(y0, y1 + 1, dtype=np.float64))
        ct, st = math.cos(pk.r[i]), math.sin(pk.r[i])   # raster.py:159-172
        dx, dy = xx - x, yy - y
        u = (ct * dx + st * dy) / s
        v = (-st * dx + ct * dy) / (s * q)
        t = int(pk.tid[i])
        wt, ht = int(pk.tw[t]), int(pk.th[t])
        U = (u + 1.0) * 0.5 * (wt - 1)                  # raster.py:175-179
        V = (v + 1.0) * 0.5 * (ht - 1)
        rgba_t = pk.tex[pk.toff[t]: pk.toff[t] + wt * ht].reshape(ht, wt, 4)

        def plane(ch):                                  # raster.py:182-200
            pl = rgba_t[:, :, ch]
            inside = (U >= 0.0) & (U <= wt - 1.0) & (V >= 0.0) & (V <= ht - 1.0)
            u0 = np.clip(np.floor(U).astype(np.int64), 0, wt - 1)
            v0 = np.clip(np.floor(V).astype(np.int64), 0, ht - 1)
            u1, v1 = np.minimum(u0 + 1, wt - 1), np.minimum(v0 + 1, ht - 1)
            wu, wv = np.clip(U - u0, 0.0, 1.0), np.clip(V - v0, 0.0, 1.0)
            val = ((1.0 - wu) * (1.0 - wv) * pl[v0, u0] + wu * (1.0 - wv) * pl[v0, u1]
                   + (1.0 - wu) * wv * pl[v1, u0] + wu * wv * pl[v1, u1])
            return np.where(inside, val, 0.0)

        a = pk.alpha_max * _expit(pk.nu[i]) * plane(3)
        cvar = _expit(pk.cv[i])
        if pk.mu > 0.0:                                  # raster.py:214-219
            c = np.stack([pk.mu * plane(ch) + (1.0 - pk.mu) * cvar[ch] for ch in range(3)], axis=-1)
        else:
            c = np.broadcast_to(cvar, a.shape + (3,))
        rgba = np.empty(a.shape + (4,))
        rgba[:, :, :3] = a[:, :, None] * c
        rgba[:, :, 3] = a
        boxes.append((x0, y0, x1, y1))
        chunks.append(rgba.reshape(-1, 4))
        offs.append(offs[-1] + rgba.shape[0] * rgba.shape[1])
    rgba_all = np.concatenate(chunks, axis=0) if chunks else np.zeros((0, 4))
    return np.asarray(boxes, dtype=np.int64), np.asarray(offs, dtype=np.int64), rgba_all


def diff_mask(prev, cur, tau):
    """dyn.py:86-97."""
    return np.abs(np.asarray(prev, np.float64) - np.asarray(cur, np.float64)).max(axis=2) > tau


def freeze_flags(pk: Packed, mask, padding):
    """dyn.py:100-130 (the binning bbox, inclusive rounding, any change inside)."""
    out = np.empty(pk.n, dtype=bool)
    for i in range(pk.n):
        r = pk.s[i] * pk.hyp[i] + padding
        x0, x1 = max(math.ceil(pk.x[i] - r), 0), min(math.floor(pk.x[i] + r), pk.W - 1)
        y0, y1 = max(math.ceil(pk.y[i] - r), 0), min(math.floor(pk.y[i] + r), pk.H - 1)
        out[i] = not (x0 <= x1 and y0 <= y1 and mask[y0:y1 + 1, x0:x1 + 1].any())
    return out


def remove_stuck(pk: Packed, z, frozen, grid, k, tau_scale, tau_alpha, zeta, eta):
    """dyn.py:133-177 -> (new opacity logits, sorted decayed indices)."""
    rows, cols = grid
    frozen = np.zeros(pk.n, dtype=bool) if frozen is None else np.asarray(frozen, dtype=bool)
    regions = {}
    for i in range(pk.n):
        ry = min(max(int(pk.y[i] * rows / pk.H), 0), rows - 1)
        rx = min(max(int(pk.x[i] * cols / pk.W), 0), cols - 1)
        regions.setdefault((ry, rx), []).append(i)
    decayed = []
    for members in regions.values():
        zs = np.asarray([z[i] for i in members])
        scored = []
        for i in members:
            rank = int((zs > z[i]).sum())
            alpha = pk.alpha_max * float(_expit(pk.nu[i]))
            if (not frozen[i] and pk.s[i] >= tau_scale * pk.W and alpha >= tau_alpha
                    and rank >= zeta * len(members)):
                scored.append((pk.s[i] * alpha, i))
        scored.sort(key=lambda t: (-t[0], t[1]))
        decayed.extend(i for _, i in scored[:k])
    nu = pk.nu.copy()
    for i in decayed:
        nu[i] = eta * nu[i]
    return nu, sorted(decayed)
