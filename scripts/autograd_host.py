"""Diagnostics: host-side cost of the eager autograd step (cProfile, c3)."""
import cProfile
import pstats
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch

from paper_2602_22625_b200 import synth
from paper_2602_22625_b200.autograd import Renderer
from paper_2602_22625_b200.compositor import adam_launch
from paper_2602_22625_b200.fit import _cfg_gains, effective_padding
from paper_2602_22625_b200.scene import param_matrix, structure_arrays

w = synth.make_workload("c3")
sc, cfg = w.scene, w.cfg
tid, z = structure_arrays(sc)
r = Renderer(sc.templates, tid, z, sc.canvas_w, sc.canvas_h, background=tuple(sc.background),
             alpha_max=sc.alpha_max, mu_blend=sc.mu_blend, preserve_aspect=sc.preserve_aspect,
             eps_skip=cfg.eps_skip, padding=effective_padding(cfg), s_max=cfg.scale_max)
params = torch.tensor(param_matrix(sc), device="cuda", requires_grad=True)
target = torch.tensor(w.target, device="cuda", dtype=torch.float32)
m = torch.zeros(params.numel(), dtype=torch.float64, device="cuda")
v = torch.zeros_like(m)
gains = _cfg_gains(cfg)


def step(it):
    img, _ = r(params)
    loss = ((img - target) ** 2).mean()
    loss.backward()
    with torch.no_grad():
        adam_launch(params.view(-1), params.grad.view(-1), m, v, gains=gains, n=params.shape[0],
                    lr=1e-3, bc1=1 - 0.9 ** (it + 1), bc2=1 - 0.999 ** (it + 1), clamp=True,
                    s_min=cfg.scale_min, s_max=cfg.scale_max, zero_grads=True)


for it in range(5):
    step(it)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for it in range(5, 105):
    step(it)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
