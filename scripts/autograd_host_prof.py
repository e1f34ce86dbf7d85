"""Diagnostics: host cost of one eager autograd training step at c3 (fused
loss_mse + pf_adam), wall-clock per step and a cProfile of the Python side."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch

from paper_2602_22625_b200 import synth
from paper_2602_22625_b200.autograd import Renderer, loss_mse
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
n = params.shape[0]
m = torch.zeros(n * 8, dtype=torch.float64, device="cuda")
v = torch.zeros_like(m)
gains = _cfg_gains(cfg)


def step():
    img, _ = r(params)
    loss = loss_mse(img, target)
    loss.backward()
    with torch.no_grad():
        adam_launch(params.view(-1), params.grad.view(-1), m, v, gains=gains, n=n, lr=1e-4,
                    bc1=0.5, bc2=0.5, clamp=True, s_min=cfg.scale_min, s_max=cfg.scale_max,
                    zero_grads=False)
    params.grad = None


for _ in range(50):
    step()
torch.cuda.synchronize()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
t0 = time.perf_counter()
for _ in range(N):
    step()
torch.cuda.synchronize()
print(f"eager step: {(time.perf_counter() - t0) / N * 1e6:.1f} us wall per step")
pr = cProfile.Profile()
pr.enable()
for _ in range(N):
    step()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
