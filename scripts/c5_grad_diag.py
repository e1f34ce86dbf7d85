"""Diagnostics: where the c5 fused-step gradient departs from the oracle."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np

from conftest import grad_close
from paper_2602_22625_b200 import synth
from paper_2602_22625_b200.fit import StepEngine, effective_padding
from test_gpu_scale import _fused_grads
sys.path.insert(0, str(ROOT / "oracle"))
import cpu_oracle as orc  # type: ignore  (test infrastructure: the checker)

orc.build()
w = synth.make_workload(sys.argv[1] if len(sys.argv) > 1 else "c5")
sc = w.scene
rng = np.random.default_rng(7)
for p in sc.primitives:
    p.x += float(rng.uniform(-0.5, 0.5))
    p.y += float(rng.uniform(-0.5, 0.5))
    p.opacity_logit = float(rng.uniform(-2.0, 3.0))
eng = StepEngine(sc, w.cfg, w.loss, 1, use_graph=False)
g, sums, color, alpha = _fused_grads(eng)
pk = orc.Packed(sc)
off, idx = orc.bin_tiles(pk, 32, effective_padding(w.cfg))
img, a_ref, sv = orc.render_forward(pk, off, idx, 32, orc.background(sc), True, w.cfg.eps_skip)
diff = img - w.target
g_ref = orc.backward(pk, sv, 2.0 * diff / diff.size, None)
ok, err = grad_close(g, g_ref)
print("grad_close", ok, err)
colmax = np.abs(g_ref).max(axis=0, keepdims=True)
floor = np.maximum(np.maximum(1e-2 * colmax, 1e-4 * np.abs(g_ref).max()), 1e-300)
e = np.abs(g - g_ref) / np.maximum(np.abs(g_ref), floor)
worst = np.argsort(e.reshape(-1))[-12:][::-1]
tid = np.array([p.template_id for p in sc.primitives])
for k in worst:
    i, c = divmod(int(k), 8)
    p = sc.primitives[i]
    print(f"prim {i:5d} col {c} err {e[i, c]:.2e} got {g[i, c]: .4e} ref {g_ref[i, c]: .4e} "
          f"tid {tid[i]} s {p.scale:.2f} nu {p.opacity_logit:.2f} xy ({p.x:.1f},{p.y:.1f})")
print("per-column max err:", [float(f"{v:.2e}") for v in e.max(axis=0)])
print("per-template max err:", {int(t): float(f"{e[tid == t].max():.2e}") for t in np.unique(tid)})
