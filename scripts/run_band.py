"""Diagnostics: run graph-replayed fit steps of one row band (ncu target).

    python scripts/run_band.py c5 8 3 [steps]
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch

from paper_2602_22625_b200 import synth
from paper_2602_22625_b200.dist import row_bands
from paper_2602_22625_b200.fit import StepEngine

name, world, rank = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 6
w = synth.make_workload(name)
band = row_bands(-(-w.scene.canvas_h // 16), world)[rank]
w.cfg.num_iterations = steps + 2
eng = StepEngine(w.scene, w.cfg, w.loss, steps + 2, band=band, use_graph=True)
for _ in range(steps):
    eng.step()
torch.cuda.synchronize()
eng.check()
print("ok", band)
