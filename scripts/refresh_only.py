"""Diagnostics: back-to-back pf_preprocess launches at c3 (for ncu)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch

from paper_2602_22625_b200 import synth
from paper_2602_22625_b200.fit import StepEngine

w = synth.make_workload("c3")
w.cfg.num_iterations = 100
eng = StepEngine(w.scene, w.cfg, w.loss, 100, use_graph=True)
eng.run(3)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    eng.refresh()
torch.cuda.synchronize()
