"""Small driver for compute-sanitizer (racecheck / synccheck / memcheck):
eager fused fit steps (K1 -> K2 -> K34 -> K5+K1) on c1 / c3, the two-kernel
path (K3 + K4, mu_blend > 0) on c1, and two-level binning + a fused step on one
band of an 8-way split of c5.

    compute-sanitizer --tool racecheck python scripts/sanitize_step.py c3
"""

from __future__ import annotations

import dataclasses
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main() -> None:
    import torch

    from paper_2602_22625_b200 import synth
    from paper_2602_22625_b200.dist import row_bands
    from paper_2602_22625_b200.fit import StepEngine

    case = sys.argv[1] if len(sys.argv) > 1 else "c1"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    if case == "c1mu":
        w = synth.make_workload("c1")
        sc = dataclasses.replace(w.scene, mu_blend=0.3)
        eng = StepEngine(sc, w.cfg, w.loss, steps, use_graph=False)
        assert not eng.fused
    elif case == "c5band":
        w = synth.make_workload("c5")
        band = row_bands(-(-w.scene.canvas_h // 16), 8)[3]
        eng = StepEngine(w.scene, w.cfg, w.loss, steps, band=band, use_graph=False)
    else:
        w = synth.make_workload(case)
        eng = StepEngine(w.scene, w.cfg, w.loss, steps, use_graph=False)
    for _ in range(steps):
        eng.step()
    torch.cuda.synchronize()
    eng.check()
    print(f"{case}: {steps} steps ok, loss {eng.history()[-1].loss:.6f}")


if __name__ == "__main__":
    main()
