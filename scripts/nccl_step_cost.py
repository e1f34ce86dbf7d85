"""Fixed cost of the NCCL allreduce node inside the step graph, measured with a
one-rank NCCL communicator (the only one a single GPU allows): graph-replayed
steps with and without the allreduce, L2 flushed, for the full canvas and for one
band of an 8-way split (the band a rank of an 8-GPU c5 job renders).

    python scripts/nccl_step_cost.py c5 8 3
"""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch
import torch.distributed as dist

from paper_2602_22625_b200 import synth
from paper_2602_22625_b200.dist import make_allreduce, row_bands
from paper_2602_22625_b200.fit import StepEngine

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
rank = int(sys.argv[3]) if len(sys.argv) > 3 else 3
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29811")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
w = synth.make_workload(name)
nty = -(-w.scene.canvas_h // 16)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
K, WARM = 30, 4
w.cfg.num_iterations = K + WARM + 2


def step_ms(band, ar) -> float:
    eng = StepEngine(w.scene, w.cfg, w.loss, K + WARM + 2, band=band, allreduce=ar,
                     use_graph=True)
    eng.run(WARM)
    torch.cuda.synchronize()
    ts = []
    for _ in range(K):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.step()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    eng.check()
    return float(np.median(ts))


res = {"config": name, "grad_allreduce_bytes": 8 * (8 * w.scene.n + 4)}
for label, band in (("full", row_bands(nty, 1)[0]), (f"band{world}:{rank}",
                                                      row_bands(nty, world)[rank])):
    a = [step_ms(band, None) for _ in range(2)]
    b = [step_ms(band, make_allreduce()) for _ in range(2)]
    res[label] = {"no_allreduce_ms": min(a), "nccl1_allreduce_ms": min(b),
                  "node_cost_us": (min(b) - min(a)) * 1e3}
    print(label, res[label], flush=True)
Path("gpurun_out").mkdir(exist_ok=True)
Path(f"gpurun_out/nccl_step_cost_{name}.json").write_text(json.dumps(res, indent=1))
dist.destroy_process_group()
