"""Projected row-band scaling on ONE GPU: the step time of every band of an
N-way row split, measured one band at a time (graph replay, L2 flushed), so the
N-GPU step is max over bands + the gradient allreduce (not measurable here).

    python scripts/band_scaling.py c5 1 2 4 8
"""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

from paper_2602_22625_b200 import synth
from paper_2602_22625_b200.dist import row_bands, row_cost_from_bins
from paper_2602_22625_b200.fit import StepEngine

# PF_BAND_NCCL=1: every band step carries the exchange node -- a one-rank NCCL
# communicator's allreduce captured in the step graph (the fold, the NCCL kernel
# and the PDL overlap it breaks are measured; only the NVSwitch transfer is not)
NCCL = os.environ.get("PF_BAND_NCCL") == "1"
if NCCL:
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29812")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    from paper_2602_22625_b200.dist import make_allreduce
name = sys.argv[1]
worlds = [int(v) for v in sys.argv[2:]] or [1, 2, 4, 8]
w = synth.make_workload(name)
H, W = w.scene.canvas_h, w.scene.canvas_w
nty, ntx = -(-H // 16), -(-W // 16)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
K, WARM = 20, 4
w.cfg.num_iterations = K + WARM + 2


CH = 8 * 8  # chained mode: 8 graphs of StepEngine.CHUNK (8) steps, timed together


def band_chained_ms(band) -> float:
    """run_loop's own issue pattern: CHUNK-step graphs with PDL edges between
    steps, no L2 flush (the per-step graph launch of band_ms is amortised)."""
    eng = StepEngine(w.scene, w.cfg, w.loss, CH + 2 * 8 + 2, band=band, use_graph=True,
                     allreduce=make_allreduce() if NCCL else None)
    eng.run(1 + 8 + 7)  # warm-up: single-step graph, one chunk, then align
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.run(CH)
    e1.record()
    torch.cuda.synchronize()
    eng.check()
    out = e0.elapsed_time(e1) / CH
    del eng
    torch.cuda.empty_cache()
    return out


def band_ms(band) -> float:
    eng = StepEngine(w.scene, w.cfg, w.loss, K + WARM + 2, band=band, use_graph=True,
                     allreduce=make_allreduce() if NCCL else None)
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
    out = float(np.median(ts))
    del eng
    torch.cuda.empty_cache()
    return out


# full-canvas bins of the initial state for cost-balanced bands
full = StepEngine(w.scene, w.cfg, w.loss, 2, use_graph=False)
full.refresh()
full.comp.bin()
cost = row_cost_from_bins(full.comp.bin_off.cpu().numpy()[: nty * ntx + 1], ntx, nty)
del full
res = {"config": name, "n": w.scene.n, "canvas": [W, H], "grad_allreduce_bytes": 8 * (8 * w.scene.n + 4)}
base = cbase = None
for N in worlds:
    for kind, rc in (("uniform", None), ("balanced", cost)):
        if N == 1 and kind == "balanced":
            continue
        bands = row_bands(nty, N, rc)
        ms = [band_ms(b) for b in bands]
        cms = [band_chained_ms(b) for b in bands]
        if N == 1:
            base, cbase = ms[0], cms[0]
        eff = base / (N * max(ms)) if base else None
        ceff = cbase / (N * max(cms)) if cbase else None
        res[f"N{N}_{kind}"] = {"band_ms": [round(m, 4) for m in ms], "max_ms": max(ms),
                              "projected_eff_no_allreduce": eff,
                              "chained_band_ms": [round(m, 4) for m in cms],
                              "chained_max_ms": max(cms), "chained_eff_no_allreduce": ceff}
        print(f"N={N} {kind:8s} max {max(ms) * 1e3:8.1f} us  mean {np.mean(ms) * 1e3:8.1f} us  "
              f"eff(no allreduce) {eff:.3f} | chained max {max(cms) * 1e3:8.1f} us  "
              f"eff {ceff:.3f}", flush=True)
Path("gpurun_out").mkdir(exist_ok=True)
res["exchange_node"] = "one-rank NCCL allreduce in every step graph" if NCCL else "none"
Path(f"gpurun_out/band_scaling_{name}{'_nccl' if NCCL else ''}.json").write_text(
    json.dumps(res, indent=1))
