"""Diagnostics: kernel timeline of graph-replayed fit steps (PF_TIMELINE=1)."""
import ctypes as C
import os
import sys
from pathlib import Path

os.environ["PF_TIMELINE"] = "1"
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

from paper_2602_22625_b200 import _native as nat, synth
from paper_2602_22625_b200.fit import StepEngine

w = synth.make_workload(sys.argv[1] if len(sys.argv) > 1 else "c3")
w.cfg.num_iterations = 60
hostio = "hostio" in sys.argv[2:]
band = None
for a in sys.argv[2:]:
    if a.startswith("band="):  # band=N:r -- rank r of an N-way uniform row split
        from paper_2602_22625_b200.dist import row_bands
        N, r = (int(v) for v in a[5:].split(":"))
        band = row_bands(-(-w.scene.canvas_h // 16), N)[r]
eng = StepEngine(w.scene, w.cfg, w.loss, 60, use_graph=True, host_io=hostio, band=band)
if hostio:  # the e2e graph: refresh from host parameters, bin, step, Adam only
    eng.run(2)
    eng.capture_host_io_step()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
lib = nat.load()
names = {0: "k_bin_rows", 1: "k_step", 2: "k_prim<adam>", 3: "k_prim<pre>", 4: " .adam done",
         5: " .fold done", 6: " .records done", 7: " .ticket done", 8: " bin.scan / K1 records stored",
         9: " bin.list / K1 scatter done", 10: " bin.counts done", 11: "k_row_counts", 12: "k_row_scatter", 13: "k_row_offsets",
         14: " .lists sorted", 15: " .barrier passed"}
for rep in range(12):
    flush.zero_()
    torch.cuda.synchronize()
    lib.pf_timeline_reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.host_step() if hostio else eng.step()
    e1.record()
    torch.cuda.synchronize()
    buf = np.zeros(64, dtype=np.uint64)
    lib.pf_timeline_dump(buf.ctypes.data_as(C.c_void_p))
if True:
    b = buf.reshape(16, 4).astype(np.float64)
    valid = [k for k in range(16) if b[k, 3] > 0 or b[k, 2] > 0]
    t0 = min(b[k, 0] for k in valid if b[k, 3] > 0)
    print(f"step (events) {e0.elapsed_time(e1) * 1e3:.1f} us; kernels (start / wait-done min..max / end, us from first start):")
    for k in valid:
        if b[k, 3] > 0:
            print(f"  {names[k]:14s} start {(b[k,0]-t0)/1e3:6.1f}  wait {(b[k,1]-t0)/1e3:6.1f}..{(b[k,2]-t0)/1e3:6.1f}  end {(b[k,3]-t0)/1e3:6.1f}")
        else:
            print(f"  {names[k]:14s} min {(b[k,1]-t0)/1e3:6.1f}  max {(b[k,2]-t0)/1e3:6.1f}")
