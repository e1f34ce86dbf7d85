"""Diagnostics: per-warp wait/work cycles of pf_fit_step (PF_STEP_PROF=1 build path)."""
import ctypes as C
import os
import sys
from pathlib import Path

os.environ["PF_STEP_PROF"] = "1"
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

from paper_2602_22625_b200 import _native as nat, synth
from paper_2602_22625_b200.fit import StepEngine

w = synth.make_workload(sys.argv[1] if len(sys.argv) > 1 else "c3")
w.cfg.num_iterations = 40
band = None
for arg in sys.argv[2:]:
    if arg.startswith("band="):  # band=N:r -- rank r of an N-way uniform row split
        from paper_2602_22625_b200.dist import row_bands
        N, r = (int(v) for v in arg[5:].split(":"))
        band = row_bands(-(-w.scene.canvas_h // 16), N)[r]
eng = StepEngine(w.scene, w.cfg, w.loss, 40, use_graph=False, band=band)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for _ in range(12):
    flush.zero_()
    eng.step()
torch.cuda.synchronize()
lib = nat.load()
lib.pf_step_prof_dump.restype = C.c_int
buf = np.zeros((148 * 32, 6), dtype=np.uint64)
n = lib.pf_step_prof_dump(buf.ctypes.data_as(C.c_void_p), 148 * 32)
buf = buf[:n][buf[:n, 3] > 0]  # padding warps leave their slot empty
n = len(buf)
d = buf.astype(np.float64)
kind = buf[:n, 5] & 1
first = (buf[:n, 5] >> 1).astype(np.float64)
prod = kind == 1
cons = ~prod
t0 = d[:, 3].min()
print(f"slots {n}: kernel span {(d[:, 4].max() - t0) / 1e3:.1f} us; start spread {(d[:, 3].max() - t0) / 1e3:.1f} us")
for name, m in (("consumer", cons), ("producer", prod)):
    x = d[m]
    print(f"{name}: wait {x[:, 0].mean() / 1965:.1f} us  work {x[:, 1].mean() / 1965:.1f} us  n {x[:, 2].mean():.2f}  "
          f"end spread {(x[:, 4].min() - t0) / 1e3:.1f}..{(x[:, 4].max() - t0) / 1e3:.1f} us  "
          f"first {first[m].mean() / 1965:.1f} us")

xe = (d[cons][:, 4] - t0) / 1e3
xs = (d[cons][:, 3] - t0) / 1e3
print("consumer end percentiles (us) p0/p10/p50/p90/p100:",
      [round(float(np.percentile(xe, q)), 1) for q in (0, 10, 50, 90, 100)])
print("consumer start percentiles (us):", [round(float(np.percentile(xs, q)), 1) for q in (0, 50, 100)])
busy = d[cons][:, 1].sum() / 1965 / 1e0
print(f"total consumer work {busy / 1e3:.1f} ms-warp; ideal span at {cons.sum()} warps {busy / cons.sum():.1f} us")
nt = eng.comp.n_tiles
tb = np.zeros((nt, 8), dtype=np.uint64)
lib.pf_step_prof_tiles(tb.ctypes.data_as(C.c_void_p), nt)
dur = (tb & 0xffffffff).astype(np.float64) / 1965.0  # us per (tile, warp)
endt = (tb >> 32).astype(np.float64)
if eng.comp.slots is not None:  # slot mode: the lists of the current parameters
    eng.refresh()
    off, _ = eng.comp.slot_lists()
else:
    off = eng.comp.bin_off.cpu().numpy()
L = np.diff(off)
tmax = dur.max(axis=1)
print(f"tile max-warp time: mean {tmax.mean():.2f} p50 {np.median(tmax):.2f} p90 {np.percentile(tmax, 90):.2f} max {tmax.max():.2f} us; warp mean {dur.mean():.2f}")
print("corr(L, tmax)", np.corrcoef(L, tmax)[0, 1])
for lo, hi in ((0, 8), (8, 16), (16, 24), (24, 33), (33, 999)):
    m = (L >= lo) & (L < hi)
    if m.any():
        print(f"  L in [{lo},{hi}): n={m.sum():5d} tmax mean {tmax[m].mean():.2f} us")
# which tiles finish last
e = endt.max(axis=1)
order = np.argsort(e)[-10:]
print("last tiles:", [(int(t), int(L[t]), round(float(tmax[t]), 1)) for t in order])

# slot-mode prologue span per CTA (wait done -> lists sorted)
allp = np.zeros(148 * 6, dtype=np.uint64)
lib.pf_step_prof_prologue(allp.ctypes.data_as(C.c_void_p), 148)
pro = allp[: 2 * 148].reshape(148, 2)
ph = allp[2 * 148 :].reshape(148, 4).astype(np.float64)
ok = pro[:, 1] > 0
if ok.any():
    p0 = pro[ok].astype(np.float64)
    span = (p0[:, 1] - p0[:, 0]) / 1e3
    st = (p0[:, 0] - p0[:, 0].min()) / 1e3
    print("prologue span per CTA (us) p0/p50/p90/p100:",
          [round(float(np.percentile(span, q)), 2) for q in (0, 50, 90, 100)],
          " start offset max", round(float(st.max()), 2),
          " slowest CTAs:", list(np.argsort(span)[-5:]))
    okp = ok & (ph[:, 0] > 0)
    if okp.any():
        b0 = pro[okp, 0].astype(np.float64)
        for k, name in enumerate(("first batch landed", "tiles sorted", "classes written")):
            d = (ph[okp, k] - b0) / 1e3
            print(f"  {name:20s} after prologue start: p50 {np.median(d):.2f} max {d.max():.2f} us")
