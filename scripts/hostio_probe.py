"""Diagnostics: cost of the zero-copy host parameter read / write at c3."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch

from paper_2602_22625_b200 import synth
from paper_2602_22625_b200.fit import StepEngine

w = synth.make_workload("c3")
w.cfg.num_iterations = 4000
eng = StepEngine(w.scene, w.cfg, w.loss, 4000, use_graph=True)
eh = StepEngine(w.scene, w.cfg, w.loss, 4000, use_graph=True, host_io=True)
eng.run(3)
eh.run(3)
eh.capture_host_io_step()
torch.cuda.synchronize()


def ev_time(fn, k=200):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k * 1e3


print(f"refresh (device params)      {ev_time(eng.refresh):7.2f} us")
print(f"refresh (host params)        {ev_time(eh.refresh):7.2f} us")


def g_dev():
    eng.graph.replay(); eng.done += 1


def g_host():
    eh.host_graph.replay(); eh.done += 1


def g_host_noref():
    eh.graph.replay(); eh.done += 1


print(f"device step graph            {ev_time(g_dev, 100):7.2f} us")
print(f"host_io step graph (no sync) {ev_time(g_host, 100):7.2f} us")
print(f"host_io w/o refresh          {ev_time(g_host_noref, 100):7.2f} us")
