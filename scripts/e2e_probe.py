"""Diagnostics: where the e2e (host-driven step) time goes at c3."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

from paper_2602_22625_b200 import synth
from paper_2602_22625_b200.fit import StepEngine

w = synth.make_workload("c3")
w.cfg.num_iterations = 2000
eng = StepEngine(w.scene, w.cfg, w.loss, 2000, use_graph=True)
eng.run(5)
torch.cuda.synchronize()
n = eng.n
hp = torch.empty(n * 8, dtype=torch.float64, pin_memory=True)
hp.copy_(eng.params.view(-1).cpu())
hl = torch.empty(n * 8 + eng.adam_blocks * 3, dtype=torch.float64, pin_memory=True)
eng.capture_host_step(hp, hl)


def timeit(name, fn, k=100):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / k * 1e6
    print(f"{name:40s} {dt:7.1f} us")


def graph_only():
    eng.graph.replay(); eng.done += 1


def graph_sync():
    eng.graph.replay(); eng.done += 1
    torch.cuda.current_stream().synchronize()


def host_step_sync():
    eng.host_step()
    torch.cuda.current_stream().synchronize()


def h2d_only():
    eng.params.view(-1).copy_(hp, non_blocking=True)
    torch.cuda.current_stream().synchronize()


def d2h_only():
    hp.copy_(eng.params.view(-1), non_blocking=True)
    torch.cuda.current_stream().synchronize()


def refresh_only():
    eng.refresh()
    torch.cuda.current_stream().synchronize()


timeit("graph replay (no sync)", graph_only)
timeit("graph replay + sync", graph_sync)
timeit("host step graph + sync", host_step_sync)
timeit("H2D 320 KB + sync", h2d_only)
timeit("D2H 320 KB + sync", d2h_only)
timeit("refresh kernel + sync", refresh_only)
timeit("empty sync", lambda: torch.cuda.current_stream().synchronize())

# zero-copy host buffer engine
eh = StepEngine(w.scene, w.cfg, w.loss, 2000, use_graph=True, host_io=True)
eh.run(5)
torch.cuda.synchronize()
eh.capture_host_io_step()
hv = eh.io.numpy()


def host_io_step():
    eh.host_step()
    torch.cuda.current_stream().synchronize()
    float(hv[eh.n * 8 :: 3].sum())


def host_io_dev_graph():
    eh.graph.replay(); eh.done += 1
    torch.cuda.current_stream().synchronize()


timeit("host_io step (zero-copy) + sync", host_io_step, 300)
timeit("host_io device graph + sync", host_io_dev_graph, 300)
timeit("host step graph + sync (again)", host_step_sync, 300)
# parity: the two engines ran the same number of steps from the same init
eng2 = StepEngine(w.scene, w.cfg, w.loss, 2000, use_graph=True)
eh2 = StepEngine(w.scene, w.cfg, w.loss, 2000, use_graph=True, host_io=True)
eng2.run(20); eh2.run(20)
torch.cuda.synchronize()
print("host_io vs device params max abs diff:",
      float((eng2.params.cpu() - eh2.params.cpu()).abs().max()))
