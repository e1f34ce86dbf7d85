#!/usr/bin/env python
"""Benchmark: optimisation steps/s (bin + fwd + loss + bwd + Adam + psnr) of the
B200 compositor on BASELINE.json's metric config (c3: 1024x809, 3000
fingerprint + 2000 autograph primitives) with synthetic, seeded inputs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

Prints ONE JSON line (rank 0).  --impl reference times the reference's CPU
algorithm (the C/OpenMP oracle port, oracle/) on the host cores instead.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

METRIC = "optimisation steps/sec (fwd+bwd+Adam) at 1024x809, 5000 prims; % HBM roofline"
UNIT = "steps/s"
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2


def _peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "src": "measured"}
    return {"hbm_gbs": 6650.0, "src": "fallback"}


def algorithmic_bytes(P: int, K16: int, N: int, atlas_texels: int) -> dict:
    """B_step = 68 P + 12 K16 + 288 N + A, A = 16 * texels (the
    fp32 model of the reference's per-step tensors), split by the kernel that
    does that work in this implementation:
      bin   (K2)    the bin index written                       4 K16
      step  (K34)   every per-pixel term (the render, loss and
                    backward all run in it), the index read by
                    forward and backward, the gradient write, A  68 P + 8 K16 + 32 N + A
      adam  (K1+K5) parameter read in preprocess + the Adam
                    touches (p r/w, m r/w, v r/w, g r)          256 N
    The two-kernel path splits `step` into forward 48 P + 4 K16 + A and
    backward 20 P + 4 K16 + 32 N."""
    A = 16 * atlas_texels
    return {
        "total": 68 * P + 12 * K16 + 288 * N + A,
        "bin": 4 * K16,
        "step": 68 * P + 8 * K16 + 32 * N + A,
        "adam": 256 * N,
        "forward": 48 * P + 4 * K16 + A,
        "backward": 20 * P + 4 * K16 + 32 * N,
    }


def compulsory_bytes(P: int, K16: int, N: int, atlas_texels: int) -> int:
    """This implementation's own compulsory HBM traffic of the fused K34 launch
    (target in, per-entry index + staged records, atlas; the image, dL/dI and the
    contribution lists never leave the SM): 16 P + 4 K16 + 256 N + A.  Reported
    beside the §8(d) figure; ncu's dram bytes per launch sit close to it."""
    return 16 * P + 4 * K16 + 256 * N + 16 * atlas_texels


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling via NVML during the timed region."""

    def __init__(self, index: int = 0, period: float = 0.05):
        self.samples: list[tuple[int, int]] = []
        self.reasons_seen: set[str] = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        self.ok = False
        try:
            import pynvml as nv

            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.period = period
            self.ok = True
        except Exception:
            self.ok = False

    _REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
        "display_clock_setting": 0x100,
    }

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((sm, rs))
                for name, bit in self._REASONS.items():
                    if rs & bit and name != "gpu_idle":
                        self.reasons_seen.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def start(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self) -> dict:
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml-unavailable"]}
        self._stop.set()
        if self._t:
            self._t.join()
        sm = [s for s, _ in self.samples]
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons_seen), "samples": len(sm)}


def cpu_baseline(config: str, max_seconds: float = 15.0, max_steps: int = 20) -> dict:
    """The reference's CPU algorithm (C/OpenMP oracle port) on this host, bounded sample."""
    import cpu_oracle as orc

    from paper_2602_22625_b200 import synth
    from paper_2602_22625_b200.fit import effective_padding

    orc.build()
    w = synth.make_workload(config)
    loop = orc.Loop(w.scene, w.target, w.cfg, effective_padding(w.cfg), tile=32)
    total = w.steps
    loop.step(0, total)  # untimed warm-up step (reference protocol: warmup + untimed step)
    times = []
    t_all = time.perf_counter()
    it = 1
    while it < total and len(times) < max_steps and time.perf_counter() - t_all < max_seconds:
        t0 = time.perf_counter()
        loop.step(it, total)
        times.append(time.perf_counter() - t0)
        it += 1
    med = float(np.median(times))
    return {"value": 1.0 / med, "unit": UNIT, "cores": orc.threads(), "kind": "port",
            "sample": f"{config}: {len(times)} timed run_loop-body steps (median; after 1 untimed)",
            "ms_per_step": med * 1e3, "cpu_model": _cpu_model()}


def numba_reference_baseline(config: str, timeout_s: float = 300.0) -> dict | None:
    """The UNMODIFIED numba reference (baseline/_ref) timed on its own run_loop
    body (scripts/numba_ref_step.py, subprocess: numba's pool owns every core),
    or None when it is not installed / not importable on this host."""
    import subprocess

    if not (ROOT / "baseline" / "_ref" / "primfit").is_dir():
        return None
    try:
        r = subprocess.run([sys.executable, str(ROOT / "scripts" / "numba_ref_step.py"), config,
                            "5", "15"], capture_output=True, text=True, timeout=timeout_s)
        out = json.loads(r.stdout.strip().splitlines()[-1])
        out["cpu_model"] = _cpu_model()
        return out
    except Exception as exc:  # noqa: BLE001 - a reported reading, never the product
        return {"unavailable": f"{type(exc).__name__}: {exc}"[:200]}


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import cpu_oracle as orc

    from paper_2602_22625_b200 import synth
    from paper_2602_22625_b200.fit import effective_padding

    orc.build()
    w = synth.make_workload(args.config)
    loop = orc.Loop(w.scene, w.target, w.cfg, effective_padding(w.cfg), tile=32)
    total = max(w.steps, args.warmup + args.steps)
    for it in range(args.warmup):
        loop.step(it, total)
    t0 = time.perf_counter()
    for it in range(args.warmup, args.warmup + args.steps):
        loop.step(it, total)
    dt = time.perf_counter() - t0
    v = args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": _config(args.config, w),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": orc.threads(), "kind": "port",
                         "sample": f"{args.config}: {args.steps} run_loop-body steps after "
                                   f"{args.warmup} warm-up (C/OpenMP port of the reference, "
                                   f"float64, bit-identical to it on golden vectors)",
                         "cpu_model": _cpu_model()},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "cpu_baseline_reference": numba_reference_baseline(args.config),
    }
    print(json.dumps(line), flush=True)


def _config(name: str, w) -> dict:
    sc = w.scene
    return {"workload": f"{name}: {sc.canvas_w}x{sc.canvas_h}, {sc.n} prims, "
                        f"{len(sc.templates)} templates, loss {w.loss.kind}",
            "canvas": [sc.canvas_w, sc.canvas_h], "primitives": sc.n,
            "templates": len(sc.templates), "render_tile": 16,
            "l2": "flushed (256 MiB write) before every timed step"}


KNAME = {"step": "k_step", "forward": "k_forward", "backward": "k_backward"}


def ncu_summary(kernel_prefix: str, config: str = "c3") -> dict | None:
    """The named kernel's entry of the newest committed ncu --set full summary
    of this config under profiles/ (scripts/ncu_extract.py), or None."""
    import re

    def version(f: Path) -> tuple:  # r02b_* after r02_* after r01_*_v11
        m = re.match(r"r(\d+)([a-z]?)_", f.stem)
        tail = f.stem.rsplit("_v", 1)
        return (int(m.group(1)) if m else -1, m.group(2) if m else "",
                int(tail[1]) if len(tail) == 2 and tail[1].isdigit() else -1)

    files = sorted((ROOT / "profiles").glob("*ncu_kernels*.json"), key=version)
    # summaries named for a config (r02*_ncu_kernels_<config>.json) count only for it
    files = [f for f in files if not re.search(r"_c\d", f.stem) or f.stem.endswith("_" + config)]
    for f in reversed(files):
        try:
            d = json.loads(f.read_text())
        except (OSError, ValueError):
            continue
        for name, v in d.items():
            if kernel_prefix in name and "dram_traffic_bytes" in v:
                return v
    return None


def issue_frac(kernel_prefix: str, config: str = "c3", sms: int = 148,
               mhz: float = 1965.0) -> float | None:
    """Issued warp instructions per SM per cycle / 4 (one issue per SMSP per cycle)
    for the named kernel, from the committed ncu summary (duration at SM clock)."""
    v = ncu_summary(kernel_prefix, config)
    if not v or not v.get("warp_instructions") or not v.get("duration_ns"):
        return None
    cycles = float(v["duration_ns"]) * 1e-9 * mhz * 1e6
    return float(v["warp_instructions"]) / (sms * cycles) / 4.0


def ncu_traffic(kernel_prefix: str, config: str = "c3") -> float | None:
    """dram bytes (read + write) per launch of the named kernel (ncu summary), or None."""
    v = ncu_summary(kernel_prefix, config)
    return float(v["dram_traffic_bytes"]) if v else None


def autograd_bench(w, steps: int, warmup: int, flush) -> dict:
    """The north_star's autograd entry point in a plain training loop: the
    Renderer's torch.autograd.Function (K1+K2+K3 forward; backward = the fit-step
    kernel on the upstream gradients) under a torch MSE loss, then the device Adam
    (pf_adam table mode), no host sync per step (s_max bounds the capacity).
    Again with the fused ``autograd.loss_mse`` in place of the torch loss.
    CUDA-event timed, L2 flushed per step."""
    import torch

    from paper_2602_22625_b200.autograd import Renderer, loss_mse
    from paper_2602_22625_b200.compositor import adam_launch
    from paper_2602_22625_b200.fit import _cfg_gains, effective_padding, lr_schedule
    from paper_2602_22625_b200.scene import param_matrix, structure_arrays

    sc, cfg = w.scene, w.cfg
    tid, z = structure_arrays(sc)
    r = Renderer(sc.templates, tid, z, sc.canvas_w, sc.canvas_h,
                 background=tuple(sc.background), alpha_max=sc.alpha_max,
                 mu_blend=sc.mu_blend, preserve_aspect=sc.preserve_aspect,
                 eps_skip=cfg.eps_skip, padding=effective_padding(cfg), s_max=cfg.scale_max)
    dev = torch.device("cuda")
    params = torch.tensor(param_matrix(sc), device=dev, requires_grad=True)
    target = torch.tensor(w.target, device=dev, dtype=torch.float32)
    n = params.shape[0]
    m = torch.zeros(n * 8, dtype=torch.float64, device=dev)
    v = torch.zeros_like(m)
    total = 4 * (warmup + steps) + 8  # eager warm-up + timed, then the graphed run (x2)
    lr = torch.tensor([lr_schedule(i, total, cfg.learning_rate) for i in range(total)],
                      dtype=torch.float64, device=dev)
    bc1 = torch.tensor([1 - 0.9 ** (i + 1) for i in range(total)], dtype=torch.float64, device=dev)
    bc2 = torch.tensor([1 - 0.999 ** (i + 1) for i in range(total)], dtype=torch.float64,
                       device=dev)
    it = torch.zeros(1, dtype=torch.int32, device=dev)
    ctr = torch.zeros(1, dtype=torch.int32, device=dev)
    gains = _cfg_gains(cfg)

    fused = [False]

    def step():
        img, _ = r(params)
        loss = loss_mse(img, target) if fused[0] else ((img - target) ** 2).mean()
        loss.backward()
        with torch.no_grad():
            adam_launch(params.view(-1), params.grad.view(-1), m, v, gains=gains, n=n,
                        lr_table=lr, bc1_table=bc1, bc2_table=bc2, iter_counter=it, counter=ctr,
                        clamp=True, s_min=cfg.scale_min, s_max=cfg.scale_max, zero_grads=False)
        params.grad = None  # (torch's zero_grad(set_to_none=True))

    def measure() -> tuple[float, float]:
        for _ in range(warmup):
            step()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps)]
        for e0, e1 in evs:
            flush.zero_()
            e0.record()
            step()
            e1.record()
        torch.cuda.synchronize()
        r.check()
        ms = sum(a.elapsed_time(b) for a, b in evs) / steps
        # the same training step captured once in a CUDA graph (torch.cuda.graph
        # recipe: side-stream warm-up, capture, replay) -- the launch-bound eager
        # loop without its Python / ctypes overhead
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(2):
                step()
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        for _ in range(warmup):
            g.replay()
        torch.cuda.synchronize()
        gevs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in range(steps)]
        for e0, e1 in gevs:
            flush.zero_()
            e0.record()
            g.replay()
            e1.record()
        torch.cuda.synchronize()
        r.check()
        return ms, sum(a.elapsed_time(b) for a, b in gevs) / steps

    ms, gms = measure()
    fused[0] = True
    fms, fgms = measure()
    return {"value": 1e3 / ms, "unit": UNIT, "ms_per_step": ms,
            "path": "autograd.Renderer forward (K1+K2+K3) + torch MSE + backward (the fit-step "
                    "kernel on the upstream gradients) + pf_adam; no host sync per step",
            "graphed": {"value": 1e3 / gms, "unit": UNIT, "ms_per_step": gms,
                        "path": "the same step captured in one CUDA graph (torch.cuda.graph)"},
            "fused_loss": {"value": 1e3 / fms, "unit": UNIT, "ms_per_step": fms,
                           "graphed": {"value": 1e3 / fgms, "unit": UNIT, "ms_per_step": fgms},
                           "path": "the same step with autograd.loss_mse (fused MSE op) in "
                                   "place of the torch loss"},
            "l2": "flushed (256 MiB write) before every timed step"}


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_2602_22625_b200 import synth
    from paper_2602_22625_b200.dist import make_allreduce, row_bands
    from paper_2602_22625_b200.fit import StepEngine

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # (diagnostics: PF_DIST_BACKEND=gloo runs the N > 1 code path with every rank on
    # one device -- the c4 frame replicas only: a gloo allreduce cannot be captured
    # in the row-band step graph)
    backend = os.environ.get("PF_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    w = synth.make_workload(args.config)
    sc = w.scene
    H, W = sc.canvas_h, sc.canvas_w
    nty = -(-H // 16)
    # c4 (video frames) is sharded by frames (BASELINE.json configs[3]): every rank
    # fits its own frame -- a replica of the full-canvas step, no collective;
    # the other configs split the canvas into row bands + a gradient allreduce
    frames = args.config == "c4" and world > 1
    band = row_bands(nty, 1 if frames else world)[0 if frames else rank]
    reduce = make_allreduce() if world > 1 and not frames else None
    prof_steps = 20
    e2e_steps = max(10, args.steps // 2)  # per e2e mode (two modes)
    loop_chunks = 10
    total = max(w.steps, args.warmup + args.steps + prof_steps + 2 * e2e_steps + 2 +
                loop_chunks * StepEngine.CHUNK + StepEngine.CHUNK)
    w.cfg.num_iterations = total
    eng = StepEngine(sc, w.cfg, w.loss, total, band=band, allreduce=reduce, use_graph=True)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")

    # warm-up (step 0 eager + CUDA-graph capture, then replays)
    eng.run(args.warmup)
    torch.cuda.synchronize()
    eng.check()
    K16 = int(eng.comp.status[0].item())

    # timed region: K graph replays, L2 flushed (untimed) before each
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    for e0, e1 in evs:
        flush.zero_()
        e0.record()
        eng.step()
        e1.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    ms_total = sum(e0.elapsed_time(e1) for e0, e1 in evs)
    t = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    ms_step = ms_total / args.steps
    # whole-job steps/s: every rank advances the same step (row bands), or its own
    # frame's step (c4 frame sharding: world frame-steps per step time)
    value = (world if frames else 1) * 1e3 / ms_step

    # per-stage timing (eager, events on the launching stream, L2 flushed)
    stage_ms: dict[str, float] = {}
    for _ in range(prof_steps):
        flush.zero_()
        marks = [("start", torch.cuda.Event(enable_timing=True))]
        marks[0][1].record()

        def mark(name):
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            marks.append((name, ev))

        eng.launch_step(mark)
        torch.cuda.synchronize()
        eng.done += 1
        for (_, e0), (name, e1) in zip(marks, marks[1:]):
            stage_ms[name] = stage_ms.get(name, 0.0) + e0.elapsed_time(e1) / prof_steps

    # end-to-end through the public step API with HOST buffers each step: the
    # parameter vector and the loss partials live in pinned host memory
    # (StepEngine(host_io=True)); one graph per step reads the parameters over
    # the host link (preprocess), bins, renders, runs the backward and Adam, and
    # writes the updated vector + the step's loss partials back to host memory
    # (zero-copy), then a host synchronisation: the host holds the step's result
    # (the next step's input) before the next.
    eh = StepEngine(sc, w.cfg, w.loss, total, band=band, allreduce=reduce, use_graph=True,
                    host_io=True)
    eh.run(args.warmup)
    torch.cuda.synchronize()
    eh.capture_host_io_step()
    n = eh.n
    nb = eh.adam_blocks
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # (1) pipelined, the headline: the host enqueues step k, then reads step
    #     k-1's loss (waiting for that step only), so at most two steps are in
    #     flight and the host's launch / read latency overlaps the device work
    # (2) synchronous: the host waits for every step before enqueueing the next
    def e2e_run(pipelined: bool) -> float:
        e_start = torch.cuda.Event(enable_timing=True)
        e_end = torch.cuda.Event(enable_timing=True)
        losses = []
        e_start.record()
        for k in range(e2e_steps):
            eh.host_step()
            if not pipelined:
                losses.append(float(eh.host_loss_part(-1)[:, 0].sum()))
            elif k > 0:
                losses.append(float(eh.host_loss_part(-2)[:, 0].sum()))
        if pipelined:
            losses.append(float(eh.host_loss_part(-1)[:, 0].sum()))
        e_end.record()
        torch.cuda.synchronize()
        assert len(losses) == e2e_steps and np.isfinite(losses).all()
        ms = e_start.elapsed_time(e_end) / e2e_steps
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    e2e_sync_ms = e2e_run(False)
    e2e_ms = e2e_run(True)
    eng.check()
    eh.check()

    # run_loop's own issue pattern (informative, not the headline): CHUNK-step
    # graphs back to back, no L2 flush between steps
    loop = None
    if world == 1:
        eng.run(StepEngine.CHUNK)  # captures the chunk graph
        torch.cuda.synchronize()
        l0, l1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0.record()
        eng.run(loop_chunks * StepEngine.CHUNK)
        l1.record()
        torch.cuda.synchronize()
        loop_ms = l0.elapsed_time(l1) / (loop_chunks * StepEngine.CHUNK)
        loop = {"value": 1e3 / loop_ms, "unit": UNIT, "steps_per_graph": StepEngine.CHUNK,
                "l2": "not flushed (back-to-back steps, as run_loop issues them)"}
        eng.check()

    autograd = None
    if world == 1 and not args.no_autograd:
        autograd = autograd_bench(w, max(10, args.steps // 2), 3, flush)

    nodes = eng.kernels_per_step
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    peaks = _peaks()
    ab = algorithmic_bytes(eng.P, K16, n, eng.atlas.texels)
    dom = max(("forward", "backward", "step"), key=lambda k: stage_ms.get(k, 0.0))
    achieved = ab[dom] / (stage_ms[dom] * 1e-3) / 1e9
    comp_b = compulsory_bytes(eng.P, K16, n, eng.atlas.texels)
    cpu = cpu_baseline(args.config) if (world == 1 and not args.no_cpu) else None
    cpu_ref = numba_reference_baseline(args.config) if (world == 1 and not args.no_cpu) else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak" if frames else "strong", "vs_baseline": None,
        "dtype": "mixed (f64 decisions/params/Adam, f32 compositing/gradients)",
        "data": "synthetic (seeded structure-aware init; procedural templates; smooth random target)",
        "config": {**_config(args.config, w),
                   "parallelism": f"frames{world}" if frames else f"rowband{world}",
                   "K16": K16, "band": [band.ty_begin, band.ty_end]},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved,
                     "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / peaks["hbm_gbs"],
                     "traffic": ncu_traffic(KNAME[dom], args.config),
                     "peak_src": peaks["src"], "algorithmic_bytes": ab[dom],
                     "bytes_model": "SURVEY 8(d) share of the dominant kernel: "
                                    "68 P + 8 K16 + 32 N + 16 texels",
                     "kernel_ms": stage_ms[dom],
                     # the whole step: 8(d) B_step over the device-timed step
                     "step_frac": ab["total"] * value / 1e9 / peaks["hbm_gbs"],
                     "step_bytes": ab["total"],
                     # this implementation's compulsory traffic of the same launch
                     "compulsory_bytes": comp_b,
                     "compulsory_frac": comp_b / (stage_ms[dom] * 1e-3) / 1e9 / peaks["hbm_gbs"],
                     # what does bound it: instruction issue (ncu summary of the
                     # same kernel: warp instructions per SM cycle against 4)
                     "issue_frac": issue_frac(KNAME[dom], args.config)},
        # SURVEY 8(d) secondary unit: binned (pixel, list entry) evaluations per
        # second (256 pixels per tile-list entry at tile 16), plus the ncu L1/tex
        # hit rate and warp execution efficiency of the dominant kernel
        "secondary": {"pair_evals_per_s": 256.0 * K16 * value, "unit": "pairs/s",
                      "ncu": {k: (ncu_summary(KNAME[dom], args.config) or {}).get(k)
                              for k in ("l1tex_hit_pct", "warp_exec_efficiency_threads",
                                        "fp64_pipe_pct", "warps_active_pct")}},
        "run_loop": loop,
        "autograd": autograd,
        "stage_ms": stage_ms,
        "e2e": {"value": (world if frames else 1) * 1e3 / e2e_ms, "unit": UNIT,
                "h2d_bytes_per_step": n * 8 * 8,
                "d2h_bytes_per_step": n * 8 * 8 + nb * 3 * 8,
                "mode": "pipelined host loop (step k enqueued, then step k-1's loss read)",
                "sync_value": (world if frames else 1) * 1e3 / e2e_sync_ms},
        "gpu_launches": (nodes * args.steps) if nodes else None,
        "kernels_per_step": nodes,
        "clocks": clk,
        "cpu_baseline": cpu,
        # second CPU reading: the unmodified numba reference itself (slower than
        # the port above, which stays the baseline)
        "cpu_baseline_reference": cpu_ref,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--no-autograd", action="store_true", help="skip the autograd sub-line")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
