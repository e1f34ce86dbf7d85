"""The multi-rank fit step executed, on one GPU.

1. Real ranks: 2 and 4 processes share cuda:0, each a ``StepEngine`` on its row
   band with ``allreduce = dist.make_allreduce()`` over a ``gloo`` process group
   (gloo reduces CUDA tensors through host memory; NCCL refuses two ranks on one
   device).  Every rank must end with bit-identical parameters and history, and
   the run must equal the single-rank engine under the Adam-noise bar of
   test_step_engine_matches_oracle_loop.
2. Graph capture around a foreign kernel: ``LocalBandGroup`` runs all bands of a
   split in one process, with the allreduce replaced by the in-stream band sum
   (pf_sum_bands), the whole group step captured in ONE CUDA graph (PDL edges
   between the engines' kernels and the sum kernel).
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
STEPS = 6


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _single_rank(name: str, steps: int):
    from paper_2602_22625_b200 import synth
    from paper_2602_22625_b200.fit import StepEngine

    w = synth.make_workload(name)
    w.cfg.num_iterations = steps
    eng = StepEngine(w.scene, w.cfg, w.loss, steps, use_graph=False)
    for _ in range(steps):
        eng.step()
    eng.check()
    return eng.params_host().reshape(-1, 8), np.array([h.loss for h in eng.history()])


def _rank_main(rank, world, name, steps, out_dir):
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2602_22625_b200 import synth
    from paper_2602_22625_b200.dist import make_allreduce, row_bands
    from paper_2602_22625_b200.fit import StepEngine

    w = synth.make_workload(name)
    w.cfg.num_iterations = steps
    nty = -(-w.scene.canvas_h // 16)
    band = row_bands(nty, world)[rank]
    eng = StepEngine(w.scene, w.cfg, w.loss, steps, band=band, allreduce=make_allreduce(),
                     use_graph=False)
    for _ in range(steps):
        eng.step()
    eng.check()
    st = eng.sync_state()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), params=eng.params_host(),
             loss=np.array([h.loss for h in eng.history()]),
             psnr=np.array([h.psnr for h in eng.history()]), m=st.m, v=st.v,
             band=np.array([band.ty_begin, band.ty_end]))
    dist.barrier()
    dist.destroy_process_group()


def _adam_bar(p, p_ref, cfg, steps):
    # Adam normalises each gradient by its own RMS: a component that is zero up
    # to round-off takes a +-lr*gain step whose sign is atomic-order noise
    close = np.isclose(p, p_ref, rtol=1e-4, atol=1e-4)
    assert close.mean() > 0.99, close.mean()
    gains = np.asarray([10, 10, 10, 1, 1.5, 1, 1, 1.0])
    assert np.all(np.abs(p - p_ref) <= 2 * cfg.learning_rate * gains[None, :] * steps)


@pytest.mark.parametrize("world", [2, 4])
def test_multirank_step_engine_gloo(torch_cuda, tmp_path, world):
    import torch.multiprocessing as mp

    from paper_2602_22625_b200 import synth

    os.environ["MASTER_PORT"] = str(29600 + (os.getpid() % 1000) + world)
    mp.spawn(_rank_main, args=(world, "c3", STEPS, str(tmp_path)), nprocs=world, join=True)
    runs = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]
    bands = [tuple(r["band"]) for r in runs]
    assert bands[0][0] == 0 and all(a[1] == b[0] for a, b in zip(bands, bands[1:]))
    for r in runs[1:]:  # replicas identical bit for bit
        np.testing.assert_array_equal(r["params"], runs[0]["params"])
        np.testing.assert_array_equal(r["loss"], runs[0]["loss"])
        np.testing.assert_array_equal(r["m"], runs[0]["m"])
        np.testing.assert_array_equal(r["v"], runs[0]["v"])
    p1, loss1 = _single_rank("c3", STEPS)
    np.testing.assert_allclose(runs[0]["loss"], loss1, rtol=1e-5)
    cfg = synth.make_workload("c3").cfg
    _adam_bar(runs[0]["params"].reshape(-1, 8), p1, cfg, STEPS)


@pytest.mark.parametrize("name,world", [("c3", 2), ("c3", 4), ("c5", 8)])
def test_local_band_group_graph(torch_cuda, name, world):
    """All bands in one process, the allreduce replaced by the in-stream band sum,
    the group step captured in one CUDA graph: bands bit-identical, equal to the
    single-rank engine under the Adam-noise bar."""
    torch = torch_cuda
    from paper_2602_22625_b200 import synth
    from paper_2602_22625_b200.dist import LocalBandGroup

    steps = 4 if name == "c5" else STEPS
    w = synth.make_workload(name)
    w.cfg.num_iterations = steps
    grp = LocalBandGroup(w.scene, w.cfg, w.loss, steps, world, use_graph=True)
    for _ in range(steps):
        grp.step()
    torch.cuda.synchronize()
    assert grp.graph is not None
    for e in grp.engines:
        e.check()
    ref = grp.engines[0]
    for e in grp.engines[1:]:
        np.testing.assert_array_equal(e.params_host(), ref.params_host())
        assert [h.loss for h in e.history()] == [h.loss for h in ref.history()]
    p1, loss1 = _single_rank(name, steps)
    np.testing.assert_allclose([h.loss for h in ref.history()], loss1, rtol=1e-5)
    _adam_bar(ref.params_host().reshape(-1, 8), p1, w.cfg, steps)


def test_sum_bands_fixed_order(torch_cuda):
    """pf_sum_bands: fixed-order float64 sum written to every destination, slices."""
    torch = torch_cuda
    from paper_2602_22625_b200.dist import sum_bands

    g = torch.Generator(device="cpu").manual_seed(3)
    bufs = [(torch.randn(10007, generator=g, dtype=torch.float64) * 10 ** k).cuda()
            for k in range(5)]
    ref = bufs[0].cpu().clone()
    for b in bufs[1:]:
        ref += b.cpu()
    outs = [torch.zeros_like(bufs[0]) for _ in range(3)]
    sum_bands(bufs, outs, 0, 5000)
    sum_bands(bufs, outs, 5000, 10007)
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o.cpu(), ref)
    sum_bands(bufs)  # in place
    for b in bufs:
        assert torch.equal(b.cpu(), ref)


def _video_frames():
    from paper_2602_22625_b200 import synth

    w = synth.make_workload("c1")
    f0 = w.target
    frames = [f0]
    for k in range(1, 4):  # a region that changes from frame to frame
        f = frames[-1].copy()
        f[40 * k : 40 * k + 50, 30:90] = 1.0 - f[40 * k : 40 * k + 50, 30:90]
        frames.append(f)
    return w, frames


def _video_cfg(w):
    import copy

    cfg = copy.deepcopy(w.cfg)
    cfg.num_iterations, cfg.sequential_iterations = 8, 6
    cfg.freeze_static = True
    return cfg


def _video_rank_main(rank, world, out_dir):
    sys.path.insert(0, str(ROOT))
    import copy

    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2602_22625_b200 import video
    from paper_2602_22625_b200.scene import pack_params

    w, frames = _video_frames()
    scenes, hists = video.optimize_video_sharded(frames, copy.deepcopy(w.scene), _video_cfg(w))
    np.savez(os.path.join(out_dir, f"video{rank}.npz"),
             params=np.stack([pack_params(s)[0] for s in scenes]),
             loss=np.concatenate([[h.loss for h in hi] for hi in hists]),
             lens=np.array([len(h) for h in hists]))
    dist.barrier()
    dist.destroy_process_group()


def test_video_frames_sharded_across_ranks(torch_cuda, tmp_path):
    """BASELINE c4's frame sharding: 2 ranks (gloo, one GPU) each run the
    warm-start chain on their chunk of 4 frames; every rank gathers the same
    per-frame results, and each chunk equals optimize_video on that chunk alone
    (chunk 0 with the sequential reference's rng)."""
    import copy

    import torch.multiprocessing as mp

    from paper_2602_22625_b200 import video
    from paper_2602_22625_b200.scene import pack_params

    os.environ["MASTER_PORT"] = str(29700 + (os.getpid() % 1000))
    mp.spawn(_video_rank_main, args=(2, str(tmp_path)), nprocs=2, join=True)
    runs = [dict(np.load(tmp_path / f"video{r}.npz")) for r in range(2)]
    np.testing.assert_array_equal(runs[0]["params"], runs[1]["params"])
    np.testing.assert_array_equal(runs[0]["loss"], runs[1]["loss"])
    assert list(runs[0]["lens"]) == [8, 6, 8, 6]  # chunk starts run the frame-0 budget
    w, frames = _video_frames()
    cfg = _video_cfg(w)
    for c, chunk in enumerate(video.frame_chunks(4, 2)):
        sc, _ = video.optimize_video([frames[i] for i in chunk], copy.deepcopy(w.scene), cfg,
                                     rng=video.chunk_rng(cfg.seed, c))
        for j, i in enumerate(chunk):
            _adam_bar(runs[0]["params"][i].reshape(-1, 8), pack_params(sc[j])[0].reshape(-1, 8),
                      cfg, 14)


def _nccl_rank_main(rank, world, name, steps, out_dir):
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", 0))
    from paper_2602_22625_b200 import synth
    from paper_2602_22625_b200.dist import make_allreduce, row_bands
    from paper_2602_22625_b200.fit import StepEngine

    w = synth.make_workload(name)
    w.cfg.num_iterations = steps
    nty = -(-w.scene.canvas_h // 16)
    eng = StepEngine(w.scene, w.cfg, w.loss, steps, band=row_bands(nty, world)[rank],
                     allreduce=make_allreduce(), use_graph=True)
    eng.run(steps)  # one single-step graph, then CHUNK-step graphs (a collective per step)
    torch.cuda.synchronize()
    eng.check()
    np.savez(os.path.join(out_dir, f"nccl{rank}.npz"), params=eng.params_host(),
             loss=np.array([h.loss for h in eng.history()]), graph=np.bool_(eng.graph is not None))
    dist.barrier()
    dist.destroy_process_group()


def test_nccl_allreduce_in_step_graph(torch_cuda, tmp_path):
    """The multi-GPU step's exact code path on hardware with the one GPU there
    is: an NCCL process group (world 1: NCCL refuses two ranks on one device),
    the gradient + loss allreduce captured inside the step's CUDA graph between
    the fit-step kernel and the Adam + records launch, also in run()'s CHUNK-step
    graphs (a collective per captured step).  A one-rank sum is the
    identity, so the run equals the engine without an allreduce (under the
    Adam-noise bar of the float64 gradient atomics' order)."""
    import torch.multiprocessing as mp

    from paper_2602_22625_b200 import synth
    from paper_2602_22625_b200.fit import StepEngine

    os.environ["MASTER_PORT"] = str(29700 + (os.getpid() % 1000))
    steps = 1 + 2 * StepEngine.CHUNK + 1
    mp.spawn(_nccl_rank_main, args=(1, "c3", steps, str(tmp_path)), nprocs=1, join=True)
    r = dict(np.load(tmp_path / "nccl0.npz"))
    assert bool(r["graph"])
    w = synth.make_workload("c3")
    w.cfg.num_iterations = steps
    eng = StepEngine(w.scene, w.cfg, w.loss, steps, use_graph=True)
    for _ in range(steps):
        eng.step()
    eng.check()
    np.testing.assert_allclose(r["loss"], [h.loss for h in eng.history()], rtol=1e-5)
    _adam_bar(r["params"].reshape(-1, 8), eng.params_host().reshape(-1, 8), w.cfg, steps)
