"""Multi-process (world size 2, gloo, CPU) checks of the row-band sharding logic.

Row-band sharding: every rank renders its band of tile rows and
contributes partial gradients + loss sums to one buffer; a SUM allreduce makes
them equal to the full-canvas values.  Here the per-band partials come from the
CPU oracle (test infrastructure) so the partition and the collective plumbing
are exercised without a GPU.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def test_row_bands_partition_and_balance():
    sys.path.insert(0, str(ROOT))
    from paper_2602_22625_b200.dist import row_bands

    for nty, world in ((51, 2), (51, 8), (135, 8), (8, 8), (10, 3)):
        bands = row_bands(nty, world)
        assert bands[0].ty_begin == 0 and bands[-1].ty_end == nty
        for a, b in zip(bands, bands[1:]):
            assert a.ty_end == b.ty_begin
        assert all(b.ty_end > b.ty_begin for b in bands)
    cost = np.ones(40)
    cost[:10] = 10.0  # busy top rows -> the first band is narrower
    bands = row_bands(40, 2, cost)
    assert bands[0].ty_end < 20


def _band_grads(rank, world, case, out):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "oracle"))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import cpu_oracle as orc
    from conftest import load_case, scene_from
    from paper_2602_22625_b200.dist import make_allreduce, row_bands

    d = load_case(case)
    sc = scene_from(d)
    pk = orc.Packed(sc)
    off, idx = orc.bin_tiles(pk, 16, 2.0)
    bg = orc.background(sc)
    img, alpha, sv = orc.render_forward(pk, off, idx, 16, bg, True, 1 / 1024)
    H, W = sc.canvas_h, sc.canvas_w
    band = row_bands(-(-H // 16), world)[rank]
    y0, y1 = band.ty_begin * 16, min(band.ty_end * 16, H)
    # this rank's share: loss pull-back restricted to its band's pixel rows
    dI = np.zeros_like(img)
    dI[y0:y1] = 2.0 * (img[y0:y1] - d["target"][y0:y1]) / img.size
    g = orc.backward(pk, sv, dI, None).reshape(-1)
    sse = float(((img[y0:y1] - d["target"][y0:y1]) ** 2).sum())
    buf = torch.from_numpy(np.concatenate([g, [sse, 0.0, 0.0, 0.0]]))
    make_allreduce()(buf)
    if rank == 0:
        np.save(out, buf.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("case", ["medium_n300", "random_s2"])
def test_allreduced_band_gradients_equal_full_canvas(tmp_path, case):
    sys.path.insert(0, str(ROOT / "oracle"))
    sys.path.insert(0, str(ROOT / "tests"))
    import cpu_oracle as orc
    from conftest import load_case, scene_from

    orc.build()
    port = 29500 + (os.getpid() % 2000)
    os.environ["MASTER_PORT"] = str(port)
    out = str(tmp_path / "buf.npy")
    mp.spawn(_band_grads, args=(2, case, out), nprocs=2, join=True)
    buf = np.load(out)
    d = load_case(case)
    sc = scene_from(d)
    pk = orc.Packed(sc)
    off, idx = orc.bin_tiles(pk, 16, 2.0)
    img, _, sv = orc.render_forward(pk, off, idx, 16, orc.background(sc), True, 1 / 1024)
    _, dI = orc.loss_mse(img, d["target"])
    g_full = orc.backward(pk, sv, dI, None).reshape(-1)
    n8 = g_full.size
    np.testing.assert_allclose(buf[:n8], g_full, rtol=1e-9, atol=1e-15)
    np.testing.assert_allclose(buf[n8], ((img - d["target"]) ** 2).sum(), rtol=1e-12)
