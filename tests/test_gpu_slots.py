"""Slot binning (the fit step's tile lists without pf_bin).

K1 scatters every (tile, primitive) pair into per-tile slots in arrival order;
pf_fit_step's producer warps sort each list by z rank.  Checked here:

1. The slot lists, sorted by z rank, are bit-identical to the oracle's
   bin_tiles (raster.py:227-265) on c1-c5 and on every band of an 8-way split
   of c5 -- also with a tiny slot count, so that most pairs take the overflow
   list.
2. The fused step on slot lists equals the step on pf_bin's CSR lists:
   gradients and loss sums within fp64 atomic-order noise, K identical; also on
   the producers' general path (slot_m forced to 4: lists longer than the slots
   and overflowed) and on c2's long lists.
3. A host-edited step (pf_preprocess_sync re-scatters edited primitives next to
   their stale entries: the dirty-step validation + de-duplication) gives the
   same step as a fresh engine on the edited parameters.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _engine(w, monkeypatch, *, csr=False, slot_m=None, band=None, total=4, **kw):
    from paper_2602_22625_b200.fit import StepEngine

    monkeypatch.setenv("PF_CSR_STEP", "1" if csr else "0")
    if slot_m is None:
        monkeypatch.delenv("PF_SLOT_M", raising=False)
    else:
        monkeypatch.setenv("PF_SLOT_M", str(slot_m))
    return StepEngine(w.scene, w.cfg, w.loss, total, band=band, use_graph=False, **kw)


@pytest.mark.parametrize("name,slot_m", [("c1", None), ("c2", None), ("c3", None), ("c3", 4),
                                         ("c4", None), ("c5", None)])
def test_slot_lists_equal_oracle_bins(torch_cuda, oracle, monkeypatch, name, slot_m):
    from paper_2602_22625_b200 import synth
    from paper_2602_22625_b200.dist import row_bands
    from paper_2602_22625_b200.fit import effective_padding

    w = synth.make_workload(name)
    sc = w.scene
    off, idx = oracle.bin_tiles(oracle.Packed(sc), 16, effective_padding(w.cfg))
    nty, ntx = -(-sc.canvas_h // 16), -(-sc.canvas_w // 16)
    bands = [None] + (row_bands(nty, 8) if name == "c5" else [])
    for band in bands:
        eng = _engine(w, monkeypatch, slot_m=slot_m, band=band)
        assert eng.comp.slots is not None
        eng.refresh()
        o, i = eng.comp.slot_lists()
        t0, t1 = (0, nty * ntx) if band is None else (band.ty_begin * ntx, band.ty_end * ntx)
        np.testing.assert_array_equal(o, off[t0 : t1 + 1] - off[t0])
        np.testing.assert_array_equal(i, idx[off[t0] : off[t1]])
        del eng


def _one_step(eng):
    """K1 (refresh) + K34 on the engine's current parameters; no Adam."""
    eng.refresh()
    c = eng.comp
    c.bin()
    eng.gbuf.zero_()
    c.fit_step(eng.gbuf, eng.sums, eps_skip=eng.eps_skip, bg_rgb=eng.bg_rgb, bg4=eng.bg4,
               loss_kind=eng.loss_kind, tgt4=eng.tgt4, alpha_w=eng.alpha_w, w_mse=eng.w_mse,
               w_gray=eng.w_gray, P_total=eng.P)
    k = c.check_overflow()
    return eng.grads.view(-1, 8).cpu().numpy(), eng.sums.cpu().numpy(), k


def _close(a, b, rtol=1e-9):
    scale = np.maximum(np.abs(b), 1e-6 * np.abs(b).max(axis=0, keepdims=True))
    return float((np.abs(a - b) / np.maximum(scale, 1e-300)).max())


@pytest.mark.parametrize("name,slot_m", [("c1", None), ("c2", None), ("c3", None), ("c3", 4),
                                         ("c2", 8)])
def test_slot_step_equals_csr_step(torch_cuda, monkeypatch, name, slot_m):
    from paper_2602_22625_b200 import synth

    w = synth.make_workload(name)
    g_csr, s_csr, k_csr = _one_step(_engine(w, monkeypatch, csr=True))
    eng = _engine(w, monkeypatch, slot_m=slot_m)
    g, s, k = _one_step(eng)
    assert k == k_csr
    np.testing.assert_allclose(s, s_csr, rtol=1e-12)
    assert _close(g, g_csr) < 1e-9
    # the slots were consumed: a second step on the same parameters is identical
    g2, s2, k2 = _one_step(eng)
    assert k2 == k_csr
    np.testing.assert_allclose(s2, s_csr, rtol=1e-12)
    assert _close(g2, g_csr) < 1e-9


@pytest.mark.parametrize("slot_m", [None, 4])
def test_slot_dirty_step_after_host_edit(torch_cuda, monkeypatch, slot_m):
    """host_io engine: Adam writes the next records + slots, the host then edits
    some primitives (moved across tiles); the next graph step re-scatters them
    (dirty) -- the loss of that step must equal a fresh engine's on the edited
    parameters."""
    from paper_2602_22625_b200 import synth

    w = synth.make_workload("c1")
    w.cfg.num_iterations = 6
    eng = _engine(w, monkeypatch, slot_m=slot_m, total=6, host_io=True)
    eng.step()
    eng.capture_host_io_step()
    eng.host_step()
    vec = eng.host_vector()
    rng = np.random.default_rng(5)
    sel = rng.choice(eng.n, size=max(1, eng.n // 5), replace=False)
    v8 = vec.reshape(-1, 8)
    v8[sel, 0] += rng.uniform(-40, 40, size=len(sel))
    v8[sel, 1] += rng.uniform(-40, 40, size=len(sel))
    edited = v8.copy()
    eng.host_step()
    part = eng.host_loss_part(-1)
    loss_dirty = part.sum(axis=0)

    # reference: a fresh engine on the edited parameters, one step
    from paper_2602_22625_b200.scene import ParamLayout, unpack_params

    w.scene = unpack_params(edited.reshape(-1), ParamLayout(eng.n), w.scene)
    ref = _engine(w, monkeypatch, csr=True, total=2)
    _, sums, _ = _one_step(ref)
    np.testing.assert_allclose(loss_dirty[0], sums[0], rtol=1e-12)
