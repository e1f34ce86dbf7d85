"""CPU checks of the layered export's file side (exportio.py:345-512).

The layer buffers come from the oracle's restatement of render_layer (test
infrastructure, pinned to the reference's goldens in test_oracle_golden.py);
the files are written by the product writer ``export.write_export`` (the same
function the GPU ``export_layers`` calls).  Then:
  * the manifest round-trips through the package's parse_manifest;
  * when the reference package is importable (this build container, not the GPU
    box) the REFERENCE's own parse_manifest reads the manifest back and its
    compose_layers re-composites the PNGs to within PNG quantisation of the
    scaled render (the reference's own bar, test_export.py:250-254).
"""

from __future__ import annotations

import dataclasses
import os
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import load_case, scene_from

REF_SRC = Path("/root/reference/pkg/src")


def _reference_exportio():
    if not REF_SRC.is_dir():
        pytest.skip("reference package not present (GPU box)")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    try:
        from primfit import exportio
    except Exception as exc:  # pragma: no cover - depends on the container
        pytest.skip(f"reference not importable: {exc}")
    return exportio


def _oracle_export(oracle, sc, rho, outdir):
    from paper_2602_22625_b200 import export

    pk = oracle.Packed(sc)
    boxes, offs, rgba = oracle.export_layers_arrays(pk, rho)

    def layer(i):
        if boxes[i, 0] < 0:
            raise export.DegenerateBBox(f"primitive {i} lies fully off-canvas")
        x0, y0, x1, y1 = (int(v) for v in boxes[i])
        return (x0, y0, x1, y1), rgba[offs[i]:offs[i + 1]].reshape(y1 - y0 + 1, x1 - x0 + 1, 4)

    scaled = export.scale_scene(sc, rho)
    spk = oracle.Packed(scaled)
    off, idx = oracle.bin_tiles(spk, 32, 2.0)
    bg_rgb = (1.0, 1.0, 1.0) if isinstance(sc.background, str) else tuple(sc.background)
    bg = np.broadcast_to(np.asarray(bg_rgb), (scaled.canvas_h, scaled.canvas_w, 3)).copy()
    img, alpha, _ = oracle.render_forward(spk, off, idx, 32, bg, False, 0.0)
    man = export.write_export(sc, rho, outdir, layer, img)
    return man, img, alpha


def _scene_with_offcanvas():
    sc = scene_from(load_case("export_random"))
    prims = list(sc.primitives)
    prims[2] = dataclasses.replace(prims[2], x=-500.0, y=-500.0)
    return dataclasses.replace(sc, primitives=prims)


@pytest.mark.parametrize("rho", [1, 2])
def test_export_files_round_trip(oracle, tmp_path, rho):
    from paper_2602_22625_b200 import export

    sc = _scene_with_offcanvas()
    man, img, alpha = _oracle_export(oracle, sc, rho, tmp_path)
    assert (tmp_path / "manifest.txt").read_text().startswith("format primfit-layers\nversion 1\n")
    back = export.read_manifest(tmp_path / "manifest.txt")
    assert back == man
    assert [r.z for r in man.layers] == list(range(sc.n))
    assert [r.prim for r in man.layers if r.file is None] == [2]
    front = min(range(sc.n), key=lambda i: sc.primitives[i].z)
    assert man.layers[-1].prim == front  # the front-most primitive paints last
    for r in man.layers:
        p = sc.primitives[r.prim]
        assert r.params == (p.x, p.y, p.scale, p.rotation, p.opacity_logit, *p.color_logits)
    composed = export.compose_layers(man, tmp_path)
    assert np.abs(composed.color - img).max() < 5e-4
    assert np.abs(composed.alpha - alpha).max() < 5e-4
    comp_png, _ = export.load_image(tmp_path / "composite.png")
    assert np.abs(comp_png - img).max() <= 0.5 / 255.0 + 1e-12


@pytest.mark.parametrize("rho", [1, 2])
def test_reference_reads_and_composes_export(oracle, tmp_path, rho):
    """The reference's own parse_manifest / compose_layers consume our files."""
    ref = _reference_exportio()
    sc = _scene_with_offcanvas()
    man, img, alpha = _oracle_export(oracle, sc, rho, tmp_path)
    rman = ref.read_manifest(tmp_path / "manifest.txt")
    assert (rman.scale, rman.canvas_w, rman.canvas_h, rman.background, rman.composite) == (
        man.scale, man.canvas_w, man.canvas_h, man.background, man.composite)
    assert [(r.z, r.prim, r.params, r.bbox, r.file) for r in rman.layers] == [
        (r.z, r.prim, r.params, r.bbox, r.file) for r in man.layers]
    composed = ref.compose_layers(rman, tmp_path)
    assert np.abs(composed.color - img).max() < 5e-4
    assert np.abs(composed.alpha - alpha).max() < 5e-4


def test_manifest_rejects_malformed():
    from paper_2602_22625_b200 import export

    with pytest.raises(ValueError, match="not a layer manifest"):
        export.parse_manifest("format something-else\n")
    good = ("format primfit-layers\nversion 1\nscale 1\ncanvas 4 4\n"
            "background 0.0 0.0 0.0\ncomposite c.png\nlayers 1\n")
    with pytest.raises(ValueError):
        export.parse_manifest(good + "layer 0 prim 0 bbox 0 0 1 1 file a.png params 1 2 3\n")
    m = export.parse_manifest(good + "layer 0 prim 0 skipped off-canvas params 1 2 3 4 5 6 7 8\n")
    assert m.layers[0].bbox is None and m.layers[0].params == (1, 2, 3, 4, 5, 6, 7, 8)
