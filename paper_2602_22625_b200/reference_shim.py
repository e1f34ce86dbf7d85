"""Route the reference package's hot-path callers to the B200 implementation.

The reference (``primfit``) has no plugin layer: its callers bind the hot-path
functions by name at import time, so rebinding only the
defining module misses them.  ``enable()`` rebinds every module-level name a
§8(b) caller resolves at call time:

  defining modules   raster.bin_tiles / render_forward (raster.py:227, 290),
                     grad.backward (grad.py:134), fit.adam_step / run_loop /
                     optimize (fit.py:195, 403, 524), dyn.diff_mask / freeze_flags /
                     remove_stuck / optimize_video (dyn.py:86-238),
                     exportio.export_layers (exportio.py:345)
  by-name importers  fit.{bin_tiles, render_forward, backward} (fit.py:28, 38),
                     dyn.run_loop (dyn.py:22-29),
                     cli.{render_forward, backward, export_layers, optimize_video,
                     optimize}
                     (cli.py:20-33: run_bench 180-230, _cmd_render 64-70,
                     _final_composite 249-260),
                     exportio.render_forward (exportio.py:54-62, the composite),
                     estimator.{render_forward, optimize_video, optimize}
                     (estimator.py:19-22)
  package surface    primfit.<name> re-exports (__init__.py:32-100)

``run_gradcheck`` (grad.py:396-398) imports raster.render_forward inside the
function and calls the module global ``backward``, ``warmup_kernels``
(raster.py:402-415) calls the raster global and ``grad.backward``: both follow
the defining-module rebinds.  The finite-difference side of the gradcheck
stays on the reference's float64 ``render_naive`` (not rebound).

``disable()`` restores the originals.  The B200 functions accept the
reference's own Scene / LossSpec / OptimState / FitConfig objects (duck-typed).
"""

from __future__ import annotations

import importlib
from types import ModuleType

from . import export as _export
from . import fit as _fit
from . import grad as _grad
from . import raster as _raster
from . import video as _video

# (reference module, attribute) -> B200 replacement
REBINDS: dict[tuple[str, str], object] = {
    ("raster", "bin_tiles"): _raster.bin_tiles,
    ("raster", "render_forward"): _raster.render_forward,
    ("grad", "backward"): _grad.backward,
    ("fit", "adam_step"): _fit.adam_step,
    ("fit", "run_loop"): _fit.run_loop,
    ("fit", "optimize"): _fit.optimize,
    ("fit", "bin_tiles"): _raster.bin_tiles,
    ("fit", "render_forward"): _raster.render_forward,
    ("fit", "backward"): _grad.backward,
    ("dyn", "run_loop"): _fit.run_loop,
    ("dyn", "diff_mask"): _video.diff_mask,
    ("dyn", "freeze_flags"): _video.freeze_flags,
    ("dyn", "remove_stuck"): _video.remove_stuck,
    ("dyn", "optimize_video"): _video.optimize_video,
    ("exportio", "render_forward"): _raster.render_forward,
    ("exportio", "export_layers"): _export.export_layers,
    ("cli", "render_forward"): _raster.render_forward,
    ("cli", "backward"): _grad.backward,
    ("cli", "export_layers"): _export.export_layers,
    ("cli", "optimize_video"): _video.optimize_video,
    ("cli", "optimize"): _fit.optimize,
    ("estimator", "render_forward"): _raster.render_forward,
    ("estimator", "optimize_video"): _video.optimize_video,
    ("estimator", "optimize"): _fit.optimize,
}
# names the package re-exports at its top level
PACKAGE_NAMES = ("bin_tiles", "render_forward", "backward", "adam_step", "run_loop", "optimize",
                 "diff_mask", "freeze_flags", "remove_stuck", "optimize_video", "export_layers")

_saved: dict[tuple[str, str], object] = {}


def _module(pkg: str, name: str) -> ModuleType:
    return importlib.import_module(f"{pkg}.{name}")


def enable(pkg: str = "primfit") -> dict[tuple[str, str], object]:
    """Rebind the reference's hot-path names to the B200 functions; returns the
    originals (also kept for disable())."""
    root = importlib.import_module(pkg)
    for (mod, attr), fn in REBINDS.items():
        m = _module(pkg, mod)
        if not hasattr(m, attr):
            raise AttributeError(f"{pkg}.{mod} has no {attr}: reference layout changed")
        _saved.setdefault((mod, attr), getattr(m, attr))
        setattr(m, attr, fn)
    for attr in PACKAGE_NAMES:
        if hasattr(root, attr):
            src = next(fn for (mod, a), fn in REBINDS.items() if a == attr)
            _saved.setdefault(("", attr), getattr(root, attr))
            setattr(root, attr, src)
    return dict(_saved)


def disable(pkg: str = "primfit") -> None:
    """Restore every name enable() replaced."""
    root = importlib.import_module(pkg)
    for (mod, attr), orig in _saved.items():
        setattr(root if mod == "" else _module(pkg, mod), attr, orig)
    _saved.clear()
