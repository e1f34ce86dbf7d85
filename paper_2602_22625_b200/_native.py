"""ctypes binding of the C ABI in include/primfit_b200.h.

The shared library is built in-tree by ``paper_2602_22625_b200.build`` into
``paper_2602_22625_b200/_lib/libprimfit_b200.so``.  There is no fallback: if
the library is missing or fails to load, every compute entry point raises
``NativeUnavailable``.  (The reference's equivalent layer is the set of numba
kernels in pkg/src/primfit/_kernels.py, bound positionally from raster.py and
grad.py.)
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_DIR = Path(__file__).resolve().parent / "_lib"
LIB_PATH = LIB_DIR / "libprimfit_b200.so"
# the diagnostics build (PF_DIAG=1: globaltimer timeline, per-warp step profile)
# is a second library; the product build compiles that code out (4 % of the
# fit-step kernel's time).  PF_TIMELINE / PF_STEP_PROF select it.
LIB_DIAG_PATH = LIB_DIR / "libprimfit_b200_diag.so"
if os.environ.get("PF_TIMELINE") or os.environ.get("PF_STEP_PROF"):
    LIB_PATH = LIB_DIAG_PATH
# diagnostics: PF_LIB=<path> loads another build (A/B runs on one box)
if os.environ.get("PF_LIB"):
    LIB_PATH = Path(os.environ["PF_LIB"])

PF_OK = 0
PF_ERR_ARG = 1001
PF_ERR_SCRATCH = 1002
PF_ERR_TILE = 1003
PF_LOSS_NONE = 0
PF_LOSS_MSE = 1
PF_LOSS_SPATIAL = 2
PF_LOSS_COMBINED = 3
PF_LOSS_EXTERN = 4
PF_LOSS_RENDER = 5

_P = C.c_void_p
_I = C.c_int
_D = C.c_double
_Z = C.c_size_t

# name -> (restype, argtypes); mirrors include/primfit_b200.h one to one
SIGNATURES: dict[str, tuple] = {
    "pf_abi_version": (_I, []),
    "pf_diag_reload": (_I, []),
    "pf_record_bytes": (_Z, []),
    "pf_render_tile": (_I, []),
    "pf_bin_scratch_bytes": (_Z, [_I, _I, _I]),
    "pf_bin_launches": (_I, [_I, _I, _I, _I, _I, _I]),
    "pf_saved_capacity": (C.c_longlong, [_I]),
    "pf_saved_bytes": (_Z, [_I]),
    "pf_preprocess": (_I, [_P, _I, _D, _D, _D, _I, _I, _I, _I, _I, _I, _P, _P, _Z, _P, _I, _P,
                           _P]),
    "pf_preprocess_sync": (_I, [_P, _P, _I, _D, _D, _D, _I, _I, _I, _I, _I, _I, _P, _P, _Z, _P,
                                _I, _P, _P]),
    "pf_slot_bytes": (_Z, [_I, _I, _I]),
    "pf_pack_grad4": (_I, [_P, _P, _I, _P, _P]),
    "pf_mse4": (_I, [_P, _P, _I, _P, _P, _P]),
    "pf_mse4_grad": (_I, [_P, _P, _I, _P, _P, _P]),
    "pf_slot_reset": (_I, [_P, _I, _I, _I, _P, _P]),
    "pf_scratch_init": (_I, [_P, _Z, _P, _P, _I, _P, _P, _P, _P, _P, _P, _I, _I, _P]),
    "pf_adam_blocks": (_I, [_I]),
    "pf_adam_preprocess": (
        _I,
        [_P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _D, _D, _P, _P, _I, _P, _P, _I, _D, _D, _D, _I,
         _I, _I, _I, _I, _I, _P, _P, _Z, _P, _P, _I, _P, _P],
    ),
    "pf_atlas_quad": (_I, [_P, _I, _P, _P, _P, _I, _P, _P]),
    "pf_atlas_pad": (_I, [_P, _I, _P, _P, _P, _P, _I, _I, _P, _P]),
    "pf_bin": (_I, [_I, _I, _I, _I, _I, _I, _I, _P, _Z, _P, _P, _P, _P, _P]),
    "pf_forward": (
        _I,
        [_P, _I, _P, _P, _I, _P, _P, _P, _I, _I, _I, _I, _D, _D, _D, _D, _D, _P,
         _P, C.c_longlong, _P, _P, _I, _P, _D, _D, _D, _D, _D, _P, _P, _P],
    ),
    "pf_step_spill_bytes": (_Z, [_I]),
    "pf_fit_step": (
        _I,
        [_P, _I, _P, _P, _P, _I, _I, _P, _P, _P, _I, _I, _I, _I, _D, _D, _D, _D, _P, _I, _P, _D,
         _D, _D, _D, _D, _P, _P, _P, _P, _P, _P, _I, _P, _Z, _I, _P, _I, _P],
    ),
    "pf_fold_loss": (_I, [_P, _I, _P, _P, _P]),
    "pf_fold_scratch_bytes": (_Z, [_I]),
    "pf_sum_bands": (_I, [_P, _I, _P, _I, C.c_longlong, C.c_longlong, _P]),
    "pf_backward": (
        _I,
        [_P, _I, _P, _P, _I, _P, _P, _P, _P, C.c_longlong, _P, _P, _D, _D, _D, _P, _D,
         _I, _I, _I, _I, _P, _P, _P, _P],
    ),
    "pf_layer_bboxes": (_I, [_P, _P, _P, _I, _I, _I, _I, _P, _P, _P, _P]),
    "pf_render_layers": (
        _I, [_P, _P, _P, _I, _P, _P, _P, _P, _I, _D, _D, _I, _P, _P, _P, _P]),
    "pf_diff_mask": (_I, [_P, _P, _I, _I, _D, _P, _P]),
    "pf_freeze_flags": (_I, [_P, _P, _P, _I, _I, _I, _D, _P, _P, _P]),
    "pf_stuck_scratch_bytes": (_Z, [_I, _I]),
    "pf_remove_stuck": (
        _I, [_P, _P, _P, _I, _I, _I, _I, _I, _I, _D, _D, _D, _D, _D, _P, _P, _Z, _P]),
    "pf_adam": (
        _I,
        [_P, _P, _P, _P, _P, _P, _I, _P, _P, _P, _P, _D, _D, _D, _I, _D, _D, _I,
         _P, _I, _D, _D, _D, _P, _P, _P, _P],
    ),
}


class NativeUnavailable(RuntimeError):
    """The CUDA extension is not built or cannot be loaded."""


class NativeError(RuntimeError):
    """A C-ABI call returned a nonzero status."""


_lib = None


def load(path: str | os.PathLike | None = None) -> C.CDLL:
    """Load (once) and return the native library with typed signatures."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise NativeUnavailable(
            f"{p} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    try:
        lib = C.CDLL(str(p))
    except OSError as exc:  # pragma: no cover - depends on the box
        raise NativeUnavailable(f"cannot load {p}: {exc}") from exc
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def check(status: int, what: str) -> None:
    if status != PF_OK:
        raise NativeError(f"{what} failed with status {status}")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()
