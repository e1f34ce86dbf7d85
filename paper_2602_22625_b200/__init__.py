"""B200-native differentiable bitmap compositor (DiffBMP / reference package ``primfit``).

Host side mirrors the reference's renderer API (raster/grad/fit modules with
the same names); every pixel operation runs in hand-written sm_100a CUDA
kernels behind the C ABI in include/primfit_b200.h.  There is no CPU path.
"""

from .errors import (  # noqa: F401
    BadChannelRange, BadTemplateRef, BinOverflow, InvalidScale, LayoutMismatch, LengthMismatch,
    MissingAlphaTarget, NonPermutationZ, PrimfitError, ShapeMismatch, StaleSavedState,
)
from .scene import (  # noqa: F401
    PARAM_GROUPS, ParamLayout, PrimitiveParams, PrimitiveTemplate, Scene, pack_params,
    scene_fingerprint, unpack_params, validate_scene,
)

__version__ = "0.1.0"
