"""Exception types raised at the renderer boundary.

Names and meanings follow the reference package (pkg/src/primfit/errors.py:11-82)
so callers' ``except`` clauses keep working; ``BinOverflow`` is new (the GPU
bins into preallocated capacity).
"""

from __future__ import annotations


class PrimfitError(Exception):
    """Base class for all package-specific errors."""


class InvalidScale(PrimfitError):
    """A primitive scale is not finite and positive."""


class BadTemplateRef(PrimfitError):
    """A primitive references a template index that does not exist."""


class NonPermutationZ(PrimfitError):
    """Depth values are not a permutation of 0..N-1."""


class BadChannelRange(PrimfitError):
    """A template texel lies outside [0, 1] or is not finite."""


class LengthMismatch(PrimfitError):
    """Collections that must have equal length do not."""


class ShapeMismatch(PrimfitError):
    """An array does not have the shape the canvas/layout requires."""


class LayoutMismatch(PrimfitError):
    """A packed vector does not match its layout."""


class StaleSavedState(PrimfitError):
    """Saved forward state does not belong to this scene/background."""


class MissingAlphaTarget(PrimfitError):
    """A loss needs a target alpha that was not supplied."""


class BinOverflow(PrimfitError):
    """Tile binning produced more entries than the preallocated capacity."""
