"""Error taxonomy of the hot path, mirroring negfgw/errors.py:11-42 so callers
catching the reference's exception names keep working."""

from __future__ import annotations


class NegfError(Exception):
    """Root of every structured error raised on the hot path."""


class BlockStructureError(NegfError):
    """Block layout / band / storage-mode violation (errors.py:15)."""


class SingularBlockError(NegfError):
    """A pivot block was exactly singular or non-finite (errors.py:20)."""


class ConvergenceError(NegfError):
    """An iterative solver ran out of budget or diverged (errors.py:24)."""


class SpectralRadiusError(NegfError):
    """Contraction solver given an operator with spectral radius >= 1 (errors.py:28)."""
