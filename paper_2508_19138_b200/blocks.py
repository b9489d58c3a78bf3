"""Block-banded complex container (drop-in for negfgw.blocks.BlockMatrix,
blocks.py:34-274) plus the conversions to the batched device layout.

The hot path never walks blocks in Python: a BlockMatrix is converted once
to stacked complex128 tensors ``diag (n_b, bs, bs)``, ``upper/lower
(n_b-1, bs, bs)`` (and an energy axis in front for batches), which is the
memory layout the C-ABI consumes. The container only exists so code written
against the reference's per-energy API keeps working.
"""

from __future__ import annotations

import numpy as np
import torch

from .errors import BlockStructureError

FULL = "full"
LG_COMPRESSED = "lg_compressed"


class BlockMatrix:
    """Square block matrix with odd block bandwidth (reference semantics:
    implied lower blocks in ``lg_compressed`` mode read as ``-X[j,i]^dag``,
    never-written in-band blocks read as zeros, writes below the diagonal
    of compressed storage are rejected)."""

    __slots__ = ("n_blocks", "block_size", "block_bandwidth", "storage_mode", "_b")

    def __init__(self, n_blocks: int, block_size: int, block_bandwidth: int = 3,
                 storage_mode: str = FULL) -> None:
        if n_blocks < 1 or block_size < 1:
            raise BlockStructureError(f"need n_blocks, block_size >= 1, got {n_blocks}, {block_size}")
        if block_bandwidth % 2 == 0 or not 1 <= block_bandwidth <= 2 * n_blocks - 1:
            raise BlockStructureError(f"invalid block bandwidth {block_bandwidth} for {n_blocks} blocks")
        if storage_mode not in (FULL, LG_COMPRESSED):
            raise BlockStructureError(f"unknown storage mode {storage_mode!r}")
        self.n_blocks, self.block_size = n_blocks, block_size
        self.block_bandwidth, self.storage_mode = block_bandwidth, storage_mode
        self._b: dict[tuple[int, int], np.ndarray] = {}

    @property
    def half_bandwidth(self) -> int:
        return self.block_bandwidth // 2

    def in_band(self, i: int, j: int) -> bool:
        return 0 <= min(i, j) and max(i, j) < self.n_blocks and abs(i - j) <= self.half_bandwidth

    def get_block(self, i: int, j: int) -> np.ndarray:
        if not self.in_band(i, j):
            raise BlockStructureError(f"block ({i}, {j}) outside the band")
        if self.storage_mode == LG_COMPRESSED and j < i:
            up = self._b.get((j, i))
            return np.zeros((self.block_size,) * 2, complex) if up is None else -up.conj().T
        blk = self._b.get((i, j))
        return np.zeros((self.block_size,) * 2, complex) if blk is None else blk

    def set_block(self, i: int, j: int, value) -> None:
        if not self.in_band(i, j):
            raise BlockStructureError(f"block ({i}, {j}) outside the band")
        if self.storage_mode == LG_COMPRESSED and j < i:
            raise BlockStructureError(f"write into implied triangle ({i}, {j})")
        v = np.asarray(value, dtype=complex)
        if v.shape != (self.block_size,) * 2:
            raise BlockStructureError(f"block ({i}, {j}) has shape {v.shape}")
        self._b[(i, j)] = v

    def add_to_block(self, i: int, j: int, value) -> None:
        self.set_block(i, j, self.get_block(i, j) + value)

    def stored_keys(self) -> list[tuple[int, int]]:
        return sorted(self._b)

    def to_dense(self) -> np.ndarray:
        bs, n = self.block_size, self.n_blocks
        out = np.zeros((n * bs, n * bs), complex)
        for i in range(n):
            for j in range(max(0, i - self.half_bandwidth), min(n, i + self.half_bandwidth + 1)):
                out[i * bs:(i + 1) * bs, j * bs:(j + 1) * bs] = self.get_block(i, j)
        return out

    def copy(self) -> "BlockMatrix":
        out = BlockMatrix(self.n_blocks, self.block_size, self.block_bandwidth, self.storage_mode)
        out._b = {k: v.copy() for k, v in self._b.items()}
        return out


def _band_get(m, i: int, j: int, bs: int) -> np.ndarray:
    if m.in_band(i, j):
        return np.asarray(m.get_block(i, j), dtype=complex)
    return np.zeros((bs, bs), complex)


def tridiag_arrays(m) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(diag, upper, lower) stacks of any object with the BlockMatrix API
    (ours or the reference's)."""
    n, bs = m.n_blocks, m.block_size
    d = np.stack([_band_get(m, i, i, bs) for i in range(n)])
    u = np.stack([_band_get(m, i, i + 1, bs) for i in range(n - 1)]) if n > 1 else np.zeros((0, bs, bs), complex)
    lo = np.stack([_band_get(m, i + 1, i, bs) for i in range(n - 1)]) if n > 1 else np.zeros((0, bs, bs), complex)
    return d, u, lo


def lg_arrays(m) -> tuple[np.ndarray, np.ndarray]:
    """(diag, upper) stacks of a lesser/greater source (lower implied)."""
    d, u, _ = tridiag_arrays(m)
    return d, u


def to_device(a: np.ndarray, device) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex128)).to(device)
