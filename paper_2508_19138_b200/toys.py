"""Seeded synthetic device inputs (restates negfgw/toys.py:89-132 so the GPU
box can generate the named benchmark shapes without the reference). Input
generation only -- not part of the hot path."""

from __future__ import annotations

import numpy as np


def chain_device(n_blocks: int, block_size: int, t: float = 0.4, onsite_seed: int = 7,
                 onsite_scale: float = 0.15):
    """Homogeneous chain (toys.py:89-108) as (diag, upper, lower) block stacks."""
    rng = np.random.default_rng(onsite_seed)
    g = lambda: rng.standard_normal((block_size, block_size)) + 1j * rng.standard_normal((block_size, block_size))
    a = g()
    onsite = onsite_scale * 0.5 * (a + a.conj().T)
    coup = t * np.eye(block_size, dtype=complex) + 0.05 * g()
    diag = np.repeat(onsite[None], n_blocks, axis=0)
    upper = np.repeat(coup[None], n_blocks - 1, axis=0)
    lower = np.repeat(coup.conj().T[None], n_blocks - 1, axis=0)
    return diag, upper, lower


def coulomb_matrix(n_blocks: int, block_size: int, v0: float = 1e-3, seed: int = 11):
    """Replicated real symmetric interaction (toys.py:111-132) as block stacks."""
    rng = np.random.default_rng(seed)
    d = rng.standard_normal((block_size, block_size))
    on = (v0 * (np.eye(block_size) + 0.1 * (d + d.T))).astype(complex)
    off = (v0 * 0.3 * rng.standard_normal((block_size, block_size))).astype(complex)
    return (np.repeat(on[None], n_blocks, axis=0), np.repeat(off[None], n_blocks - 1, axis=0),
            np.repeat(off.T[None], n_blocks - 1, axis=0))
