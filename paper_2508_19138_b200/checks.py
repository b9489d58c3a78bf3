"""ScbaOptions.oracle_mode diagnostics (scba.py:913-915, 988-998, 412-430):
every selected solve is compared with a dense inversion + triple product
(rgf.py:246-267 dense_selected_oracle) and every P / Sigma convolution with
the direct O(N_E^2) sum (convolve.py:74-98 convolve_energy_direct).

These are run-time self-checks of the product path, computed on the device
with torch (cuSOLVER inverse, elementwise sums) -- an independent second
evaluation, not the repository's test oracle (oracle/). Like the reference
they are meant for small systems: the dense check refuses systems above
MAX_DENSE orbitals.
"""

from __future__ import annotations

import torch

MAX_DENSE = 4096


def _dense(d, u, lo):
    """(n_e, n_b, bs, bs) diag + (n_e, n_b-1, bs, bs) upper/lower -> dense (n_e, N, N)."""
    n_e, n_b, bs = d.shape[0], d.shape[1], d.shape[-1]
    out = torch.zeros((n_e, n_b * bs, n_b * bs), dtype=d.dtype, device=d.device)
    for i in range(n_b):
        out[:, i * bs:(i + 1) * bs, i * bs:(i + 1) * bs] = d[:, i]
        if i + 1 < n_b:
            out[:, i * bs:(i + 1) * bs, (i + 1) * bs:(i + 2) * bs] = u[:, i]
            out[:, (i + 1) * bs:(i + 2) * bs, i * bs:(i + 1) * bs] = lo[:, i]
    return out


def _h(x):
    return x.conj().transpose(-1, -2)


def dense_solution_deviation(m, b_lg: dict, x_r, x_lg: dict, chunk: int = 8) -> tuple[float, float]:
    """scba.py:440-453 _solution_deviation against dense_selected_oracle.

    m = (diag, upper, lower) of the closed system; b_lg[kind] = (diag, upper)
    lg-compressed sources (lower = -upper^dag); x_r = (diag, upper, lower) and
    x_lg[kind] = (diag, upper) the selected solution (symmetrized). Returns
    (max deviation, max reference magnitude) over all blocks and energies."""
    n_e, n_b, bs = m[0].shape[0], m[0].shape[1], m[0].shape[-1]
    if n_b * bs > MAX_DENSE:
        raise ValueError(f"oracle_mode dense check supports at most {MAX_DENSE} orbitals, got {n_b * bs}")
    dev = scale = 0.0

    def acc(a, ref):
        nonlocal dev, scale
        if ref.numel():
            dev = max(dev, float((a - ref).abs().max()))
            scale = max(scale, float(ref.abs().max()))

    def cut(full, i, j):
        return full[:, i * bs:(i + 1) * bs, j * bs:(j + 1) * bs]

    for e0 in range(0, n_e, chunk):
        s = slice(e0, min(n_e, e0 + chunk))
        g = torch.linalg.inv(_dense(m[0][s], m[1][s], m[2][s]))
        for i in range(n_b):
            acc(x_r[0][s][:, i], cut(g, i, i))
            if i + 1 < n_b:
                acc(x_r[1][s][:, i], cut(g, i, i + 1))
                acc(x_r[2][s][:, i], cut(g, i + 1, i))
        for kind, (bd, bu) in b_lg.items():
            bfull = _dense(bd[s], bu[s], -_h(bu[s]))
            full = g @ bfull @ _h(g)
            xd, xu = x_lg[kind]
            for i in range(n_b):
                blk = cut(full, i, i)
                acc(xd[s][:, i], 0.5 * (blk - _h(blk)))  # symmetrize (rgf.py:82-88)
                if i + 1 < n_b:
                    acc(xu[s][:, i], cut(full, i, i + 1))
        del g
    return dev, scale


def _direct(x1, x2, mode: str):
    """convolve.py:74-98: sum_m x1[m] x2[k - m] (convolution) or
    sum_m x1[m] x2[m - k] (correlation), k = 0..n-1, over the last axis."""
    n = x1.shape[-1]
    out = torch.empty_like(x1)
    for k in range(n):
        if mode == "convolution":
            out[:, k] = (x1[:, :k + 1] * x2[:, :k + 1].flip(-1)).sum(-1)
        else:
            out[:, k] = (x1[:, k:] * x2[:, :n - k]).sum(-1)
    return out


def _proj(x, diag):
    if diag is None:
        return x
    y = x.clone()
    y[diag.bool()] = 1j * y[diag.bool()].imag
    return y


def polarization_deviation(gl, gg, pl, pg, diag, de: float) -> tuple[float, float]:
    """fft_vs_direct for P^< and P^> (scba.py:1035-1042), C_P = -i/2pi; the
    fused kernel's outputs are diagonal-projected, so is the direct sum."""
    c = -1j / (2 * torch.pi) * de
    dev = scale = 0.0
    for got, a, b in ((pl, gl, gg), (pg, gg, gl)):
        ref = _proj(c * _direct(a, -b.conj(), "correlation"), diag)
        if ref.numel():
            dev = max(dev, float((got - ref).abs().max()))
            scale = max(scale, float(ref.abs().max()))
    return dev, scale


def self_energy_deviation(gl, gg, wl, wg, sl, sg, diag, de: float) -> tuple[float, float]:
    """fft_vs_direct for Sigma^< and Sigma^> (scba.py:1118-1126), C_Sigma = i/2pi."""
    c = 1j / (2 * torch.pi) * de
    dev = scale = 0.0
    for got, a, w in ((sl, gl, wl), (sg, gg, wg)):
        ref = _proj(c * _direct(a, w, "convolution"), diag)
        if ref.numel():
            dev = max(dev, float((got - ref).abs().max()))
            scale = max(scale, float(ref.abs().max()))
    return dev, scale
