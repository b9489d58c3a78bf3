"""GPU parity of the energy convolutions (convolve.py:39-129 and the fused
P / Sigma stages of scba.py:1035-1048, 1118-1132). Bar 1e-9 relative
Frobenius; observed ~1e-15."""

import numpy as np
import pytest
import torch

import negf_oracle as orc
from paper_2508_19138_b200 import conv

pytestmark = pytest.mark.gpu
TOL = 1e-9


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("ne", [24, 128, 129, 1000])
def test_convolve_and_retarded_match_reference_golden(golden, cuda, ne):
    g = golden("golden_conv.npz")
    x1, x2 = g[f"n{ne}_x1"], g[f"n{ne}_x2"]
    assert rel(conv.convolve_energy(x1, x2, "convolution", 0.7 - 0.2j, 0.01), g[f"n{ne}_conv"]) < TOL
    assert rel(conv.convolve_energy(x1, x2, "correlation", -0.3 + 1.1j, 0.02), g[f"n{ne}_corr"]) < TOL
    assert rel(conv.retarded_from_lg(x1, x2), g[f"n{ne}_ret"]) < TOL


@pytest.mark.parametrize("ne", [1, 2, 3, 16, 32, 64, 100, 256, 1024, 2048, 2049, 4096])
def test_convolutions_match_oracle_sizes(cuda, ne):
    """The reference-signature drop-ins: N_E > 2048 (L > 4096) take the
    cuFFT path (conv.MAX_L_GENERIC); the fused P / Sigma kernels below run
    natively up to N_E = 4096."""
    rng = np.random.default_rng(ne)
    x1 = rng.standard_normal((5, ne)) + 1j * rng.standard_normal((5, ne))
    x2 = rng.standard_normal((5, ne)) + 1j * rng.standard_normal((5, ne))
    for mode in ("convolution", "correlation"):
        assert rel(conv.convolve_energy(x1, x2, mode, 1.0, 0.1), orc.convolve_energy(x1, x2, mode, 1.0, 0.1)) < TOL
    assert rel(conv.retarded_from_lg(x1, x2), orc.retarded_from_lg(x1, x2)) < TOL


@pytest.mark.parametrize("ne,rows", [(3, 517), (8, 37), (16, 37), (16, 1001), (128, 37), (300, 75), (2048, 37),
                                     (2049, 11), (2100, 9), (3000, 21), (4096, 5), (4096, 40)])
def test_fused_polarization_and_sigma_match_oracle(cuda, ne, rows):
    """Short series pack several entry rows per CTA (ragged last CTA covered);
    2048 < N_E <= 4096 (L = 8192) runs on cluster pairs of CTAs splitting the
    even / odd frequency bins (conv.cu pol_kernel_x2 / sigma_kernel_x2)."""
    rng = np.random.default_rng(7 + ne)
    mk = lambda: rng.standard_normal((rows, ne)) + 1j * rng.standard_normal((rows, ne))
    gl, gg, wl, wg = mk(), mk(), mk(), mk()
    diag = rng.random(rows) < 0.3
    de = 4.0 / (ne - 1)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(cuda)
    dm = torch.from_numpy(diag.astype(np.uint8)).to(cuda)
    got = conv.polarization(t(gl), t(gg), dm, de)
    ref = orc.polarization(gl, gg, diag, de)
    for a, b in zip(got, ref):
        assert rel(a.cpu().numpy(), b) < TOL
    # Sigma with a W row gather (w_to_g)
    w_rows = rng.integers(0, rows, size=rows)
    got = conv.self_energy(t(gl), t(gg), t(wl), t(wg), torch.from_numpy(w_rows).to(cuda), dm, de)
    ref = orc.self_energy(gl, gg, wl[w_rows], wg[w_rows], diag, de)
    for a, b in zip(got, ref):
        assert rel(a.cpu().numpy(), b) < TOL
