"""Energy convolutions on the GPU (drop-in for negfgw.convolve).

``ConvPlan`` holds the per-N_E tables (twiddles, causal-kernel spectra);
``polarization`` / ``self_energy`` are the fused per-entry-row kernels of the
GW step; ``convolve_energy`` / ``retarded_from_lg`` keep the reference
signatures (convolve.py:39, :101) for numpy or torch inputs.
"""

from __future__ import annotations

import numpy as np
import torch
from scipy.fft import next_fast_len

from . import _lib
from .constants import C_POLARIZATION, C_SIGMA

MODE_CONVOLUTION = "convolution"
MODE_CORRELATION = "correlation"

_PLANS: dict[tuple, "ConvPlan"] = {}


def retarded_padding(n: int) -> int:
    """convolve.py:118-121: m = next_fast_len(2N), forced even."""
    m = next_fast_len(2 * n)
    if m % 2 == 1:
        m = next_fast_len(m + 1)
    return m


class ConvPlan:
    """Tables for series of length n on a power-of-two circular grid
    L >= max(8, 2n-1): twiddles exp(-2 pi i k / L), k < L, and the causal
    kernel spectra in natural order."""

    def __init__(self, n: int, device) -> None:
        self.n = n
        self.dev = torch.device(device)
        L = 8
        while L < 2 * n - 1:
            L *= 2
        self.L = L
        k = np.arange(L)
        tw = np.exp(-2j * np.pi * k / L)
        m = retarded_padding(n)
        theta = np.zeros(m)
        theta[0] = theta[m // 2] = 0.5
        theta[1:m // 2] = 1.0
        km = np.fft.ifft(theta)  # causal kernel on the reference's m-grid
        kc = np.zeros(L, dtype=complex)
        kc[:n] = km[:n]
        if n > 1:
            kc[L - np.arange(1, n)] = km[m - np.arange(1, n)]
        kf = np.fft.fft(kc)
        kcf = np.fft.fft(np.conj(kc))
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex128)).to(self.dev)
        self.tw, self.kf, self.kcf = t(tw), t(kf), t(kcf)

    @classmethod
    def get(cls, n: int, device) -> "ConvPlan":
        dev = torch.device(device)
        key = (n, dev.type, dev.index)
        if key not in _PLANS:
            _PLANS[key] = cls(n, dev)
        return _PLANS[key]


def _rows(x: torch.Tensor) -> int:
    return int(np.prod(x.shape[:-1])) if x.dim() > 1 else 1


def _check(*ts):
    for t in ts:
        if t is not None and (t.dtype != torch.complex128 or not t.is_cuda or not t.is_contiguous()):
            raise ValueError("expected contiguous complex128 CUDA tensors")


def polarization(gl: torch.Tensor, gg: torch.Tensor, diag: torch.Tensor | None, de: float,
                 prefactor: complex = C_POLARIZATION, out=None):
    """scba.py:1035-1048 for rows of entry-major G^<, G^> (n_rows, n_e):
    returns (P^<, P^>, P^R_up, P^R_lo)."""
    _check(gl, gg)
    n = gl.shape[-1]
    plan = ConvPlan.get(n, gl.device)
    out = out or tuple(torch.empty_like(gl) for _ in range(4))
    sc = complex(prefactor) * de
    lib = _lib.load()
    rc = lib.negf_conv_polarization(_rows(gl), n, plan.L, gl.data_ptr(), gg.data_ptr(), plan.tw.data_ptr(),
                                    plan.kf.data_ptr(), plan.kcf.data_ptr(), _lib.ptr(diag), sc.real, sc.imag,
                                    *(o.data_ptr() for o in out), _lib.stream_ptr(gl.device))
    _lib.check(rc, "negf_conv_polarization")
    return out


def self_energy(gl: torch.Tensor, gg: torch.Tensor, wl: torch.Tensor, wg: torch.Tensor,
                w_rows: torch.Tensor | None, diag: torch.Tensor | None, de: float,
                prefactor: complex = C_SIGMA, out=None):
    """scba.py:1118-1132: returns (Sigma^<, Sigma^>, Sigma^R_up, Sigma^R_lo)."""
    _check(gl, gg, wl, wg)
    n = gl.shape[-1]
    plan = ConvPlan.get(n, gl.device)
    out = out or tuple(torch.empty_like(gl) for _ in range(4))
    sc = complex(prefactor) * de
    lib = _lib.load()
    rc = lib.negf_conv_sigma(_rows(gl), n, plan.L, gl.data_ptr(), gg.data_ptr(), wl.data_ptr(), wg.data_ptr(),
                             _lib.ptr(w_rows), plan.tw.data_ptr(), plan.kf.data_ptr(), plan.kcf.data_ptr(),
                             _lib.ptr(diag), sc.real, sc.imag, *(o.data_ptr() for o in out),
                             _lib.stream_ptr(gl.device))
    _lib.check(rc, "negf_conv_sigma")
    return out


def _as_dev(x, device="cuda"):
    if isinstance(x, torch.Tensor):
        return x.to(dtype=torch.complex128).contiguous(), True
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=complex))).to(device), False


def convolve_energy(x1, x2, mode: str, prefactor: complex, de: float):
    """convolve.py:39-71 signature. numpy in -> numpy out; CUDA tensors stay on device."""
    a, is_t = _as_dev(x1)
    b, _ = _as_dev(x2, a.device)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch {tuple(a.shape)} vs {tuple(b.shape)}")
    if mode not in (MODE_CONVOLUTION, MODE_CORRELATION):
        raise ValueError(f"unknown mode {mode!r}")
    n = a.shape[-1]
    plan = ConvPlan.get(n, a.device)
    out = torch.empty_like(a)
    sc = complex(prefactor) * de
    rc = _lib.load().negf_convolve_energy(_rows(a), n, plan.L, a.data_ptr(), b.data_ptr(),
                                          0 if mode == MODE_CONVOLUTION else 1, sc.real, sc.imag,
                                          plan.tw.data_ptr(), out.data_ptr(), _lib.stream_ptr(a.device))
    _lib.check(rc, "negf_convolve_energy")
    return out if is_t else out.cpu().numpy()


def retarded_from_lg(x_lesser, x_greater):
    """convolve.py:101-129 signature."""
    a, is_t = _as_dev(x_lesser)
    b, _ = _as_dev(x_greater, a.device)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch {tuple(a.shape)} vs {tuple(b.shape)}")
    n = a.shape[-1]
    plan = ConvPlan.get(n, a.device)
    out = torch.empty_like(a)
    rc = _lib.load().negf_retarded_from_lg(_rows(a), n, plan.L, a.data_ptr(), b.data_ptr(), plan.tw.data_ptr(),
                                           plan.kf.data_ptr(), out.data_ptr(), _lib.stream_ptr(a.device))
    _lib.check(rc, "negf_retarded_from_lg")
    return out if is_t else out.cpu().numpy()
