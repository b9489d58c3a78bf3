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


# Longest circular grid of the fused P / Sigma kernels: 4096 on one CTA (two
# L-point complex arrays per row in shared memory), 8192 (N_E <= 4096, C4's
# 4096 energies) on a cluster pair of CTAs splitting the even / odd bins
# (conv.cu pol_kernel_x2 / sigma_kernel_x2). The reference-signature drop-ins
# convolve_energy / retarded_from_lg run the one-CTA engine up to 4096. Longer
# series (beyond every BASELINE config) run the same algebra through cuFFT
# (torch.fft on the device) in row chunks.
_MAX_L_ENV = int(__import__("os").environ.get("NEGF_CONV_MAX_L", "8192"))  # env: tests of the cuFFT leg
MAX_L_NATIVE = _MAX_L_ENV
MAX_L_GENERIC = min(_MAX_L_ENV, 4096)
_CHUNK_BYTES = 1 << 30


def _chunks(n_rows: int, L: int):
    step = max(1, _CHUNK_BYTES // (16 * L * 4))
    for r0 in range(0, n_rows, step):
        yield slice(r0, min(n_rows, r0 + step))


def _proj_rows(x: torch.Tensor, diag) -> torch.Tensor:
    if diag is not None:
        m = diag.bool()
        x[m] = 1j * x[m].imag
    return x


def _retarded_tail_fft(d: torch.Tensor, plan: "ConvPlan", up: torch.Tensor | None, lo: torch.Tensor | None) -> None:
    """r_up = K*d, r_lo = -conj(conj(K)*d) on the L-grid (as retarded_tail in conv.cu)."""
    n = d.shape[-1]
    D = torch.fft.fft(d, n=plan.L, dim=-1)
    if up is not None:
        up.copy_(torch.fft.ifft(D * plan.kf, dim=-1)[:, :n])
    if lo is not None:
        lo.copy_(-torch.fft.ifft(D * plan.kcf, dim=-1)[:, :n].conj())


def _pol_fft(gl, gg, diag, sc: complex, plan, out) -> None:
    n, L = gl.shape[-1], plan.L
    g2 = lambda x: x.reshape(-1, n)
    gl2, gg2 = g2(gl), g2(gg)
    o2 = [g2(o) for o in out]
    for s in _chunks(gl2.shape[0], L):
        a = torch.fft.fft(gl2[s], n=L, dim=-1)
        b = torch.fft.fft(gg2[s], n=L, dim=-1)
        p = torch.fft.ifft(a * -b.conj(), dim=-1)
        dg = diag[s] if diag is not None else None
        pl = _proj_rows(sc * p[:, :n], dg)
        rev = torch.roll(torch.flip(p, dims=[-1]), 1, dims=-1)  # p[(L - k) % L]
        pg = _proj_rows(sc * rev[:, :n].conj(), dg)
        o2[0][s], o2[1][s] = pl, pg
        _retarded_tail_fft(pg - pl, plan, o2[2][s] if out[2] is not None else None,
                           o2[3][s] if out[3] is not None else None)


def _sigma_fft(gl, gg, wl, wg, w_rows, diag, sc: complex, plan, out) -> None:
    n, L = gl.shape[-1], plan.L
    g2 = lambda x: x.reshape(-1, n)
    gl2, gg2, wl2, wg2 = g2(gl), g2(gg), g2(wl), g2(wg)
    o2 = [g2(o) for o in out]
    for s in _chunks(gl2.shape[0], L):
        dg = diag[s] if diag is not None else None
        res = []
        for gx, wx in ((gl2, wl2), (gg2, wg2)):
            w = wx[w_rows[s]] if w_rows is not None else wx[s]
            x = torch.fft.ifft(torch.fft.fft(gx[s], n=L, dim=-1) * torch.fft.fft(w, n=L, dim=-1), dim=-1)
            res.append(_proj_rows(sc * x[:, :n], dg))
        o2[0][s], o2[1][s] = res
        _retarded_tail_fft(res[1] - res[0], plan, o2[2][s] if out[2] is not None else None,
                           o2[3][s] if out[3] is not None else None)


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
    if plan.L > MAX_L_NATIVE:
        _pol_fft(gl, gg, diag, sc, plan, out)
        return out
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
    if plan.L > MAX_L_NATIVE:
        _sigma_fft(gl, gg, wl, wg, w_rows, diag, sc, plan, out)
        return out
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
    if plan.L > MAX_L_GENERIC:
        a2, b2, o2 = a.reshape(-1, n), b.reshape(-1, n), out.reshape(-1, n)
        for s in _chunks(a2.shape[0], plan.L):
            y = b2[s] if mode == MODE_CONVOLUTION else torch.roll(torch.flip(
                torch.nn.functional.pad(b2[s], (0, plan.L - n)), dims=[-1]), 1, dims=-1)  # y[j] = b[-j]
            x = torch.fft.ifft(torch.fft.fft(a2[s], n=plan.L, dim=-1) * torch.fft.fft(y, n=plan.L, dim=-1), dim=-1)
            o2[s] = sc * x[:, :n]
        return out if is_t else out.cpu().numpy()
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
    if plan.L > MAX_L_GENERIC:
        a2, b2, o2 = a.reshape(-1, n), b.reshape(-1, n), out.reshape(-1, n)
        for s in _chunks(a2.shape[0], plan.L):
            _retarded_tail_fft(b2[s] - a2[s], plan, o2[s], None)
        return out if is_t else out.cpu().numpy()
    rc = _lib.load().negf_retarded_from_lg(_rows(a), n, plan.L, a.data_ptr(), b.data_ptr(), plan.tw.data_ptr(),
                                           plan.kf.data_ptr(), out.data_ptr(), _lib.stream_ptr(a.device))
    _lib.check(rc, "negf_retarded_from_lg")
    return out if is_t else out.cpu().numpy()
