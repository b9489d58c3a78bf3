"""Open-boundary contact self-energies on the GPU (drop-in for negfgw.obc).

Batched native API: ``sancho_batched`` (many surface problems in one call)
and ``sigma_lg_obc_batched``. Reference-signature shims: ``obc_sancho_rubio``
(obc.py:144), ``sigma_lg_obc`` (obc.py:460), ``fixed_point_step`` (obc.py:138).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
from scipy.special import expit

from . import _lib
from .errors import ConvergenceError, SingularBlockError, SpectralRadiusError

SIDE_LEFT = "left"
SIDE_RIGHT = "right"

OBC_OK, OBC_SINGULAR, OBC_NOT_CONVERGED, OBC_RESIDUAL = 0, 1, 2, 3


def fermi(e, mu: float, kT: float):
    """device.py:32-36: overflow-safe Fermi-Dirac occupation."""
    if kT <= 0.0:
        raise ValueError(f"kT must be positive, got {kT}")
    return expit(-(np.asarray(e, dtype=float) - mu) / kT)


@dataclass(frozen=True)
class ContactBlocks:
    """obc.py:50-81: boundary cell m, coupling n into the lead, reverse n'."""

    m: np.ndarray
    n: np.ndarray
    n_prime: np.ndarray
    side: str = SIDE_LEFT
    subsystem: str = "G"


@dataclass
class SurfaceResult:
    x_r: np.ndarray
    iters: int
    converged: bool
    residual: float = float("nan")


@dataclass
class ObcSigma:
    sigma_r: np.ndarray
    sigma_lesser: np.ndarray
    sigma_greater: np.ndarray


def raise_on_obc_status(status: np.ndarray, iters: np.ndarray, resid: np.ndarray | None,
                        max_iter: int, tol: float, what: str = "surface") -> None:
    bad = np.flatnonzero(status)
    if not bad.size:
        return
    b = int(bad[0])
    code = int(status[b])
    if code == OBC_SINGULAR:
        raise SingularBlockError(f"singular block in {what} problem {b}")
    if code == OBC_NOT_CONVERGED:
        raise ConvergenceError(f"surface decimation did not converge in {max_iter} sweeps ({what} problem {b})")
    r = float("nan") if resid is None else float(resid[b])
    raise ConvergenceError(
        f"decimation closed but residual {r:.3e} exceeds {10 * max(tol, 1e-14):.3e} ({what} problem {b})")


def sancho_batched(m: torch.Tensor, n: torch.Tensor, n_prime: torch.Tensor, tol: float = 1e-12,
                   max_iter: int = 100, check: bool = True):
    """Sancho-Rubio for a batch (batch, bs, bs) of complex128 CUDA tensors.
    Returns (x, iters, status, resid) tensors."""
    if tol <= 0:
        raise ValueError(f"tol must be positive, got {tol}")
    lib = _lib.load()
    batch, bs = m.shape[0], m.shape[-1]
    for t in (m, n, n_prime):
        if t.dtype != torch.complex128 or not t.is_cuda or tuple(t.shape) != (batch, bs, bs) or not t.is_contiguous():
            raise ValueError("m, n, n_prime must be contiguous complex128 CUDA tensors of one shape")
    dev = m.device
    x = torch.empty_like(m)
    status = torch.zeros(batch, dtype=torch.int32, device=dev)
    iters = torch.zeros(batch, dtype=torch.int32, device=dev)
    resid = torch.zeros(batch, dtype=torch.float64, device=dev)
    nbytes = lib.negf_sancho_workspace_bytes(batch, bs)
    ws = _lib.workspace(nbytes, dev)
    rc = lib.negf_obc_sancho_batched(batch, bs, m.data_ptr(), n.data_ptr(), n_prime.data_ptr(), tol,
                                     max_iter, x.data_ptr(), status.data_ptr(), iters.data_ptr(),
                                     resid.data_ptr(), ws.data_ptr(), nbytes, _lib.stream_ptr(dev))
    _lib.check(rc, "negf_obc_sancho_batched")
    if check:
        raise_on_obc_status(status.cpu().numpy(), iters.cpu().numpy(), resid.cpu().numpy(), max_iter, tol)
    return x, iters, status, resid


def sigma_lg_obc_batched(x_r: torch.Tensor, n: torch.Tensor, n_prime: torch.Tensor, f: torch.Tensor):
    """(Sigma^R, Sigma^<, Sigma^>) for a batch; f = contact occupation per problem."""
    lib = _lib.load()
    batch, bs = x_r.shape[0], x_r.shape[-1]
    dev = x_r.device
    sr, sl, sg = torch.empty_like(x_r), torch.empty_like(x_r), torch.empty_like(x_r)
    f = f.to(device=dev, dtype=torch.float64).contiguous()
    nbytes = lib.negf_sigma_lg_obc_workspace_bytes(batch, bs)
    ws = _lib.workspace(nbytes, dev)
    rc = lib.negf_sigma_lg_obc_batched(batch, bs, x_r.data_ptr(), n.data_ptr(), n_prime.data_ptr(),
                                       f.data_ptr(), sr.data_ptr(), sl.data_ptr(), sg.data_ptr(),
                                       ws.data_ptr(), nbytes, _lib.stream_ptr(dev))
    _lib.check(rc, "negf_sigma_lg_obc_batched")
    return sr, sl, sg


def _t(a, dev) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=complex))).to(dev)


def obc_sancho_rubio(c, tol: float = 1e-12, max_iter: int = 100, device="cuda") -> SurfaceResult:
    """obc.py:144-182 signature (single problem)."""
    dev = torch.device(device)
    x, iters, _, resid = sancho_batched(_t(c.m, dev)[None], _t(c.n, dev)[None], _t(c.n_prime, dev)[None],
                                        tol, max_iter)
    return SurfaceResult(x[0].cpu().numpy(), int(iters[0]), True, float(resid[0]))


def sigma_lg_obc(x_r, contact_mu: float, kT: float, energy: float, couplings, device="cuda") -> ObcSigma:
    """obc.py:460-486 signature (single problem)."""
    if not np.all(np.isfinite(x_r)):
        raise ValueError("non-finite surface block")
    dev = torch.device(device)
    n, n_prime = couplings
    f = torch.tensor([float(fermi(energy, contact_mu, kT))], dtype=torch.float64)
    sr, sl, sg = sigma_lg_obc_batched(_t(x_r, dev)[None], _t(n, dev)[None], _t(n_prime, dev)[None], f)
    return ObcSigma(sr[0].cpu().numpy(), sl[0].cpu().numpy(), sg[0].cpu().numpy())


def stein_batched(a: torch.Tensor, q: torch.Tensor, tol: float = 1e-12, max_iter: int = 100, check: bool = True):
    """Geometric Stein w - a w a^dag = q for a batch (batch, bs, bs)."""
    lib = _lib.load()
    batch, bs = a.shape[0], a.shape[-1]
    dev = a.device
    w = torch.empty_like(q)
    status = torch.zeros(batch, dtype=torch.int32, device=dev)
    iters = torch.zeros(batch, dtype=torch.int32, device=dev)
    nbytes = lib.negf_stein_workspace_bytes(batch, bs)
    ws = _lib.workspace(nbytes, dev)
    v0 = _lib.power_start_vector(bs, dev)
    rc = lib.negf_stein_batched(batch, bs, a.data_ptr(), q.data_ptr(), w.data_ptr(), tol, max_iter, v0.data_ptr(),
                                status.data_ptr(), iters.data_ptr(), ws.data_ptr(), nbytes, _lib.stream_ptr(dev))
    _lib.check(rc, "negf_stein_batched")
    if check:
        st = status.cpu().numpy()
        if np.any(st == 4):
            raise SpectralRadiusError("spectral radius estimate >= 1; geometric series diverges")
        if np.any(st):
            raise ConvergenceError(f"geometric Stein did not reach tol {tol} in {max_iter} squarings")
    return w, iters


def stein_geometric(a, q, tol: float = 1e-12, max_iter: int = 100, device="cuda"):
    """obc.py:427-447 signature (single problem)."""
    dev = torch.device(device)
    w, _ = stein_batched(_t(a, dev)[None], _t(q, dev)[None], tol, max_iter)
    return w[0].cpu().numpy()


def fixed_point_step(c, x, device="cuda"):
    """obc.py:138-141: one surface update (m - n x n')^-1 on the device."""
    lib = _lib.load()
    dev = torch.device(device)
    m, n, npr, xx = (_t(v, dev) for v in (c.m, c.n, c.n_prime, x))
    bs = m.shape[-1]
    t = torch.empty_like(m)
    s_ = t.clone()
    st = _lib.stream_ptr(dev)
    rc = lib.negf_zgemm_batched(bs, bs, bs, 1, 1.0, 0.0, n.data_ptr(), 0, bs, 0, xx.data_ptr(), 0, bs, 0, 0.0, 0.0,
                                None, 0, bs, t.data_ptr(), 0, bs, st)
    _lib.check(rc, "negf_zgemm_batched")
    rc = lib.negf_zgemm_batched(bs, bs, bs, 1, -1.0, 0.0, t.data_ptr(), 0, bs, 0, npr.data_ptr(), 0, bs, 0, 1.0, 0.0,
                                m.data_ptr(), 0, bs, s_.data_ptr(), 0, bs, st)
    _lib.check(rc, "negf_zgemm_batched")
    out = torch.empty_like(m)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    nbytes = lib.negf_zinv_workspace_bytes(bs, 1)
    ws = _lib.workspace(nbytes, dev)
    rc = lib.negf_zinv_batched(bs, 1, s_.data_ptr(), out.data_ptr(), status.data_ptr(), None, ws.data_ptr(), nbytes, st)
    _lib.check(rc, "negf_zinv_batched")
    if int(status.item()):
        raise SingularBlockError("singular surface update")
    return out.cpu().numpy()
