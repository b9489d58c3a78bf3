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
                   max_iter: int = 100, check: bool = True, select: torch.Tensor | None = None,
                   out: torch.Tensor | None = None):
    """Sancho-Rubio for a batch (batch, bs, bs) of complex128 CUDA tensors.
    Returns (x, iters, status, resid) tensors. ``select`` (int32 per problem)
    restricts the solve to select != 0; the others keep ``out``'s values."""
    if tol <= 0:
        raise ValueError(f"tol must be positive, got {tol}")
    lib = _lib.load()
    batch, bs = m.shape[0], m.shape[-1]
    for t in (m, n, n_prime):
        if t.dtype != torch.complex128 or not t.is_cuda or tuple(t.shape) != (batch, bs, bs) or not t.is_contiguous():
            raise ValueError("m, n, n_prime must be contiguous complex128 CUDA tensors of one shape")
    dev = m.device
    x = torch.empty_like(m) if out is None else out
    status = torch.zeros(batch, dtype=torch.int32, device=dev)
    iters = torch.zeros(batch, dtype=torch.int32, device=dev)
    resid = torch.zeros(batch, dtype=torch.float64, device=dev)
    nbytes = lib.negf_sancho_workspace_bytes(batch, bs)
    ws = _lib.workspace(nbytes, dev)
    rc = lib.negf_obc_sancho_batched(batch, bs, m.data_ptr(), n.data_ptr(), n_prime.data_ptr(), tol,
                                     max_iter, x.data_ptr(), status.data_ptr(), iters.data_ptr(),
                                     resid.data_ptr(), _lib.ptr(select), ws.data_ptr(), nbytes,
                                     _lib.stream_ptr(dev))
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


def stein_batched(a: torch.Tensor, q: torch.Tensor, tol: float = 1e-12, max_iter: int = 100, check: bool = True,
                  select: torch.Tensor | None = None, out: torch.Tensor | None = None):
    """Geometric Stein w - a w a^dag = q for a batch (batch, bs, bs);
    ``select`` / ``out`` as in sancho_batched."""
    lib = _lib.load()
    batch, bs = a.shape[0], a.shape[-1]
    dev = a.device
    w = torch.empty_like(q) if out is None else out
    status = torch.zeros(batch, dtype=torch.int32, device=dev)
    iters = torch.zeros(batch, dtype=torch.int32, device=dev)
    nbytes = lib.negf_stein_workspace_bytes(batch, bs)
    ws = _lib.workspace(nbytes, dev)
    v0 = _lib.power_start_vector(bs, dev)
    rc = lib.negf_stein_batched(batch, bs, a.data_ptr(), q.data_ptr(), w.data_ptr(), tol, max_iter, v0.data_ptr(),
                                status.data_ptr(), iters.data_ptr(), _lib.ptr(select), ws.data_ptr(), nbytes,
                                _lib.stream_ptr(dev))
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


# -- runtime memoization (obc.py:490-608) --------------------------------------

MEMO_SURFACE, MEMO_STEIN = 0, 1


class SurfaceCache:
    """obc.py:498-515 on the device: cached surface / Stein blocks in slots
    named (subsystem, kind-class), each (n_seg, ld, bs, bs) complex128 with
    (n_seg, ld) int32 has/used flags -- the reference's dict keyed by
    (subsystem, side, energy index, kind), laid out so one batch of energies
    is a strided slab. ``stats`` counts direct and memoized calls like the
    reference (read lazily: one device reduction per snapshot)."""

    def __init__(self, n_fpi_retarded: int = 20, n_fpi_lg: int = 10) -> None:
        if n_fpi_retarded < 2 or n_fpi_lg < 2:
            raise ValueError("refresh budgets must be at least 2")
        self.n_fpi_retarded, self.n_fpi_lg = n_fpi_retarded, n_fpi_lg
        self.slots: dict[tuple, tuple[torch.Tensor, torch.Tensor, torch.Tensor]] = {}
        self._calls = 0
        self._memo = None

    def n_fpi(self, kind: str) -> int:
        return self.n_fpi_retarded if kind == "R" else self.n_fpi_lg

    def slot(self, name: tuple, n_seg: int, ld: int, bs: int, device):
        s = self.slots.get(name)
        if s is None:
            dev = torch.device(device)
            s = (torch.zeros((n_seg, ld, bs, bs), dtype=torch.complex128, device=dev),
                 torch.zeros((n_seg, ld), dtype=torch.int32, device=dev),
                 torch.zeros((n_seg, ld), dtype=torch.int32, device=dev))
            self.slots[name] = s
            if self._memo is None:
                self._memo = torch.zeros((), dtype=torch.int64, device=dev)
        return s

    def record(self, used: torch.Tensor, e0: int, n_e: int) -> None:
        """Count the calls of one batch (columns e0:e0+n_e of a used array)."""
        u = used[:, e0:e0 + n_e]
        self._calls += u.numel()
        self._memo += u.sum()

    @property
    def stats(self) -> dict[str, int]:
        memo = int(self._memo.item()) if self._memo is not None else 0
        return {"direct_calls": self._calls - memo, "memoized_calls": memo}

    def hit_rate(self) -> float:
        st = self.stats
        total = st["direct_calls"] + st["memoized_calls"]
        return st["memoized_calls"] / total if total else 0.0


def memo_refresh_batched(kind: int, x0: torch.Tensor, has: torch.Tensor, n_fpi: int, tol: float,
                         m=None, n=None, n_prime=None, a=None, q=None, n_kind: int = 1):
    """The refresh leg of memoized_obc for a batch (negf_memo_refresh_batched).
    Returns (out, need_direct, used); out holds the accepted iterates."""
    lib = _lib.load()
    p_all, bs = x0.shape[0], x0.shape[-1]
    n_side = p_all // n_kind
    dev = x0.device
    out = torch.zeros_like(x0)
    need = torch.zeros(p_all, dtype=torch.int32, device=dev)
    used = torch.zeros(p_all, dtype=torch.int32, device=dev)
    nbytes = lib.negf_memo_workspace_bytes(kind, n_side, n_kind, bs)
    ws = _lib.workspace(nbytes, dev)
    p = _lib.ptr
    rc = lib.negf_memo_refresh_batched(kind, n_side, n_kind, bs, p(m), p(n), p(n_prime), p(a), p(q), n_fpi, tol,
                                       p(x0), p(has), p(out), p(need), p(used), p(ws), nbytes, _lib.stream_ptr(dev))
    _lib.check(rc, "negf_memo_refresh_batched")
    return out, need, used


def memoized_surface_batched(m: torch.Tensor, n: torch.Tensor, n_prime: torch.Tensor, x0: torch.Tensor,
                             has: torch.Tensor, n_fpi: int = 20, tol: float = 1e-6, surface_tol: float = 1e-8,
                             max_iter: int = 100):
    """memoized_obc (obc.py:519-608) for a batch of surface problems with the
    fixed_point_step refresh and Sancho-Rubio as the direct solver.
    Returns (x, used): used[b] = 1 where the cached block was refreshed."""
    out, need, used = memo_refresh_batched(MEMO_SURFACE, x0, has, n_fpi, tol, m=m, n=n, n_prime=n_prime)
    sancho_batched(m, n, n_prime, surface_tol, max_iter, select=need, out=out)
    return out, used


def memoized_stein_batched(a: torch.Tensor, q: torch.Tensor, w0: torch.Tensor, has: torch.Tensor,
                           n_fpi: int = 10, tol: float = 1e-6, stein_tol: float = 1e-12, max_iter: int = 100):
    """memoized_obc with the Stein map w <- q + a w a^dag and the geometric
    Stein solve as the direct solver (scba.py:647-658)."""
    out, need, used = memo_refresh_batched(MEMO_STEIN, w0, has, n_fpi, tol, a=a, q=q)
    stein_batched(a, q, stein_tol, max_iter, select=need, out=out)
    return out, used


# -- Beyn contour-integral solver (obc.py:184-296) ---------------------------------

BEYN_PROBE_SEED = 1278  # obc.py:47


@dataclass
class BeynResult:
    """obc.py:89-94."""

    x_r: np.ndarray
    n_modes: int
    residual: float
    no_modes_warning: bool = False


_PROBES: dict = {}


def _probe(bs: int, dev, seed: int = BEYN_PROBE_SEED) -> torch.Tensor:
    key = (bs, dev.type, dev.index, seed)
    if key not in _PROBES:
        rng = np.random.default_rng(seed)
        pr = rng.standard_normal((bs, bs)) + 1j * rng.standard_normal((bs, bs))
        _PROBES[key] = torch.from_numpy(pr).to(dev)
    return _PROBES[key]


def beyn_batched(m: torch.Tensor, n: torch.Tensor, n_prime: torch.Tensor, n_quad: int = 16, radius: float = 1.0,
                 center: complex = 0.0, svd_tol: float = 1e-8):
    """obc_beyn for a batch (batch, bs, bs) of nearest-neighbour leads
    (stencil [n', m, n]). Contour moments on the device
    (negf_beyn_moments: batched P(z)^-1 over the quadrature nodes), then per
    problem the rank-revealing SVD, the reduced eigenproblem and the
    pseudo-inverse (cuSOLVER via torch.linalg, rcond 1e-15 like numpy),
    and x = (m + n F)^-1 with the library's batched inverse.
    Returns (x, n_modes) -- n_modes = 0 marks the reference's fallback
    x = m^-1 (decoupled lead, zero rank or no decaying modes)."""
    if n_quad < 8:
        raise ValueError(f"need at least 8 quadrature nodes, got {n_quad}")
    if not 0 < radius <= 1:
        raise ValueError(f"radius must lie in (0, 1], got {radius}")
    lib = _lib.load()
    batch, bs = m.shape[0], m.shape[-1]
    dev = m.device
    zs = center + radius * np.exp(2j * np.pi * np.arange(n_quad) / n_quad)
    ws_ = (zs - center) / n_quad
    zh = np.ascontiguousarray(np.stack([zs.real, zs.imag], 1).reshape(-1))
    wh = np.ascontiguousarray(np.stack([ws_.real, ws_.imag], 1).reshape(-1))
    a0, a1 = torch.empty_like(m), torch.empty_like(m)
    status = torch.zeros(batch, dtype=torch.int32, device=dev)
    nbytes = lib.negf_beyn_workspace_bytes(batch, bs)
    ws = _lib.workspace(nbytes, dev)
    import ctypes

    dp = ctypes.POINTER(ctypes.c_double)
    rc = lib.negf_beyn_moments(batch, bs, n_quad, m.data_ptr(), n.data_ptr(), n_prime.data_ptr(),
                               zh.ctypes.data_as(dp), wh.ctypes.data_as(dp), _probe(bs, dev).data_ptr(),
                               a0.data_ptr(), a1.data_ptr(), status.data_ptr(), ws.data_ptr(), nbytes,
                               _lib.stream_ptr(dev))
    _lib.check(rc, "negf_beyn_moments")
    st = status.cpu().numpy()
    if np.any(st):
        b = int(np.flatnonzero(st)[0])
        raise SingularBlockError(f"singular contour node {int(st[b]) - 1} (Beyn problem {b})")
    u, sig, vh = torch.linalg.svd(a0)
    sig_h = sig.cpu().numpy()
    decoupled = (n.abs().amax(dim=(1, 2)) == 0).cpu().numpy()
    target = m.clone()
    modes = np.zeros(batch, dtype=np.int64)
    f_all = torch.zeros_like(m)
    # Reduced problems batched by numerical rank (cuSOLVER batched SVD /
    # eig / pinv through torch.linalg): the decaying modes (|mu| < 1) are
    # selected by zeroing the other eigenvector columns -- pinv of [Phi 0] is
    # [pinv(Phi); 0], so F = Phi diag(mu) Phi^+ equals the per-problem form
    # that drops them (obc.py:260-296).
    valid = (~decoupled) & (sig_h[:, 0] > 0)
    ranks = np.where(valid, np.sum(sig_h > svd_tol * sig_h[:, :1], axis=1), 0)
    for r in np.unique(ranks[ranks > 0]):
        idx_h = np.flatnonzero(ranks == r)
        idx = torch.from_numpy(idx_h).to(dev)
        ub = u[idx, :, :r]
        w_red = vh[idx].conj().transpose(-1, -2)[:, :, :r]
        b_small = (ub.conj().transpose(-1, -2) @ a1[idx] @ w_red) / sig[idx, :r].unsqueeze(-2)
        mu, vecs = torch.linalg.eig(b_small)
        keep = mu.abs() < 1.0 - 1e-8
        mu = mu * keep
        phi = ub @ (vecs * keep.unsqueeze(-2))
        f = (phi * mu.unsqueeze(-2)) @ torch.linalg.pinv(phi, rtol=1e-15)
        n_keep = keep.sum(-1)
        has = n_keep > 0
        f_all[idx[has]] = f[has]
        modes[idx_h] = n_keep.cpu().numpy()
    # x = (m + n F)^-1 (problems without modes keep F = 0: x = m^-1)
    st_ = _lib.stream_ptr(dev)
    rc = lib.negf_zgemm_batched(bs, bs, bs, batch, 1.0, 0.0, n.data_ptr(), bs * bs, bs, 0, f_all.data_ptr(),
                                bs * bs, bs, 0, 1.0, 0.0, m.data_ptr(), bs * bs, bs, target.data_ptr(), bs * bs, bs,
                                st_)
    _lib.check(rc, "negf_zgemm_batched")
    x = torch.empty_like(m)
    inv_status = torch.zeros(batch, dtype=torch.int32, device=dev)
    nbytes = lib.negf_zinv_workspace_bytes(bs, batch)
    ws = _lib.workspace(nbytes, dev)
    rc = lib.negf_zinv_batched(bs, batch, target.data_ptr(), x.data_ptr(), inv_status.data_ptr(), None,
                               ws.data_ptr(), nbytes, st_)
    _lib.check(rc, "negf_zinv_batched")
    if int(inv_status.amax().item()):
        raise SingularBlockError("singular surface matrix m + n F")
    return x, modes


def obc_beyn(m_tilde_blocks, contour: dict | None = None, svd_tol: float = 1e-8, probe_seed: int = BEYN_PROBE_SEED,
             device="cuda") -> BeynResult:
    """obc.py:198-296 signature for a nearest-neighbour stencil [n', m, n]
    (N_U = 1; longer stencils are outside the hot path)."""
    if len(m_tilde_blocks) != 3:
        raise ValueError("the GPU Beyn solver takes nearest-neighbour stencils [n', m, n]")
    if probe_seed != BEYN_PROBE_SEED:
        raise ValueError("only the reference probe seed is supported")
    params = {"radius": 1.0, "center": 0.0, "n_quad": 16}
    params.update(contour or {})
    dev = torch.device(device)
    npr, m, n = (_t(b, dev)[None] for b in m_tilde_blocks)
    x, modes = beyn_batched(m, n, npr, int(params["n_quad"]), float(params["radius"]), complex(params["center"]),
                            svd_tol)
    return BeynResult(x[0].cpu().numpy(), int(modes[0]), float("nan"), no_modes_warning=int(modes[0]) == 0)


def fixed_point_batched(m: torch.Tensor, n: torch.Tensor, n_prime: torch.Tensor, x0: torch.Tensor | None = None,
                        tol: float = 1e-10, max_iter: int = 5000):
    """obc_fixed_point for a batch: returns (x, iters, status, resid) tensors
    (status 0 converged, 1 singular update, 2 not converged)."""
    if tol <= 0:
        raise ValueError(f"tol must be positive, got {tol}")
    lib = _lib.load()
    batch, bs = m.shape[0], m.shape[-1]
    dev = m.device
    x = torch.empty_like(m)
    status = torch.zeros(batch, dtype=torch.int32, device=dev)
    iters = torch.zeros(batch, dtype=torch.int32, device=dev)
    resid = torch.full((batch,), float("nan"), dtype=torch.float64, device=dev)
    nbytes = lib.negf_fixed_point_workspace_bytes(batch, bs)
    ws = _lib.workspace(nbytes, dev)
    rc = lib.negf_obc_fixed_point_batched(batch, bs, m.data_ptr(), n.data_ptr(), n_prime.data_ptr(), _lib.ptr(x0),
                                          tol, max_iter, x.data_ptr(), status.data_ptr(), iters.data_ptr(),
                                          resid.data_ptr(), ws.data_ptr(), nbytes, _lib.stream_ptr(dev))
    _lib.check(rc, "negf_obc_fixed_point_batched")
    return x, iters, status, resid


def obc_fixed_point(c, x0=None, max_iter: int = 5000, tol: float = 1e-10, device="cuda") -> SurfaceResult:
    """obc.py:108-135 signature: direct iteration x <- (m - n x n')^-1 from x0
    (default 0); not converging is reported (converged=False), not raised."""
    dev = torch.device(device)
    x, iters, status, resid = fixed_point_batched(_t(c.m, dev)[None], _t(c.n, dev)[None], _t(c.n_prime, dev)[None],
                                                  None if x0 is None else _t(x0, dev)[None], tol, max_iter)
    st, it = int(status[0]), int(iters[0])
    if st == OBC_SINGULAR:
        raise SingularBlockError(f"singular surface update at fixed-point iteration {it}")
    return SurfaceResult(x[0].cpu().numpy(), it, st == OBC_OK, float(resid[0]))


def solve_surfaces(m: torch.Tensor, n: torch.Tensor, n_prime: torch.Tensor, method: str, memo=None,
                   slot: tuple = ("G", "R"), surface_tol: float = 1e-8, beyn=None) -> torch.Tensor:
    """_retarded_surface (scba.py:577-614) for a batch of contact cells
    stacked [2 sides][n_e]: the direct solver ``method`` ("beyn" or
    "fixed_point"; Sancho runs inside the library's closure kernels), through
    the memoizer when ``memo`` = (SurfaceCache, ld, e0, tol_memo) is given:
    cached problems are refreshed with fixed_point_step, the direct solver
    runs on the rest only, and every result goes back to the cache."""
    if method == "beyn":
        o = beyn
        direct = lambda a, b_, c_: beyn_batched(a, b_, c_, o.n_quad, o.radius, 0.0, o.svd_tol)[0]
    elif method == "fixed_point":
        def direct(a, b_, c_):
            x, it, st, _ = fixed_point_batched(a, b_, c_, None, surface_tol)
            stn = st.cpu().numpy()
            if np.any(stn == OBC_SINGULAR):
                b0 = int(np.flatnonzero(stn == OBC_SINGULAR)[0])
                raise SingularBlockError(f"singular surface update at fixed-point iteration {int(it[b0])}")
            return x  # like the reference, an unconverged iterate is used as is
    else:
        raise ValueError(f"unknown retarded method {method!r}")
    if memo is None:
        return direct(m, n, n_prime)
    cache, ld, e0, tol_memo = memo
    ne = m.shape[0] // 2
    xs, hs, us = cache.slot(slot, 2, ld, m.shape[-1], m.device)
    x0 = torch.cat([xs[0, e0:e0 + ne], xs[1, e0:e0 + ne]])
    has = torch.cat([hs[0, e0:e0 + ne], hs[1, e0:e0 + ne]]).contiguous()
    x, need, used = memo_refresh_batched(MEMO_SURFACE, x0, has, cache.n_fpi("R"), tol_memo, m=m, n=n, n_prime=n_prime)
    idx = torch.nonzero(need).flatten()
    if idx.numel():
        x[idx] = direct(m[idx].contiguous(), n[idx].contiguous(), n_prime[idx].contiguous())
    xs[0, e0:e0 + ne], xs[1, e0:e0 + ne] = x[:ne], x[ne:]
    hs[:, e0:e0 + ne] = 1
    us[0, e0:e0 + ne], us[1, e0:e0 + ne] = used[:ne], used[ne:]
    cache.record(us, e0, ne)
    return x


def contact_cells(m_diag: torch.Tensor, m_upper: torch.Tensor, m_lower: torch.Tensor):
    """_lead_cell (scba.py:558-574) for both sides, stacked [2 sides][n_e]:
    left m = M_00, n = M_10, n' = M_01; right m = M_{N-1,N-1},
    n = M_{N-2,N-1}, n' = M_{N-1,N-2}."""
    nb = m_diag.shape[1]
    m = torch.cat([m_diag[:, 0], m_diag[:, nb - 1]])
    n = torch.cat([m_lower[:, 0], m_upper[:, nb - 2]])
    npr = torch.cat([m_upper[:, 0], m_lower[:, nb - 2]])
    return m, n, npr
