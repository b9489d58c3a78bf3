"""Selected block-tridiagonal solve on the GPU (drop-in for negfgw.rgf).

Two entry levels:

* ``selected_solve_batched`` -- the native API: stacked complex128 CUDA
  tensors for a whole batch of energies, one C-ABI call
  (``negf_rgf_selected_solve_batched``, include/negf_b200.h) that runs the
  fused retarded + lesser + greater forward and backward sweeps.
* ``selected_solve`` / ``SelectedSolution`` -- the reference's per-energy
  signature (rgf.py:232-243, rgf.py:61-110), implemented as a batch of one.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .blocks import FULL, LG_COMPRESSED, BlockMatrix, lg_arrays, to_device, tridiag_arrays
from .errors import SingularBlockError

KIND_LESSER = "<"
KIND_GREATER = ">"
_KEYS = {KIND_LESSER: "xl", KIND_GREATER: "xg"}


def _check_bt(t: torch.Tensor, shape: tuple, name: str) -> None:
    if t.dtype != torch.complex128 or not t.is_cuda:
        raise ValueError(f"{name} must be a complex128 CUDA tensor")
    if tuple(t.shape) != shape:
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {shape}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def alloc_outputs(n_e: int, n_b: int, bs: int, kinds, device) -> dict[str, torch.Tensor]:
    z = dict(dtype=torch.complex128, device=device)
    out = {
        "xr_diag": torch.empty((n_e, n_b, bs, bs), **z),
        "xr_upper": torch.empty((n_e, max(n_b - 1, 0), bs, bs), **z),
        "xr_lower": torch.empty((n_e, max(n_b - 1, 0), bs, bs), **z),
    }
    for k in kinds:
        out[_KEYS[k] + "_diag"] = torch.empty((n_e, n_b, bs, bs), **z)
        out[_KEYS[k] + "_upper"] = torch.empty((n_e, max(n_b - 1, 0), bs, bs), **z)
    return out


def selected_solve_batched(
    m_diag: torch.Tensor,
    m_upper: torch.Tensor,
    m_lower: torch.Tensor,
    b_lesser: tuple[torch.Tensor, torch.Tensor] | None = None,
    b_greater: tuple[torch.Tensor, torch.Tensor] | None = None,
    symmetrize: bool = False,
    out: dict[str, torch.Tensor] | None = None,
    check: bool = True,
    u_spread: torch.Tensor | None = None,
    status: torch.Tensor | None = None,
    lg_anti_hermitian: bool = False,
) -> dict[str, torch.Tensor]:
    """Batched selected inverse of M (n_e, n_b, bs, bs) and X^lg = M^-1 B M^-dag.

    Returns tensors ``xr_diag/xr_upper/xr_lower`` and, per present kind,
    ``xl_*`` (lesser) / ``xg_*`` (greater) with diag + upper blocks. With
    ``check`` the per-energy status is read back and a singular Schur
    complement raises ``SingularBlockError`` naming the forward step like
    rgf.py:121-126 (this synchronises the stream). ``lg_anti_hermitian``
    declares the B^lg diagonal blocks anti-Hermitian (true of every lesser /
    greater source of the NEGF/GW solver), which lets the anti-Hermitian
    forward products run on half the tiles; the reference takes any B.
    """
    lib = _lib.load()
    n_e, n_b, bs = m_diag.shape[0], m_diag.shape[1], m_diag.shape[2]
    dev = m_diag.device
    _check_bt(m_diag, (n_e, n_b, bs, bs), "m_diag")
    off = (n_e, max(n_b - 1, 0), bs, bs)
    _check_bt(m_upper, off, "m_upper")
    _check_bt(m_lower, off, "m_lower")
    kinds = []
    for k, b in ((KIND_LESSER, b_lesser), (KIND_GREATER, b_greater)):
        if b is not None:
            _check_bt(b[0], (n_e, n_b, bs, bs), f"b{k}_diag")
            _check_bt(b[1], off, f"b{k}_upper")
            kinds.append(k)
    if out is None:
        out = alloc_outputs(n_e, n_b, bs, kinds, dev)
    if status is None:
        status = torch.zeros(n_e, dtype=torch.int32, device=dev)
    else:
        status.zero_()
    ws_bytes = lib.negf_rgf_workspace_bytes(n_e, n_b, bs)
    ws = _lib.workspace(ws_bytes, dev)
    p = _lib.ptr
    bl = b_lesser or (None, None)
    bg = b_greater or (None, None)
    rc = lib.negf_rgf_selected_solve_batched(
        n_e, n_b, bs,
        p(m_diag), p(m_upper), p(m_lower),
        p(bl[0]), p(bl[1]), p(bg[0]), p(bg[1]),
        p(out["xr_diag"]), p(out["xr_upper"]), p(out["xr_lower"]),
        p(out.get("xl_diag")) if b_lesser is not None else None,
        p(out.get("xl_upper")) if b_lesser is not None else None,
        p(out.get("xg_diag")) if b_greater is not None else None,
        p(out.get("xg_upper")) if b_greater is not None else None,
        (1 if symmetrize else 0) | (2 if lg_anti_hermitian else 0), p(status), p(u_spread), p(ws), ws_bytes,
        _lib.stream_ptr(dev),
    )
    _lib.check(rc, "negf_rgf_selected_solve_batched")
    out["status"] = status
    if check:
        raise_on_status(status)
    return out


def raise_on_status(status: torch.Tensor, energy_offset: int = 0) -> None:
    st = status.cpu().numpy()
    bad = np.flatnonzero(st)
    if bad.size:
        e = int(bad[0])
        raise SingularBlockError(
            f"singular Schur complement at forward step {int(st[e]) - 1} "
            f"(energy index {e + energy_offset})"
        )


# -- reference-signature shims (per energy) ---------------------------------


@dataclass
class SelectedSolution:
    """rgf.py:61-110: diagonal and first off-diagonal blocks of X^R and X^lg
    (numpy arrays; lower lesser/greater blocks implied)."""

    n_blocks: int
    block_size: int
    x_r_diag: list = field(default_factory=list)
    x_r_upper: list = field(default_factory=list)
    x_r_lower: list = field(default_factory=list)
    x_lg_diag: dict = field(default_factory=dict)
    x_lg_upper: dict = field(default_factory=dict)

    def lg_lower(self, kind: str, i: int) -> np.ndarray:
        return -self.x_lg_upper[kind][i].conj().T

    def symmetrize(self) -> None:
        for kind, diag in self.x_lg_diag.items():
            self.x_lg_diag[kind] = [0.5 * (b - b.conj().T) for b in diag]

    def retarded_block_matrix(self) -> BlockMatrix:
        out = BlockMatrix(self.n_blocks, self.block_size, min(3, 2 * self.n_blocks - 1))
        for i, b in enumerate(self.x_r_diag):
            out.set_block(i, i, b)
        for i in range(self.n_blocks - 1):
            out.set_block(i, i + 1, self.x_r_upper[i])
            out.set_block(i + 1, i, self.x_r_lower[i])
        return out

    def lg_block_matrix(self, kind: str, storage_mode: str = LG_COMPRESSED) -> BlockMatrix:
        out = BlockMatrix(self.n_blocks, self.block_size, min(3, 2 * self.n_blocks - 1), storage_mode)
        for i, b in enumerate(self.x_lg_diag[kind]):
            out.set_block(i, i, b)
        for i, b in enumerate(self.x_lg_upper[kind]):
            out.set_block(i, i + 1, b)
            if storage_mode == FULL:
                out.set_block(i + 1, i, -b.conj().T)
        return out


def _solution_from(out: dict, e: int, n: int, bs: int, kinds) -> SelectedSolution:
    host = {k: v[e].cpu().numpy() for k, v in out.items() if k != "status"}
    sol = SelectedSolution(n, bs)
    sol.x_r_diag = list(host["xr_diag"])
    sol.x_r_upper = list(host["xr_upper"])
    sol.x_r_lower = list(host["xr_lower"])
    for k in kinds:
        sol.x_lg_diag[k] = list(host[_KEYS[k] + "_diag"])
        sol.x_lg_upper[k] = list(host[_KEYS[k] + "_upper"])
    return sol


def selected_solve(m_tilde, b_lesser=None, b_greater=None, device="cuda") -> SelectedSolution:
    """rgf.py:232-243 signature: one energy, BlockMatrix in, SelectedSolution out
    (not symmetrized, like the reference)."""
    n, bs = m_tilde.n_blocks, m_tilde.block_size
    d, u, lo = tridiag_arrays(m_tilde)
    dev = torch.device(device)
    md, mu, ml = (to_device(x[None], dev) for x in (d, u, lo))
    srcs = []
    for b in (b_lesser, b_greater):
        if b is None:
            srcs.append(None)
        else:
            bd, bu = lg_arrays(b)
            srcs.append((to_device(bd[None], dev), to_device(bu[None], dev)))
    out = selected_solve_batched(md, mu, ml, srcs[0], srcs[1])
    kinds = [k for k, b in ((KIND_LESSER, b_lesser), (KIND_GREATER, b_greater)) if b is not None]
    return _solution_from(out, 0, n, bs, kinds)


# -- the sweeps separately (rgf.py:113-229 signatures) ----------------------


@dataclass
class RetardedPass:
    """rgf.py:37-49: forward intermediates x_fwd[i] and the pivot spread."""

    x_fwd: list = field(default_factory=list)
    u_spread: list = field(default_factory=list)


@dataclass
class LgPass:
    """rgf.py:52-58. ``b_fwd`` (effective sources) is not materialised by the
    device recursion; no caller on the hot path reads it (dist.py uses
    x_fwd_lg only)."""

    x_fwd_lg: list = field(default_factory=list)
    b_fwd: list = field(default_factory=list)


def _sweeps(mode: int, m_tilde, b_lg: dict, xr_diag: np.ndarray | None = None, xl: dict | None = None,
            fwd_given: bool = False, symmetrize: bool = False, device="cuda"):
    """One call of negf_rgf_sweeps_batched for a single energy. ``xr_diag`` /
    ``xl`` pre-fill the in/out diagonal arrays (modes 1 with fwd_given, and 2)."""
    lib = _lib.load()
    dev = torch.device(device)
    n, bs = m_tilde.n_blocks, m_tilde.block_size
    d, u, lo = tridiag_arrays(m_tilde)
    md, mu, ml = (to_device(x[None], dev) for x in (d, u, lo))
    z = dict(dtype=torch.complex128, device=dev)
    out = {"xr_diag": torch.zeros((1, n, bs, bs), **z) if xr_diag is None else to_device(xr_diag[None], dev),
           "xr_upper": torch.zeros((1, max(n - 1, 0), bs, bs), **z),
           "xr_lower": torch.zeros((1, max(n - 1, 0), bs, bs), **z)}
    srcs = {}
    for kind, b in b_lg.items():
        bd, bu = lg_arrays(b)
        srcs[kind] = (to_device(bd[None], dev), to_device(bu[None], dev))
        pre = None if xl is None else xl.get(kind)
        out[_KEYS[kind] + "_diag"] = torch.zeros((1, n, bs, bs), **z) if pre is None else to_device(pre[None], dev)
        out[_KEYS[kind] + "_upper"] = torch.zeros((1, max(n - 1, 0), bs, bs), **z)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    spread = torch.zeros((1, n), dtype=torch.float64, device=dev)
    nbytes = lib.negf_rgf_workspace_bytes(1, n, bs)
    ws = _lib.workspace(nbytes, dev)
    p = _lib.ptr
    bl = srcs.get(KIND_LESSER, (None, None))
    bg = srcs.get(KIND_GREATER, (None, None))
    rc = lib.negf_rgf_sweeps_batched(
        mode, 1 if fwd_given else 0, 1, n, bs, p(md), p(mu), p(ml), p(bl[0]), p(bl[1]), p(bg[0]), p(bg[1]),
        p(out["xr_diag"]), p(out["xr_upper"]), p(out["xr_lower"]), p(out.get("xl_diag")), p(out.get("xl_upper")),
        p(out.get("xg_diag")), p(out.get("xg_upper")), 1 if symmetrize else 0, p(status), p(spread), p(ws), nbytes,
        _lib.stream_ptr(dev))
    _lib.check(rc, "negf_rgf_sweeps_batched")
    raise_on_status(status)
    host = {k: v[0].cpu().numpy() for k, v in out.items()}
    return host, spread[0].cpu().numpy()


def forward_retarded(m_tilde, device="cuda") -> RetardedPass:
    """rgf.py:113-129."""
    host, spread = _sweeps(1, m_tilde, {}, device=device)
    return RetardedPass(list(host["xr_diag"]), [float(x) for x in spread])


def forward_lg(m_tilde, b_lg, fwd: RetardedPass, device="cuda") -> LgPass:
    """rgf.py:132-149, riding on the given retarded intermediates."""
    host, _ = _sweeps(1, m_tilde, {KIND_LESSER: b_lg}, xr_diag=np.stack(fwd.x_fwd), fwd_given=True, device=device)
    return LgPass(list(host["xl_diag"]), [])


def rgf_retarded(m_tilde, fwd: RetardedPass | None = None, x_last=None, device="cuda"):
    """rgf.py:152-183: backward sweep (forward pass computed unless given);
    ``x_last`` seeds the exact last diagonal block."""
    if fwd is None:
        fwd = forward_retarded(m_tilde, device=device)
    xr = np.stack(fwd.x_fwd).copy()
    if x_last is not None:
        xr[-1] = x_last
    host, _ = _sweeps(2, m_tilde, {}, xr_diag=xr, device=device)
    n, bs = m_tilde.n_blocks, m_tilde.block_size
    sol = SelectedSolution(n, bs, list(host["xr_diag"]), list(host["xr_upper"]), list(host["xr_lower"]))
    return sol, fwd


def rgf_lesser_greater(m_tilde, b_lg, fwd: RetardedPass, sol: SelectedSolution, kind: str,
                       lg: LgPass | None = None, x_last=None, device="cuda") -> LgPass:
    """rgf.py:186-229: stores X^lg blocks of ``kind`` into ``sol`` (not
    symmetrized) and returns the forward intermediates. The retarded chain is
    re-run on the device from ``fwd`` with sol's last retarded block as seed,
    which reproduces sol's X^R."""
    if lg is None:
        lg = forward_lg(m_tilde, b_lg, fwd, device=device)
    xr = np.stack(fwd.x_fwd).copy()
    xr[-1] = sol.x_r_diag[-1]
    xl = np.stack(lg.x_fwd_lg).copy()
    if x_last is not None:
        xl[-1] = x_last
    host, _ = _sweeps(2, m_tilde, {KIND_LESSER: b_lg}, xr_diag=xr, xl={KIND_LESSER: xl}, device=device)
    sol.x_lg_diag[kind] = list(host["xl_diag"])
    sol.x_lg_upper[kind] = list(host["xl_upper"])
    return lg
