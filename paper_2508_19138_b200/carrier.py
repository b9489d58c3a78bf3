"""Carrier (G) solve for a batch of energies, entirely on the GPU.

One ``CarrierSolver.solve`` call replaces, for every energy of the batch,
the body of scba_run's G loop (scba.py:965-1000):
  _assemble_g_system  scba.py:730-775  -> negf_g_assemble + negf_g_obc_apply
  selected_solve      rgf.py:232-243   -> negf_rgf_selected_solve_batched
  sol.symmetrize()    rgf.py:82-88     -> fused (symmetrize=1)
Buffers are allocated once per (n_e, n_b, bs) and reused across batches, so
a sweep over many energy batches does no allocation on the hot path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ConvergenceError, SingularBlockError
from .obc import fermi, raise_on_obc_status
from .rgf import raise_on_status

Z = torch.complex128


@dataclass(frozen=True)
class Contacts:
    """scba.py:101-121 ContactConfig."""

    mu_left: float
    mu_right: float
    kT: float = 0.02585

    @property
    def mu_mean(self) -> float:
        return 0.5 * (self.mu_left + self.mu_right)


def _dev_tensor(a, dev) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=Z).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=complex))).to(dev)


class CarrierSolver:
    """Batched G solve for a fixed Hamiltonian H (block tridiagonal)."""

    def __init__(self, h, eta: float, contacts: Contacts, surface_tol: float = 1e-8,
                 max_sweeps: int = 100, device="cuda", streams: int = 1,
                 greater: str = "recursion", retarded_method: str = "sancho", beyn=None) -> None:
        """``greater``: "recursion" runs the greater Keldysh pass like the
        reference; "identity" derives G^> = G^< + G^R - G^R^dag on the
        selected blocks (exact for the carrier system), saving
        ~40% of the RGF work."""
        if greater not in ("recursion", "identity"):
            raise ValueError(f"unknown greater mode {greater!r}")
        if retarded_method not in ("sancho", "beyn", "fixed_point"):
            raise ValueError(f"unknown retarded method {retarded_method!r}")
        self.retarded_method = retarded_method
        if beyn is None:
            from .scba import BeynOptions

            beyn = BeynOptions()
        self.beyn = beyn
        self.greater = greater
        self.dev = torch.device(device)
        self.lib = _lib.load()
        hd, hu, hl = h
        self.h = tuple(_dev_tensor(x, self.dev) for x in (hd, hu, hl))
        self.n_b, self.bs = self.h[0].shape[0], self.h[0].shape[-1]
        if self.n_b < 2:
            raise ValueError("need at least two blocks for two-terminal boundaries")
        self.eta = float(eta)
        self.contacts = contacts
        self.surface_tol = float(surface_tol)
        self.max_sweeps = int(max_sweeps)
        self._buf: dict | None = None
        self._n_e = 0
        self.dd = None  # (PartitionPlan, Comm): spatial domain decomposition of the RGF (scba_run plan=)
        self.streams = streams
        self._side_streams = [torch.cuda.Stream(self.dev) for _ in range(streams)] if streams > 1 else []

    def set_hamiltonian(self, h) -> None:
        """Copy new H blocks (host or device) into the resident device tensors."""
        for dst, src in zip(self.h, h):
            if isinstance(src, torch.Tensor):
                dst.copy_(src, non_blocking=True)
            else:
                dst.copy_(torch.from_numpy(np.ascontiguousarray(np.asarray(src, dtype=complex))))

    def check_status(self, b: dict) -> None:
        raise_on_obc_status(b["obc_status"].cpu().numpy(), b["obc_iters"].cpu().numpy(),
                            b["obc_resid"].cpu().numpy(), self.max_sweeps, self.surface_tol, "G contact")
        raise_on_status(b["rgf_status"])

    # -- buffers -----------------------------------------------------------
    def buffers(self, n_e: int) -> dict[str, torch.Tensor]:
        """Device buffers for a batch of n_e energies. A smaller batch than the
        allocated one (the last, partial batch of a run) gets leading-energy
        views of the same arrays instead of a reallocation."""
        if self._buf is not None and self._n_e == n_e:
            return self._buf
        if self._buf is not None and n_e < self._n_e:
            cut = {k: (2 * n_e if k.startswith("obc_") else n_e) for k in self._buf}
            return {k: v[:cut[k]] for k, v in self._buf.items()}
        self._buf = None
        torch.cuda.empty_cache()
        nb, bs, dev = self.n_b, self.bs, self.dev
        d = (n_e, nb, bs, bs)
        o = (n_e, nb - 1, bs, bs)
        c = (n_e, bs, bs)
        b = {k: torch.empty(d, dtype=Z, device=dev) for k in
             ("m_diag", "bl_diag", "bg_diag", "xr_diag", "xl_diag", "xg_diag")}
        b.update({k: torch.empty(o, dtype=Z, device=dev) for k in
                  ("m_upper", "m_lower", "bl_upper", "bg_upper", "xr_upper", "xr_lower", "xl_upper", "xg_upper")})
        b.update({k: torch.empty(c, dtype=Z, device=dev) for k in
                  ("sl_left", "sg_left", "sl_right", "sg_right")})
        b["energy"] = torch.empty(n_e, dtype=torch.float64, device=dev)
        b["f_bath"] = torch.empty(n_e, dtype=torch.float64, device=dev)
        b["f_left"] = torch.empty(n_e, dtype=torch.float64, device=dev)
        b["f_right"] = torch.empty(n_e, dtype=torch.float64, device=dev)
        b["obc_status"] = torch.zeros(2 * n_e, dtype=torch.int32, device=dev)
        b["obc_iters"] = torch.zeros(2 * n_e, dtype=torch.int32, device=dev)
        b["obc_resid"] = torch.zeros(2 * n_e, dtype=torch.float64, device=dev)
        b["rgf_status"] = torch.zeros(n_e, dtype=torch.int32, device=dev)
        self._buf, self._n_e = b, n_e
        return b

    @staticmethod
    def bytes_per_energy(n_b: int, bs: int) -> int:
        blk = 16 * bs * bs
        outputs = (6 * n_b + 8 * (n_b - 1) + 4) * blk
        rgf_ws = 14 * blk
        obc_ws = 2 * (6 + 10) * blk
        return outputs + rgf_ws + obc_ws

    # -- solve -------------------------------------------------------------
    def solve(self, energies, sigma: dict | None = None, n_e: int | None = None,
              check: bool = True, energies_dev: torch.Tensor | None = None,
              memo: tuple | None = None) -> dict[str, torch.Tensor]:
        """Solve the carrier system at ``energies`` (host array). ``sigma`` holds
        scattering self-energy blocks, energy-major: keys sr_diag/sr_upper/
        sr_lower, sl_diag/sl_upper, sg_diag/sg_upper (any subset). ``memo`` =
        (SurfaceCache, ld, e0, tol_memo) routes the contact surfaces through
        the OBC memoizer (scba.py:577-614), cache columns e0:e0+n_e of ld."""
        lib, p = self.lib, _lib.ptr
        energies = np.asarray(energies, dtype=np.float64)
        ne = len(energies)
        b = self.buffers(n_e or ne)
        if ne != b["energy"].shape[0]:
            raise ValueError("energy batch size does not match the allocated buffers")
        c = self.contacts
        host = np.stack([energies, fermi(energies, c.mu_mean, c.kT), fermi(energies, c.mu_left, c.kT),
                         fermi(energies, c.mu_right, c.kT)])
        dev_host = torch.from_numpy(host)
        for i, k in enumerate(("energy", "f_bath", "f_left", "f_right")):
            b[k].copy_(dev_host[i], non_blocking=False)
        s = sigma or {}
        st = _lib.stream_ptr(self.dev)
        hd, hu, hl = self.h
        # with G^> from the identity the greater source B^> is never read
        bg_d, bg_u = (None, None) if self.greater == "identity" else (p(b["bg_diag"]), p(b["bg_upper"]))
        rc = lib.negf_g_assemble(
            ne, self.n_b, self.bs, p(hd), p(hu), p(hl), p(b["energy"]), p(b["f_bath"]), self.eta,
            p(s.get("sr_diag")), p(s.get("sr_upper")), p(s.get("sr_lower")),
            p(s.get("sl_diag")), p(s.get("sl_upper")), p(s.get("sg_diag")), p(s.get("sg_upper")),
            p(b["m_diag"]), p(b["m_upper"]), p(b["m_lower"]), p(b["bl_diag"]), p(b["bl_upper"]),
            bg_d, bg_u, st)
        _lib.check(rc, "negf_g_assemble")
        nbytes = lib.negf_g_obc_workspace_bytes(ne, self.bs)
        ws = _lib.workspace(nbytes, self.dev)
        mc = mh = mu_ = None
        ld, n_fpi, tol_memo = 0, 20, 0.0
        x_surface = None
        if self.retarded_method != "sancho":
            from .obc import contact_cells, solve_surfaces

            x_surface = solve_surfaces(*contact_cells(b["m_diag"], b["m_upper"], b["m_lower"]),
                                       self.retarded_method, memo, ("G", "R"), self.surface_tol, self.beyn)
        elif memo is not None:
            cache, ld, e0, tol_memo = memo
            xs, hs, us = cache.slot(("G", "R"), 2, ld, self.bs, self.dev)
            mc, mh, mu_ = xs[0, e0], hs[0, e0:], us[0, e0:]
            n_fpi = cache.n_fpi("R")
        rc = lib.negf_g_obc_apply(
            ne, self.n_b, self.bs, p(b["m_diag"]), p(b["m_upper"]), p(b["m_lower"]), p(b["bl_diag"]),
            bg_d, p(b["f_left"]), p(b["f_right"]), self.surface_tol, self.max_sweeps,
            p(b["sl_left"]), p(b["sg_left"]), p(b["sl_right"]), p(b["sg_right"]),
            p(b["obc_status"]), p(b["obc_iters"]), p(b["obc_resid"]), p(mc), p(mh), p(mu_), ld, n_fpi,
            tol_memo, p(x_surface), p(ws), nbytes, st)
        _lib.check(rc, "negf_g_obc_apply")
        if memo is not None and x_surface is None:
            cache.record(us, e0, ne)
        if check:
            raise_on_obc_status(b["obc_status"].cpu().numpy(), b["obc_iters"].cpu().numpy(),
                                b["obc_resid"].cpu().numpy(), self.max_sweeps, self.surface_tol, "G contact")
        b["rgf_status"].zero_()
        if self.dd is not None:  # spatial mode of scba_run: all ranks solve this batch jointly
            from .dd import dd_solve_into

            dd_solve_into(b, *self.dd, kinds=("bl",) if self.greater == "identity" else ("bl", "bg"))
            if self.greater == "identity":
                rc = lib.negf_greater_from_identity(ne, self.n_b, self.bs, p(b["xl_diag"]), p(b["xl_upper"]),
                                                    p(b["xr_diag"]), p(b["xr_upper"]), p(b["xr_lower"]),
                                                    p(b["xg_diag"]), p(b["xg_upper"]), st)
                _lib.check(rc, "negf_greater_from_identity")
        elif self.greater == "identity":
            rgf_selected_solve_split(lib, b, ne, self.n_b, self.bs, self.dev, self.streams, self._side_streams,
                                     kinds=("bl",))
            rc = lib.negf_greater_from_identity(ne, self.n_b, self.bs, p(b["xl_diag"]), p(b["xl_upper"]),
                                                p(b["xr_diag"]), p(b["xr_upper"]), p(b["xr_lower"]),
                                                p(b["xg_diag"]), p(b["xg_upper"]), st)
            _lib.check(rc, "negf_greater_from_identity")
        else:
            rgf_selected_solve_split(lib, b, ne, self.n_b, self.bs, self.dev, self.streams, self._side_streams)
        if check:
            raise_on_status(b["rgf_status"])
        return b


def rgf_selected_solve_split(lib, b: dict, ne: int, n_b: int, bs: int, dev, streams: int, side_streams,
                             prefix: tuple = ("m", "bl", "bg", "xr", "xl", "xg"), symmetrize: int = 3,
                             kinds: tuple = ("bl", "bg")) -> None:
    """RGF over the batch in ``b``, split into ``streams`` energy slices on
    side streams so the latency-bound inversion panels of one slice overlap
    the DMMA GEMMs of another (energies are independent). ``symmetrize``:
    bit 0 symmetrizes the Keldysh diagonal blocks (rgf.py:82-88), bit 1
    declares the B^lg diagonal blocks anti-Hermitian -- true of the carrier
    sources Sigma^lg +- 2i eta f I and the contact terms."""
    m, bl, bg, xr, xl, xg = prefix
    p = _lib.ptr
    main = torch.cuda.current_stream(dev)
    parts = streams if streams > 1 and ne >= 2 * streams else 1
    bounds = [ne * k // parts for k in range(parts + 1)]
    ev = main.record_event() if parts > 1 else None
    for k in range(parts):
        a, z = bounds[k], bounds[k + 1]
        st_obj = side_streams[k] if parts > 1 else main
        if ev is not None:
            st_obj.wait_event(ev)
        with torch.cuda.stream(st_obj):
            nbytes = lib.negf_rgf_workspace_bytes(z - a, n_b, bs)
            ws = _lib.workspace(nbytes, dev)
            sl = lambda key: p(b[key][a:z])
            rc = lib.negf_rgf_selected_solve_batched(
                z - a, n_b, bs, sl(f"{m}_diag"), sl(f"{m}_upper"), sl(f"{m}_lower"),
                sl(f"{bl}_diag") if "bl" in kinds else None, sl(f"{bl}_upper") if "bl" in kinds else None,
                sl(f"{bg}_diag") if "bg" in kinds else None, sl(f"{bg}_upper") if "bg" in kinds else None,
                sl(f"{xr}_diag"), sl(f"{xr}_upper"), sl(f"{xr}_lower"),
                sl(f"{xl}_diag") if "bl" in kinds else None, sl(f"{xl}_upper") if "bl" in kinds else None,
                sl(f"{xg}_diag") if "bg" in kinds else None, sl(f"{xg}_upper") if "bg" in kinds else None, symmetrize, p(b["rgf_status"][a:z]), None, p(ws), nbytes,
                st_obj.cuda_stream)
            _lib.check(rc, "negf_rgf_selected_solve_batched")
    if parts > 1:
        for k in range(parts):
            main.wait_stream(side_streams[k])


RESULT_KEYS = {
    "g_r_diag": "xr_diag", "g_r_upper": "xr_upper", "g_r_lower": "xr_lower",
    "g_lesser_diag": "xl_diag", "g_lesser_upper": "xl_upper",
    "g_greater_diag": "xg_diag", "g_greater_upper": "xg_upper",
    "sigma_obc_lesser_left": "sl_left", "sigma_obc_greater_left": "sg_left",
    "sigma_obc_lesser_right": "sl_right", "sigma_obc_greater_right": "sg_right",
}


def ballistic_run(h, energies, eta: float, contacts: Contacts, surface_tol: float = 1e-8,
                  batch: int | None = None, device="cuda", greater: str = "recursion") -> dict[str, np.ndarray]:
    """scba_run(v_mat=None) equivalent (scba.py:951-1011): host arrays with
    the ScbaResult field names."""
    solver = CarrierSolver(h, eta, contacts, surface_tol, device=device, greater=greater)
    energies = np.asarray(energies, dtype=float)
    ne = len(energies)
    batch = batch or ne
    out = {k: [] for k in RESULT_KEYS}
    for s in range(0, ne, batch):
        chunk = energies[s:s + batch]
        b = solver.solve(chunk, n_e=len(chunk))
        for k, src in RESULT_KEYS.items():
            out[k].append(b[src].cpu().numpy())
    return {k: np.concatenate(v) for k, v in out.items()}


# -- observables -----------------------------------------------------------

C_OBSERVABLE = 1.0 / (2.0 * np.pi)


class ObservableAccumulator:
    """Per-energy traces reduced on the device (negf_observables), gathered
    across energy batches. Finalises to the reference's observables
    (scba.py:1313-1376): dos, electron_density, current_spectrum,
    terminal_current(left/right)."""

    def __init__(self, n_e_total: int, n_b: int, de: float, device) -> None:
        self.dev = torch.device(device)
        self.n_b, self.de = n_b, de
        self.tr_gr = torch.zeros((n_e_total, n_b), dtype=Z, device=self.dev)
        self.tr_gl = torch.zeros((n_e_total, n_b), dtype=Z, device=self.dev)
        self.cur = torch.zeros((n_e_total, max(n_b - 1, 1)), dtype=torch.float64, device=self.dev)
        self.term = torch.zeros((n_e_total, 2), dtype=Z, device=self.dev)

    def reset(self) -> None:
        for t in (self.tr_gr, self.tr_gl, self.cur, self.term):
            t.zero_()

    def add(self, solver: "CarrierSolver", b: dict, e0: int, ne: int) -> None:
        p = _lib.ptr
        rc = solver.lib.negf_observables(
            ne, solver.n_b, solver.bs, p(b["xr_diag"]), p(b["xl_diag"]), p(b["xg_diag"]),
            p(b["xl_upper"]), p(solver.h[1]), p(b["sl_left"]), p(b["sg_left"]), p(b["sl_right"]),
            p(b["sg_right"]), p(self.tr_gr[e0:]), p(self.tr_gl[e0:]), p(self.cur[e0:]),
            p(self.term[e0:]), _lib.stream_ptr(self.dev))
        _lib.check(rc, "negf_observables")

    def to_host(self) -> dict[str, np.ndarray]:
        tr_gr = self.tr_gr.cpu().numpy()
        tr_gl = self.tr_gl.cpu().numpy()
        term = self.term.cpu().numpy()
        return {
            "dos": -tr_gr.imag / np.pi,
            "density": (C_OBSERVABLE * self.de * (-1j * tr_gl).sum(axis=0)).real,
            "current_spectrum": self.cur.cpu().numpy()[:, : self.n_b - 1],
            "terminal_left": float(C_OBSERVABLE * self.de * term[:, 0].real.sum()),
            "terminal_right": float(C_OBSERVABLE * self.de * term[:, 1].real.sum()),
        }

    def d2h_bytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in (self.tr_gr, self.tr_gl, self.cur, self.term))


def ballistic_observables(h, energies, eta: float, contacts: Contacts, surface_tol: float = 1e-8,
                          batch: int | None = None, device="cuda", solver: CarrierSolver | None = None,
                          greater: str = "recursion"):
    """Public end-to-end ballistic API: host H blocks + energy grid in, host
    observables out. Every G block is computed on the device; only the
    reduced observables cross back to the host."""
    energies = np.asarray(energies, dtype=float)
    if solver is None:
        solver = CarrierSolver(h, eta, contacts, surface_tol, device=device, greater=greater)
    else:
        solver.set_hamiltonian(h)
    ne = len(energies)
    batch = batch or ne
    de = (energies[-1] - energies[0]) / (ne - 1) if ne > 1 else 0.0
    acc = ObservableAccumulator(ne, solver.n_b, de, solver.dev)
    for s in range(0, ne, batch):
        chunk = energies[s:s + batch]
        b = solver.solve(chunk, n_e=len(chunk), check=False)
        acc.add(solver, b, s, len(chunk))
        solver.check_status(b)
    return acc.to_host()
