"""Self-consistent Born (GW) iteration on the GPU (drop-in for the hot path
of negfgw.scba.scba_run, scba.py:865-1216).

One iteration, every stage a call into libnegf_b200.so:
  1. carrier solve per energy batch (carrier.CarrierSolver): Sigma entries ->
     blocks (negf_unpack_*), assembly, contact closure, RGF, symmetrize;
     G^<> blocks -> entry-major series (negf_pack_lg)           scba.py:965-1029
  2. polarization, fused FFT kernel (negf_conv_polarization)   scba.py:1035-1048
  3. screened interaction per batch: P entries -> blocks, W assembly
     (negf_w_assemble), W contact closure (negf_w_obc_apply), RGF, pack W^<>
                                                                scba.py:1059-1116
  4. self-energy, fused FFT kernel (negf_conv_sigma)           scba.py:1118-1132
  5. mixing + residual on per-block traces (negf_mix, negf_diag_traces)
                                                                scba.py:1155-1177
Entry-major state stays resident in HBM across iterations; only the
per-block traces (n_b x N_E) come back to the host for the residual.

Single-GPU driver; the multi-GPU energy-sharded version (E <-> nnz
transposes over NCCL all-to-all) is in ``dist.py``.
"""

from __future__ import annotations

import os

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .carrier import RESULT_KEYS, CarrierSolver, Contacts, rgf_selected_solve_split
from .conv import polarization, self_energy
from .dist import Comm, Transposer
from .errors import ConvergenceError, SpectralRadiusError
from .obc import raise_on_obc_status
from .results import EntryPattern, ScbaResult, SigmaState, TranspositionStats, count_transpose_bytes
from .rgf import raise_on_status

Z = torch.complex128


@dataclass(frozen=True)
class BeynOptions:
    """scba.py:124-140: contour parameters of the Beyn boundary solver."""

    n_quad: int = 16
    radius: float = 1.0
    svd_tol: float = 1e-8

    def __post_init__(self) -> None:
        if self.n_quad < 8:
            raise ValueError(f"need at least 8 quadrature nodes, got {self.n_quad}")
        if not 0 < self.radius <= 1:
            raise ValueError(f"radius must lie in (0, 1], got {self.radius}")
        if self.svd_tol <= 0:
            raise ValueError(f"svd_tol must be positive, got {self.svd_tol}")

    def contour(self) -> dict:
        return {"radius": self.radius, "center": 0.0, "n_quad": self.n_quad}


@dataclass(frozen=True)
class MemoizerOptions:
    """scba.py:143-154: budgets of the runtime direct-vs-refresh choice."""

    enabled: bool = True
    n_fpi_retarded: int = 20
    n_fpi_lg: int = 10

    def __post_init__(self) -> None:
        if self.n_fpi_retarded < 2 or self.n_fpi_lg < 2:
            raise ValueError("refresh budgets must be at least 2")


@dataclass(frozen=True)
class ScbaOptions:
    """scba.py:157-190, same defaults (incl. retarded_method="beyn",
    scba.py:165). The memoizer tolerance is tol / 10 as in the reference
    (scba.py:911)."""

    max_iter: int = 50
    tol: float = 1e-5
    mixing: float = 0.3
    surface_tol: float = 1e-8
    stein_tol: float = 1e-12
    stein_max_iter: int = 100
    batch: int | None = None  # energies per device batch (None: all)
    memoizer: MemoizerOptions = field(default_factory=MemoizerOptions)
    # carrier retarded surfaces (scba.py:577-614): "beyn" (the reference's
    # default, kept for drop-in parity although SURVEY §0.4 finds it wrong in
    # band at eta = 1e-3), "sancho" (what the parity tests and benches use)
    # or "fixed_point"
    retarded_method: str = "beyn"
    # W retarded surface: "sancho" (default; equal to Beyn on the reference's
    # weak-V inputs) or "beyn" (the reference's choice, scba.py:844)
    w_retarded_method: str = "sancho"
    beyn: BeynOptions = field(default_factory=lambda: BeynOptions())
    # scba.py:943: a warm-start initial_sigma is used only when reset_sigma is False
    reset_sigma: bool = True
    # scba.py:171, 913-915: compare every selected solve with a dense inverse
    # and every P / Sigma convolution with the direct sum (checks.py);
    # ScbaResult.oracle_deviations = {"solve_vs_dense", "fft_vs_direct"}
    oracle_mode: bool = False
    # Deviation (off by default): restrict the entry set of G^<>, P, W and
    # Sigma to |row - col| <= entry_cutoff orbitals -- the paper's r_cut
    # nonzero set (the reference applies r_cut to V only,
    # driver.py:276-277, and keeps the full band, scba.py:917). None = the
    # reference's full band. What makes a 2048-energy C3 iteration fit in HBM.
    entry_cutoff: int | None = None
    # Deviation (off by default): "identity" derives the carrier G^> from
    # G^> = G^< + G^R - G^R^dag instead of its own Keldysh recursion (the
    # reference runs all three, rgf.py:232-243; its identity_defects show the
    # identity holds to ~1e-15 for G, P and Sigma). 0.6x the carrier RGF work.
    greater: str = "recursion"
    # energy slices per device batch solved on side streams, so the inversion
    # panels of one slice (a few SMs each at small batches) overlap the GEMMs
    # of another (1: one stream)
    rgf_streams: int = 1

    def __post_init__(self) -> None:
        if self.max_iter < 1:
            raise ValueError(f"max_iter must be at least 1, got {self.max_iter}")
        if self.tol <= 0:
            raise ValueError(f"tol must be positive, got {self.tol}")
        if not 0 < self.mixing <= 1:
            raise ValueError(f"mixing must lie in (0, 1], got {self.mixing}")
        if self.surface_tol <= 0:
            raise ValueError(f"surface_tol must be positive, got {self.surface_tol}")
        if self.w_retarded_method not in ("sancho", "beyn", "fixed_point"):
            raise ValueError(f"unknown W retarded method {self.w_retarded_method!r}")
        if self.retarded_method not in ("sancho", "beyn", "fixed_point"):
            raise ValueError(f"unknown retarded method {self.retarded_method!r}")
        if self.entry_cutoff is not None and self.entry_cutoff < 0:
            raise ValueError(f"entry_cutoff must be >= 0 orbitals, got {self.entry_cutoff}")
        if self.greater not in ("recursion", "identity"):
            raise ValueError(f"unknown greater mode {self.greater!r}")
        if self.rgf_streams < 1:
            raise ValueError(f"rgf_streams must be at least 1, got {self.rgf_streams}")


class EntryLayout:
    """Device tables of the entry-major pattern and where its entries live in
    the block stacks.

    Default: the reference's compressed bandwidth-3 EntryPattern
    (convolve.py:135-187) on the stacks' own blocking -- structured kernels.
    Table mode (negf_*_table) for everything else:
      * ``cutoff``: keep only entries with |row - col| <= cutoff orbitals (the
        paper's r_cut nonzero set of G, P, W and Sigma, on
        the 1D orbital chain of the synthetic devices) -- a documented
        deviation; cutoff=None is the reference's full band;
      * ``target_bs``: the stacks use a coarser blocking (the W grid,
        bs_w = k bs, scba.py:893-937)."""

    def __init__(self, n_b: int, bs: int, device, cutoff: int | None = None, target_bs: int | None = None) -> None:
        self.n_b, self.bs = n_b, bs
        self.dev = torch.device(device)
        self.cutoff = cutoff
        self.target_bs = target_bs or bs
        if self.target_bs % bs or (n_b * bs) % self.target_bs:
            raise ValueError(f"target block size {self.target_bs} is not a multiple of {bs} dividing {n_b * bs}")
        self.n_bt = n_b * bs // self.target_bs
        self.table = cutoff is not None or self.target_bs != bs
        r, c = np.triu_indices(bs)
        self.tri_q = torch.from_numpy((r * bs + c).astype(np.int32)).to(self.dev)
        if not self.table:
            self.n_entries = int(_lib.load().negf_pattern_entries(n_b, bs))
            t = len(r)
            per_row = t + bs * bs
            diag = np.zeros(self.n_entries, dtype=np.uint8)
            rows = []
            for b in range(n_b):
                base = b * per_row
                on = np.flatnonzero(r == c)
                diag[base + on] = 1
                rows.append(base + on)
            self.diag = torch.from_numpy(diag).to(self.dev)
            self.diag_rows = torch.from_numpy(np.stack(rows).astype(np.int64)).to(self.dev)  # (n_b, bs)
            return
        from .results import EntryPattern

        pat = EntryPattern(n_b, bs, 3, True, cutoff)
        rows, cols = pat.rows, pat.cols
        self.n_entries = int(rows.size)
        bt = self.target_bs
        R, C = rows // bt, cols // bt
        code = (2 * R + (C - R)).astype(np.int32)
        q = ((rows % bt) * bt + cols % bt).astype(np.int32)
        self.code = torch.from_numpy(code).to(self.dev)
        self.q = torch.from_numpy(q).to(self.dev)
        on = rows == cols
        self.diag = torch.from_numpy(on.astype(np.uint8)).to(self.dev)
        idx = np.flatnonzero(on)  # every diagonal entry survives any cutoff (distance 0)
        self.diag_rows = torch.from_numpy(idx.reshape(n_b, bs).astype(np.int64)).to(self.dev)

    def pack(self, x_diag, x_upper, out, e0):
        if self.table:
            rc = _lib.load().negf_pack_lg_table(x_diag.shape[0], self.n_entries, self.n_bt, self.target_bs,
                                                self.code.data_ptr(), self.q.data_ptr(), x_diag.data_ptr(),
                                                x_upper.data_ptr(), out.data_ptr(), out.shape[-1], e0,
                                                _lib.stream_ptr(self.dev))
            _lib.check(rc, "negf_pack_lg_table")
            return
        rc = _lib.load().negf_pack_lg(x_diag.shape[0], self.n_b, self.bs, self.tri_q.data_ptr(), x_diag.data_ptr(),
                                      x_upper.data_ptr(), out.data_ptr(), out.shape[-1], e0,
                                      _lib.stream_ptr(self.dev))
        _lib.check(rc, "negf_pack_lg")

    def pack_p2p(self, x_diag, x_upper, peers, col0: int) -> None:
        """pack fused with the E -> nnz transpose into the owners' symmetric
        entry-major buffers (dist.PeerEntryMajor)."""
        _, ptrs, _ = peers[1]
        tr = peers[0].tr
        rc = _lib.load().negf_pack_lg_p2p(x_diag.shape[0], self.n_b, self.bs, self.tri_q.data_ptr(),
                                          x_diag.data_ptr(), x_upper.data_ptr(), tr.comm.size, ptrs.data_ptr(),
                                          peers[0].row_start.data_ptr(), tr.n_e, col0, _lib.stream_ptr(self.dev))
        _lib.check(rc, "negf_pack_lg_p2p")

    def unpack_p2p(self, peer, names, col0: int, n_e: int, x_diag, x_upper, x_lower=None) -> None:
        """unpack fused with the nnz -> E transpose: reads the entry owners'
        symmetric arrays (names: ("lg",) or (upper, lower) for retarded)."""
        ptrs = [peer.buffer(k)[1] for k in names]
        ret = len(names) == 2
        rc = _lib.load().negf_unpack_p2p(n_e, self.n_b, self.bs, self.tri_q.data_ptr(), int(ret), peer.tr.comm.size,
                                         ptrs[0].data_ptr(), ptrs[1].data_ptr() if ret else None,
                                         peer.row_start.data_ptr(), peer.tr.n_e, col0, x_diag.data_ptr(),
                                         x_upper.data_ptr(), x_lower.data_ptr() if ret else None,
                                         _lib.stream_ptr(self.dev))
        _lib.check(rc, "negf_unpack_p2p")

    def _unpack_table(self, up, lo, e0, n_e, x_diag, x_upper, x_lower):
        ret = lo is not None
        rc = _lib.load().negf_unpack_table(n_e, self.n_entries, self.n_bt, self.target_bs, self.code.data_ptr(),
                                           self.q.data_ptr(), int(ret), up.data_ptr(),
                                           lo.data_ptr() if ret else None, up.shape[-1], e0, x_diag.data_ptr(),
                                           x_upper.data_ptr(), x_lower.data_ptr() if ret else None, 1,
                                           _lib.stream_ptr(self.dev))
        _lib.check(rc, "negf_unpack_table")

    def unpack_lg(self, src, e0, n_e, x_diag, x_upper):
        if self.table:
            return self._unpack_table(src, None, e0, n_e, x_diag, x_upper, None)
        rc = _lib.load().negf_unpack_lg(n_e, self.n_b, self.bs, self.tri_q.data_ptr(), src.data_ptr(), src.shape[-1],
                                        e0, x_diag.data_ptr(), x_upper.data_ptr(), _lib.stream_ptr(self.dev))
        _lib.check(rc, "negf_unpack_lg")

    def unpack_retarded(self, up, lo, e0, n_e, x_diag, x_upper, x_lower):
        if self.table:
            return self._unpack_table(up, lo, e0, n_e, x_diag, x_upper, x_lower)
        rc = _lib.load().negf_unpack_retarded(n_e, self.n_b, self.bs, self.tri_q.data_ptr(), up.data_ptr(),
                                              lo.data_ptr(), up.shape[-1], e0, x_diag.data_ptr(),
                                              x_upper.data_ptr(), x_lower.data_ptr(), _lib.stream_ptr(self.dev))
        _lib.check(rc, "negf_unpack_retarded")

    def traces(self, x) -> torch.Tensor:
        tr = torch.empty((self.n_b, x.shape[-1]), dtype=Z, device=self.dev)
        rc = _lib.load().negf_diag_traces(x.data_ptr(), x.shape[-1], x.shape[-1], self.diag_rows.data_ptr(),
                                          self.n_b, self.bs, tr.data_ptr(), _lib.stream_ptr(self.dev))
        _lib.check(rc, "negf_diag_traces")
        return tr


class ScreenedSolver:
    """Batched W solve: assembly + contact closure + RGF (scba.py:1059-1103)."""

    def __init__(self, v, options: ScbaOptions, device) -> None:
        self.dev = torch.device(device)
        self.lib = _lib.load()
        self.v = tuple(torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=complex))).to(self.dev) for x in v)
        self.n_b, self.bs = self.v[0].shape[0], self.v[0].shape[-1]
        # a V with exactly zero imaginary part (the reference's coulomb_matrix)
        # lets the 3M GEMM skip its ai*bi product on every assembly term
        self.v_real = all(bool(torch.all(x.imag == 0)) for x in self.v)
        # a Hermitian V makes the diagonal W sources (V P V)_ii anti-Hermitian
        # (formed on half the tiles, negf_w_assemble bit 1)
        vd, vu, vl = self.v
        self.v_herm = bool(torch.equal(vd, vd.conj().transpose(-1, -2))) and bool(
            torch.equal(vl, vu.conj().transpose(-1, -2)))
        self.opt = options
        self._side_streams = ([torch.cuda.Stream(self.dev) for _ in range(options.rgf_streams)]
                              if options.rgf_streams > 1 else [])
        self.dd = None  # (PartitionPlan, Comm) in the spatial mode of scba_run
        self._buf, self._n_e = None, 0

    def buffers(self, n_e: int, pool=()) -> dict:
        """Block stacks of one energy batch. ``pool``: tensors of another stage
        that is never live at the same time as the W solve (scba_run passes
        the carrier's stacks), reused by shape so G and W do not both hold
        C3-size block memory."""
        if self._buf is not None and self._n_e == n_e:
            return self._buf
        self._buf = None
        nb, bs, dev = self.n_b, self.bs, self.dev
        d, o = (n_e, nb, bs, bs), (n_e, nb - 1, bs, bs)
        free = [x for x in pool if x.dtype == Z and x.is_contiguous()]

        def take(shape):
            for i, x in enumerate(free):
                if tuple(x.shape) == shape:
                    return free.pop(i)
            return torch.empty(shape, dtype=Z, device=dev)

        b = {k: take(d) for k in ("pr_diag", "pl_diag", "pg_diag", "m_diag", "bl_diag", "bg_diag")}
        b.update({k: take(o) for k in
                  ("pr_upper", "pr_lower", "pl_upper", "pg_upper", "m_upper", "m_lower", "bl_upper", "bg_upper")})
        # P blocks are dead once M_W and B_W are assembled: the RGF writes W
        # into them (7 fewer block stacks per batch)
        for part in ("diag", "upper", "lower"):
            b["wr_" + part] = b["pr_" + part]
        for part in ("diag", "upper"):
            b["wl_" + part], b["wg_" + part] = b["pl_" + part], b["pg_" + part]
        b["obc_status"] = torch.zeros(2 * n_e, dtype=torch.int32, device=dev)
        b["obc_iters"] = torch.zeros(2 * n_e, dtype=torch.int32, device=dev)
        b["stein_status"] = torch.zeros(4 * n_e, dtype=torch.int32, device=dev)
        b["stein_iters"] = torch.zeros(4 * n_e, dtype=torch.int32, device=dev)
        b["rgf_status"] = torch.zeros(n_e, dtype=torch.int32, device=dev)
        self._buf, self._n_e = b, n_e
        return b

    def solve(self, n_e: int, check: bool = True, timer=None, memo: tuple | None = None) -> dict:
        """Inputs in buffers pr_*/pl_*/pg_* (filled by the caller; the W outputs
        wr_*/wl_*/wg_* reuse their storage). ``memo`` =
        (SurfaceCache, ld, e0, tol_memo) as in CarrierSolver.solve."""
        import contextlib

        T = timer or (lambda name: contextlib.nullcontext())
        b = self.buffers(n_e)
        with T("W: assembly"):
            self._assemble(b, n_e)
        with T("W: OBC (Sancho+Stein)"):
            self._closure(b, n_e, memo, check)
        with T("W: RGF"):
            self._rgf(b, n_e)
        if check:
            raise_on_status(b["rgf_status"])
        return b

    def _assemble(self, b: dict, n_e: int) -> None:
        """scba.py:784-796: M_W = I - trunc3(V P^R), B^<> = trunc3((V P^<>) V)."""
        lib, p = self.lib, _lib.ptr
        vd, vu, vl = self.v
        nbytes = lib.negf_w_assemble_workspace_bytes(n_e, self.n_b, self.bs)
        ws = _lib.workspace(nbytes, self.dev)
        rc = lib.negf_w_assemble(n_e, self.n_b, self.bs, p(vd), p(vu), p(vl), p(b["pr_diag"]), p(b["pr_upper"]),
                                 p(b["pr_lower"]), p(b["pl_diag"]), p(b["pl_upper"]), p(b["pg_diag"]),
                                 p(b["pg_upper"]), p(b["m_diag"]), p(b["m_upper"]), p(b["m_lower"]),
                                 p(b["bl_diag"]), p(b["bl_upper"]), p(b["bg_diag"]), p(b["bg_upper"]),
                                 int(self.v_real) | (2 if self.v_herm else 0), p(ws), nbytes,
                                 _lib.stream_ptr(self.dev))
        _lib.check(rc, "negf_w_assemble")

    def _closure(self, b: dict, n_e: int, memo, check: bool) -> None:
        """scba.py:839-858: surfaces (Sancho, or Beyn like the reference), Stein
        corner sources, both through the memoizer when it is on."""
        lib, p, o = self.lib, _lib.ptr, self.opt
        nbytes = lib.negf_w_obc_workspace_bytes(n_e, self.bs)
        ws = _lib.workspace(nbytes, self.dev)
        memo_args = [None] * 6 + [0, 20, 10, 0.0]
        if memo is not None:
            cache, ld, e0, tol_memo = memo
            xr, hr, ur = cache.slot(("W", "R"), 2, ld, self.bs, self.dev)
            xl, hl, ul = cache.slot(("W", "lg"), 4, ld, self.bs, self.dev)
            memo_args = [p(xr[0, e0]), p(hr[0, e0:]), p(ur[0, e0:]), p(xl[0, e0]), p(hl[0, e0:]), p(ul[0, e0:]),
                         ld, cache.n_fpi("R"), cache.n_fpi("<"), tol_memo]
        x_surface = None
        if o.w_retarded_method != "sancho":  # the reference's Beyn (scba.py:844)
            from .obc import contact_cells, solve_surfaces

            x_surface = solve_surfaces(*contact_cells(b["m_diag"], b["m_upper"], b["m_lower"]),
                                       o.w_retarded_method, memo, ("W", "R"), o.surface_tol, o.beyn)
            memo_args[:3] = [None] * 3
        rc = lib.negf_w_obc_apply(n_e, self.n_b, self.bs, p(b["m_diag"]), p(b["m_upper"]), p(b["m_lower"]),
                                  p(b["bl_diag"]), p(b["bl_upper"]), p(b["bg_diag"]), p(b["bg_upper"]),
                                  o.surface_tol, 100, o.stein_tol, o.stein_max_iter,
                                  p(_lib.power_start_vector(self.bs, self.dev)), p(b["obc_status"]),
                                  p(b["obc_iters"]), p(b["stein_status"]), p(b["stein_iters"]), *memo_args,
                                  p(x_surface), p(ws), nbytes, _lib.stream_ptr(self.dev))
        _lib.check(rc, "negf_w_obc_apply")
        if memo is not None:
            if x_surface is None:
                cache.record(ur, e0, n_e)
            cache.record(ul, e0, n_e)
        if check:
            raise_on_obc_status(b["obc_status"].cpu().numpy(), b["obc_iters"].cpu().numpy(), None, 100,
                                o.surface_tol, "W contact")
            ss = b["stein_status"].cpu().numpy()
            if np.any(ss == 4):
                raise SpectralRadiusError("W boundary Stein: spectral radius estimate >= 1 (Kronecker fallback not ported)")
            if np.any(ss):
                raise ConvergenceError(f"geometric Stein did not reach tol {o.stein_tol} in {o.stein_max_iter} squarings")

    def _rgf(self, b: dict, n_e: int) -> None:
        """Selected solve of the W system, symmetrized (scba.py:1084-1087)."""
        lib, p = self.lib, _lib.ptr
        if self.dd is not None:  # spatial mode: all ranks solve the batch jointly (scba.py:1073-1083)
            from .dd import dd_solve_into

            dd_solve_into(b, *self.dd, prefix=("m", "bl", "bg", "wr", "wl", "wg"))
            return
        b["rgf_status"].zero_()
        # a Hermitian V makes the W sources anti-Hermitian (symmetrize bit 1)
        rgf_selected_solve_split(lib, b, n_e, self.n_b, self.bs, self.dev, self.opt.rgf_streams, self._side_streams,
                                 prefix=("m", "bl", "bg", "wr", "wl", "wg"), symmetrize=1 | (2 if self.v_herm else 0))


@dataclass
class ScbaState:
    """Entry-major scattering self-energy (scba.py:459-489 SigmaState)."""

    lesser: torch.Tensor
    greater: torch.Tensor
    ret_upper: torch.Tensor
    ret_lower: torch.Tensor

    @classmethod
    def zeros(cls, n_entries: int, n_e: int, device) -> "ScbaState":
        z = lambda: torch.zeros((n_entries, n_e), dtype=Z, device=device)
        return cls(z(), z(), z(), z())

    def as_tuple(self):
        return self.lesser, self.greater, self.ret_upper, self.ret_lower


@dataclass(frozen=True)
class EnergyGrid:
    """device.py:39-73: uniform energy axis (linspace) with broadening eta."""

    e_min: float
    e_max: float
    n_e: int
    eta: float = 1e-3

    def __post_init__(self) -> None:
        if self.n_e < 2:
            raise ValueError(f"n_e must be at least 2, got {self.n_e}")
        if not self.e_max > self.e_min:
            raise ValueError(f"need e_max > e_min, got [{self.e_min}, {self.e_max}]")
        if not self.eta > 0.0:
            raise ValueError(f"eta must be positive, got {self.eta}")

    @property
    def de(self) -> float:
        return (self.e_max - self.e_min) / (self.n_e - 1)

    @property
    def energies(self) -> np.ndarray:
        return np.linspace(self.e_min, self.e_max, self.n_e)


def _stacks(m):
    """Block stacks from either (diag, upper, lower) arrays or any object with
    the BlockMatrix API (ours or the reference's)."""
    if hasattr(m, "get_block"):
        from .blocks import tridiag_arrays

        if m.block_bandwidth > 3:
            raise ValueError("the hot path takes block-tridiagonal H and V")
        return tridiag_arrays(m)
    return m


def g_identity_defect(b: dict, n_e: int, n_b: int, bs: int, out: torch.Tensor) -> None:
    """scba.py:1223-1238 on the device: accumulates max |X^> - X^< - (X^R - X^R^dag)|
    and max |X^R - X^R^dag| over the stored blocks into out[0:2] (max-combined)."""
    up = lambda k: b[k].data_ptr() if n_b > 1 else None
    rc = _lib.load().negf_g_identity_defect(n_e, n_b, bs, b["xr_diag"].data_ptr(), up("xr_upper"), up("xr_lower"),
                                            b["xl_diag"].data_ptr(), up("xl_upper"), b["xg_diag"].data_ptr(),
                                            up("xg_upper"), out.data_ptr(), _lib.stream_ptr(out.device))
    _lib.check(rc, "negf_g_identity_defect")


def entry_identity_defect(lesser, greater, ret_upper, ret_lower, out: torch.Tensor) -> None:
    """scba.py:1241-1248 on the device for entry-major series (P or Sigma rows)."""
    for x in (lesser, greater, ret_upper, ret_lower):
        if x.dtype != Z or not x.is_contiguous() or x.shape != lesser.shape:
            raise ValueError("identity defect needs contiguous complex128 series of one shape")
    rc = _lib.load().negf_entry_identity_defect(lesser.numel(), lesser.data_ptr(), greater.data_ptr(),
                                                ret_upper.data_ptr(), ret_lower.data_ptr(), out.data_ptr(),
                                                _lib.stream_ptr(out.device))
    _lib.check(rc, "negf_entry_identity_defect")


def scba_run_reference_api(h_mat, v_mat, grid, contacts, options: ScbaOptions | None = None,
                           comm: Comm | None = None, plan=None, initial_sigma: ScbaState | None = None,
                           device="cuda") -> dict:
    """scba.py:865 signature: BlockMatrix H / V (or None), an EnergyGrid-like
    grid (energies, eta), a ContactConfig-like object (mu_left, mu_right,
    kT), ``comm`` for energy sharding and ``plan`` (dd.PartitionPlan) for
    the spatial mode."""
    c = Contacts(contacts.mu_left, contacts.mu_right, contacts.kT)
    res = scba_run(_stacks(h_mat), None if v_mat is None else _stacks(v_mat), grid.energies, grid.eta, c,
                   options, device=device, comm=comm, initial_sigma=initial_sigma, plan=plan)
    res.grid, res.contacts = grid, contacts  # the caller's objects, like the reference's result
    return res


def scba_run(h, v, energies, eta: float, contacts: Contacts, options: ScbaOptions | None = None,
             device="cuda", keep_g: bool = True, initial_sigma: ScbaState | None = None,
             comm: Comm | None = None, profile: bool = False, sigma_to_host: bool = True,
             plan=None) -> "ScbaResult":
    """SCBA on one GPU or energy-sharded over ``comm`` (one rank per GPU).

    ``h``/``v`` are (diag, upper, lower) block stacks; ``v=None`` runs the
    ballistic single pass. Each rank solves its energy chunk
    (energy_chunks, scba.py:243-249) and owns an entry chunk for the
    convolutions; the E<->nnz switches are NCCL all-to-alls (dist.py).
    Returns host arrays named like ScbaResult fields for this rank's
    energies (G of the last iteration's carrier solve when keep_g), the
    mixed Sigma columns of this rank's energies ('sigma_lesser', ...),
    'residuals' (global) and 'energy_slice'.

    With ``plan.p_s > 1`` (a dd.PartitionPlan, p_s == comm.size) every energy
    is solved jointly by all ranks over the spatial partitions (dd.py, the
    reference's spatial mode, scba.py:878-880, 971-979, 1073-1083): Sigma is
    replicated, P and Sigma are all-gathered after the convolutions, and each
    rank still owns its energy chunk of the entry-major layout."""
    options = options or ScbaOptions()
    comm = comm or Comm()
    dev = torch.device(device)
    energies = np.asarray(energies, dtype=float)
    ne = len(energies)
    de = (energies[-1] - energies[0]) / (ne - 1)
    carrier = CarrierSolver(h, eta, contacts, options.surface_tol, device=dev, greater=options.greater,
                            retarded_method=options.retarded_method, beyn=options.beyn,
                            streams=options.rgf_streams)
    n_b, bs = carrier.n_b, carrier.bs
    lay = EntryLayout(n_b, bs, dev, cutoff=options.entry_cutoff)
    tr = Transposer(comm, lay.n_entries, ne)
    spatial = plan is not None and plan.p_s > 1
    if spatial:
        from .dd import PartitionError, make_partition_plan

        if options.oracle_mode:
            raise ValueError("oracle_mode supports only sequential solves")
        if plan.n_blocks != n_b:
            raise PartitionError(f"plan covers {plan.n_blocks} blocks, matrix has {n_b}")
        if plan.p_s != comm.size:
            raise PartitionError(f"plan has {plan.p_s} partitions but communicator has {comm.size} ranks")
        carrier.dd = (plan, comm)
    # multi-GPU GW: every E <-> nnz switch runs through symmetric (NVLink-
    # mapped) memory inside the layout kernels -- G^<> and W^<> are written
    # into their entry owners' arrays by the pack, P is read from its owners
    # by the W unpack and Sigma by the mixing; stream-ordered barriers order
    # writers and readers. NEGF_PEER_TRANSPOSE=0 selects NCCL all-to-all.
    peer = None
    if (comm.size > 1 and v is not None and not spatial and not lay.table
            and os.environ.get("NEGF_PEER_TRANSPOSE", "1") != "0"):
        from .dist import PeerEntryMajor

        peer = PeerEntryMajor.try_create(tr, dev)  # None (-> NCCL all-to-all) off NCCL / without P2P
    own = tr.own_e
    n_own = tr.n_own_e
    # energies this rank solves: its chunk, or all of them in the spatial mode
    s0, n_sol = (0, ne) if spatial else (own.start, n_own)
    my_e = energies[s0:s0 + n_sol]
    diag_rows = lay.diag[tr.own_r].contiguous()
    batch = options.batch or max(n_sol, 1)
    sig = ScbaState.zeros(lay.n_entries, n_sol, dev)
    if initial_sigma is not None and not options.reset_sigma:
        # scba.py:942-949: any object with lesser / greater / ret_upper /
        # ret_lower (the reference's SigmaState, ours, or a device ScbaState),
        # either the full (n_entries, N_E) array like the reference or this
        # rank's own (n_entries, n_own) columns
        parts = [getattr(initial_sigma, k) for k in ("lesser", "greater", "ret_upper", "ret_lower")]
        shape = tuple(parts[0].shape)
        if shape == (lay.n_entries, ne) and n_sol != ne:
            parts = [x[:, s0:s0 + n_sol] for x in parts]
        elif shape not in ((lay.n_entries, n_sol), (lay.n_entries, ne)):
            raise ValueError(f"warm-start state has shape {shape}, expected {(lay.n_entries, ne)}")
        sig = ScbaState(*(torch.as_tensor(x, dtype=Z, device=dev).clone().contiguous() for x in parts))
    if v is None:
        max_iter = 1
    else:
        max_iter = options.max_iter
        screened = ScreenedSolver(v, options, dev)
        # scba.py:893-903 preconditions, same messages
        if screened.n_b * screened.bs != n_b * bs:
            raise ValueError(f"screening layout {screened.n_b}x{screened.bs} does not match carrier layout "
                             f"{n_b}x{bs}")
        if screened.bs % bs != 0:
            raise ValueError("screening block size must be a multiple of the carrier block size, got "
                             f"{screened.bs} and {bs}")
        if spatial and screened.bs != bs:
            raise ValueError("the spatial mode takes equal G and W blockings")
    # P goes into the W stacks and W^<> comes back at G-pattern coordinates
    # (scba.py:925-937 _scatter_groups(pat_g, bs_w) / w_to_g): with a coarser
    # W grid through the table-driven layout on the W blocking
    lay_w = lay
    if v is not None and screened.bs != bs:
        lay_w = EntryLayout(n_b, bs, dev, cutoff=options.entry_cutoff, target_bs=screened.bs)
        peer = None
        if spatial:  # the W chain gets its own even split (scba.py:930)
            screened.dd = (make_partition_plan(n_b, plan.p_s), comm)
    cols = lambda: torch.empty((lay.n_entries, n_own), dtype=Z, device=dev)
    result: dict = {}
    residuals = []
    identity_defects: list[dict[str, float]] = []
    converged = v is None
    n_iter = 0
    blocks = None
    timings: dict[str, float] = {}
    import time as _time

    class _T:  # stage timer (scba.py:85-94 KernelTimers categories); syncs only when profiling
        def __init__(self, name):
            self.name = name

        def __enter__(self):
            if profile:
                torch.cuda.synchronize(dev)
                self.t0 = _time.perf_counter()

        def __exit__(self, *a):
            if profile:
                torch.cuda.synchronize(dev)
                timings[self.name] = timings.get(self.name, 0.0) + _time.perf_counter() - self.t0

    iter_times = []
    cache = None
    if options.memoizer.enabled:
        from .obc import SurfaceCache

        cache = SurfaceCache(options.memoizer.n_fpi_retarded, options.memoizer.n_fpi_lg)
    tol_memo = options.tol / 10.0
    stats_by_it = []
    odev = {"solve_vs_dense": 0.0, "fft_vs_direct": 0.0} if options.oracle_mode else None

    def solve_check(bb, w: bool) -> None:
        from .checks import dense_solution_deviation

        x = "w" if w else "x"
        dv, sc = dense_solution_deviation(
            (bb["m_diag"], bb["m_upper"], bb["m_lower"]),
            {"<": (bb["bl_diag"], bb["bl_upper"]), ">": (bb["bg_diag"], bb["bg_upper"])},
            (bb[x + "r_diag"], bb[x + "r_upper"], bb[x + "r_lower"]),
            {"<": (bb[x + "l_diag"], bb[x + "l_upper"]), ">": (bb[x + "g_diag"], bb[x + "g_upper"])})
        odev["solve_vs_dense"] = max(odev["solve_vs_dense"], dv / (sc + 1e-300))

    memo = (lambda e0: (cache, max(n_sol, 1), e0, tol_memo)) if cache is not None else (lambda e0: None)

    def own_part(e0: int, nb_: int):
        """(offset in the batch, count, column in the own chunk) of the batch's own energies."""
        if not spatial:
            return 0, nb_, e0
        lo, hi = max(e0, own.start), min(e0 + nb_, own.stop)
        return lo - e0, max(hi - lo, 0), lo - own.start

    def pack_own(xd, xu, out, e0: int, nb_: int, layout=None) -> None:
        a, n, c = own_part(e0, nb_)
        if n:
            (layout or lay).pack(xd[a:a + n], xu[a:a + n], out, c)
    timings_by_it = []
    # reference observables of each iteration's G solve (scba.py:1313-1376),
    # reduced on the device per batch; the last iteration's are reported
    from .carrier import ObservableAccumulator

    obs_acc = ObservableAccumulator(max(n_sol, 1), n_b, de, dev)
    stats = TranspositionStats()
    pattern = EntryPattern(n_b, bs, 3, True, options.entry_cutoff)
    full_count = pattern.full_entry_count()
    w_count = (lay.n_entries, full_count)
    if v is not None and screened.bs != bs:
        pat_w = EntryPattern(screened.n_b, screened.bs, 3, True, options.entry_cutoff)
        w_count = (pat_w.n_entries, pat_w.full_entry_count())
    for it in range(max_iter):
        n_iter = it + 1
        torch.cuda.synchronize(dev)
        t_iter = _time.perf_counter()
        t_snap = dict(timings)
        obs_acc.reset()
        # identity-defect accumulators (G, P, Sigma) x (defect, scale), scba.py:1002-1006
        defects = torch.zeros(6, dtype=torch.float64, device=dev)
        g_host = {k: [] for k in RESULT_KEYS} if keep_g else None
        if peer is not None:  # E -> nnz fused into the pack (peer memory)
            p_gl, p_gg = peer.buffer("gl"), peer.buffer("gg")
            peer.barrier()  # every peer is done with last iteration's arrays
            gl_c = gg_c = None
        else:
            gl_c, gg_c = cols(), cols()
        # 1. carrier solve per energy batch of this rank
        for e0 in range(0, n_sol, batch):
            e1 = min(n_sol, e0 + batch)
            nb_ = e1 - e0
            if blocks is None or blocks["sr_diag"].shape[0] != nb_:
                d, o = (nb_, n_b, bs, bs), (nb_, n_b - 1, bs, bs)
                blocks = {k: torch.empty(d, dtype=Z, device=dev) for k in ("sr_diag", "sl_diag", "sg_diag")}
                blocks.update({k: torch.empty(o, dtype=Z, device=dev) for k in
                               ("sr_upper", "sr_lower", "sl_upper", "sg_upper")})
            with _T("layout"):
                lay.unpack_retarded(sig.ret_upper, sig.ret_lower, e0, nb_, blocks["sr_diag"], blocks["sr_upper"],
                                    blocks["sr_lower"])
                lay.unpack_lg(sig.lesser, e0, nb_, blocks["sl_diag"], blocks["sl_upper"])
                lay.unpack_lg(sig.greater, e0, nb_, blocks["sg_diag"], blocks["sg_upper"])
            with _T("G: OBC+RGF"):
                b = carrier.solve(my_e[e0:e1], sigma=blocks, n_e=nb_, memo=memo(e0))
            g_identity_defect(b, nb_, n_b, bs, defects[0:2])
            obs_acc.add(carrier, b, e0, nb_)
            if odev is not None:
                solve_check(b, False)
            with _T("layout"):
                if peer is not None:
                    lay.pack_p2p(b["xl_diag"], b["xl_upper"], (peer, p_gl), own.start + e0)
                    lay.pack_p2p(b["xg_diag"], b["xg_upper"], (peer, p_gg), own.start + e0)
                    peer.count(2 * nb_)
                else:
                    pack_own(b["xl_diag"], b["xl_upper"], gl_c, e0, nb_)
                    pack_own(b["xg_diag"], b["xg_upper"], gg_c, e0, nb_)
            if keep_g:
                a_, n_, _c = own_part(e0, nb_)
                for k, src in RESULT_KEYS.items():
                    g_host[k].append(b[src][a_:a_ + n_].cpu().numpy())
        if keep_g and n_own:
            result = {k: np.concatenate(vv) for k, vv in g_host.items()}
        if v is None:
            d = comm.allreduce_max(defects[0:2].tolist(), dev)
            identity_defects.append({"G": d[0] / (d[1] + 1e-300)})
            residuals.append(0.0)
            if cache is not None:
                stats_by_it.append(cache.stats)
            break
        # logical transposition volume of this iteration, counted like the
        # reference's replicated exchanges (scba.py:1028-1141, _count_bytes):
        # G^<>, P^<>, W^<>, Sigma^<> lg-compressed; P^R, Sigma^R plain
        for _ in range(6):
            count_transpose_bytes(stats, True, lay.n_entries, ne, full_count)
        for _ in range(2):  # W^<> travel on the W pattern in the reference (pat_w)
            count_transpose_bytes(stats, True, w_count[0], ne, w_count[1])
        for _ in range(4):
            count_transpose_bytes(stats, False, lay.n_entries, ne, 0)
        # 2. G^<> to entry-major (all-to-all), polarization on own entry rows
        with _T("transpose"):
            if peer is not None:
                peer.barrier()
                gl, gg = p_gl[0], p_gg[0]
            else:
                gl, gg = tr.to_entry_major(gl_c), tr.to_entry_major(gg_c)
        del gl_c, gg_c
        with _T("convolution"):
            p_out = tuple(peer.buffer(k)[0] for k in ("pl", "pg", "pru", "prl")) if peer is not None else None
            p_rows = polarization(gl, gg, diag_rows, de, out=p_out)
        entry_identity_defect(*p_rows, defects[2:4])
        if odev is not None:
            from .checks import polarization_deviation

            dv, sc = polarization_deviation(gl, gg, p_rows[0], p_rows[1], diag_rows, de)
            odev["fft_vs_direct"] = max(odev["fft_vs_direct"], dv / (sc + 1e-300))
        with _T("transpose"):
            if peer is not None:  # the W unpack reads the owners' P rows directly
                peer.barrier()
                peer.count(4 * n_own)
                pl = pg = pru = prl = None
            else:
                pl, pg, pru, prl = ((tr.rows_to_full(x) if spatial else tr.to_energy_major(x)) for x in p_rows)
        del p_rows
        # 3. screened interaction per batch of own energies
        if peer is not None:
            p_wl, p_wg = peer.buffer("wl"), peer.buffer("wg")
            wl_c = wg_c = None
        else:
            wl_c, wg_c = cols(), cols()
        for e0 in range(0, n_sol, batch):
            e1 = min(n_sol, e0 + batch)
            nb_ = e1 - e0
            # the carrier's stacks of this batch size are dead during the W stage
            pool = list(blocks.values()) if blocks is not None and blocks["sr_diag"].shape[0] == nb_ else []
            cb = carrier._buf if carrier._buf is not None and carrier._n_e >= nb_ else {}
            pool += [x[:nb_] for x in cb.values() if x.dim() == 4]  # leading views for a partial last batch
            wb = screened.buffers(nb_, pool)
            with _T("layout"):
                if peer is not None:
                    c0 = own.start + e0
                    lay.unpack_p2p(peer, ("pru", "prl"), c0, nb_, wb["pr_diag"], wb["pr_upper"], wb["pr_lower"])
                    lay.unpack_p2p(peer, ("pl",), c0, nb_, wb["pl_diag"], wb["pl_upper"])
                    lay.unpack_p2p(peer, ("pg",), c0, nb_, wb["pg_diag"], wb["pg_upper"])
                else:
                    lay_w.unpack_retarded(pru, prl, e0, nb_, wb["pr_diag"], wb["pr_upper"], wb["pr_lower"])
                    lay_w.unpack_lg(pl, e0, nb_, wb["pl_diag"], wb["pl_upper"])
                    lay_w.unpack_lg(pg, e0, nb_, wb["pg_diag"], wb["pg_upper"])
            wb = screened.solve(nb_, timer=_T, memo=memo(e0))
            if odev is not None:
                solve_check(wb, True)
            with _T("layout"):
                if peer is not None:
                    lay.pack_p2p(wb["wl_diag"], wb["wl_upper"], (peer, p_wl), own.start + e0)
                    lay.pack_p2p(wb["wg_diag"], wb["wg_upper"], (peer, p_wg), own.start + e0)
                    peer.count(2 * nb_)
                else:
                    pack_own(wb["wl_diag"], wb["wl_upper"], wl_c, e0, nb_, lay_w)
                    pack_own(wb["wg_diag"], wb["wg_upper"], wg_c, e0, nb_, lay_w)
        del pl, pg, pru, prl
        with _T("transpose"):
            if peer is not None:
                peer.barrier()
                wl, wg = p_wl[0], p_wg[0]
            else:
                wl, wg = tr.to_entry_major(wl_c), tr.to_entry_major(wg_c)
        del wl_c, wg_c
        # 4. self-energy on own entry rows, back to energy-major columns
        with _T("convolution"):
            s_out = tuple(peer.buffer(k)[0] for k in ("sl", "sg", "sru", "srl")) if peer is not None else None
            s_rows = self_energy(gl, gg, wl, wg, None, diag_rows, de, out=s_out)
        entry_identity_defect(*s_rows, defects[4:6])
        if odev is not None:
            from .checks import self_energy_deviation

            dv, sc = self_energy_deviation(gl, gg, wl, wg, s_rows[0], s_rows[1], diag_rows, de)
            odev["fft_vs_direct"] = max(odev["fft_vs_direct"], dv / (sc + 1e-300))
        with _T("transpose"):
            if peer is not None:  # the mixing reads the owners' Sigma rows directly
                peer.barrier()
                peer.count(4 * n_own)
                raw = None
            else:
                raw = tuple((tr.rows_to_full(x) if spatial else tr.to_energy_major(x)) for x in s_rows)
        del s_rows
        del wl, wg, gl, gg
        # 5. mixing + residual (scba.py:1155-1177), max over ranks
        tr_old = [lay.traces(sig.lesser), lay.traces(sig.greater)]
        if peer is not None:
            src = torch.cat([peer.buffer(k)[1] for k in ("sl", "sg", "sru", "srl")])
            rc = _lib.load().negf_mix_p2p(lay.n_entries, n_own, options.mixing, *(x.data_ptr() for x in sig.as_tuple()),
                                          comm.size, src.data_ptr(), peer.row_start.data_ptr(), ne, own.start,
                                          _lib.stream_ptr(dev))
            _lib.check(rc, "negf_mix_p2p")
        else:
            rc = _lib.load().negf_mix(sig.lesser.numel(), options.mixing, *(x.data_ptr() for x in sig.as_tuple()),
                                      *(x.data_ptr() for x in raw), _lib.stream_ptr(dev))
            _lib.check(rc, "negf_mix")
        tr_new = [lay.traces(sig.lesser), lay.traces(sig.greater)]
        to = [t.cpu().numpy() for t in tr_old]
        tn = [t.cpu().numpy() for t in tr_new]
        mx = lambda arrs: max((float(np.max(np.abs(a))) if a.size else 0.0) for a in arrs)
        delta = mx([a - b_ for a, b_ in zip(tn, to)])
        scale = max(mx(to), mx(tn))
        delta, scale = comm.allreduce_max([delta, scale], dev)
        residuals.append(delta / (scale + 1e-300))
        d = comm.allreduce_max(defects.tolist(), dev)
        identity_defects.append({k: d[2 * j] / (d[2 * j + 1] + 1e-300) for j, k in enumerate(("G", "P", "Sigma"))})
        del raw
        if cache is not None:
            stats_by_it.append(cache.stats)
        iter_times.append(_time.perf_counter() - t_iter)
        timings_by_it.append({k: x - t_snap.get(k, 0.0) for k, x in timings.items()})
        if residuals[-1] < options.tol:
            converged = True
            break
        if len(residuals) >= 11 and residuals[-1] > 5.0 * residuals[-11]:
            raise ConvergenceError(f"residual grew from {residuals[-11]:.3e} to {residuals[-1]:.3e} over 10 iterations")
    sigma_host = None
    if v is not None and sigma_to_host:
        sigma_host = SigmaState(*((t[:, own] if spatial else t).cpu().numpy() for t in sig.as_tuple()))
    observables = _gather_observables(obs_acc, comm, spatial, n_sol, dev)
    oracle_devs = {}
    if odev is not None:
        o = comm.allreduce_max([odev["solve_vs_dense"], odev["fft_vs_direct"]], dev)
        oracle_devs = {"solve_vs_dense": o[0], "fft_vs_direct": o[1]}
    try:
        grid = EnergyGrid(float(energies[0]), float(energies[-1]), ne, eta)
    except ValueError:
        grid = None
    return ScbaResult(
        grid=grid, contacts=contacts, options=options, n_blocks=n_b, block_size=bs, converged=converged,
        n_iter=n_iter, residuals=np.asarray(residuals), identity_defects=identity_defects,
        **{k: result.get(k) for k in RESULT_KEYS},
        sigma=sigma_host, sigma_pattern=pattern, timings=timings, wall_total=float(sum(iter_times)),
        transposition=stats,
        cache_stats=cache.stats if cache is not None else {"direct_calls": 0, "memoized_calls": 0},
        cache_stats_by_iteration=stats_by_it, dist_stats=None, comm_bytes=int(tr.bytes_moved),
        oracle_deviations=oracle_devs, state=sig, energy_slice=own, iteration_s=iter_times,
        timings_by_iteration=timings_by_it, observables=observables)


def _gather_observables(acc, comm: Comm, spatial: bool, n_sol: int, dev) -> dict:
    """This rank's device-reduced observables -> the whole grid's: per-energy
    arrays concatenated over the energy chunks, energy integrals summed
    (all_gather_object of the small host arrays)."""
    if n_sol == 0:
        loc = None
    else:
        loc = acc.to_host()
        loc["dos"] = loc["dos"][:n_sol]
        loc["current_spectrum"] = loc["current_spectrum"][:n_sol]
    if comm.size == 1 or spatial:
        return loc or {}
    import torch.distributed as dist

    parts = [None] * comm.size
    dist.all_gather_object(parts, loc, group=comm.group)
    parts = [p_ for p_ in parts if p_ is not None]
    return {"dos": np.concatenate([p_["dos"] for p_ in parts]),
            "density": np.sum([p_["density"] for p_ in parts], axis=0),
            "current_spectrum": np.concatenate([p_["current_spectrum"] for p_ in parts]),
            "terminal_left": float(sum(p_["terminal_left"] for p_ in parts)),
            "terminal_right": float(sum(p_["terminal_right"] for p_ in parts))}

