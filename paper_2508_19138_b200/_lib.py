"""ctypes binding of ``libnegf_b200.so`` (the C ABI in include/negf_b200.h).

There is deliberately no CPU fallback: if the shared library is missing or
no CUDA device is visible, every hot-path call raises. The library is built
in-tree by ``paper_2508_19138_b200/build.py`` (``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import torch

import os

# NEGF_B200_LIB: load another build of the library (kernel experiments)
_LIB_PATH = Path(os.environ.get("NEGF_B200_LIB", Path(__file__).resolve().parent / "libnegf_b200.so"))
_lib: C.CDLL | None = None

_vp = C.c_void_p
_i = C.c_int
_ll = C.c_longlong
_d = C.c_double
_sz = C.c_size_t

# name -> (restype, argtypes)
_SIGNATURES: dict[str, tuple] = {
    "negf_abi_version": (_i, []),
    "negf_set_gemm_algo": (_i, [_i]),
    "negf_set_rgf_overlap": (_i, [_i]),
    "negf_rgf_workspace_bytes": (_sz, [_i, _i, _i]),
    "negf_rgf_selected_solve_batched": (
        _i,
        [_i, _i, _i] + [_vp] * 14 + [_i, _vp, _vp, _vp, _sz, _vp],
    ),
    "negf_rgf_sweeps_batched": (
        _i,
        [_i, _i, _i, _i, _i] + [_vp] * 14 + [_i, _vp, _vp, _vp, _sz, _vp],
    ),
    "negf_greater_from_identity": (_i, [_i, _i, _i] + [_vp] * 8),
    "negf_zgemm_batched": (
        _i,
        [_i, _i, _i, _i, _d, _d, _vp, _ll, _i, _i, _vp, _ll, _i, _i, _d, _d, _vp, _ll, _i, _vp, _ll, _i, _vp],
    ),
    "negf_zinv_workspace_bytes": (_sz, [_i, _i]),
    "negf_zinv_batched": (_i, [_i, _i, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "negf_sancho_workspace_bytes": (_sz, [_i, _i]),
    "negf_obc_sancho_batched": (_i, [_i, _i, _vp, _vp, _vp, _d, _i, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "negf_fixed_point_workspace_bytes": (_sz, [_i, _i]),
    "negf_obc_fixed_point_batched": (_i, [_i, _i] + [_vp] * 4 + [_d, _i] + [_vp] * 4 + [_vp, _sz, _vp]),
    "negf_sigma_lg_obc_workspace_bytes": (_sz, [_i, _i]),
    "negf_sigma_lg_obc_batched": (_i, [_i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "negf_stein_workspace_bytes": (_sz, [_i, _i]),
    "negf_stein_batched": (_i, [_i, _i, _vp, _vp, _vp, _d, _i, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "negf_beyn_workspace_bytes": (_sz, [_i, _i]),
    "negf_beyn_moments": (_i, [_i, _i, _i] + [_vp] * 3 + [_vp, _vp] + [_vp] * 4 + [_vp, _sz, _vp]),
    "negf_memo_workspace_bytes": (_sz, [_i, _i, _i, _i]),
    "negf_memo_refresh_batched": (_i, [_i, _i, _i, _i] + [_vp] * 5 + [_i, _d] + [_vp] * 6 + [_sz, _vp]),
    "negf_g_obc_workspace_bytes": (_sz, [_i, _i]),
    "negf_g_obc_apply": (
        _i,
        [_i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _d, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
         _vp, _vp, _vp, _ll, _i, _d, _vp, _vp, _sz, _vp],
    ),
    "negf_g_assemble": (_i, [_i, _i, _i, _vp, _vp, _vp, _vp, _vp, _d] + [_vp] * 7 + [_vp] * 7 + [_vp]),
    "negf_observables": (_i, [_i, _i, _i] + [_vp] * 14),
    "negf_conv_polarization": (_i, [_ll, _i, _i] + [_vp] * 6 + [_d, _d] + [_vp] * 5),
    "negf_conv_sigma": (_i, [_ll, _i, _i] + [_vp] * 9 + [_d, _d] + [_vp] * 5),
    "negf_convolve_energy": (_i, [_ll, _i, _i, _vp, _vp, _i, _d, _d, _vp, _vp, _vp]),
    "negf_retarded_from_lg": (_i, [_ll, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp]),
    "negf_pattern_entries": (_ll, [_i, _i]),
    "negf_pack_lg": (_i, [_i, _i, _i, _vp, _vp, _vp, _vp, _ll, _i, _vp]),
    "negf_unpack_lg": (_i, [_i, _i, _i, _vp, _vp, _ll, _i, _vp, _vp, _vp]),
    "negf_unpack_retarded": (_i, [_i, _i, _i, _vp, _vp, _vp, _ll, _i, _vp, _vp, _vp, _vp]),
    "negf_pack_lg_table": (_i, [_i, _ll, _i, _i, _vp, _vp, _vp, _vp, _vp, _ll, _i, _vp]),
    "negf_unpack_table": (_i, [_i, _ll, _i, _i, _vp, _vp, _i, _vp, _vp, _ll, _i, _vp, _vp, _vp, _i, _vp]),
    "negf_w_assemble_workspace_bytes": (_sz, [_i, _i, _i]),
    "negf_w_assemble": (_i, [_i, _i, _i] + [_vp] * 17 + [_i, _vp, _sz, _vp]),
    "negf_w_obc_workspace_bytes": (_sz, [_i, _i]),
    "negf_w_obc_apply": (_i, [_i, _i, _i] + [_vp] * 7 + [_d, _i, _d, _i] + [_vp] * 5 + [_vp] * 6
                         + [_ll, _i, _i, _d, _vp, _vp, _sz, _vp]),
    "negf_dd_workspace_bytes": (_sz, [_i, _i]),
    "negf_dd_schur_tail": (_i, [_i, _i, _i] + [_vp] * 13 + [_vp, _sz, _vp]),
    "negf_dd_middle_sweep": (_i, [_i, _i, _i] + [_vp] * 10 + [_vp, _vp, _sz, _vp]),
    "negf_dd_fold_corner": (_i, [_i, _i, _i, _i, _i] + [_vp] * 10 + [_vp, _sz, _vp]),
    "negf_dd_reverse_chain": (_i, [_i, _i, _i] + [_vp] * 7),
    "negf_g_identity_defect": (_i, [_i, _i, _i] + [_vp] * 9),
    "negf_entry_identity_defect": (_i, [_ll] + [_vp] * 6),
    "negf_pack_lg_p2p": (_i, [_i, _i, _i, _vp, _vp, _vp, _i, _vp, _vp, _ll, _i, _vp]),
    "negf_unpack_p2p": (_i, [_i, _i, _i, _vp, _i, _i, _vp, _vp, _vp, _ll, _i, _vp, _vp, _vp, _vp]),
    "negf_mix_p2p": (_i, [_ll, _i, _d, _vp, _vp, _vp, _vp, _i, _vp, _vp, _ll, _i, _vp]),
    "negf_mix": (_i, [_ll, _d] + [_vp] * 9),
    "negf_diag_traces": (_i, [_vp, _ll, _i, _vp, _i, _i, _vp, _vp]),
    "negf_prof_enable": (None, [_i]),
    "negf_launch_count": (_ll, []),
    "negf_prof_reset": (None, []),
    "negf_prof_query": (_i, [_i, _vp, _vp, _vp, _vp]),
}


class NativeLibraryError(RuntimeError):
    """The CUDA library is missing or the call failed."""


def lib_path() -> Path:
    return _LIB_PATH


def load(require_gpu: bool = True) -> C.CDLL:
    """Load the shared library (idempotent). Raises if absent."""
    global _lib
    if require_gpu and not torch.cuda.is_available():
        raise NativeLibraryError(
            "negf_b200 hot path needs a CUDA device (sm_100a); there is no CPU fallback"
        )
    if _lib is None:
        if not _LIB_PATH.exists():
            raise NativeLibraryError(
                f"{_LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = C.CDLL(str(_LIB_PATH))
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        algo = os.environ.get("NEGF_GEMM_ALGO")  # experiments: 0 = 4M, 2 = 3M cp.async, 3 = 3M bulk copies
        if algo is not None and lib.negf_set_gemm_algo(int(algo)) != 0:
            raise NativeLibraryError(f"NEGF_GEMM_ALGO={algo} is not a GEMM algorithm of this library")
        _lib = lib
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


_CODES = {-1: "invalid argument", -2: "unsupported leading dimension", -4: "workspace too small",
          -5: "size above the kernel's limit (pivoted inverse: 4096 orbitals; fused convolutions: 4096 energies)",
          -6: "could not set the kernel's shared-memory attribute"}


def check(rc: int, what: str) -> None:
    if rc != 0:
        raise NativeLibraryError(f"{what} failed with code {rc} ({_CODES.get(rc, 'CUDA error')})")


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


_V0: dict = {}


def power_start_vector(n: int, device) -> torch.Tensor:
    """obc.py:329-331: the seeded start vector of spectral_radius_estimate."""
    import numpy as np

    dev = torch.device(device)
    key = (n, dev.type, dev.index)
    if key not in _V0:
        rng = np.random.default_rng(5)
        v = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        v /= np.linalg.norm(v)
        _V0[key] = torch.from_numpy(v).to(dev)
    return _V0[key]


def stream_ptr(device: torch.device | None = None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


_WS: dict[tuple, torch.Tensor] = {}


def workspace(nbytes: int, device: torch.device) -> torch.Tensor:
    """Per-device cached scratch buffer (grown on demand, stream-ordered use)."""
    key = (device.type, device.index, torch.cuda.current_stream(device).cuda_stream)
    buf = _WS.get(key)
    if buf is None or buf.numel() < nbytes:
        _WS.pop(key, None)
        buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
        _WS[key] = buf
    return buf
