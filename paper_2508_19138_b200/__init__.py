"""B200-native NEGF+GW hot path (arxiv 2508.19138 / QuaTrEx restatement ``negfgw``).

Public names mirror the reference package's solver API (negfgw/__init__.py)
for the hot path only: the selected solve (RGF), the contact boundary
solvers, and the energy convolutions. All compute runs in the sm_100a
library ``libnegf_b200.so`` through the C ABI in include/negf_b200.h.
"""

from .blocks import FULL, LG_COMPRESSED, BlockMatrix
from .constants import C_OBSERVABLE, C_POLARIZATION, C_SIGMA, KT_DEFAULT
from .errors import (
    BlockStructureError,
    ConvergenceError,
    NegfError,
    SingularBlockError,
    SpectralRadiusError,
)
from .rgf import (
    KIND_GREATER,
    KIND_LESSER,
    LgPass,
    RetardedPass,
    SelectedSolution,
    forward_lg,
    forward_retarded,
    rgf_lesser_greater,
    rgf_retarded,
    selected_solve,
    selected_solve_batched,
)

__all__ = [
    "FULL", "LG_COMPRESSED", "BlockMatrix",
    "C_OBSERVABLE", "C_POLARIZATION", "C_SIGMA", "KT_DEFAULT",
    "BlockStructureError", "ConvergenceError", "NegfError", "SingularBlockError", "SpectralRadiusError",
    "KIND_GREATER", "KIND_LESSER", "LgPass", "RetardedPass", "SelectedSolution", "forward_lg",
    "forward_retarded", "rgf_lesser_greater", "rgf_retarded", "selected_solve", "selected_solve_batched",
]
