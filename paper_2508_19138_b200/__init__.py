"""B200-native NEGF+GW hot path (arxiv 2508.19138 / QuaTrEx restatement ``negfgw``).

Public names mirror the reference package's solver API (negfgw/__init__.py)
for the hot path only: the selected solve (RGF) and its spatial domain
decomposition, the contact boundary solvers (Sancho-Rubio, Beyn, Stein,
memoizer), the energy convolutions, the E<->nnz redistribution and the
SCBA driver. All compute runs in the sm_100a
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

from .carrier import Contacts, ballistic_observables, ballistic_run
from .conv import convolve_energy, retarded_from_lg
from .dd import PartitionPlan, balanced_partition_plan, dist_selected_solve, make_partition_plan
from .dist import energy_chunks, transpose_distribution
from .obc import (
    ContactBlocks,
    ObcSigma,
    SurfaceCache,
    SurfaceResult,
    beyn_batched,
    fixed_point_batched,
    fixed_point_step,
    memoized_stein_batched,
    memoized_surface_batched,
    obc_beyn,
    obc_sancho_rubio,
    obc_fixed_point,
    sancho_batched,
    sigma_lg_obc,
    stein_geometric,
)
from .scba import BeynOptions, EnergyGrid, MemoizerOptions, ScbaOptions, ScbaResult, scba_run, scba_run_reference_api

ContactConfig = Contacts  # scba.py:101-121 name

__all__ = [
    "Contacts", "ContactConfig", "ballistic_observables", "ballistic_run", "convolve_energy", "retarded_from_lg",
    "PartitionPlan", "balanced_partition_plan", "dist_selected_solve", "make_partition_plan", "energy_chunks",
    "transpose_distribution", "ContactBlocks", "ObcSigma", "SurfaceCache", "SurfaceResult", "beyn_batched",
    "fixed_point_batched", "fixed_point_step", "memoized_stein_batched", "memoized_surface_batched", "obc_beyn", "obc_fixed_point", "obc_sancho_rubio",
    "sancho_batched", "sigma_lg_obc", "stein_geometric", "BeynOptions", "EnergyGrid", "MemoizerOptions",
    "ScbaOptions", "ScbaResult", "scba_run", "scba_run_reference_api",
    "FULL", "LG_COMPRESSED", "BlockMatrix",
    "C_OBSERVABLE", "C_POLARIZATION", "C_SIGMA", "KT_DEFAULT",
    "BlockStructureError", "ConvergenceError", "NegfError", "SingularBlockError", "SpectralRadiusError",
    "KIND_GREATER", "KIND_LESSER", "LgPass", "RetardedPass", "SelectedSolution", "forward_lg",
    "forward_retarded", "rgf_lesser_greater", "rgf_retarded", "selected_solve", "selected_solve_batched",
]
