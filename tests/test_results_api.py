"""Reference-shaped results (scba.py:492-528) and observables
(scba.py:1313-1376) on the host: our observables on a ScbaResult built from
the reference's own golden arrays, and -- when the reference package is
present (build container only) -- the REFERENCE's observable functions run
unchanged on our ScbaResult object (drop-in check). No GPU needed."""

from pathlib import Path

import numpy as np
import pytest

import negf_oracle as orc
from paper_2508_19138_b200.results import (EntryPattern, ScbaResult, SigmaState, current_spectrum, dos,
                                           electron_density, terminal_current)
from paper_2508_19138_b200.scba import EnergyGrid, ScbaOptions
from paper_2508_19138_b200.carrier import Contacts

GOLDEN = Path(__file__).parent / "golden"
REF = Path("/root/reference/pkg/src")
FIELDS = ["g_r_diag", "g_r_upper", "g_r_lower", "g_lesser_diag", "g_lesser_upper", "g_greater_diag",
          "g_greater_upper", "sigma_obc_lesser_left", "sigma_obc_greater_left", "sigma_obc_lesser_right",
          "sigma_obc_greater_right"]


def result_from_golden(g, nb, bs, ne):
    return ScbaResult(grid=EnergyGrid(-2.0, 2.0, ne, 1e-3), contacts=Contacts(0.1, -0.1, 0.05),
                      options=ScbaOptions(), n_blocks=nb, block_size=bs, converged=True, n_iter=1,
                      residuals=np.array([0.0]), identity_defects=[], **{f: g[f] for f in FIELDS},
                      sigma=SigmaState.zeros(EntryPattern(nb, bs).n_entries, ne), sigma_pattern=EntryPattern(nb, bs))


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


def test_observables_match_reference_goldens():
    g = np.load(GOLDEN / "golden_ballistic_small.npz")
    res = result_from_golden(g, 5, 3, 16)
    h = orc.chain_device(5, 3)
    assert rel(dos(res), g["obs_dos"]) < 1e-12
    assert rel(electron_density(res), g["obs_density"]) < 1e-12
    assert rel(current_spectrum(res, h), g["obs_current_spectrum"]) < 1e-12
    assert abs(terminal_current(res, "left") - float(g["obs_terminal_left"])) < 1e-12
    assert abs(terminal_current(res, "right") - float(g["obs_terminal_right"])) < 1e-12
    with pytest.raises(ValueError):
        terminal_current(res, "top")


@pytest.mark.skipif(not REF.exists(), reason="reference package only in the build container")
def test_reference_observables_run_on_our_result():
    import sys

    sys.path.insert(0, str(REF))
    sys.dont_write_bytecode = True
    from negfgw import scba as ref_scba, toys as ref_toys

    g = np.load(GOLDEN / "golden_ballistic_small.npz")
    res = result_from_golden(g, 5, 3, 16)
    assert rel(ref_scba.dos(res), g["obs_dos"]) < 1e-12
    assert rel(ref_scba.electron_density(res), g["obs_density"]) < 1e-12
    assert rel(ref_scba.current_spectrum(res, ref_toys.chain_device(5, 3)), g["obs_current_spectrum"]) < 1e-12
    assert abs(ref_scba.terminal_current(res, "left") - float(g["obs_terminal_left"])) < 1e-12
    # the result's pattern enumerates entries exactly like the reference's EntryPattern
    from negfgw.convolve import EntryPattern as RefPattern

    rp = RefPattern(4, 5, 3, True)
    assert np.array_equal(res.sigma_pattern.rows, RefPattern(5, 3, 3, True).rows)
    assert np.array_equal(EntryPattern(4, 5).cols, rp.cols) and EntryPattern(4, 5).n_entries == rp.n_entries
    assert EntryPattern(4, 5).full_entry_count() == rp.full_entry_count()
