"""Host-side option validation (scba.py:124-190): same ValueErrors as the
reference's ScbaOptions / BeynOptions / MemoizerOptions; no GPU needed."""

import pytest

from paper_2508_19138_b200.scba import BeynOptions, MemoizerOptions, ScbaOptions, ScbaResult


@pytest.mark.parametrize("kw,msg", [
    ({"max_iter": 0}, "max_iter"), ({"tol": 0.0}, "tol"), ({"mixing": 0.0}, "mixing"),
    ({"mixing": 1.5}, "mixing"), ({"surface_tol": -1.0}, "surface_tol"),
    ({"retarded_method": "lu"}, "retarded method"), ({"w_retarded_method": "x"}, "W retarded"),
    ({"greater": "dense"}, "greater mode"), ({"entry_cutoff": -1}, "entry_cutoff"),
    ({"rgf_streams": 0}, "rgf_streams"),
])
def test_scba_options_reject(kw, msg):
    with pytest.raises(ValueError, match=msg):
        ScbaOptions(**kw)


def test_scba_options_defaults_follow_reference():
    o = ScbaOptions()
    assert (o.max_iter, o.tol, o.mixing, o.surface_tol, o.reset_sigma, o.oracle_mode) == (50, 1e-5, 0.3, 1e-8, True,
                                                                                        False)
    assert o.retarded_method == "beyn"  # scba.py:165
    assert o.greater == "recursion" and o.entry_cutoff is None  # the reference's algorithm and entry set
    assert o.memoizer.enabled and (o.memoizer.n_fpi_retarded, o.memoizer.n_fpi_lg) == (20, 10)
    assert BeynOptions().contour() == {"radius": 1.0, "center": 0.0, "n_quad": 16}


@pytest.mark.parametrize("kw", [{"n_quad": 4}, {"radius": 0.0}, {"radius": 1.2}, {"svd_tol": 0.0}])
def test_beyn_options_reject(kw):
    with pytest.raises(ValueError):
        BeynOptions(**kw)


def test_memoizer_options_reject():
    with pytest.raises(ValueError, match="at least 2"):
        MemoizerOptions(n_fpi_retarded=1)


def test_scba_result_attribute_and_key_access():
    import numpy as np

    from paper_2508_19138_b200.results import EntryPattern, SigmaState

    r = ScbaResult(grid=None, contacts=None, options=ScbaOptions(), n_blocks=2, block_size=3, converged=True,
                   n_iter=1, residuals=np.array([1.0]), identity_defects=[], sigma=SigmaState.zeros(5, 4),
                   sigma_pattern=EntryPattern(2, 3))
    assert r.converged and list(r["residuals"]) == [1.0]
    assert r["sigma_lesser"].shape == (5, 4) and "sigma_ret_lower" in r
    assert "g_r_diag" not in r
    with pytest.raises(KeyError):
        r["missing"]
    with pytest.raises(AttributeError):
        r.missing


def test_entry_pattern_matches_reference_order():
    """convolve.py:135-187 order (vectorised here), incl. n_entries and the
    uncompressed in-band count."""
    import numpy as np

    from paper_2508_19138_b200.results import EntryPattern

    p = EntryPattern(3, 4)
    rows, cols = [], []
    for bi in range(3):
        for bj in range(max(0, bi - 1), min(3, bi + 2)):
            if bj < bi:
                continue
            for r in range(4):
                for c in range(4):
                    if bi == bj and c < r:
                        continue
                    rows.append(bi * 4 + r)
                    cols.append(bj * 4 + c)
    assert np.array_equal(p.rows, rows) and np.array_equal(p.cols, cols)
    assert p.n_entries == len(rows) == 3 * 10 + 2 * 16
    assert p.full_entry_count() == (3 + 4) * 16
