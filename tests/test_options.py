"""Host-side option validation (scba.py:124-190): same ValueErrors as the
reference's ScbaOptions / BeynOptions / MemoizerOptions; no GPU needed."""

import pytest

from paper_2508_19138_b200.scba import BeynOptions, MemoizerOptions, ScbaOptions, ScbaResult


@pytest.mark.parametrize("kw,msg", [
    ({"max_iter": 0}, "max_iter"), ({"tol": 0.0}, "tol"), ({"mixing": 0.0}, "mixing"),
    ({"mixing": 1.5}, "mixing"), ({"surface_tol": -1.0}, "surface_tol"),
    ({"retarded_method": "lu"}, "retarded method"), ({"w_retarded_method": "x"}, "W retarded"),
])
def test_scba_options_reject(kw, msg):
    with pytest.raises(ValueError, match=msg):
        ScbaOptions(**kw)


def test_scba_options_defaults_follow_reference():
    o = ScbaOptions()
    assert (o.max_iter, o.tol, o.mixing, o.surface_tol, o.reset_sigma, o.oracle_mode) == (50, 1e-5, 0.3, 1e-8, True,
                                                                                        False)
    assert o.memoizer.enabled and (o.memoizer.n_fpi_retarded, o.memoizer.n_fpi_lg) == (20, 10)
    assert BeynOptions().contour() == {"radius": 1.0, "center": 0.0, "n_quad": 16}


@pytest.mark.parametrize("kw", [{"n_quad": 4}, {"radius": 0.0}, {"radius": 1.2}, {"svd_tol": 0.0}])
def test_beyn_options_reject(kw):
    with pytest.raises(ValueError):
        BeynOptions(**kw)


def test_memoizer_options_reject():
    with pytest.raises(ValueError, match="at least 2"):
        MemoizerOptions(n_fpi_retarded=1)


def test_scba_result_attribute_access():
    r = ScbaResult({"converged": True, "residuals": [1.0]})
    assert r.converged and r["residuals"] == [1.0]
    with pytest.raises(AttributeError):
        r.missing
