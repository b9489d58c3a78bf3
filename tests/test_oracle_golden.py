"""The CPU oracle (oracle/negf_oracle.py) against golden vectors produced by
running the reference package itself (tests/golden/make_golden.py)."""

import numpy as np
import pytest

import negf_oracle as orc


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _case(g, c):
    p = f"c{c}_"
    m = (g[p + "m_diag"][None], g[p + "m_upper"][None], g[p + "m_lower"][None])
    b = {"<": (g[p + "bl_diag"][None], g[p + "bl_upper"][None]),
         ">": (g[p + "bg_diag"][None], g[p + "bg_upper"][None])}
    return p, m, b


def test_random_bt_system_reproduces_reference_inputs(golden):
    g = golden("golden_rgf.npz")
    for c in range(int(g["n_cases"])):
        p, m, b = _case(g, c)
        seed, nb, bs, mb, mbs = (int(x) for x in g[p + "seed"])
        md, mu, ml, src = orc.random_bt_system(seed, None if nb < 0 else nb, None if bs < 0 else bs, mb, mbs)
        np.testing.assert_array_equal(md, m[0])
        np.testing.assert_array_equal(mu, m[1])
        np.testing.assert_array_equal(ml, m[2])
        np.testing.assert_array_equal(src["<"][0], b["<"][0])
        np.testing.assert_array_equal(src[">"][1], b[">"][1])


@pytest.mark.parametrize("c", range(8))
def test_oracle_rgf_matches_reference(golden, c):
    g = golden("golden_rgf.npz")
    p, m, b = _case(g, c)
    out = orc.rgf_selected(*m, b)
    for key, ref in (("xr_diag", "xr_diag"), ("xr_upper", "xr_upper"), ("xr_lower", "xr_lower"),
                     ("x<_diag", "xl_diag"), ("x<_upper", "xl_upper"),
                     ("x>_diag", "xg_diag"), ("x>_upper", "xg_upper")):
        if g[p + ref].size == 0:
            continue
        assert rel(out[key][0], g[p + ref]) < 1e-13, key
    sym = orc.rgf_selected(*m, b, symmetrize=True)
    assert rel(sym["x<_diag"][0], g[p + "sym_xl_diag"]) < 1e-13
    assert rel(sym["x>_diag"][0], g[p + "sym_xg_diag"]) < 1e-13


@pytest.mark.parametrize("c", range(8))
def test_oracle_rgf_matches_dense(golden, c):
    g = golden("golden_rgf.npz")
    p, m, b = _case(g, c)
    a = orc.rgf_selected(*m, b)
    d = orc.dense_selected(*m, b)
    for k in d:
        if d[k].size:
            assert rel(a[k], d[k]) < 1e-11, k
