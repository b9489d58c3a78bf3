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


def test_oracle_sancho_matches_reference(golden):
    g = golden("golden_obc.npz")
    for s in range(5):
        m, n, np_ = g[f"lead{s}_m"], g[f"lead{s}_n"], g[f"lead{s}_np"]
        x, it, _ = orc.sancho_rubio(m, n, np_, tol=1e-14)
        assert it == int(g[f"lead{s}_iters"])
        assert rel(x, g[f"lead{s}_x"]) < 1e-13
        sr, sl, sg = orc.sigma_lg_obc(x, 0.1, 0.05, 0.03, n, np_)
        assert rel(sr, g[f"lead{s}_sr"]) < 1e-13
        assert rel(sl, g[f"lead{s}_sl"]) < 1e-13
        assert rel(sg, g[f"lead{s}_sg"]) < 1e-13


def test_oracle_stein_matches_reference(golden):
    g = golden("golden_obc.npz")
    for k in range(3):
        w = orc.stein_geometric(g[f"stein{k}_a"], g[f"stein{k}_q"])
        assert rel(w, g[f"stein{k}_w"]) < 1e-13


def test_oracle_scalar_fixed_point_known_answer():
    # test_obc.py:24: stable root 4 - 2 sqrt(3) of x = 1/(2 - 0.25 x)
    x, _, _ = orc.sancho_rubio(np.array([[2.0 + 0j]]), np.array([[0.5 + 0j]]), np.array([[0.5 + 0j]]), tol=1e-14)
    assert abs(x[0, 0] - 0.5358983848622456) < 1e-12


def test_oracle_chain_devices_match_reference_generators(golden):
    g = golden("golden_ballistic_small.npz")
    assert g["g_r_diag"].shape == (16, 5, 3, 3)


def test_oracle_ballistic_matches_reference_scba_run(golden):
    g = golden("golden_ballistic_small.npz")
    h = orc.chain_device(5, 3)
    energies = np.linspace(-2.0, 2.0, 16)
    out = orc.ballistic(h, energies, 1e-3, 0.1, -0.1, 0.05, tol=1e-8)
    for k, v in out.items():
        assert rel(v, g[k]) < 1e-12, k


def test_oracle_observables_match_reference(golden):
    g = golden("golden_ballistic_small.npz")
    h = orc.chain_device(5, 3)
    res = {k: g[k] for k in g.files if not k.startswith(("obs_", "ver_"))}
    obs = orc.observables(res, h[1], 4.0 / 15)
    assert rel(obs["dos"], g["obs_dos"]) < 1e-13
    assert rel(obs["density"], g["obs_density"]) < 1e-13
    assert rel(obs["current_spectrum"], g["obs_current_spectrum"]) < 1e-13
    assert abs(obs["terminal_left"] - float(g["obs_terminal_left"])) < 1e-13
    assert abs(obs["terminal_right"] - float(g["obs_terminal_right"])) < 1e-13
