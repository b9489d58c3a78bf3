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


@pytest.mark.parametrize("ne", [24, 128, 129, 1000])
def test_oracle_convolutions_match_reference(golden, ne):
    g = golden("golden_conv.npz")
    x1, x2 = g[f"n{ne}_x1"], g[f"n{ne}_x2"]
    assert rel(orc.convolve_energy(x1, x2, "convolution", 0.7 - 0.2j, 0.01), g[f"n{ne}_conv"]) < 1e-14
    assert rel(orc.convolve_energy(x1, x2, "correlation", -0.3 + 1.1j, 0.02), g[f"n{ne}_corr"]) < 1e-14
    assert rel(orc.retarded_from_lg(x1, x2), g[f"n{ne}_ret"]) < 1e-14
    assert rel(orc.convolve_energy_direct(x1, x2, "convolution", 0.7 - 0.2j, 0.01), g[f"n{ne}_direct_conv"]) < 1e-12
    assert rel(orc.convolve_energy_direct(x1, x2, "correlation", -0.3 + 1.1j, 0.02), g[f"n{ne}_direct_corr"]) < 1e-12


def test_oracle_scba_small_matches_reference(golden):
    """Full SCBA (3 iterations, 6x4 chain + Coulomb, 32 energies) vs scba_run."""
    g = golden("golden_scba_small.npz")
    h = orc.chain_device(6, 4)
    v = orc.coulomb_matrix(6, 4)
    res = orc.scba(h, v, np.linspace(-2.0, 2.0, 32), 1e-3, 0.1, -0.1, 0.05, max_iter=3, tol=1e-12)
    for k in g.files:
        if k.startswith(("ver_", "config")):
            continue
        assert rel(res[k], g[k]) < 1e-11, k


def test_oracle_entry_layout_roundtrip():
    rng = np.random.default_rng(0)
    n_b, bs, ne = 4, 3, 5
    d = rng.standard_normal((ne, n_b, bs, bs)) + 1j * rng.standard_normal((ne, n_b, bs, bs))
    d = 0.5 * (d - np.conj(np.swapaxes(d, -1, -2)))
    u = rng.standard_normal((ne, n_b - 1, bs, bs)) + 0j
    vals = orc.gather_entries(d, u)
    rows, cols = orc.entry_pattern(n_b, bs)
    assert vals.shape == (len(rows), ne) and np.all(rows <= cols)
    d2, u2 = orc.scatter_lg(vals, n_b, bs)
    np.testing.assert_allclose(d2, d, atol=0)
    np.testing.assert_allclose(u2, u, atol=0)


def test_oracle_scba_c1_matches_reference(golden):
    """C1 (16 blocks x 32 orbitals, 128 energies, 1 SCBA iteration) vs the
    reference scba_run: energy slices + weighted checksums of every array."""
    g = golden("golden_scba_c1.npz")
    res = orc.scba(orc.chain_device(16, 32), orc.coulomb_matrix(16, 32), np.linspace(-2.0, 2.0, 128),
                   1e-3, 0.1, -0.1, 0.05, max_iter=1)
    check_c1(res, g)


def check_c1(res, g, tol=1e-10):
    sel = g["sel"]
    rng = np.random.default_rng(99)
    for f in ["g_r_diag", "g_r_upper", "g_r_lower", "g_lesser_diag", "g_lesser_upper", "g_greater_diag",
              "g_greater_upper", "sigma_obc_lesser_left", "sigma_obc_greater_left", "sigma_obc_lesser_right",
              "sigma_obc_greater_right"]:
        a = res[f]
        assert rel(a[sel], g[f + "_sel"]) < tol, f
        w = rng.standard_normal(a.shape[1:])
        assert rel(np.tensordot(a, w, axes=a.ndim - 1), g[f + "_chk"]) < tol, f
    for f in ("lesser", "greater", "ret_upper", "ret_lower"):
        a = res["sigma_" + f]
        assert rel(a[:, sel], g["sigma_" + f + "_sel"]) < tol, f
        assert rel(a.T @ rng.standard_normal(a.shape[0]), g["sigma_" + f + "_chk"]) < tol, f
        assert abs(np.linalg.norm(a) - float(g["sigma_" + f + "_fro"])) < tol * float(g["sigma_" + f + "_fro"])
    assert rel(res["residuals"], g["residuals"]) < tol


def test_oracle_memoized_obc_matches_reference(golden):
    """memoized_obc (obc.py:519-608): same refresh/direct decision and value
    as the reference on primed caches (surface fixed point and Stein)."""
    g = golden("golden_memo.npz")
    for k in range(int(g["n_r"])):
        p = f"r{k}_"
        m, n, npr = g[p + "m"], g[p + "n"], g[p + "np"]
        n_fpi, tol = int(g[p + "cfg"][0]), float(g[p + "cfg"][1])
        cache = orc.SurfaceCache()
        cache.entries["k"] = g[p + "x0"]
        x = orc.memoized_obc("k", lambda: orc.sancho_rubio(m, n, npr, tol=1e-8)[0],
                             lambda x: orc.fixed_point_step(m, n, npr, x), cache, n_fpi, tol)
        assert cache.stats["memoized_calls"] == int(g[p + "memoized"]), k
        assert rel(x, g[p + "x"]) < 1e-12, k
    for k in range(int(g["n_s"])):
        p = f"s{k}_"
        a, q = g[p + "a"], g[p + "q"]
        cache = orc.SurfaceCache()
        cache.entries["k"] = g[p + "w0"]
        w = orc.memoized_obc("k", lambda: orc.stein_direct(a, q), lambda w: q + a @ w @ a.conj().T, cache, 10, 1e-6)
        assert cache.stats["memoized_calls"] == int(g[p + "memoized"]), k
        assert rel(w, g[p + "w"]) < 1e-12, k


def test_oracle_scba_memoizer_matches_reference(golden):
    """scba_run with the OBC memoizer on (reference default, tol 1e-5): 4
    iterations, per-iteration direct/memoized counts and every array."""
    g = golden("golden_scba_memo_small.npz")
    res = orc.scba(orc.chain_device(6, 4), orc.coulomb_matrix(6, 4), np.linspace(-2.0, 2.0, 32), 1e-3, 0.1, -0.1,
                   0.05, max_iter=4, tol=1e-5, memoizer=(20, 10))
    stats = np.array([[s["direct_calls"], s["memoized_calls"]] for s in res["cache_stats_by_iteration"]])
    np.testing.assert_array_equal(stats, g["cache_stats"])
    for k in g.files:
        if k.startswith(("ver_", "config", "cache_stats")):
            continue
        assert rel(res[k], g[k]) < 1e-9, k


@pytest.mark.parametrize("c", range(5))
def test_oracle_dd_matches_reference_dist_selected_solve(golden, c):
    """dist_selected_solve (dist.py:750) run by the reference over spmd_run
    ranks vs the oracle's partition-by-partition restatement; plans equal."""
    g = golden("golden_dd.npz")
    p = f"c{c}_"
    seed, nb, bs, p_s = (int(x) for x in g[p + "cfg"])
    ranges = orc.make_partition_plan(nb, p_s)
    assert [tuple(r) for r in g[p + "ranges"].tolist()] == ranges
    m = (g[p + "m_diag"][None], g[p + "m_upper"][None], g[p + "m_lower"][None])
    b = {"<": (g[p + "bl_diag"][None], g[p + "bl_upper"][None]),
         ">": (g[p + "bg_diag"][None], g[p + "bg_upper"][None])}
    out = orc.dd_selected(*m, b, ranges)
    for key, ref in (("xr_diag", "xr_diag"), ("xr_upper", "xr_upper"), ("xr_lower", "xr_lower"),
                     ("x<_diag", "xl_diag"), ("x<_upper", "xl_upper"), ("x>_diag", "xg_diag"),
                     ("x>_upper", "xg_upper")):
        assert rel(out[key][0], g[p + ref]) < 1e-12, key
    seq = orc.rgf_selected(*m, b)
    assert rel(out["x<_diag"], seq["x<_diag"]) < 1e-10


def test_oracle_beyn_matches_reference(golden):
    """obc_beyn (obc.py:198-296) vs the oracle restatement: same mode count,
    same surface block. (On these in-band random leads Beyn keeps fewer
    decaying modes than bs and differs from the Sancho-Rubio fixed point --
    the reference behaviour SURVEY §0.4 documents; the goldens pin it.)"""
    g = golden("golden_beyn.npz")
    for k in range(int(g["n_b"])):
        p = f"b{k}_"
        x, modes = orc.beyn(g[p + "m"], g[p + "n"], g[p + "np"])
        assert modes == int(g[p + "modes"]), k
        assert rel(x, g[p + "x"]) < 1e-12, k


def test_oracle_entry_cutoff_infinite_is_full_band():
    """The oracle's r_cut hook (entry_cutoff, test infrastructure for the
    paper's nonzero-set deviation) is the identity for cutoff >= the band."""
    h, v = orc.chain_device(4, 3), orc.coulomb_matrix(4, 3)
    e = np.linspace(-2.0, 2.0, 12)
    a = orc.scba(h, v, e, 1e-3, 0.1, -0.1, 0.05, max_iter=2)
    b = orc.scba(h, v, e, 1e-3, 0.1, -0.1, 0.05, max_iter=2, entry_cutoff=100)
    for k in a:
        if k != "cache_stats_by_iteration":
            assert np.array_equal(a[k], b[k]), k
    c = orc.scba(h, v, e, 1e-3, 0.1, -0.1, 0.05, max_iter=2, entry_cutoff=1)
    rows, cols = orc.entry_pattern(4, 3)
    assert np.all(c["sigma_lesser"][np.abs(rows - cols) > 1] == 0)
    assert np.any(c["sigma_lesser"] != a["sigma_lesser"])
