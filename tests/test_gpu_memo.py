"""GPU OBC memoizer (obc.py:519-608) against the reference: refresh/direct
decisions and values on primed caches, and scba_run with the memoizer on
(reference default) including the per-iteration direct/memoized counts."""

import numpy as np
import pytest
import torch

import negf_oracle as orc
from paper_2508_19138_b200.carrier import Contacts
from paper_2508_19138_b200.obc import memoized_stein_batched, memoized_surface_batched
from paper_2508_19138_b200.scba import MemoizerOptions, ScbaOptions, scba_run
from test_oracle_golden import rel

pytestmark = pytest.mark.gpu
TOL = 1e-9


def t(a, dev):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=complex))).to(dev)


def _roundoff_case(f, x0) -> bool:
    """A cache already at the fixed point to machine precision: the two trial
    updates are pure roundoff (delta ~1e-14), so rho -- and with it the
    refresh/direct choice -- is decided by summation order, not by the
    algorithm. Either choice returns the fixed point to ~1e-14; only the
    value is checked for such cases."""
    x1 = f(x0)
    return np.linalg.norm(x1 - x0) / np.linalg.norm(x1) < 1e-12


def test_memoized_surface_matches_reference(golden, cuda):
    g = golden("golden_memo.npz")
    groups: dict = {}
    for k in range(int(g["n_r"])):
        cfg = (int(g[f"r{k}_cfg"][0]), float(g[f"r{k}_cfg"][1]))
        groups.setdefault(cfg, []).append(k)
    for (n_fpi, tol), ks in groups.items():
        st = lambda key: torch.stack([t(g[f"r{k}_{key}"], cuda) for k in ks])
        has = torch.ones(len(ks), dtype=torch.int32, device=cuda)
        x, used = memoized_surface_batched(st("m"), st("n"), st("np"), st("x0"), has, n_fpi, tol, surface_tol=1e-8)
        used = used.cpu().numpy()
        for i, k in enumerate(ks):
            if not _roundoff_case(lambda x: orc.fixed_point_step(g[f"r{k}_m"], g[f"r{k}_n"], g[f"r{k}_np"], x),
                                  g[f"r{k}_x0"]):
                assert used[i] == int(g[f"r{k}_memoized"]), k
            assert rel(x[i].cpu().numpy(), g[f"r{k}_x"]) < 1e-10, k


def test_memoized_stein_matches_reference(golden, cuda):
    g = golden("golden_memo.npz")
    ks = range(int(g["n_s"]))
    st = lambda key: torch.stack([t(g[f"s{k}_{key}"], cuda) for k in ks])
    has = torch.ones(len(ks), dtype=torch.int32, device=cuda)
    w, used = memoized_stein_batched(st("a"), st("q"), st("w0"), has, 10, 1e-6)
    used = used.cpu().numpy()
    for i, k in enumerate(ks):
        a, q = g[f"s{k}_a"], g[f"s{k}_q"]
        if not _roundoff_case(lambda w: q + a @ w @ a.conj().T, g[f"s{k}_w0"]):
            assert used[i] == int(g[f"s{k}_memoized"]), k
        assert rel(w[i].cpu().numpy(), g[f"s{k}_w"]) < 1e-10, k


def test_memoized_surface_without_cache_goes_direct(cuda):
    md, mu, ml, _ = orc.random_bt_system(3, n_blocks=2, block_size=8)
    c = (md[0, 0], ml[0, 0], mu[0, 0])
    m, n, npr = (t(x, cuda)[None].repeat(4, 1, 1) for x in c)
    has = torch.tensor([0, 1, 0, 1], dtype=torch.int32, device=cuda)
    x_ref, _, _ = orc.sancho_rubio(*c, tol=1e-8)
    x0 = torch.stack([t(x_ref, cuda)] * 4)
    x0[1] *= 1.0 + 1e-8  # a near (not roundoff-exact) cache: refreshed
    x0[3] = float("nan")  # non-finite cache -> direct
    x, used = memoized_surface_batched(m, n, npr, x0, has, 20, 1e-6)
    assert used.cpu().tolist() == [0, 1, 0, 0]
    for i in range(4):
        assert rel(x[i].cpu().numpy(), x_ref) < 1e-7


def _stats(res):
    return np.array([[s["direct_calls"], s["memoized_calls"]] for s in res["cache_stats_by_iteration"]])


def test_scba_memoizer_small_matches_reference(golden, cuda):
    """4 iterations, memoizer on (tol 1e-5 -> tol_memo 1e-6), batches of 10."""
    g = golden("golden_scba_memo_small.npz")
    res = scba_run(orc.chain_device(6, 4), orc.coulomb_matrix(6, 4), np.linspace(-2.0, 2.0, 32), 1e-3,
                   Contacts(0.1, -0.1, 0.05), ScbaOptions(retarded_method="sancho", max_iter=4, batch=10), device=cuda)
    np.testing.assert_array_equal(_stats(res), g["cache_stats"])
    for k in g.files:
        if k.startswith(("ver_", "config", "cache_stats")):
            continue
        assert rel(res[k], g[k]) < TOL, k


def test_scba_memoizer_c1_matches_reference(golden, cuda):
    """C1, 3 iterations with the memoizer: weighted checksums of every array
    and the direct/memoized counts per iteration."""
    g = golden("golden_scba_memo_c1.npz")
    res = scba_run(orc.chain_device(16, 32), orc.coulomb_matrix(16, 32), np.linspace(-2.0, 2.0, 128), 1e-3,
                   Contacts(0.1, -0.1, 0.05), ScbaOptions(retarded_method="sancho", max_iter=3, batch=64), device=cuda)
    np.testing.assert_array_equal(_stats(res), g["cache_stats"])
    rng = np.random.default_rng(98)
    for f in ["g_r_diag", "g_r_upper", "g_r_lower", "g_lesser_diag", "g_lesser_upper", "g_greater_diag",
              "g_greater_upper", "sigma_obc_lesser_left", "sigma_obc_greater_left", "sigma_obc_lesser_right",
              "sigma_obc_greater_right"]:
        a = res[f]
        assert rel(np.tensordot(a, rng.standard_normal(a.shape[1:]), axes=a.ndim - 1), g[f + "_chk"]) < TOL, f
    for f in ("lesser", "greater", "ret_upper", "ret_lower"):
        a = res["sigma_" + f]
        assert rel(a.T @ rng.standard_normal(a.shape[0]), g["sigma_" + f + "_chk"]) < TOL, f
    assert rel(res["residuals"], g["residuals"]) < TOL


def test_scba_memoizer_off_counts_direct_calls(cuda):
    res = scba_run(orc.chain_device(4, 3), orc.coulomb_matrix(4, 3), np.linspace(-1.0, 1.0, 12), 1e-3,
                   Contacts(0.1, -0.1, 0.05), ScbaOptions(retarded_method="sancho", max_iter=2, memoizer=MemoizerOptions(enabled=False)),
                   device=cuda)
    assert res["cache_stats_by_iteration"] == []


def test_scba_memoizer_with_beyn_w_surface(golden, cuda):
    """Memoizer on with Beyn as the W surfaces' direct solver -- the reference's
    exact configuration: arrays and per-iteration call counts."""
    g = golden("golden_scba_memo_small.npz")
    res = scba_run(orc.chain_device(6, 4), orc.coulomb_matrix(6, 4), np.linspace(-2.0, 2.0, 32), 1e-3,
                   Contacts(0.1, -0.1, 0.05), ScbaOptions(retarded_method="sancho", max_iter=4, batch=10, w_retarded_method="beyn"),
                   device=cuda)
    np.testing.assert_array_equal(_stats(res), g["cache_stats"])
    for k in g.files:
        if k.startswith(("ver_", "config", "cache_stats")):
            continue
        assert rel(res[k], g[k]) < TOL, k
