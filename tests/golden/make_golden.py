"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (the reference is read-only at /root/reference
and does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes tests/golden/*.npz. Versions of numpy/scipy used are stored in every
file (the reference pins only lower bounds).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import scipy

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
sys.dont_write_bytecode = True

from negfgw import rgf, obc, convolve, scba, toys  # noqa: E402
from negfgw.blocks import BlockMatrix  # noqa: E402
from negfgw.device import EnergyGrid  # noqa: E402
from threadpoolctl import threadpool_limits  # noqa: E402

OUT = Path(__file__).resolve().parent
VERS = dict(numpy=np.__version__, scipy=scipy.__version__)


def stack_bt(m: BlockMatrix):
    n = m.n_blocks
    d = np.stack([m.get_block(i, i) for i in range(n)])
    u = np.stack([m.get_block(i, i + 1) for i in range(n - 1)])
    lo = np.stack([m.get_block(i + 1, i) for i in range(n - 1)])
    return d, u, lo


def sol_arrays(sol, prefix: str, out: dict):
    out[prefix + "xr_diag"] = np.stack(sol.x_r_diag)
    out[prefix + "xr_upper"] = np.stack(sol.x_r_upper)
    out[prefix + "xr_lower"] = np.stack(sol.x_r_lower)
    for k, tag in (("<", "l"), (">", "g")):
        out[prefix + f"x{tag}_diag"] = np.stack(sol.x_lg_diag[k])
        out[prefix + f"x{tag}_upper"] = np.stack(sol.x_lg_upper[k])


def make_rgf():
    out = {}
    cases = [(17 * k, None, None, 8, 6) for k in range(5)] + [(101, 6, 32, 10, 8), (202, 2, 40, 10, 8), (303, 2, 1, 10, 8)]
    out["n_cases"] = np.array(len(cases))
    for c, (seed, nb, bs, mb, mbs) in enumerate(cases):
        m, bl, bg = toys.random_bt_system(seed, n_blocks=nb, block_size=bs, max_blocks=mb, max_block_size=mbs)
        p = f"c{c}_"
        out[p + "m_diag"], out[p + "m_upper"], out[p + "m_lower"] = stack_bt(m)
        for tag, b in (("l", bl), ("g", bg)):
            n = b.n_blocks
            out[p + f"b{tag}_diag"] = np.stack([b.get_block(i, i) for i in range(n)])
            out[p + f"b{tag}_upper"] = np.stack([b.get_block(i, i + 1) for i in range(n - 1)])
        out[p + "seed"] = np.array([seed, -1 if nb is None else nb, -1 if bs is None else bs, mb, mbs])
        sol = rgf.selected_solve(m, b_lesser=bl, b_greater=bg)
        sol_arrays(sol, p, out)
        sol.symmetrize()
        out[p + "sym_xl_diag"] = np.stack(sol.x_lg_diag["<"])
        out[p + "sym_xg_diag"] = np.stack(sol.x_lg_diag[">"])
        fwd = rgf.forward_retarded(m)
        out[p + "u_spread"] = np.asarray(fwd.u_spread)
    np.savez_compressed(OUT / "golden_rgf.npz", **out, **{f"ver_{k}": v for k, v in VERS.items()})


def make_obc():
    out = {}
    for seed in range(5):
        c = toys.random_lead(seed=seed, block_size=5, eta=0.02)
        r = obc.obc_sancho_rubio(c, tol=1e-14)
        out[f"lead{seed}_m"], out[f"lead{seed}_n"], out[f"lead{seed}_np"] = c.m, c.n, c.n_prime
        out[f"lead{seed}_x"] = r.x_r
        out[f"lead{seed}_iters"] = np.array(r.iters)
        s = obc.sigma_lg_obc(r.x_r, 0.1, 0.05, 0.03, (c.n, c.n_prime))
        out[f"lead{seed}_sr"], out[f"lead{seed}_sl"], out[f"lead{seed}_sg"] = s.sigma_r, s.sigma_lesser, s.sigma_greater
    # stein geometric
    rng = np.random.default_rng(3)
    for k in range(3):
        a = 0.3 * (rng.standard_normal((6, 6)) + 1j * rng.standard_normal((6, 6))) / np.sqrt(6)
        q = rng.standard_normal((6, 6)) + 1j * rng.standard_normal((6, 6))
        out[f"stein{k}_a"], out[f"stein{k}_q"] = a, q
        out[f"stein{k}_w"] = obc.stein_geometric(a, q)
    np.savez_compressed(OUT / "golden_obc.npz", **out, **{f"ver_{k}": v for k, v in VERS.items()})


def make_conv():
    out = {}
    rng = np.random.default_rng(5)
    for ne in (24, 128, 129, 1000):
        x1 = rng.standard_normal((3, ne)) + 1j * rng.standard_normal((3, ne))
        x2 = rng.standard_normal((3, ne)) + 1j * rng.standard_normal((3, ne))
        out[f"n{ne}_x1"], out[f"n{ne}_x2"] = x1, x2
        out[f"n{ne}_conv"] = convolve.convolve_energy(x1, x2, "convolution", 0.7 - 0.2j, 0.01)
        out[f"n{ne}_corr"] = convolve.convolve_energy(x1, x2, "correlation", -0.3 + 1.1j, 0.02)
        out[f"n{ne}_ret"] = convolve.retarded_from_lg(x1, x2)
        out[f"n{ne}_direct_conv"] = convolve.convolve_energy_direct(x1, x2, "convolution", 0.7 - 0.2j, 0.01)
        out[f"n{ne}_direct_corr"] = convolve.convolve_energy_direct(x1, x2, "correlation", -0.3 + 1.1j, 0.02)
    np.savez_compressed(OUT / "golden_conv.npz", **out, **{f"ver_{k}": v for k, v in VERS.items()})


def scba_case(nb, bs, ne, iters, ballistic=False, memo=False, method="sancho"):
    h = toys.chain_device(nb, bs)
    v = None if ballistic else toys.coulomb_matrix(nb, bs)
    grid = EnergyGrid(-2.0, 2.0, ne, eta=1e-3)
    contacts = scba.ContactConfig(mu_left=0.1, mu_right=-0.1, kT=0.05)
    opts = scba.ScbaOptions(max_iter=iters, tol=1e-5 if memo else 1e-12, mixing=0.3, retarded_method=method,
                            memoizer=scba.MemoizerOptions(enabled=memo))
    with threadpool_limits(1):
        return scba.scba_run(h, v, grid, contacts, opts)


RESULT_FIELDS = ["g_r_diag", "g_r_upper", "g_r_lower", "g_lesser_diag", "g_lesser_upper",
                 "g_greater_diag", "g_greater_upper", "sigma_obc_lesser_left",
                 "sigma_obc_greater_left", "sigma_obc_lesser_right", "sigma_obc_greater_right"]


def make_scba_coarse_w():
    """W grid coarser than the G grid (scba.py:893-903, 925-937): G on
    chain_device(8, 4), V = coulomb_matrix(4, 8) (bs_w = 2 bs), 3 iterations."""
    h = toys.chain_device(8, 4)
    v = toys.coulomb_matrix(4, 8)
    grid = EnergyGrid(-2.0, 2.0, 32, eta=1e-3)
    contacts = scba.ContactConfig(mu_left=0.1, mu_right=-0.1, kT=0.05)
    opts = scba.ScbaOptions(max_iter=3, tol=1e-12, mixing=0.3, retarded_method="sancho",
                            memoizer=scba.MemoizerOptions(enabled=False))
    with threadpool_limits(1):
        res = scba.scba_run(h, v, grid, contacts, opts)
    out = {f: getattr(res, f) for f in RESULT_FIELDS}
    for f in ("lesser", "greater", "ret_upper", "ret_lower"):
        out["sigma_" + f] = getattr(res.sigma, f)
    out["residuals"] = np.asarray(res.residuals)
    out["config"] = np.array([8, 4, 4, 8, 32, 3])
    np.savez_compressed(OUT / "golden_scba_coarse_w.npz", **out, **{f"ver_{k}": v for k, v in VERS.items()})


def make_ballistic():
    out = {}
    res = scba_case(5, 3, 16, 1, ballistic=True)
    for f in RESULT_FIELDS:
        out[f] = getattr(res, f)
    h = toys.chain_device(5, 3)
    out["obs_dos"] = scba.dos(res)
    out["obs_density"] = scba.electron_density(res)
    out["obs_current_spectrum"] = scba.current_spectrum(res, h)
    out["obs_terminal_left"] = np.array(scba.terminal_current(res, "left"))
    out["obs_terminal_right"] = np.array(scba.terminal_current(res, "right"))
    out["obs_landauer"] = np.array(scba.landauer_current(h, res.grid, res.contacts))
    np.savez_compressed(OUT / "golden_ballistic_small.npz", **out, **{f"ver_{k}": v for k, v in VERS.items()})


def make_scba():
    # small: every array in full
    out = {}
    res = scba_case(6, 4, 32, 3)
    for f in RESULT_FIELDS:
        out[f] = getattr(res, f)
    for f in ("lesser", "greater", "ret_upper", "ret_lower"):
        out["sigma_" + f] = getattr(res.sigma, f)
    out["residuals"] = np.asarray(res.residuals)
    out["config"] = np.array([6, 4, 32, 3])
    np.savez_compressed(OUT / "golden_scba_small.npz", **out, **{f"ver_{k}": v for k, v in VERS.items()})
    # C1 (16 x 32, 128 energies, 1 iteration): energy slices + weighted checksums
    out = {}
    res = scba_case(16, 32, 128, 1)
    sel = np.array([0, 37, 64, 101, 127])
    out["sel"] = sel
    rng = np.random.default_rng(99)
    for f in RESULT_FIELDS:
        a = getattr(res, f)
        out[f + "_sel"] = a[sel]
        w = rng.standard_normal(a.shape[1:])
        out[f + "_chk"] = np.tensordot(a, w, axes=a.ndim - 1)  # per-energy weighted sums
    for f in ("lesser", "greater", "ret_upper", "ret_lower"):
        a = getattr(res.sigma, f)
        out["sigma_" + f + "_sel"] = a[:, sel]
        out["sigma_" + f + "_chk"] = a.T @ rng.standard_normal(a.shape[0])
        out["sigma_" + f + "_fro"] = np.array(np.linalg.norm(a))
    out["residuals"] = np.asarray(res.residuals)
    out["config"] = np.array([16, 32, 128, 1])
    np.savez_compressed(OUT / "golden_scba_c1.npz", **out, **{f"ver_{k}": v for k, v in VERS.items()})
    # ballistic small
    out = {}
    res = scba_case(5, 3, 16, 1, ballistic=True)
    for f in RESULT_FIELDS:
        out[f] = getattr(res, f)
    h = toys.chain_device(5, 3)
    out["obs_dos"] = scba.dos(res)
    out["obs_density"] = scba.electron_density(res)
    out["obs_current_spectrum"] = scba.current_spectrum(res, h)
    out["obs_terminal_left"] = np.array(scba.terminal_current(res, "left"))
    out["obs_terminal_right"] = np.array(scba.terminal_current(res, "right"))
    out["obs_landauer"] = np.array(scba.landauer_current(h, res.grid, res.contacts))
    np.savez_compressed(OUT / "golden_ballistic_small.npz", **out, **{f"ver_{k}": v for k, v in VERS.items()})


def make_memo():
    """memoized_obc (obc.py:519-608) decisions and values, and scba_run with
    the memoizer on (reference default; tol 1e-5 -> tol_memo 1e-6)."""
    out = {}
    k = 0
    for seed in range(4):
        for de, eta, n_fpi, tol in ((0.0, 0.05, 20, 1e-6), (1e-7, 0.05, 20, 1e-6), (1e-4, 0.05, 20, 1e-6),
                                    (1e-3, 0.02, 10, 1e-8), (3e-2, 0.05, 20, 1e-6), (0.4, 0.05, 20, 1e-6),
                                    (1e-3, 1e-3, 20, 1e-6)):
            c0 = toys.random_lead(seed, 6, energy=0.2, eta=eta)
            c1 = toys.random_lead(seed, 6, energy=0.2 + de, eta=eta)
            cache = obc.SurfaceCache()
            key = ("G", "left", 0, "R")
            obc.memoized_obc(key, lambda: obc.obc_sancho_rubio(c0, tol=1e-8).x_r,
                             lambda x: obc.fixed_point_step(c0, x), cache, n_fpi, tol)
            x0 = np.array(cache.entries[key].value)
            x = obc.memoized_obc(key, lambda: obc.obc_sancho_rubio(c1, tol=1e-8).x_r,
                                 lambda x: obc.fixed_point_step(c1, x), cache, n_fpi, tol)
            p = f"r{k}_"
            out[p + "m"], out[p + "n"], out[p + "np"] = c1.m, c1.n, c1.n_prime
            out[p + "x0"], out[p + "x"] = x0, np.asarray(x)
            out[p + "cfg"] = np.array([n_fpi, tol])
            out[p + "memoized"] = np.array(cache.stats["memoized_calls"])
            k += 1
    out["n_r"] = np.array(k)
    rng = np.random.default_rng(21)
    k = 0
    for rad in (0.3, 0.7, 0.95):
        for pert in (0.0, 1e-9, 1e-5, 1e-2, 1.0):
            a = rng.standard_normal((5, 5)) + 1j * rng.standard_normal((5, 5))
            a *= rad / max(abs(np.linalg.eigvals(a)))
            q = rng.standard_normal((5, 5)) + 1j * rng.standard_normal((5, 5))
            q = q + q.conj().T
            w0 = obc.stein_geometric(a, q) + pert * (rng.standard_normal((5, 5)) + 0j)
            cache = obc.SurfaceCache()
            key = ("W", "left", 0, "<")
            cache.entries[key] = obc.CacheEntry(w0)
            w = obc.memoized_obc(key, lambda: scba._stein_direct(a, q),
                                 lambda w: q + a @ w @ a.conj().T, cache, 10, 1e-6)
            p = f"s{k}_"
            out[p + "a"], out[p + "q"], out[p + "w0"], out[p + "w"] = a, q, w0, np.asarray(w)
            out[p + "memoized"] = np.array(cache.stats["memoized_calls"])
            k += 1
    out["n_s"] = np.array(k)
    np.savez_compressed(OUT / "golden_memo.npz", **out, **{f"ver_{k}": v for k, v in VERS.items()})
    # scba_run, memoizer on
    out = {}
    res = scba_case(6, 4, 32, 4, memo=True)
    for f in RESULT_FIELDS:
        out[f] = getattr(res, f)
    for f in ("lesser", "greater", "ret_upper", "ret_lower"):
        out["sigma_" + f] = getattr(res.sigma, f)
    out["residuals"] = np.asarray(res.residuals)
    out["cache_stats"] = np.array([[s_["direct_calls"], s_["memoized_calls"]] for s_ in res.cache_stats_by_iteration])
    out["config"] = np.array([6, 4, 32, 4])
    np.savez_compressed(OUT / "golden_scba_memo_small.npz", **out, **{f"ver_{k}": v for k, v in VERS.items()})
    out = {}
    res = scba_case(16, 32, 128, 3, memo=True)
    rng = np.random.default_rng(98)
    for f in RESULT_FIELDS:
        a = getattr(res, f)
        out[f + "_chk"] = np.tensordot(a, rng.standard_normal(a.shape[1:]), axes=a.ndim - 1)
    for f in ("lesser", "greater", "ret_upper", "ret_lower"):
        a = getattr(res.sigma, f)
        out["sigma_" + f + "_chk"] = a.T @ rng.standard_normal(a.shape[0])
        out["sigma_" + f + "_fro"] = np.array(np.linalg.norm(a))
    out["residuals"] = np.asarray(res.residuals)
    out["cache_stats"] = np.array([[s_["direct_calls"], s_["memoized_calls"]] for s_ in res.cache_stats_by_iteration])
    out["config"] = np.array([16, 32, 128, 3])
    np.savez_compressed(OUT / "golden_scba_memo_c1.npz", **out, **{f"ver_{k}": v for k, v in VERS.items()})


def make_dd():
    """dist_selected_solve (dist.py:750-784) run by the reference itself over
    spmd_run thread ranks: partition plans, full solutions and the
    sequential selected_solve of the same systems."""
    from negfgw import dist

    out = {}
    cases = [(11, 8, 5, 2), (12, 9, 4, 3), (13, 12, 6, 4), (14, 10, 3, 4), (15, 7, 8, 3)]
    out["n_cases"] = np.array(len(cases))
    for c, (seed, nb, bs, p_s) in enumerate(cases):
        m, bl, bg = toys.random_bt_system(seed, n_blocks=nb, block_size=bs)
        plan = dist.make_partition_plan(nb, p_s)

        def body(comm):
            return dist.dist_selected_solve(m, bl, bg, plan=plan, comm=comm)

        sol, _ = dist.spmd_run(body, p_s)[0]
        p = f"c{c}_"
        out[p + "cfg"] = np.array([seed, nb, bs, p_s])
        out[p + "ranges"] = np.array(plan.ranges)
        out[p + "m_diag"], out[p + "m_upper"], out[p + "m_lower"] = stack_bt(m)
        for tag, b in (("l", bl), ("g", bg)):
            out[p + f"b{tag}_diag"] = np.stack([b.get_block(i, i) for i in range(nb)])
            out[p + f"b{tag}_upper"] = np.stack([b.get_block(i, i + 1) for i in range(nb - 1)])
        sol_arrays(sol, p, out)
    np.savez_compressed(OUT / "golden_dd.npz", **out, **{f"ver_{k}": v for k, v in VERS.items()})


def make_beyn():
    """obc_beyn (obc.py:198-296) on random leads and on the W-side cells of
    the small SCBA case (stencil [n_up, m, n_dn], BeynOptions defaults)."""
    out = {}
    k = 0
    for seed, bs, eta, e in ((0, 5, 0.02, 0.1), (1, 6, 0.05, -0.3), (2, 4, 1e-3, 0.0), (3, 8, 0.01, 0.5),
                             (4, 3, 0.1, 1.2)):
        c = toys.random_lead(seed, bs, energy=e, eta=eta)
        r = obc.obc_beyn([c.n_prime, c.m, c.n], contour={"radius": 1.0, "center": 0.0, "n_quad": 16},
                         svd_tol=1e-8)
        p = f"b{k}_"
        out[p + "m"], out[p + "n"], out[p + "np"] = c.m, c.n, c.n_prime
        out[p + "x"], out[p + "modes"] = r.x_r, np.array(r.n_modes)
        k += 1
    out["n_b"] = np.array(k)
    np.savez_compressed(OUT / "golden_beyn.npz", **out, **{f"ver_{k}": v for k, v in VERS.items()})


def make_methods():
    """scba_run with the other carrier retarded methods (scba.py:577-614):
    the reference default "beyn" and "fixed_point", 6x4 chain, 32 energies,
    2 GW iterations, memoizer off."""
    for method in ("beyn", "fixed_point"):
        out = {}
        res = scba_case(6, 4, 32, 2, method=method)
        for f in RESULT_FIELDS:
            out[f] = getattr(res, f)
        for f in ("lesser", "greater", "ret_upper", "ret_lower"):
            out["sigma_" + f] = getattr(res.sigma, f)
        out["residuals"] = np.asarray(res.residuals)
        np.savez_compressed(OUT / f"golden_scba_{method}.npz", **out, **{f"ver_{k}": v for k, v in VERS.items()})


if __name__ == "__main__":
    which = sys.argv[1:] or ["rgf", "obc", "conv", "scba"]
    for w in which:
        globals()["make_" + w]()
        print("wrote", w, flush=True)
