"""GPU parity of the full SCBA (GW) iteration and its layout/W stages
against reference golden vectors and the pinned oracle. Bar: 1e-9 relative
Frobenius per quantity (north_star)."""

import numpy as np
import pytest
import torch

import negf_oracle as orc
from paper_2508_19138_b200.carrier import Contacts
from paper_2508_19138_b200.scba import EntryLayout, MemoizerOptions, ScbaOptions, ScreenedSolver, scba_run

MEMO_OFF = MemoizerOptions(enabled=False)
from test_oracle_golden import check_c1

pytestmark = pytest.mark.gpu
TOL = 1e-9


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def t(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def test_pack_unpack_match_oracle(cuda):
    rng = np.random.default_rng(1)
    n_b, bs, ne, tot = 5, 7, 9, 40
    lay = EntryLayout(n_b, bs, cuda)
    d = rng.standard_normal((ne, n_b, bs, bs)) + 1j * rng.standard_normal((ne, n_b, bs, bs))
    u = rng.standard_normal((ne, n_b - 1, bs, bs)) + 1j * rng.standard_normal((ne, n_b - 1, bs, bs))
    out = torch.zeros((lay.n_entries, tot), dtype=torch.complex128, device=cuda)
    lay.pack(t(d, cuda), t(u, cuda), out, 13)
    ref = orc.gather_entries(d, u)
    np.testing.assert_array_equal(out[:, 13:13 + ne].cpu().numpy(), ref)
    assert torch.count_nonzero(out[:, :13]).item() == 0
    vals = rng.standard_normal((lay.n_entries, tot)) + 1j * rng.standard_normal((lay.n_entries, tot))
    dd = torch.empty((ne, n_b, bs, bs), dtype=torch.complex128, device=cuda)
    uu = torch.empty((ne, n_b - 1, bs, bs), dtype=torch.complex128, device=cuda)
    ll = torch.empty_like(uu)
    lay.unpack_lg(t(vals, cuda), 5, ne, dd, uu)
    rd, ru = orc.scatter_lg(vals[:, 5:5 + ne], n_b, bs)
    np.testing.assert_array_equal(dd.cpu().numpy(), rd)
    np.testing.assert_array_equal(uu.cpu().numpy(), ru)
    lo = rng.standard_normal((lay.n_entries, tot)) + 1j * rng.standard_normal((lay.n_entries, tot))
    lay.unpack_retarded(t(vals, cuda), t(lo, cuda), 2, ne, dd, uu, ll)
    rd, ru, rl = orc.scatter_retarded(vals[:, 2:2 + ne], lo[:, 2:2 + ne], n_b, bs)
    np.testing.assert_array_equal(dd.cpu().numpy(), rd)
    np.testing.assert_array_equal(uu.cpu().numpy(), ru)
    np.testing.assert_array_equal(ll.cpu().numpy(), rl)


@pytest.mark.parametrize("n_b,bs,ne", [(4, 6, 5), (6, 40, 3), (3, 80, 2)])
def test_screened_solve_matches_oracle(cuda, n_b, bs, ne):
    rng = np.random.default_rng(n_b * bs)
    v = orc.coulomb_matrix(n_b, bs)
    mk = lambda *s: 0.3 * (rng.standard_normal(s) + 1j * rng.standard_normal(s))
    pr = (mk(ne, n_b, bs, bs) - 1j * np.eye(bs), mk(ne, n_b - 1, bs, bs), mk(ne, n_b - 1, bs, bs))
    def lg():
        d = mk(ne, n_b, bs, bs)
        return 0.5 * (d - np.conj(np.swapaxes(d, -1, -2))), mk(ne, n_b - 1, bs, bs)
    pl, pg = lg(), lg()
    mw, srcs = orc.w_system(v, pr, pl, pg)
    orc.w_closure(mw, srcs, 1e-8)
    ref = orc.rgf_selected(*mw, srcs, symmetrize=True)
    solver = ScreenedSolver(v, ScbaOptions(retarded_method="sancho"), cuda)
    b = solver.buffers(ne)
    for k, a in (("pr_diag", pr[0]), ("pr_upper", pr[1]), ("pr_lower", pr[2]), ("pl_diag", pl[0]),
                 ("pl_upper", pl[1]), ("pg_diag", pg[0]), ("pg_upper", pg[1])):
        b[k].copy_(t(a, cuda))
    b = solver.solve(ne)
    for k, rk in (("wr_diag", "xr_diag"), ("wr_upper", "xr_upper"), ("wl_diag", "x<_diag"),
                  ("wl_upper", "x<_upper"), ("wg_diag", "x>_diag"), ("wg_upper", "x>_upper")):
        assert rel(b[k].cpu().numpy(), ref[rk]) < TOL, k


@pytest.mark.parametrize("complex_v,bs", [(False, 24), (False, 23), (True, 24)])
def test_w_assembly_real_v_path(cuda, complex_v, bs):
    """A real V (ScreenedSolver.v_real) takes the real x complex kernel from a
    double copy of V (even block sizes) or the 2-product Gauss path (odd),
    and a Hermitian V forms the anti-Hermitian diagonal sources on half the
    tiles (v_herm): equal to the general full 3-product path to roundoff; a
    complex non-Hermitian V is detected; all match the oracle's W system.
    P^<> are anti-Hermitian like every lg-compressed quantity of the solver."""
    rng = np.random.default_rng(3)
    n_b, ne = 5, 3
    v = orc.coulomb_matrix(n_b, bs)
    if complex_v:
        v = tuple(x + 1e-4j * rng.standard_normal(x.shape) for x in v)
    mk = lambda *s: 0.3 * (rng.standard_normal(s) + 1j * rng.standard_normal(s))
    ah = lambda x: 0.5 * (x - np.conj(np.swapaxes(x, -1, -2)))
    pr = (mk(ne, n_b, bs, bs) - 1j * np.eye(bs), mk(ne, n_b - 1, bs, bs), mk(ne, n_b - 1, bs, bs))
    pl = (ah(mk(ne, n_b, bs, bs)), mk(ne, n_b - 1, bs, bs))
    pg = (ah(mk(ne, n_b, bs, bs)), mk(ne, n_b - 1, bs, bs))
    outs = []
    for force_complex in (False, True):
        solver = ScreenedSolver(v, ScbaOptions(retarded_method="sancho"), cuda)
        assert solver.v_real == (not complex_v) and solver.v_herm == (not complex_v)
        if force_complex:
            solver.v_real = solver.v_herm = False
        b = solver.buffers(ne)
        for k, a in (("pr_diag", pr[0]), ("pr_upper", pr[1]), ("pr_lower", pr[2]), ("pl_diag", pl[0]),
                     ("pl_upper", pl[1]), ("pg_diag", pg[0]), ("pg_upper", pg[1])):
            b[k].copy_(t(a, cuda))
        solver._assemble(b, ne)
        outs.append({k: b[k].cpu().numpy() for k in ("m_diag", "m_upper", "m_lower", "bl_diag", "bl_upper",
                                                       "bg_diag", "bg_upper")})
    for k in outs[0]:
        assert rel(outs[0][k], outs[1][k]) < 1e-14, k
    mw, srcs = orc.w_system(v, pr, pl, pg)
    for k, ref in (("m_diag", mw[0]), ("m_upper", mw[1]), ("m_lower", mw[2]), ("bl_diag", srcs["<"][0]),
                   ("bl_upper", srcs["<"][1]), ("bg_diag", srcs[">"][0]), ("bg_upper", srcs[">"][1])):
        assert rel(outs[0][k], ref) < 1e-12, k


def test_scba_small_matches_reference_scba_run(golden, cuda):
    """3 GW iterations, 6x4 chain + Coulomb, 32 energies (batches of 10)."""
    g = golden("golden_scba_small.npz")
    res = scba_run(orc.chain_device(6, 4), orc.coulomb_matrix(6, 4), np.linspace(-2.0, 2.0, 32), 1e-3,
                   Contacts(0.1, -0.1, 0.05), ScbaOptions(retarded_method="sancho", max_iter=3, tol=1e-12, batch=10, memoizer=MEMO_OFF), device=cuda)
    for k in g.files:
        if k.startswith(("ver_", "config")):
            continue
        assert rel(res[k], g[k]) < TOL, k


def test_scba_c1_matches_reference_scba_run(golden, cuda):
    """C1: 16 blocks x 32 orbitals, 128 energies, one GW iteration."""
    g = golden("golden_scba_c1.npz")
    res = scba_run(orc.chain_device(16, 32), orc.coulomb_matrix(16, 32), np.linspace(-2.0, 2.0, 128), 1e-3,
                   Contacts(0.1, -0.1, 0.05), ScbaOptions(retarded_method="sancho", max_iter=1, tol=1e-12, batch=64, memoizer=MEMO_OFF), device=cuda)
    check_c1(res, g, tol=TOL)


def test_scba_greater_identity_matches_reference(golden, cuda):
    """ScbaOptions.greater="identity" (G^> = G^< + G^R - G^R^dag instead of
    the greater recursion) still reproduces the reference's scba_run, which
    runs all three recursions: small (3 iterations) and C1."""
    g = golden("golden_scba_small.npz")
    res = scba_run(orc.chain_device(6, 4), orc.coulomb_matrix(6, 4), np.linspace(-2.0, 2.0, 32), 1e-3,
                   Contacts(0.1, -0.1, 0.05), ScbaOptions(retarded_method="sancho", max_iter=3, tol=1e-12, batch=10,
                                                          memoizer=MEMO_OFF, greater="identity"), device=cuda)
    for k in g.files:
        if k.startswith(("ver_", "config")):
            continue
        assert rel(res[k], g[k]) < TOL, k
    g = golden("golden_scba_c1.npz")
    res = scba_run(orc.chain_device(16, 32), orc.coulomb_matrix(16, 32), np.linspace(-2.0, 2.0, 128), 1e-3,
                   Contacts(0.1, -0.1, 0.05), ScbaOptions(retarded_method="sancho", max_iter=1, tol=1e-12, batch=64,
                                                          memoizer=MEMO_OFF, greater="identity"), device=cuda)
    check_c1(res, g, tol=TOL)


def test_scba_rgf_streams_matches_reference(golden, cuda):
    """ScbaOptions.rgf_streams=2 (energy slices of each batch on side streams
    for the G and W selected solves) reproduces the reference's scba_run."""
    g = golden("golden_scba_small.npz")
    res = scba_run(orc.chain_device(6, 4), orc.coulomb_matrix(6, 4), np.linspace(-2.0, 2.0, 32), 1e-3,
                   Contacts(0.1, -0.1, 0.05), ScbaOptions(retarded_method="sancho", max_iter=3, tol=1e-12, batch=10,
                                                          memoizer=MEMO_OFF, rgf_streams=2), device=cuda)
    for k in g.files:
        if k.startswith(("ver_", "config")):
            continue
        assert rel(res[k], g[k]) < TOL, k


def test_scba_c1_matches_oracle_two_iterations(cuda):
    """Second iteration (nonzero Sigma feeding the carrier assembly) vs the oracle."""
    h, v = orc.chain_device(16, 32), orc.coulomb_matrix(16, 32)
    e = np.linspace(-2.0, 2.0, 128)
    ref = orc.scba(h, v, e, 1e-3, 0.1, -0.1, 0.05, max_iter=2)
    res = scba_run(h, v, e, 1e-3, Contacts(0.1, -0.1, 0.05), ScbaOptions(retarded_method="sancho", max_iter=2, tol=1e-12, memoizer=MEMO_OFF), device=cuda)
    for k in ref:
        if k != "cache_stats_by_iteration":
            assert rel(res[k], ref[k]) < TOL, k


def test_scba_reference_api_with_blockmatrix_inputs(golden, cuda):
    """scba.py:865 call shape: BlockMatrix H/V, EnergyGrid, ContactConfig-like."""
    from paper_2508_19138_b200 import BlockMatrix
    from paper_2508_19138_b200.scba import EnergyGrid, scba_run_reference_api
    from types import SimpleNamespace

    def bm(stacks):
        d, u, l = stacks
        m = BlockMatrix(d.shape[0], d.shape[-1])
        for i in range(d.shape[0]):
            m.set_block(i, i, d[i])
            if i + 1 < d.shape[0]:
                m.set_block(i, i + 1, u[i])
                m.set_block(i + 1, i, l[i])
        return m

    g = golden("golden_scba_small.npz")
    res = scba_run_reference_api(bm(orc.chain_device(6, 4)), bm(orc.coulomb_matrix(6, 4)), EnergyGrid(-2.0, 2.0, 32),
                                 SimpleNamespace(mu_left=0.1, mu_right=-0.1, kT=0.05),
                                 ScbaOptions(retarded_method="sancho", max_iter=3, tol=1e-12, memoizer=MEMO_OFF), device=cuda)
    for k in ("g_r_diag", "g_lesser_upper", "sigma_lesser", "sigma_ret_lower", "residuals"):
        assert rel(res[k], g[k]) < TOL, k


def test_scba_with_beyn_w_surface_matches_reference(golden, cuda):
    """W retarded surface by Beyn, as the reference hard-codes (scba.py:844)."""
    g = golden("golden_scba_small.npz")
    res = scba_run(orc.chain_device(6, 4), orc.coulomb_matrix(6, 4), np.linspace(-2.0, 2.0, 32), 1e-3,
                   Contacts(0.1, -0.1, 0.05), ScbaOptions(retarded_method="sancho", max_iter=3, tol=1e-12, batch=16, memoizer=MEMO_OFF,
                                                          w_retarded_method="beyn"), device=cuda)
    for k in g.files:
        if k.startswith(("ver_", "config")):
            continue
        assert rel(res[k], g[k]) < TOL, k


@pytest.mark.parametrize("method", ["beyn", "fixed_point"])
def test_scba_carrier_retarded_methods_match_reference(golden, cuda, method):
    """retarded_method (scba.py:577-614): the reference default "beyn" and
    "fixed_point" for the carrier contacts (W by Beyn like the reference)."""
    g = golden(f"golden_scba_{method}.npz")
    res = scba_run(orc.chain_device(6, 4), orc.coulomb_matrix(6, 4), np.linspace(-2.0, 2.0, 32), 1e-3,
                   Contacts(0.1, -0.1, 0.05), ScbaOptions(max_iter=2, tol=1e-12, batch=16, memoizer=MEMO_OFF,
                                                          retarded_method=method, w_retarded_method="beyn"),
                   device=cuda)
    for k in g.files:
        if k.startswith(("ver_", "config")):
            continue
        assert rel(res[k], g[k]) < TOL, k


def _np_g_defect(xr_d, xr_u, xr_l, xl_d, xl_u, xg_d, xg_u):
    """scba.py:1223-1238 restated over stacked (n_e, n_b, bs, bs) arrays."""
    h = lambda a: np.conj(np.swapaxes(a, -1, -2))
    gam_d, gam_u = xr_d - h(xr_d), xr_u - h(xr_l)
    d = max(np.max(np.abs((xg_d - xl_d) - gam_d)), np.max(np.abs((xg_u - xl_u) - gam_u)) if xr_u.size else 0.0)
    s = max(np.max(np.abs(gam_d)), np.max(np.abs(gam_u)) if xr_u.size else 0.0)
    return d, s


@pytest.mark.parametrize("n_e,n_b,bs", [(3, 4, 7), (2, 3, 40), (1, 1, 33)])
def test_identity_defect_kernels_match_numpy(cuda, n_e, n_b, bs):
    from paper_2508_19138_b200.scba import entry_identity_defect, g_identity_defect

    rng = np.random.default_rng(n_b * bs)
    z = lambda *s: rng.standard_normal(s) + 1j * rng.standard_normal(s)
    a = dict(xr_diag=z(n_e, n_b, bs, bs), xr_upper=z(n_e, n_b - 1, bs, bs), xr_lower=z(n_e, n_b - 1, bs, bs),
             xl_diag=z(n_e, n_b, bs, bs), xl_upper=z(n_e, n_b - 1, bs, bs), xg_diag=z(n_e, n_b, bs, bs),
             xg_upper=z(n_e, n_b - 1, bs, bs))
    out = torch.zeros(2, dtype=torch.float64, device=cuda)
    g_identity_defect({k: t(v, cuda) for k, v in a.items()}, n_e, n_b, bs, out)
    d, s = _np_g_defect(*a.values())
    np.testing.assert_allclose(out.cpu().numpy(), [d, s], rtol=1e-14)
    ser = [z(57, 13) for _ in range(4)]
    out.zero_()
    entry_identity_defect(*(t(x, cuda) for x in ser), out)
    gam = ser[2] - np.conj(ser[3])
    ref = [np.max(np.abs((ser[1] - ser[0]) - gam)), np.max(np.abs(gam))]
    np.testing.assert_allclose(out.cpu().numpy(), ref, rtol=1e-14)


def test_scba_identity_defects_and_result_fields(golden, cuda):
    """ScbaResult.identity_defects (scba.py:1155-1166): one {"G","P","Sigma"}
    record per iteration at roundoff level (the reference's own run of this
    case gives 1e-16..1e-15), the G entry equal to the defect of the returned
    last-iteration G; converged / n_iter and attribute access as ScbaResult."""
    g = golden("golden_scba_small.npz")
    res = scba_run(orc.chain_device(6, 4), orc.coulomb_matrix(6, 4), np.linspace(-2.0, 2.0, 32), 1e-3,
                   Contacts(0.1, -0.1, 0.05), ScbaOptions(retarded_method="sancho", max_iter=3, tol=1e-12, batch=10, memoizer=MEMO_OFF), device=cuda)
    assert len(res.identity_defects) == 3 and res.n_iter == 3 and res.converged is False
    for d in res.identity_defects:
        assert set(d) == {"G", "P", "Sigma"} and max(d.values()) < 1e-12
    dg, sg = _np_g_defect(res.g_r_diag, res.g_r_upper, res.g_r_lower, res.g_lesser_diag, res.g_lesser_upper,
                          res.g_greater_diag, res.g_greater_upper)
    assert abs(res.identity_defects[-1]["G"] - dg / sg) <= 1e-6 * dg / sg + 1e-300
    assert rel(res.residuals, g["residuals"]) < TOL
    ball = scba_run(orc.chain_device(5, 3), None, np.linspace(-2.0, 2.0, 16), 1e-3, Contacts(0.1, -0.1, 0.05),
                    device=cuda)
    assert ball.converged and ball.n_iter == 1 and list(ball.identity_defects[0]) == ["G"]
    assert ball.identity_defects[0]["G"] < 1e-12


def test_scba_warm_start_reset_sigma(cuda):
    """scba.py:943-949: initial_sigma is ignored unless reset_sigma=False; a
    converged state fed back converges at once; a wrong shape is a ValueError."""
    h, v, e = orc.chain_device(6, 4), orc.coulomb_matrix(6, 4), np.linspace(-2.0, 2.0, 32)
    c = Contacts(0.1, -0.1, 0.05)
    first = scba_run(h, v, e, 1e-3, c, ScbaOptions(retarded_method="sancho", max_iter=80, tol=1e-8, memoizer=MEMO_OFF), device=cuda)
    assert first.converged
    cold = scba_run(h, v, e, 1e-3, c, ScbaOptions(retarded_method="sancho", max_iter=2, tol=1e-8, memoizer=MEMO_OFF), device=cuda,
                    initial_sigma=first.state)
    assert rel(cold.residuals, first.residuals[:2]) < TOL  # reset_sigma=True: cold start
    warm = scba_run(h, v, e, 1e-3, c, ScbaOptions(retarded_method="sancho", max_iter=80, tol=1e-8, memoizer=MEMO_OFF, reset_sigma=False),
                    device=cuda, initial_sigma=first.state)
    assert warm.converged and warm.n_iter <= 2
    from paper_2508_19138_b200.scba import ScbaState

    bad = ScbaState.zeros(7, 32, cuda)
    with pytest.raises(ValueError, match="warm-start"):
        scba_run(h, v, e, 1e-3, c, ScbaOptions(retarded_method="sancho", max_iter=2, reset_sigma=False, memoizer=MEMO_OFF), device=cuda,
                 initial_sigma=bad)


def test_scba_oracle_mode_deviations(golden, cuda):
    """ScbaOptions.oracle_mode (scba.py:913-915): every G and W selected solve
    against a dense inverse + triple product and every P / Sigma convolution
    against the direct sum, reported like the reference's oracle_deviations;
    results unchanged."""
    g = golden("golden_scba_small.npz")
    res = scba_run(orc.chain_device(6, 4), orc.coulomb_matrix(6, 4), np.linspace(-2.0, 2.0, 32), 1e-3,
                   Contacts(0.1, -0.1, 0.05), ScbaOptions(retarded_method="sancho", max_iter=3, tol=1e-12, batch=10, memoizer=MEMO_OFF,
                                                          oracle_mode=True), device=cuda)
    od = res.oracle_deviations
    assert set(od) == {"solve_vs_dense", "fft_vs_direct"}
    assert 0 < od["solve_vs_dense"] < 1e-10 and 0 < od["fft_vs_direct"] < 1e-10, od
    assert rel(res["sigma_lesser"], g["sigma_lesser"]) < TOL
    plain = scba_run(orc.chain_device(6, 4), orc.coulomb_matrix(6, 4), np.linspace(-2.0, 2.0, 32), 1e-3,
                     Contacts(0.1, -0.1, 0.05), ScbaOptions(retarded_method="sancho", max_iter=1, memoizer=MEMO_OFF), device=cuda)
    assert plain.oracle_deviations == {}


def test_scba_spatial_plan_preconditions(cuda):
    """scba.py:890-892 / dist.py:767-778: oracle_mode is sequential only; the
    plan must cover the chain and have one partition per rank."""
    from paper_2508_19138_b200.dd import PartitionError, make_partition_plan

    args = (orc.chain_device(6, 4), orc.coulomb_matrix(6, 4), np.linspace(-2.0, 2.0, 8), 1e-3,
            Contacts(0.1, -0.1, 0.05))
    with pytest.raises(ValueError, match="oracle_mode"):
        scba_run(*args, ScbaOptions(retarded_method="sancho", max_iter=1, oracle_mode=True), device=cuda, plan=make_partition_plan(6, 2))
    with pytest.raises(PartitionError, match="partitions"):
        scba_run(*args, ScbaOptions(retarded_method="sancho", max_iter=1), device=cuda, plan=make_partition_plan(6, 2))
    with pytest.raises(PartitionError, match="covers"):
        scba_run(*args, ScbaOptions(retarded_method="sancho", max_iter=1), device=cuda, plan=make_partition_plan(8, 2))


def test_scba_result_is_reference_shaped(golden, cuda):
    """ScbaResult carries the reference's fields (scba.py:492-528): grid,
    contacts, options, sigma: SigmaState, sigma_pattern, transposition
    counted like _count_bytes; the device-reduced observables equal the
    reference observables evaluated on the returned G blocks; a host
    SigmaState (the reference's warm-start type) warm-starts a run."""
    from paper_2508_19138_b200.results import (ScbaResult, SigmaState, current_spectrum, dos, electron_density,
                                               terminal_current)

    g = golden("golden_scba_small.npz")
    h, v, e = orc.chain_device(6, 4), orc.coulomb_matrix(6, 4), np.linspace(-2.0, 2.0, 32)
    opts = ScbaOptions(retarded_method="sancho", max_iter=3, tol=1e-12, memoizer=MEMO_OFF)
    res = scba_run(h, v, e, 1e-3, Contacts(0.1, -0.1, 0.05), opts, device=cuda)
    assert isinstance(res, ScbaResult) and isinstance(res.sigma, SigmaState)
    assert res.grid.n_e == 32 and abs(res.grid.de - 4.0 / 31) < 1e-15 and res.options is opts
    assert res.sigma_pattern.n_entries == res.sigma.lesser.shape[0] == res.sigma_pattern.rows.size
    assert rel(res.sigma.lesser, g["sigma_lesser"]) < TOL and rel(res["sigma_ret_upper"], g["sigma_ret_upper"]) < TOL
    n_ent, full = res.sigma_pattern.n_entries, res.sigma_pattern.full_entry_count()
    assert res.transposition.lg_bytes == 3 * 8 * n_ent * 32 * 16
    assert res.transposition.lg_full_bytes == 3 * 8 * full * 32 * 16
    assert res.transposition.other_bytes == 3 * 4 * n_ent * 32 * 16
    obs = res.observables
    assert rel(obs["dos"], dos(res)) < 1e-12
    assert rel(obs["density"], electron_density(res)) < 1e-12
    assert rel(obs["current_spectrum"], current_spectrum(res, h)) < 1e-12
    for side in ("left", "right"):
        assert abs(obs["terminal_" + side] - terminal_current(res, side)) < 1e-12 * max(1.0, abs(obs["terminal_" + side]))
    warm = scba_run(h, v, e, 1e-3, Contacts(0.1, -0.1, 0.05),
                    ScbaOptions(retarded_method="sancho", max_iter=1, tol=1e-12, memoizer=MEMO_OFF, reset_sigma=False),
                    device=cuda, initial_sigma=res.sigma.copy())
    # the warm run's G solve sees the returned Sigma: its first residual is the
    # 4th iteration's of a cold 4-iteration run
    cold = scba_run(h, v, e, 1e-3, Contacts(0.1, -0.1, 0.05),
                    ScbaOptions(retarded_method="sancho", max_iter=4, tol=1e-12, memoizer=MEMO_OFF), device=cuda)
    assert abs(warm.residuals[0] - cold.residuals[3]) < 1e-9 * cold.residuals[3]


def test_scba_coarse_w_grid_matches_reference(golden, cuda):
    """bs_w = 2 bs (scba.py:893-903, 925-937): P scattered from the G pattern
    into the W blocks and W read back at G-pattern coordinates through the
    table-driven layout kernels; vs the reference's scba_run."""
    g = golden("golden_scba_coarse_w.npz")
    res = scba_run(orc.chain_device(8, 4), orc.coulomb_matrix(4, 8), np.linspace(-2.0, 2.0, 32), 1e-3,
                   Contacts(0.1, -0.1, 0.05),
                   ScbaOptions(retarded_method="sancho", max_iter=3, tol=1e-12, batch=12, memoizer=MEMO_OFF),
                   device=cuda)
    for k in g.files:
        if k.startswith(("ver_", "config")):
            continue
        assert rel(res[k], g[k]) < TOL, k


def test_scba_w_grid_preconditions(cuda):
    c = Contacts(0.1, -0.1, 0.05)
    e = np.linspace(-1.0, 1.0, 8)
    with pytest.raises(ValueError, match="does not match carrier layout"):
        scba_run(orc.chain_device(8, 4), orc.coulomb_matrix(3, 8), e, 1e-3, c, ScbaOptions(retarded_method="sancho"),
                 device=cuda)
    with pytest.raises(ValueError, match="multiple of the carrier block"):
        scba_run(orc.chain_device(8, 4), orc.coulomb_matrix(16, 2), e, 1e-3, c, ScbaOptions(retarded_method="sancho"),
                 device=cuda)


@pytest.mark.parametrize("case", ["small", "c1"])
def test_scba_entry_cutoff_infinite_equals_reference(golden, cuda, case):
    """r_cut = infinity equivalence: the table-driven entry layout with a
    cutoff larger than any |row - col| reproduces the reference's full-band
    scba_run."""
    if case == "small":
        g = golden("golden_scba_small.npz")
        res = scba_run(orc.chain_device(6, 4), orc.coulomb_matrix(6, 4), np.linspace(-2.0, 2.0, 32), 1e-3,
                       Contacts(0.1, -0.1, 0.05),
                       ScbaOptions(retarded_method="sancho", max_iter=3, tol=1e-12, memoizer=MEMO_OFF,
                                   entry_cutoff=10 ** 6), device=cuda)
        for k in ("g_r_diag", "g_lesser_upper", "g_greater_diag", "sigma_lesser", "sigma_greater",
                  "sigma_ret_upper", "sigma_ret_lower", "residuals"):
            assert rel(res[k], g[k]) < TOL, k
    else:
        g = golden("golden_scba_c1.npz")
        res = scba_run(orc.chain_device(16, 32), orc.coulomb_matrix(16, 32), np.linspace(-2.0, 2.0, 128), 1e-3,
                       Contacts(0.1, -0.1, 0.05),
                       ScbaOptions(retarded_method="sancho", max_iter=1, tol=1e-12, batch=64, memoizer=MEMO_OFF,
                                   entry_cutoff=10 ** 6), device=cuda)
        check_c1(res, g, tol=TOL)


@pytest.mark.parametrize("cutoff,bs", [(5, 4), (0, 4), (40, 32)])
def test_scba_entry_cutoff_matches_oracle(cuda, cutoff, bs):
    """The paper's r_cut nonzero set (ScbaOptions.entry_cutoff, a documented
    deviation) against the oracle computing on the full band with the
    dropped entries zeroed after every gather."""
    nb = 6 if bs == 4 else 5
    h, v = orc.chain_device(nb, bs), orc.coulomb_matrix(nb, bs)
    e = np.linspace(-2.0, 2.0, 24)
    ref = orc.scba(h, v, e, 1e-3, 0.1, -0.1, 0.05, max_iter=3, entry_cutoff=cutoff)
    res = scba_run(h, v, e, 1e-3, Contacts(0.1, -0.1, 0.05),
                   ScbaOptions(retarded_method="sancho", max_iter=3, tol=1e-12, batch=7, memoizer=MEMO_OFF,
                               entry_cutoff=cutoff), device=cuda)
    rows, cols = orc.entry_pattern(nb, bs)
    keep = np.abs(rows - cols) <= cutoff
    assert res.sigma_pattern.n_entries == int(keep.sum())
    assert np.array_equal(res.sigma_pattern.rows, rows[keep])
    for k in ("g_r_diag", "g_r_upper", "g_lesser_diag", "g_lesser_upper", "g_greater_upper", "residuals"):
        assert rel(res[k], ref[k]) < TOL, k
    for k in ("lesser", "greater", "ret_upper", "ret_lower"):
        assert rel(res["sigma_" + k], ref["sigma_" + k][keep]) < TOL, k
        assert np.all(ref["sigma_" + k][~keep] == 0)
