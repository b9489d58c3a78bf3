"""Parity at the BENCHMARKED / BASELINE shapes (VERDICT r1 "pin parity at the
benchmarked shapes"): the GPU path against fixtures produced by running the
reference's own scba_run (tests/golden/make_golden_large.py) and against the
oracle restatement.

* C2 (BASELINE configs[1], the bench workload): chain_device(64, 256),
  ballistic, 4 energies over [-2, 2] eV, G^> by its own recursion (the
  reference algorithm) and by the identity (the bench's fast option).
* C3 (configs[2] device): chain_device(64, 512) + coulomb_matrix, full GW
  scba_run, 2 energies (-0.5, 0.5 eV), 2 iterations, Sancho, memoizer off.

Full arrays at these shapes are GBs, so the fixtures hold per-(energy, block)
weighted sums and norms plus 4096 sampled elements per field; all are
compared at the 1e-9 relative bar of north_star.
"""

import numpy as np
import pytest

import negf_oracle as orc
from paper_2508_19138_b200.carrier import Contacts, ballistic_observables, ballistic_run

pytestmark = pytest.mark.gpu
TOL = 1e-9


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def block_weights(bs, seed=1234):
    return np.random.default_rng(seed).standard_normal((bs, bs))


def check_field(got, g, name):
    got = np.asarray(got)
    w = block_weights(got.shape[-1])
    assert rel(np.einsum("...ij,ij->...", got, w), g[name + "_blk"]) < TOL, name + " block checksums"
    assert rel(np.linalg.norm(got, axis=(-2, -1)), g[name + "_nrm"]) < TOL, name + " block norms"
    assert rel(got.reshape(-1)[g[name + "_idx"]], g[name + "_val"]) < TOL, name + " sampled elements"


FIELDS = ["g_r_diag", "g_r_upper", "g_r_lower", "g_lesser_diag", "g_lesser_upper", "g_greater_diag",
          "g_greater_upper", "sigma_obc_lesser_left", "sigma_obc_greater_left", "sigma_obc_lesser_right",
          "sigma_obc_greater_right"]


@pytest.mark.parametrize("greater", ["recursion", "identity"])
def test_c2_ballistic_matches_reference(golden, cuda, greater):
    g = golden("golden_c2_ballistic.npz")
    nb, bs, ne, _ = (int(x) for x in g["config"])
    h = orc.chain_device(nb, bs)
    out = ballistic_run(h, np.linspace(-2.0, 2.0, ne), 1e-3, Contacts(0.1, -0.1, 0.05), 1e-8, batch=ne,
                        device=cuda, greater=greater)
    for f in FIELDS:
        check_field(out[f], g, f)


def test_c2_observables_match_reference(golden, cuda):
    """The bench's e2e API (ballistic_observables) at the C2 shape."""
    g = golden("golden_c2_ballistic.npz")
    nb, bs, ne, _ = (int(x) for x in g["config"])
    obs = ballistic_observables(orc.chain_device(nb, bs), np.linspace(-2.0, 2.0, ne), 1e-3,
                                Contacts(0.1, -0.1, 0.05), 1e-8, batch=ne, device=cuda, greater="identity")
    assert rel(obs["dos"], g["obs_dos"]) < TOL
    assert rel(obs["density"], g["obs_density"]) < TOL
    # Currents are differences of O(|H| |G^<|) terms: in the transport window
    # f_L - f_R ~ 1e-5 while G^< ~ f A is O(1), so both codes carry roundoff of
    # ~eps * |H_up| |G^<_up| per bond (1e-9 relative to the 7e-5 current; at
    # E = +-2 eV the exact current vanishes and both return 1e-13 noise).
    # The bar is therefore 1e-9 relative to that uncancelled scale, per
    # (energy, bond) -- the conditioning of the observable itself.
    h = orc.chain_device(nb, bs)
    hu = np.linalg.norm(h[1], axis=(-2, -1))  # (nb-1,)
    cscale = 2.0 / (2.0 * np.pi) * hu[None, :] * g["g_lesser_upper_nrm"]
    err = np.abs(obs["current_spectrum"] - g["obs_current_spectrum"])
    assert np.all(err <= TOL * cscale), float(np.max(err / cscale))
    de = 4.0 / (ne - 1)
    for side, c in (("left", 0), ("right", nb - 1)):
        tscale = de / (2.0 * np.pi) * np.sum(g[f"sigma_obc_lesser_{side}_nrm"] * g["g_greater_diag_nrm"][:, c]
                                             + g[f"sigma_obc_greater_{side}_nrm"] * g["g_lesser_diag_nrm"][:, c])
        assert abs(obs["terminal_" + side] - float(g["obs_terminal_" + side])) < TOL * tscale


def test_c2_shape_matches_oracle_both_recursions(cuda):
    """Same shape against the oracle restatement at two other energies
    (in-band, |E| < 1), both Keldysh kinds by recursion."""
    h = orc.chain_device(64, 256)
    e = np.array([-0.35, 0.8])
    ref = orc.ballistic(h, e, 1e-3, 0.1, -0.1, 0.05, tol=1e-8)
    out = ballistic_run(h, e, 1e-3, Contacts(0.1, -0.1, 0.05), 1e-8, batch=2, device=cuda, greater="recursion")
    for k in FIELDS:
        assert rel(out[k], ref[k]) < TOL, k


def test_c3_gw_iteration_matches_reference(golden, cuda):
    from paper_2508_19138_b200.scba import MemoizerOptions, ScbaOptions, scba_run

    from pathlib import Path

    if not (Path(__file__).parent / "golden" / "golden_c3_gw.npz").exists():
        pytest.skip("golden_c3_gw.npz not generated yet (tests/golden/make_golden_large.py c3)")
    g = golden("golden_c3_gw.npz")
    nb, bs, ne, iters = (int(x) for x in g["config"])
    e_min, e_max = (float(x) for x in g["grid"])
    res = scba_run(orc.chain_device(nb, bs), orc.coulomb_matrix(nb, bs), np.linspace(e_min, e_max, ne), 1e-3,
                   Contacts(0.1, -0.1, 0.05),
                   ScbaOptions(retarded_method="sancho", max_iter=iters, tol=1e-12, batch=ne, memoizer=MemoizerOptions(enabled=False)),
                   device=cuda)
    for f in FIELDS:
        check_field(res[f], g, f)
    for k, f in enumerate(("lesser", "greater", "ret_upper", "ret_lower")):
        a = res["sigma_" + f]
        name = "sigma_" + f
        assert rel(a[g[name + "_rows"]], g[name + "_val"]) < TOL, name
        chk = a.T @ np.random.default_rng(300 + 2 * k + 1).standard_normal(a.shape[0])
        assert rel(chk, g[name + "_chk"]) < TOL, name
        assert abs(np.linalg.norm(a) - float(g[name + "_fro"])) < TOL * float(g[name + "_fro"])
    assert rel(res["residuals"], g["residuals"]) < 1e-8
