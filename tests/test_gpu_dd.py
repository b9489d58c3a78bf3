"""Spatial domain decomposition (dist.py:750 dist_selected_solve) on the GPU
vs the reference's own distributed solve (goldens from spmd_run ranks), the
oracle restatement and the sequential solve."""

import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

import negf_oracle as orc
from paper_2508_19138_b200.dd import dd_selected_solve_local, dist_selected_solve, make_partition_plan
from test_oracle_golden import rel

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
TOL = 1e-9
KEYS = (("xr_diag", "xr_diag"), ("xr_upper", "xr_upper"), ("xr_lower", "xr_lower"), ("xl_diag", "xl_diag"),
        ("xl_upper", "xl_upper"), ("xg_diag", "xg_diag"), ("xg_upper", "xg_upper"))


def t(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


@pytest.mark.parametrize("c", range(5))
def test_dd_matches_reference_dist_selected_solve(golden, cuda, c):
    g = golden("golden_dd.npz")
    p = f"c{c}_"
    seed, nb, bs, p_s = (int(x) for x in g[p + "cfg"])
    plan = make_partition_plan(nb, p_s)
    assert [list(r) for r in plan.ranges] == g[p + "ranges"].tolist()
    md, mu, ml = (t(g[p + k][None], cuda) for k in ("m_diag", "m_upper", "m_lower"))
    src = {"<": (t(g[p + "bl_diag"][None], cuda), t(g[p + "bl_upper"][None], cuda)),
           ">": (t(g[p + "bg_diag"][None], cuda), t(g[p + "bg_upper"][None], cuda))}
    out = dd_selected_solve_local(md, mu, ml, src, plan)
    for mine, ref in KEYS:
        assert rel(out[mine][0].cpu().numpy(), g[p + ref]) < TOL, mine


@pytest.mark.parametrize("nb,bs,p_s", [(9, 40, 3), (16, 72, 4), (11, 65, 5), (8, 96, 2)])
def test_dd_batched_matches_oracle_and_sequential(cuda, nb, bs, p_s):
    ne = 3
    sys_ = [orc.random_bt_system(200 + e, n_blocks=nb, block_size=bs) for e in range(ne)]
    md, mu, ml = (np.concatenate([s[i] for s in sys_]) for i in range(3))
    src = {k: tuple(np.concatenate([s[3][k][i] for s in sys_]) for i in range(2)) for k in ("<", ">")}
    plan = make_partition_plan(nb, p_s)
    ref = orc.dd_selected(md, mu, ml, src, [tuple(r) for r in plan.ranges])
    seq = orc.rgf_selected(md, mu, ml, src)
    out = dd_selected_solve_local(t(md, cuda), t(mu, cuda), t(ml, cuda),
                                  {k: (t(d, cuda), t(u, cuda)) for k, (d, u) in src.items()}, plan)
    for mine, rk in (("xr_diag", "xr_diag"), ("xr_upper", "xr_upper"), ("xr_lower", "xr_lower"),
                     ("xl_diag", "x<_diag"), ("xl_upper", "x<_upper"), ("xg_diag", "x>_diag"),
                     ("xg_upper", "x>_upper")):
        got = out[mine].cpu().numpy()
        assert rel(got, ref[rk]) < TOL, mine
        assert rel(got, seq[rk]) < TOL, mine


def test_dd_symmetrize_and_reference_signature(golden, cuda):
    """dist_selected_solve with BlockMatrix inputs returns the full solution."""
    from paper_2508_19138_b200 import BlockMatrix
    from paper_2508_19138_b200.blocks import LG_COMPRESSED

    g = golden("golden_dd.npz")
    p = "c2_"
    nb, bs, p_s = (int(x) for x in g[p + "cfg"][1:])
    m = BlockMatrix(nb, bs)
    bl, bg = BlockMatrix(nb, bs, storage_mode=LG_COMPRESSED), BlockMatrix(nb, bs, storage_mode=LG_COMPRESSED)
    for i in range(nb):
        m.set_block(i, i, g[p + "m_diag"][i])
        bl.set_block(i, i, g[p + "bl_diag"][i])
        bg.set_block(i, i, g[p + "bg_diag"][i])
        if i + 1 < nb:
            m.set_block(i, i + 1, g[p + "m_upper"][i])
            m.set_block(i + 1, i, g[p + "m_lower"][i])
            bl.set_block(i, i + 1, g[p + "bl_upper"][i])
            bg.set_block(i, i + 1, g[p + "bg_upper"][i])
    sol, stats = dist_selected_solve(m, bl, bg, plan=make_partition_plan(nb, p_s), device=cuda)
    assert rel(np.stack(sol.x_r_diag), g[p + "xr_diag"]) < TOL
    assert rel(np.stack(sol.x_lg_upper[">"]), g[p + "xg_upper"]) < TOL


def test_dd_over_nccl_ranks(cuda):
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs (one partition per GPU)")
    for world in sorted({2, min(n, 4)}):
        out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--standalone", "--nproc-per-node",
                              str(world), str(ROOT / "tools" / "dd_check.py")],
                             capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
        assert "DD_CHECK" in out.stdout


def test_dd_balanced_plan_gives_the_same_solution(cuda):
    from paper_2508_19138_b200.dd import balanced_partition_plan

    nb, bs, ne = 20, 48, 2
    sys_ = [orc.random_bt_system(300 + e, n_blocks=nb, block_size=bs) for e in range(ne)]
    md, mu, ml = (np.concatenate([s[i] for s in sys_]) for i in range(3))
    src = {k: tuple(np.concatenate([s[3][k][i] for s in sys_]) for i in range(2)) for k in ("<", ">")}
    seq = orc.rgf_selected(md, mu, ml, src)
    for p_s in (3, 4, 5):
        plan = balanced_partition_plan(nb, p_s)
        assert plan.ranges[0][1] - plan.ranges[0][0] > plan.ranges[1][1] - plan.ranges[1][0]
        out = dd_selected_solve_local(t(md, cuda), t(mu, cuda), t(ml, cuda),
                                      {k: (t(d, cuda), t(u, cuda)) for k, (d, u) in src.items()}, plan)
        for mine, rk in (("xr_diag", "xr_diag"), ("xl_upper", "x<_upper"), ("xg_diag", "x>_diag")):
            assert rel(out[mine].cpu().numpy(), seq[rk]) < TOL, (p_s, mine)
