"""Spatial DD selected solve over N ranks (torchrun, one GPU per partition)
vs the reference's dist_selected_solve goldens and vs the oracle at a larger
batched size. Usage: torchrun --standalone --nproc-per-node N tools/dd_check.py"""
import os, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "oracle"))
import numpy as np, torch, torch.distributed as dist
import negf_oracle as orc
from paper_2508_19138_b200.dd import (assemble, dd_selected_solve_batched, make_partition_plan,
                                      partition_inputs)

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
rank, size = dist.get_rank(), dist.get_world_size()
rel = lambda a, b: np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
KEYS = (("xr_diag", "xr_diag"), ("xr_upper", "xr_upper"), ("xr_lower", "xr_lower"), ("xl_diag", "x<_diag"),
        ("xl_upper", "x<_upper"), ("xg_diag", "x>_diag"), ("xg_upper", "x>_upper"))
worst = 0.0


def run(md, mu, ml, src, plan):
    part = partition_inputs(md, mu, ml, src, plan, rank)
    loc, cr = dd_selected_solve_batched(part, plan)
    objs = [None] * size
    dist.all_gather_object(objs, ({k: v.cpu() for k, v in loc.items()},
                                  None if cr is None else {k: v.cpu() for k, v in cr.items()}))
    return assemble([o[0] for o in objs], [o[1] for o in objs], plan, list(src))


g = np.load(ROOT / "tests" / "golden" / "golden_dd.npz")
for c in range(int(g["n_cases"])):
    p = f"c{c}_"
    seed, nb, bs, p_s = (int(x) for x in g[p + "cfg"])
    if p_s != size:
        continue
    plan = make_partition_plan(nb, p_s)
    md, mu, ml = (T(g[p + k][None]) for k in ("m_diag", "m_upper", "m_lower"))
    src = {"<": (T(g[p + "bl_diag"][None]), T(g[p + "bl_upper"][None])),
           ">": (T(g[p + "bg_diag"][None]), T(g[p + "bg_upper"][None]))}
    full = run(md, mu, ml, src, plan)
    for mine, ref in KEYS:
        worst = max(worst, rel(full[mine][0].numpy(), g[p + ref.replace("x<", "xl").replace("x>", "xg")]))
# larger batched case vs the oracle's partition-by-partition restatement
ne, nb, bs = 3, 4 * size + 1, 48
sys_ = [orc.random_bt_system(100 + e, n_blocks=nb, block_size=bs) for e in range(ne)]
md, mu, ml = (np.concatenate([s[i] for s in sys_]) for i in range(3))
src_np = {k: tuple(np.concatenate([s[3][k][i] for s in sys_]) for i in range(2)) for k in ("<", ">")}
plan = make_partition_plan(nb, size)
ref = orc.dd_selected(md, mu, ml, src_np, [tuple(r) for r in plan.ranges])
full = run(T(md), T(mu), T(ml), {k: (T(d), T(u)) for k, (d, u) in src_np.items()}, plan)
for mine, rk in KEYS:
    worst = max(worst, rel(full[mine].numpy(), ref[rk]))
t = torch.tensor([worst], dtype=torch.float64, device=dev)
dist.all_reduce(t, op=dist.ReduceOp.MAX)
if rank == 0:
    print(f"DD_CHECK world={size} worst_rel={t.item():.3e}")
    assert t.item() < 1e-9
dist.destroy_process_group()
