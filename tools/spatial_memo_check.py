"""Spatial scba_run (plan=, one partition per rank) with the OBC memoizer on
(the reference default) vs the sequential run on one GPU: Sigma of every
rank's energies and the per-iteration direct/memoized call counts (every
rank solves every energy in the spatial mode, so its counts equal the
sequential run's).
Usage: torchrun --standalone --nproc-per-node N tools/spatial_memo_check.py"""
import os, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "oracle"))
import numpy as np, torch, torch.distributed as dist
import negf_oracle as orc
from paper_2508_19138_b200.carrier import Contacts
from paper_2508_19138_b200.dd import make_partition_plan
from paper_2508_19138_b200.dist import Comm
from paper_2508_19138_b200.scba import MemoizerOptions, ScbaOptions, scba_run

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
comm = Comm.from_env()
args = (orc.chain_device(16, 32), orc.coulomb_matrix(16, 32), np.linspace(-2.0, 2.0, 64), 1e-3,
        Contacts(0.1, -0.1, 0.05), ScbaOptions(retarded_method="sancho", max_iter=4, tol=1e-12, batch=32, memoizer=MemoizerOptions(enabled=True)))
res = scba_run(*args, device=dev, comm=comm, plan=make_partition_plan(16, comm.size))
sig = {f: res["sigma_" + f] for f in ("lesser", "greater", "ret_upper", "ret_lower")}
parts = [None] * comm.size
dist.all_gather_object(parts, (res["energy_slice"].start, sig))
if comm.rank == 0:
    rel = lambda a, b: np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)
    parts.sort(key=lambda x: x[0])
    one = scba_run(*args, device=dev)
    w = max(rel(np.concatenate([p[1][f] for p in parts], axis=1), one["sigma_" + f]) for f in sig)
    w = max(w, rel(res["residuals"], one["residuals"]))
    same = res["cache_stats_by_iteration"] == one["cache_stats_by_iteration"]
    print(f"SPATIAL_MEMO world={comm.size} worst_rel_vs_1gpu={w:.3e} counts_equal={same} "
          f"counts={res['cache_stats_by_iteration']}")
    assert w < 1e-9 and same
dist.destroy_process_group()
