"""Energy-sharded SCBA at N ranks (torchrun, one GPU per rank) vs the C1
reference golden: every rank checks its own energies' per-energy checksums.
Usage: torchrun --standalone --nproc-per-node N tools/dist_check.py"""
import os, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "oracle"))
import numpy as np, torch, torch.distributed as dist
import negf_oracle as orc
from paper_2508_19138_b200.carrier import Contacts
from paper_2508_19138_b200.dist import Comm
from paper_2508_19138_b200.scba import MemoizerOptions, ScbaOptions, scba_run

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
comm = Comm.from_env()
g = np.load(ROOT / "tests" / "golden" / "golden_scba_c1.npz")
res = scba_run(orc.chain_device(16, 32), orc.coulomb_matrix(16, 32), np.linspace(-2.0, 2.0, 128), 1e-3,
               Contacts(0.1, -0.1, 0.05), ScbaOptions(max_iter=1, tol=1e-12, batch=40, memoizer=MemoizerOptions(enabled=False)), device=dev, comm=comm)
own = res["energy_slice"]
rel = lambda a, b: np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)
rng = np.random.default_rng(99)
worst = 0.0
for f in ["g_r_diag", "g_r_upper", "g_r_lower", "g_lesser_diag", "g_lesser_upper", "g_greater_diag",
          "g_greater_upper", "sigma_obc_lesser_left", "sigma_obc_greater_left", "sigma_obc_lesser_right",
          "sigma_obc_greater_right"]:
    a = res[f]
    w = rng.standard_normal(a.shape[1:])
    worst = max(worst, rel(np.tensordot(a, w, axes=a.ndim - 1), g[f + "_chk"][own]))
for f in ("lesser", "greater", "ret_upper", "ret_lower"):
    a = res["sigma_" + f]
    wv = rng.standard_normal(a.shape[0])
    worst = max(worst, rel(a.T @ wv, g["sigma_" + f + "_chk"][own]))
worst = max(worst, rel(res["residuals"], g["residuals"]))
t = torch.tensor([worst], dtype=torch.float64, device=dev)
dist.all_reduce(t, op=dist.ReduceOp.MAX)
if comm.rank == 0:
    print(f"DIST_CHECK world={comm.size} worst_rel={t.item():.3e} transpose_bytes_rank0={res['transpose_bytes']}")
dist.destroy_process_group()
sys.exit(0 if t.item() < 1e-9 else 1)
