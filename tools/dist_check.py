"""Energy-sharded SCBA at N ranks (torchrun, one GPU per rank) vs the C1
reference golden: the per-energy checksums of every rank's energies are
all-gathered and compared with the golden over the whole energy axis (the
same relative-Frobenius measure as the single-GPU test; a single rank's slice
can hold a near-zero quantity, e.g. Sigma^> far below the Fermi level).
NEGF_SPATIAL=1 runs the reference's spatial mode instead (scba_run with
plan = make_partition_plan(16, N): every energy solved jointly by all ranks,
dd.py), checked the same way.
Usage: torchrun --standalone --nproc-per-node N tools/dist_check.py"""
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
spatial = os.environ.get("NEGF_SPATIAL") == "1"
plan = make_partition_plan(16, comm.size) if spatial else None
g = np.load(ROOT / "tests" / "golden" / "golden_scba_c1.npz")
res = scba_run(orc.chain_device(16, 32), orc.coulomb_matrix(16, 32), np.linspace(-2.0, 2.0, 128), 1e-3,
               Contacts(0.1, -0.1, 0.05), ScbaOptions(retarded_method="sancho", max_iter=1, tol=1e-12, batch=40,
                                                      memoizer=MemoizerOptions(enabled=False)), device=dev, comm=comm,
               plan=plan)
own = res["energy_slice"]
rel = lambda a, b: np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)
rng = np.random.default_rng(99)
mine = {}
for f in ["g_r_diag", "g_r_upper", "g_r_lower", "g_lesser_diag", "g_lesser_upper", "g_greater_diag",
          "g_greater_upper", "sigma_obc_lesser_left", "sigma_obc_greater_left", "sigma_obc_lesser_right",
          "sigma_obc_greater_right"]:
    a = res[f]
    mine[f] = np.tensordot(a, rng.standard_normal(a.shape[1:]), axes=a.ndim - 1)
for f in ("lesser", "greater", "ret_upper", "ret_lower"):
    a = res["sigma_" + f]
    mine["sigma_" + f] = a.T @ rng.standard_normal(a.shape[0])
parts = [None] * comm.size
dist.all_gather_object(parts, (own.start, mine))
parts.sort(key=lambda x: x[0])
worst, which = 0.0, ""
for f in mine:
    full = np.concatenate([p[1][f] for p in parts])
    r = rel(full, g[f + "_chk"])
    if r > worst:
        worst, which = r, f
worst = max(worst, rel(res["residuals"], g["residuals"]))
if comm.rank == 0:
    print(f"DIST_CHECK world={comm.size} spatial={int(spatial)} worst_rel={worst:.3e} ({which}) "
          f"transpose_bytes_rank0={res['transpose_bytes']}")
    assert worst < 1e-9
# three GW iterations (buffers reused across iterations) vs the same run on one GPU
opts3 = ScbaOptions(retarded_method="sancho", max_iter=3, tol=1e-12, batch=40, memoizer=MemoizerOptions(enabled=False))
args = (orc.chain_device(16, 32), orc.coulomb_matrix(16, 32), np.linspace(-2.0, 2.0, 128), 1e-3,
        Contacts(0.1, -0.1, 0.05), opts3)
res3 = scba_run(*args, device=dev, comm=comm, plan=plan)
sig = {f: res3["sigma_" + f] for f in ("lesser", "greater", "ret_upper", "ret_lower")}
parts = [None] * comm.size
dist.all_gather_object(parts, (res3["energy_slice"].start, sig))
if comm.rank == 0:
    parts.sort(key=lambda x: x[0])
    one = scba_run(*args, device=dev)
    w3 = max(rel(np.concatenate([p[1][f] for p in parts], axis=1), one["sigma_" + f]) for f in sig)
    w3 = max(w3, rel(res3["residuals"], one["residuals"]))
    print(f"DIST_CHECK_3IT world={comm.size} worst_rel_vs_1gpu={w3:.3e} peer_transpose="
          f"{os.environ.get('NEGF_PEER_TRANSPOSE', '1')} spatial={int(spatial)}")
    # spatial: the partitioned elimination rounds differently from the sequential sweep
    assert w3 < (1e-9 if spatial else 1e-12)
# energy-sharded extras (not spatial): the r_cut entry set (table-driven
# layout + NCCL all-to-all) and the gathered device observables vs one GPU
if not spatial:
    optc = ScbaOptions(retarded_method="sancho", max_iter=2, tol=1e-12, batch=40,
                       memoizer=MemoizerOptions(enabled=False), entry_cutoff=20)
    argc = args[:5] + (optc,)
    rc_ = scba_run(*argc, device=dev, comm=comm)
    sig = {f: rc_["sigma_" + f] for f in ("lesser", "greater")}
    parts = [None] * comm.size
    dist.all_gather_object(parts, (rc_["energy_slice"].start, sig))
    if comm.rank == 0:
        parts.sort(key=lambda x: x[0])
        one = scba_run(*argc, device=dev)
        wc = max(rel(np.concatenate([p[1][f] for p in parts], axis=1), one["sigma_" + f]) for f in sig)
        wc = max(wc, rel(rc_["residuals"], one["residuals"]))
        wo = max(rel(rc_.observables[k], one.observables[k]) for k in ("dos", "density", "current_spectrum"))
        wo = max(wo, abs(rc_.observables["terminal_left"] - one.observables["terminal_left"])
                 / abs(one.observables["terminal_left"]))
        print(f"DIST_CHECK_CUTOFF world={comm.size} worst_rel_vs_1gpu={wc:.3e} observables_rel={wo:.3e}")
        assert wc < 1e-12 and wo < 1e-12
dist.destroy_process_group()
