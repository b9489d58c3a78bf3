"""C3-shape SCGW rate: chain_device(64,512) + coulomb_matrix(64,512),
a small energy count per rank (the full 2048-energy job needs 816 GB per
entry-major quantity), two GW iterations, the second timed. Usage:
  python tools/c3_rate.py [n_b] [bs] [energies_per_rank] [batch]
  torchrun --nproc-per-node N tools/c3_rate.py ...   (energy-sharded)"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2508_19138_b200 import toys  # noqa: E402
from paper_2508_19138_b200.carrier import Contacts  # noqa: E402
from paper_2508_19138_b200.dist import Comm  # noqa: E402
from paper_2508_19138_b200.scba import ScbaOptions, scba_run  # noqa: E402

n_b, bs, ne, batch = (int(x) for x in (sys.argv[1:] + ["64", "512", "8", "8"][len(sys.argv) - 1:]))
import os  # noqa: E402

if int(os.environ.get("WORLD_SIZE", "1")) > 1:
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
comm = Comm.from_env()
world, rank = comm.size, comm.rank
dev = torch.device("cuda", rank % torch.cuda.device_count())
torch.cuda.set_device(dev)
h, v = toys.chain_device(n_b, bs), toys.coulomb_matrix(n_b, bs)
e = np.linspace(-2.0, 2.0, ne * world)
opts = ScbaOptions(retarded_method="sancho", max_iter=2, tol=1e-5, batch=batch,
                   greater=os.environ.get("NEGF_GREATER", "recursion"),
                   rgf_streams=int(os.environ.get("NEGF_RGF_STREAMS", "1")))
res = scba_run(h, v, e, 1e-3, Contacts(0.1, -0.1, 0.05), opts, device=dev, keep_g=False, comm=comm,
               sigma_to_host=False, profile=True)
dt = torch.tensor([res["iteration_s"][-1]], dtype=torch.float64, device=dev)
if world > 1:
    torch.distributed.all_reduce(dt, op=torch.distributed.ReduceOp.MAX)
dt = float(dt.item())
flops = 2 * 8.0 * bs ** 3 * (38 * n_b - 33) * ne * world  # SURVEY §8(d) F_RGF, G and W
if rank == 0:
    print(json.dumps({"config": f"chain_device({n_b},{bs}) + coulomb_matrix, {ne * world} energies ({ne}/rank), "
                                f"batch {batch}, x{world} GPUs, 2nd GW iteration timed, G^> by {opts.greater}",
                      "iteration_s": dt, "energies_per_s": ne * world / dt, "rgf_model_tflops_GW": flops / dt / 1e12,
                      "stage_s_both_iterations": res["timings"], "iteration_s_all": res["iteration_s"],
                      "residuals": list(map(float, res["residuals"])),
                      "identity_defects": res["identity_defects"], "cache_stats": res["cache_stats_by_iteration"],
                      "max_mem_gb": torch.cuda.max_memory_allocated(dev) / 1e9,
                      "transpose_bytes_rank0": int(res["transpose_bytes"])}))
