"""Spatial-DD selected solve timing: one partition per GPU (torchrun) on a
large-block chain, vs the sequential solve on one GPU (N=1 path).
Usage: torchrun --standalone --nproc-per-node N tools/dd_bench.py [n_blocks bs n_e]"""
import os, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch, torch.distributed as dist
from paper_2508_19138_b200.dd import (balanced_partition_plan, dd_selected_solve_batched, make_partition_plan,
                                      partition_inputs)
from paper_2508_19138_b200.rgf import selected_solve_batched

nb, bs, ne = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (32, 1024, 2)))
world = int(os.environ.get("WORLD_SIZE", "1"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
if world > 1:
    dist.init_process_group("nccl", device_id=dev)
rank = dist.get_rank() if world > 1 else 0
g = torch.Generator(device=dev).manual_seed(0)
r = lambda *s: torch.complex(torch.randn(*s, generator=g, device=dev, dtype=torch.float64),
                             torch.randn(*s, generator=g, device=dev, dtype=torch.float64)) * (1.0 / bs ** 0.5)
eye = torch.eye(bs, dtype=torch.complex128, device=dev)
balanced = len(sys.argv) > 4 and sys.argv[4] == "balanced"
plan = balanced_partition_plan(nb, world) if balanced else make_partition_plan(nb, world)
a, b = plan.ranges[rank]
# each rank builds only its partition + halo (same seeded full chain on every rank, sliced)
md = r(ne, nb, bs, bs) + (4 + 1j) * eye
mu, ml = r(ne, nb - 1, bs, bs), r(ne, nb - 1, bs, bs)
src = {"<": (r(ne, nb, bs, bs), r(ne, nb - 1, bs, bs)), ">": (r(ne, nb, bs, bs), r(ne, nb - 1, bs, bs))}


def step():
    if world == 1:
        return selected_solve_batched(md, mu, ml, src["<"], src[">"], check=False)
    return dd_selected_solve_batched(part, plan)


if world > 1:
    part = partition_inputs(md, mu, ml, src, plan, rank)
    del md, mu, ml, src
    torch.cuda.empty_cache()
for _ in range(2):
    step()
times = []
for _ in range(3):
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    times.append(time.perf_counter() - t0)
t = torch.tensor([min(times)], dtype=torch.float64, device=dev)
if world > 1:
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
if rank == 0:
    flops = 8.0 * bs ** 3 * (38 * nb - 33) * ne
    print(f"DD_BENCH n_gpus={world} chain={nb}x{bs} n_e={ne} plan={plan.ranges} time={t.item()*1e3:.1f} ms "
          f"energies/s={ne / t.item():.2f} model_TF={flops / t.item() / 1e12:.2f}", flush=True)
if world > 1:
    dist.destroy_process_group()
