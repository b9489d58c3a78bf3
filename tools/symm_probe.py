"""Probe torch symmetric memory (peer pointers over NVLink) on N ranks."""
import os

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm

rank = int(os.environ["RANK"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=dev)
t = symm.empty(1 << 20, dtype=torch.complex128, device=dev)
t.fill_(rank + 1)
h = symm.rendezvous(t, dist.group.WORLD.group_name)
print(rank, "ptrs", [hex(p) for p in h.buffer_ptrs], "world", h.world_size, "rank", h.rank, flush=True)
h.barrier()
peer = (rank + 1) % h.world_size
rt = h.get_buffer(peer, (16,), torch.complex128)
print(rank, "peer", peer, "reads", rt[:2].tolist(), flush=True)
h.barrier()
dist.destroy_process_group()
