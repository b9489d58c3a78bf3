"""Batched pivoted inverse timing (negf_zinv_batched), n x n, batch matrices."""
import sys; sys.path.insert(0, '/root/repo')
import torch
from paper_2508_19138_b200 import _lib
n, batch = (int(x) for x in (sys.argv[1:3] if len(sys.argv) > 2 else (256, 128)))
algo = int(sys.argv[3]) if len(sys.argv) > 3 else 2
dev = torch.device('cuda')
lib = _lib.load()
assert lib.negf_set_gemm_algo(algo) == 0
g = torch.Generator(device=dev).manual_seed(0)
a = torch.complex(torch.randn(batch, n, n, generator=g, device=dev, dtype=torch.float64),
                  torch.randn(batch, n, n, generator=g, device=dev, dtype=torch.float64))
a += 4 * torch.eye(n, dtype=torch.complex128, device=dev)
s, x = a.clone(), torch.empty_like(a)
st = torch.zeros(batch, dtype=torch.int32, device=dev)
nb = lib.negf_zinv_workspace_bytes(n, batch)
ws = torch.empty(nb, dtype=torch.uint8, device=dev)
def run():
    s.copy_(a)
    rc = lib.negf_zinv_batched(n, batch, s.data_ptr(), x.data_ptr(), st.data_ptr(), None, ws.data_ptr(), nb,
                               _lib.stream_ptr())
    assert rc == 0, rc
run(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 20
e0.record()
for _ in range(reps):
    run()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
err = (torch.linalg.inv(a) - x).abs().max().item()
print(f"zinv n={n} batch={batch}: {ms:.3f} ms ({8.0 * n**3 * batch / ms / 1e9:.2f} TFLOP/s incl. copy) maxerr {err:.2e} "
      f"{_lib._LIB_PATH.name} algo {algo}", flush=True)
