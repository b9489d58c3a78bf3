"""One fused P and one Sigma launch at N_E energies on synthetic rows (for ncu).
Usage: python tools/conv_one.py N_E [rows]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2508_19138_b200.conv import polarization, self_energy  # noqa: E402

ne = int(sys.argv[1])
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 15
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
mk = lambda: torch.complex(torch.randn(rows, ne, generator=g, device=dev, dtype=torch.float64),
                           torch.randn(rows, ne, generator=g, device=dev, dtype=torch.float64))
gl, gg, wl, wg = mk(), mk(), mk(), mk()
diag = torch.zeros(rows, dtype=torch.uint8, device=dev)
for _ in range(2):
    polarization(gl, gg, diag, 0.01)
    self_energy(gl, gg, wl, wg, None, diag, 0.01)
torch.cuda.synchronize()
print("ok", ne, rows)
