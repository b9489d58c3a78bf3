"""Fused P / Sigma convolution kernels alone: HBM GB/s (algorithmic bytes)."""
import sys; sys.path.insert(0, '/root/repo')
import torch
from paper_2508_19138_b200.conv import polarization, self_energy
rows, n = (int(x) for x in (sys.argv[1:3] if len(sys.argv) > 2 else (200000, 512)))
dev = torch.device('cuda')
g = torch.Generator(device=dev).manual_seed(0)
r = lambda: torch.complex(torch.randn(rows, n, generator=g, device=dev, dtype=torch.float64),
                          torch.randn(rows, n, generator=g, device=dev, dtype=torch.float64))
gl, gg, wl, wg = r(), r(), r(), r()
diag = torch.zeros(rows, dtype=torch.uint8, device=dev)
for name, fn, by in (("P", lambda: polarization(gl, gg, diag, 0.01), 96),
                     ("Sigma", lambda: self_energy(gl, gg, wl, wg, None, diag, 0.01), 128)):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{name}: rows={rows} n={n}: {ms:.2f} ms  {by * rows * n / ms / 1e6:.0f} GB/s", flush=True)
