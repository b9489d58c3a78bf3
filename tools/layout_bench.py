"""E<->nnz pack/unpack kernels alone (EntryLayout), C2-like pattern."""
import sys; sys.path.insert(0, '/root/repo')
import torch
from paper_2508_19138_b200.scba import EntryLayout
n_b, bs, ne = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (32, 128, 128)))
dev = torch.device('cuda')
lay = EntryLayout(n_b, bs, dev)
g = torch.Generator(device=dev).manual_seed(0)
r = lambda *s: torch.complex(torch.randn(*s, generator=g, device=dev, dtype=torch.float64),
                             torch.randn(*s, generator=g, device=dev, dtype=torch.float64))
xd, xu = r(ne, n_b, bs, bs), r(ne, n_b - 1, bs, bs)
cols = torch.empty((lay.n_entries, ne), dtype=torch.complex128, device=dev)
for name, fn, by in (("pack", lambda: lay.pack(xd, xu, cols, 0), 32 * lay.n_entries * ne),
                     ("unpack_lg", lambda: lay.unpack_lg(cols, 0, ne, xd, xu),
                      16 * (lay.n_entries + (2 * n_b - 1) * bs * bs) * ne)):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{name}: {n_b}x{bs} n_e={ne}: {ms:.3f} ms  {by / ms / 1e6:.0f} GB/s", flush=True)
