"""One warm RGF selected solve at a given shape (for ncu captures)."""
import sys; sys.path.insert(0, '/root/repo')
import torch
from paper_2508_19138_b200 import selected_solve_batched
nb_, bs, ne = (int(x) for x in sys.argv[1:4])
dev = torch.device('cuda')
g = torch.Generator(device=dev).manual_seed(0)
r = lambda *s: torch.complex(torch.randn(*s, generator=g, device=dev, dtype=torch.float64),
                             torch.randn(*s, generator=g, device=dev, dtype=torch.float64)) * (1.0 / bs ** 0.5)
eye = torch.eye(bs, dtype=torch.complex128, device=dev)
md = r(ne, nb_, bs, bs) + (4 + 1j) * eye
mu, ml = r(ne, nb_ - 1, bs, bs), r(ne, nb_ - 1, bs, bs)
bl = (r(ne, nb_, bs, bs), r(ne, nb_ - 1, bs, bs))
bg = (r(ne, nb_, bs, bs), r(ne, nb_ - 1, bs, bs))
for _ in range(int(sys.argv[4]) if len(sys.argv) > 4 else 2):
    out = selected_solve_batched(md, mu, ml, bl, bg, symmetrize=True)
torch.cuda.synchronize()
print("ok")
