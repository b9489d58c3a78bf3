"""Lesser RGF blocks vs the oracle on unscaled random systems (per block rel error)."""
import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import numpy as np, torch
import negf_oracle as orc
from paper_2508_19138_b200 import selected_solve_batched
dev = torch.device('cuda')
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
def rel(a, b): return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)
for nb, bs, ne in [(1, 128, 1), (2, 128, 1), (2, 64, 1), (2, 32, 1), (3, 128, 2), (2, 256, 1)]:
    md, mu, ml, src = orc.random_bt_system(1000, nb, bs)
    ref = orc.rgf_selected(md, mu, ml, src)
    out = selected_solve_batched(t(md), t(mu), t(ml), (t(src['<'][0]), t(src['<'][1])), (t(src['>'][0]), t(src['>'][1])))
    xl = out['xl_diag'].cpu().numpy()[0]
    print(nb, bs, ' '.join(f"{rel(xl[i], ref['x<_diag'][0, i]):.1e}" for i in range(nb)),
          'xr', f"{rel(out['xr_diag'].cpu().numpy(), ref['xr_diag']):.1e}",
          'antiherm(ref xl0)', f"{rel(ref['x<_diag'][0,0], -ref['x<_diag'][0,0].conj().T):.1e}", flush=True)
