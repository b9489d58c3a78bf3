"""C2-like chain (n_b x 256) carrier solve vs the oracle: per-block rel error of G^< diag."""
import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import numpy as np, torch
import negf_oracle as orc
from paper_2508_19138_b200.carrier import CarrierSolver, Contacts
dev = torch.device('cuda')
def rel(a, b): return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)
from paper_2508_19138_b200 import _lib
import os
_lib.load().negf_set_rgf_overlap(int(os.environ.get("OV", "1")))
for nb in (4, 16):
    h = orc.chain_device(nb, 256)
    e = np.array([0.05])
    ref = orc.ballistic(h, e, 1e-3, 0.1, -0.1, 0.05)
    s = CarrierSolver(h, 1e-3, Contacts(0.1, -0.1, 0.05), 1e-8, device=dev)
    b = s.solve(e, n_e=1)
    xl = b['xl_diag'].cpu().numpy()[0]
    xlf = b['xl_diag'].cpu().numpy()[0]
    print(nb, 'xl per block', ' '.join(f"{rel(xl[i], ref['g_lesser_diag'][0, i]):.1e}" for i in range(nb)), flush=True)
    print(nb, 'xr', f"{rel(b['xr_diag'].cpu().numpy()[0], ref['g_r_diag'][0]):.1e}", flush=True)
