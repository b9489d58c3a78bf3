import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import numpy as np, torch
import negf_oracle as orc
from paper_2508_19138_b200 import selected_solve_batched
dev = torch.device('cuda')
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)
rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
for shift in (0.0, 20.0):
    for bs, nb in ((128, 4), (96, 3), (64, 4), (65, 3), (256, 3)):
        md, mu, ml, src = orc.random_bt_system(1000, nb, bs)
        md = md + shift * np.eye(bs)
        ref = orc.rgf_selected(md, mu, ml, src)
        dn = orc.dense_selected(md, mu, ml, src)
        out = selected_solve_batched(t(md), t(mu), t(ml), tuple(map(t, src['<'])), None)
        g = {k: v.cpu().numpy() for k, v in out.items()}
        print(shift, bs, nb, 'xr_diag blocks', ['%.1e' % rel(g['xr_diag'][0, i], ref['xr_diag'][0, i]) for i in range(nb)],
              'up %.1e lo %.1e' % (rel(g['xr_upper'], ref['xr_upper']), rel(g['xr_lower'], ref['xr_lower'])),
              'xl %.1e' % rel(g['xl_diag'], ref['x<_diag']), 'oracle-dense %.1e' % rel(ref['xr_diag'], dn['xr_diag']),
              'gpu-dense %.1e' % rel(g['xr_diag'], dn['xr_diag']))
