import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import numpy as np, torch
import negf_oracle as orc
from paper_2508_19138_b200.scba import ScbaOptions, ScreenedSolver
cuda = torch.device('cuda')
n_b, bs, ne = 4, 6, 5
rng = np.random.default_rng(1)
v = orc.coulomb_matrix(n_b, bs)
mk = lambda *s: 0.3 * (rng.standard_normal(s) + 1j * rng.standard_normal(s))
solver = ScreenedSolver(v, ScbaOptions(retarded_method="sancho"), cuda)
b = solver.buffers(ne)
for k in b:
    if b[k].dtype == torch.complex128:
        b[k].copy_(torch.from_numpy(mk(*b[k].shape)))
b = solver.solve(ne)
print("ok")
