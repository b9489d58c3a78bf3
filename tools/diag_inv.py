import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import numpy as np, torch, scipy.linalg as sla
import negf_oracle as orc
from paper_2508_19138_b200 import _lib
lib = _lib.load(); dev = torch.device('cuda')
def ginv(a):
    n = a.shape[-1]; b = a.shape[0]
    s = torch.from_numpy(a.copy()).to(dev); x = torch.empty_like(s)
    st = torch.zeros(b, dtype=torch.int32, device=dev)
    nb = lib.negf_zinv_workspace_bytes(n, b); ws = torch.empty(max(nb,1), dtype=torch.uint8, device=dev)
    assert lib.negf_zinv_batched(n, b, s.data_ptr(), x.data_ptr(), st.data_ptr(), None, ws.data_ptr(), nb, _lib.stream_ptr()) == 0
    return x.cpu().numpy()
md, mu, ml, src = orc.random_bt_system(1000, 4, 128)
x = None
for i in range(4):
    s = md[0, i] if i == 0 else md[0, i] - ml[0, i-1] @ x @ mu[0, i-1]
    lu = sla.lu_solve(sla.lu_factor(s), np.eye(128))
    g = ginv(s[None])[0]
    print(i, 'cond %.1e' % np.linalg.cond(s), 'gpu-vs-lapack %.2e' % (np.linalg.norm(g - lu) / np.linalg.norm(lu)),
          'resid %.2e' % (np.linalg.norm(g @ s - np.eye(128))))
    x = lu
rng = np.random.default_rng(0)
for n in (64, 65, 96, 128, 256):
    a = rng.standard_normal((2, n, n)) + 1j * rng.standard_normal((2, n, n))
    g = ginv(a)
    for b in range(2):
        lu = sla.lu_solve(sla.lu_factor(a[b]), np.eye(n))
        print(n, b, 'cond %.1e' % np.linalg.cond(a[b]), 'err %.2e' % (np.linalg.norm(g[b] - lu) / np.linalg.norm(lu)))
