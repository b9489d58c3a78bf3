"""Forward-only RGF (mode 1) lesser blocks vs the oracle's forward pass, per block."""
import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import numpy as np, torch
import negf_oracle as o
from paper_2508_19138_b200 import _lib
dev = torch.device('cuda'); lib = _lib.load(); p = _lib.ptr
H = lambda x: x.conj().swapaxes(-1, -2)
r = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
n, bs = 16, 256
h = o.chain_device(n, bs); e = np.array([0.05])
m, bl, bg = o.assemble_g(e, 1e-3, h, o.fermi(e, 0.0, 0.05))
o.g_closure(m, bl, bg, e, 0.1, -0.1, 0.05, 1e-8)
md, mu, ml = m
xf, xlf = o.rgf_forward(md, mu, ml, {'<': bl})
z = dict(dtype=torch.complex128, device=dev)
out = {k: torch.zeros(s, **z) for k, s in (("xr_diag", (1, n, bs, bs)), ("xr_upper", (1, n - 1, bs, bs)), ("xr_lower", (1, n - 1, bs, bs)),
                                          ("xl_diag", (1, n, bs, bs)), ("xl_upper", (1, n - 1, bs, bs)))}
st = torch.zeros(1, dtype=torch.int32, device=dev); sp = torch.zeros((1, n), dtype=torch.float64, device=dev)
nb = lib.negf_rgf_workspace_bytes(1, n, bs); ws = _lib.workspace(nb, dev)
M = [t(x) for x in (md, mu, ml)]; B = [t(x) for x in bl]
rc = lib.negf_rgf_sweeps_batched(1, 0, 1, n, bs, p(M[0]), p(M[1]), p(M[2]), p(B[0]), p(B[1]), None, None,
                                 p(out["xr_diag"]), p(out["xr_upper"]), p(out["xr_lower"]), p(out["xl_diag"]), p(out["xl_upper"]),
                                 None, None, 0, p(st), p(sp), p(ws), nb, _lib.stream_ptr(dev))
torch.cuda.synchronize()
xl = out["xl_diag"].cpu().numpy()[0]; xr = out["xr_diag"].cpu().numpy()[0]
print('rc', rc)
print('xr fwd err', ' '.join(f"{r(xr[i], xf[i][0]):.0e}" for i in range(n)))
print('xl fwd err', ' '.join(f"{r(xl[i], xlf['<'][i][0]):.0e}" for i in range(n)))
print('xl AH dev ', ' '.join(f"{r(xl[i], -H(xl[i])):.0e}" for i in range(n)))
print('ref AH dev', ' '.join(f"{r(xlf['<'][i][0], -H(xlf['<'][i][0])):.0e}" for i in range(n)))
