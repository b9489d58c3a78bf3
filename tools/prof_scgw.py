"""Stage timings of one SCGW iteration (synchronising timers)."""
import sys; sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2508_19138_b200 import toys
from paper_2508_19138_b200.carrier import Contacts
from paper_2508_19138_b200.scba import ScbaOptions, scba_run
n_b, bs, ne = (int(x) for x in sys.argv[1].split('x'))
e = np.linspace(-2, 2, ne)
h, v = toys.chain_device(n_b, bs), toys.coulomb_matrix(n_b, bs)
opts = ScbaOptions(retarded_method="sancho", max_iter=2, tol=1e-5, batch=min(int(sys.argv[2]) if len(sys.argv) > 2 else 128, ne))
r0 = scba_run(h, v, e, 1e-3, Contacts(0.1, -0.1, 0.05), opts, keep_g=False); print("iteration_s", r0["iteration_s"])
r = scba_run(h, v, e, 1e-3, Contacts(0.1, -0.1, 0.05), opts, keep_g=False, profile=True)
tot = sum(r["timings"].values())
for k, t in sorted(r["timings"].items(), key=lambda x: -x[1]):
    print(f"{k:28s} {t:8.3f} s {100*t/tot:5.1f}%")
