"""Device time per kernel class (CUDA-event profiler in prof.cu) for one SCGW
iteration: python tools/prof_classes.py n_bxbsxne [batch]"""
import ctypes
import sys

sys.path.insert(0, '/root/repo')
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2508_19138_b200 import _lib, toys  # noqa: E402
from paper_2508_19138_b200.carrier import Contacts  # noqa: E402
from paper_2508_19138_b200.scba import ScbaOptions, scba_run  # noqa: E402

n_b, bs, ne = (int(x) for x in sys.argv[1].split('x'))
batch = int(sys.argv[2]) if len(sys.argv) > 2 else min(128, ne)
e = np.linspace(-2, 2, ne)
h, v = toys.chain_device(n_b, bs), toys.coulomb_matrix(n_b, bs)
run = lambda: scba_run(h, v, e, 1e-3, Contacts(0.1, -0.1, 0.05), ScbaOptions(retarded_method="sancho", max_iter=1, batch=batch),
                       keep_g=False, sigma_to_host=False)
run()
lib = _lib.load()
lib.negf_prof_reset()
lib.negf_prof_enable(1)
r = run()
torch.cuda.synchronize()
lib.negf_prof_enable(0)
names = {0: "zgemm K>32", 1: "zinv (other)", 2: "elementwise", 3: "other", 4: "zgemm K<=32 (sweeps)",
         5: "panel", 8: "unpermute", 9: "conv", 10: "layout"}
print("iteration_s", r["iteration_s"])
tot = 0.0
rows = []
for c in range(12):
    ms, fl, by, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_double(), ctypes.c_longlong()
    if lib.negf_prof_query(c, ctypes.byref(ms), ctypes.byref(fl), ctypes.byref(by), ctypes.byref(n)) != 0:
        continue
    if n.value:
        rows.append((c, ms.value, fl.value, by.value, n.value))
        tot += ms.value
for c, ms, fl, by, n in sorted(rows, key=lambda x: -x[1]):
    print(f"{names.get(c, c):24s} {ms:9.1f} ms {100 * ms / tot:5.1f}%  launches {n:6d}  "
          f"{fl / ms / 1e9 if ms else 0:6.1f} TF  {by / ms / 1e6 if ms else 0:7.1f} GB/s")
