"""Device-time breakdown (CUDA-event profiler classes) of one C2 carrier batch."""
import sys, ctypes; sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2508_19138_b200 import toys, _lib
from paper_2508_19138_b200.carrier import CarrierSolver, Contacts
nb_, bs, batch = (int(x) for x in sys.argv[1:4])
ov = int(sys.argv[4]) if len(sys.argv) > 4 else 0
lib = _lib.load(); lib.negf_set_rgf_overlap(ov)
greater = sys.argv[5] if len(sys.argv) > 5 else "identity"
solver = CarrierSolver(toys.chain_device(nb_, bs), 1e-3, Contacts(0.1, -0.1, 0.05), 1e-8, greater=greater)
e = np.linspace(-2, 2, batch)
solver.solve(e, n_e=batch); torch.cuda.synchronize()
lib.negf_prof_reset(); lib.negf_prof_enable(1)
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
t0.record(); solver.solve(e, n_e=batch, check=False); t1.record(); torch.cuda.synchronize()
lib.negf_prof_enable(0)
print(f"total {t0.elapsed_time(t1):.1f} ms (overlap={ov})")
for cls, name in ((0, "zgemm K>32"), (4, "zgemm K<=32"), (1, "zinv kernels"), (2, "elementwise"), (3, "other"), (5, " panel"), (6, " swap"), (7, " rows"), (8, " unpermute")):
    ms, fl, by, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_double(), ctypes.c_longlong()
    lib.negf_prof_query(cls, ctypes.byref(ms), ctypes.byref(fl), ctypes.byref(by), ctypes.byref(n))
    tf = fl.value / (ms.value * 1e-3) / 1e12 if ms.value else 0
    print(f"{name:14s} {ms.value:9.1f} ms  {n.value:6d} launches  {tf:6.2f} TF")
