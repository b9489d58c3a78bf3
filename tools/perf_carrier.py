"""C2-shape carrier throughput: assembly + Sancho OBC + RGF per energy batch."""
import sys, time; sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2508_19138_b200 import toys
from paper_2508_19138_b200.carrier import CarrierSolver, Contacts
nb_, bs = int(sys.argv[1]), int(sys.argv[2])
dev = torch.device('cuda')
h = toys.chain_device(nb_, bs)
from paper_2508_19138_b200 import _lib
for spec in sys.argv[3:]:
    batch, streams, algo, ov = (int(x.replace("m", "-")) for x in spec.split("x"))
    _lib.load().negf_set_gemm_algo(algo)
    _lib.load().negf_set_rgf_overlap(ov)
    solver = CarrierSolver(h, 1e-3, Contacts(0.1, -0.1, 0.05), 1e-8, device=dev, streams=streams,
                           greater="identity" if streams < 0 else "recursion")
    streams = abs(streams)
    e = np.linspace(-2, 2, batch)
    solver.solve(e, n_e=batch)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 2
    for _ in range(reps):
        b = solver.solve(e, n_e=batch, check=False)
    th = (time.perf_counter() - t0) / reps
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    print(f"  host enqueue {th*1e3:.1f} ms/batch", flush=True)
    solver.check_status(b)
    print(f"{nb_}x{bs} batch={batch} streams={streams} algo={algo} overlap={ov}: {dt*1e3:.1f} ms/batch  {batch/dt:.1f} energies/s  "
          f"model {8.0*bs**3*(38*nb_-33)*batch/dt/1e12:.2f} TF", flush=True)
    del solver, b
    torch.cuda.empty_cache()
