"""CPU cost of the reference's own ballistic path vs the oracle port that the
bench's reference arm times on the GPU box (the reference package cannot
travel there). Same energy, C2 device chain_device(64, 256), one BLAS thread.
Run in the build container (reads /root/reference):
    PYTHONDONTWRITEBYTECODE=1 python tools/ref_vs_port_cpu.py [n_energies]"""
import sys
import time
from pathlib import Path

import numpy as np
from threadpoolctl import threadpool_limits

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True
import negf_oracle as orc  # noqa: E402
from negfgw import scba, toys  # noqa: E402
from negfgw.device import EnergyGrid  # noqa: E402

ne = int(sys.argv[1]) if len(sys.argv) > 1 else 2
with threadpool_limits(1):
    h = toys.chain_device(64, 256)
    grid = EnergyGrid(-0.5, 0.5, ne, eta=1e-3)
    opts = scba.ScbaOptions(max_iter=1, retarded_method="sancho", memoizer=scba.MemoizerOptions(enabled=False))
    t0 = time.perf_counter()
    scba.scba_run(h, None, grid, scba.ContactConfig(mu_left=0.1, mu_right=-0.1, kT=0.05), opts)
    t_ref = time.perf_counter() - t0
    ho = orc.chain_device(64, 256)
    t0 = time.perf_counter()
    orc.ballistic(ho, np.linspace(-0.5, 0.5, ne), 1e-3, 0.1, -0.1, 0.05, 1e-8)
    t_port = time.perf_counter() - t0
print(f"REF_VS_PORT C2 chain 64x256, {ne} energies, 1 thread: reference scba_run(v_mat=None) {t_ref:.1f} s "
      f"({t_ref / ne:.2f} s/energy) | oracle port ballistic {t_port:.1f} s ({t_port / ne:.2f} s/energy) | "
      f"port/reference time {t_port / t_ref:.2f}")
