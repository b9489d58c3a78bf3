import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch
import negf_oracle as orc
from paper_2508_19138_b200.carrier import Contacts
from paper_2508_19138_b200.scba import MemoizerOptions, ScbaOptions, scba_run
from test_oracle_golden import check_c1
g = np.load('/root/repo/tests/golden/golden_scba_c1.npz')
for batch in (32, 40, 64, 16):
    res = scba_run(orc.chain_device(16, 32), orc.coulomb_matrix(16, 32), np.linspace(-2.0, 2.0, 128), 1e-3,
                   Contacts(0.1, -0.1, 0.05), ScbaOptions(retarded_method="sancho", max_iter=1, tol=1e-12, batch=batch, memoizer=MemoizerOptions(enabled=False)), device='cuda')
    try:
        check_c1(res, g, tol=1e-9); print(batch, 'ok')
    except AssertionError as e:
        print(batch, 'FAIL', str(e)[:300])
