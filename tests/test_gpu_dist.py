"""Energy-sharded GW iteration over NCCL (all-to-all E<->nnz transposes) on
>= 2 GPUs vs the C1 reference golden (tools/dist_check.py under torchrun)."""

import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_energy_sharded_scba_matches_reference(cuda):
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs (one rank per GPU; ranks never share a GPU)")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--standalone", "--nproc-per-node",
                          str(min(n, 4)), str(ROOT / "tools" / "dist_check.py")],
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "DIST_CHECK" in out.stdout
