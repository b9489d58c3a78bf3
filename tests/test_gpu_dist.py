"""Energy-sharded GW iteration on >= 2 GPUs vs the C1 reference golden and
vs the same 3-iteration run on one GPU (tools/dist_check.py under torchrun):
G^<> / W^<> reach their entry owners through the fused peer-memory pack
(negf_pack_lg_p2p), P / Sigma return by NCCL all-to-all; the all-to-all-only
path (NEGF_PEER_TRANSPOSE=0) is checked the same way."""

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
    assert "DIST_CHECK" in out.stdout and "DIST_CHECK_3IT" in out.stdout and "DIST_CHECK_CUTOFF" in out.stdout


def test_energy_sharded_scba_all_to_all_only(cuda):
    import os

    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs (one rank per GPU; ranks never share a GPU)")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--standalone", "--nproc-per-node", "2",
                          str(ROOT / "tools" / "dist_check.py")], capture_output=True, text=True, timeout=600,
                         env={**os.environ, "NEGF_PEER_TRANSPOSE": "0"})
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "peer_transpose=0" in out.stdout


def test_spatial_scba_matches_reference(cuda):
    """The reference's spatial mode (scba_run plan=, scba.py:878-880): every
    energy solved jointly by 2 ranks over the partitions (dd.py), vs the C1
    golden and vs the sequential run over 3 iterations."""
    import os

    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs (one rank per GPU; ranks never share a GPU)")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--standalone", "--nproc-per-node", "2",
                          str(ROOT / "tools" / "dist_check.py")], capture_output=True, text=True, timeout=600,
                         env={**os.environ, "NEGF_SPATIAL": "1"})
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "spatial=1" in out.stdout and "DIST_CHECK_3IT" in out.stdout


def test_spatial_scba_with_memoizer_matches_sequential(cuda):
    """Spatial mode with the OBC memoizer on (the reference default): Sigma and
    the per-iteration direct/memoized call counts equal the sequential run's."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs (one rank per GPU; ranks never share a GPU)")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--standalone", "--nproc-per-node", "2",
                          str(ROOT / "tools" / "spatial_memo_check.py")], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "SPATIAL_MEMO" in out.stdout and "counts_equal=True" in out.stdout
