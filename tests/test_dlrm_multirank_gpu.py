"""The data-parallel DLRM step (dlrm.py, world 2): two torchrun ranks sharing
the one available GPU (gloo moves the flat gradient buffer) train halves of each
batch; rank 0 checks every parameter against a single-process full-batch twin
(tools/dlrm_dp_check.py)."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_dlrm_data_parallel_two_ranks_equal_full_batch():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tools", "dlrm_dp_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT,
                       env=dict(os.environ, DP_BACKEND="gloo", DP_DEVICE="0"))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "dp ok" in r.stdout
