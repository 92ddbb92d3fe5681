"""The N>1 bench path end to end on the one available GPU: two torchrun ranks
share device 0 (BENCH_SHARE_GPU=1, gloo for the host-side collectives).  The
fused peer reduce+SGD (CUDA IPC between the two processes) and the allreduce
fallback must both run, validate replicas and print one JSON line from rank 0.
Timings are meaningless here (the ranks time-slice one GPU)."""
import json
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


@pytest.mark.parametrize("extra,want", [([], "fused-peer-reduce+sgd"),
                                        (["--nccl"], "nccl-allreduce+sgd")])
def test_two_ranks_on_one_gpu(extra, want):
    env = dict(os.environ, BENCH_SHARE_GPU="1", BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "4", "--warmup", "3",
           "--no-cpu-baseline"] + extra
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "dp2"
    assert d["execution"]["gradient_reduce"] == want
    assert d["value"] > 0 and d["e2e"]["value"] > 0


def test_two_ranks_multitable_step():
    """cfg5's 7-table step with the coalesced gradient reduction (allreduce over gloo here)."""
    env = dict(os.environ, BENCH_SHARE_GPU="1", BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "cfg5", "--steps", "2",
           "--warmup", "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["tables"] == 26 and d["config"]["tt_tables"] == 7 and d["value"] > 0
