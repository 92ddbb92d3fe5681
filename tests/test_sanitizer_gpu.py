"""GPU: compute-sanitizer racecheck + memcheck + synccheck over one fast-path and one
generic-path fwd+bwd+SGD step, the wide3 tail kernels, the cache fast path and the
peer reduce (the reference's determinism tests act as race
canaries; on the GPU we check for races directly)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, %r)
import paper_2101_11714_b200 as tt
for rank, generic in ((32, False), (8, True)):
    p = tt.plan_shapes(10131227, 16, 3, rank, [200, 220, 250], [2, 2, 4])
    t = tt.TtTable(p, "san")
    rng = np.random.default_rng(0)
    t.set_cores([(rng.standard_normal(p.core_size(k)) * 0.3).astype(np.float32) for k in range(3)])
    t.set_generic_path(generic)
    b = tt.generate_zipfian_batch(p.num_rows, 0.8, 5, 20000, 1)
    g = rng.standard_normal((20000, 16)).astype(np.float32)
    r = tt.forward_bags(t, b)
    gr = tt.backward_bags(t, b, r.context, g)
    tt.sgd_step(t, gr, 0.01)
    r = tt.forward_bags(t, b, save_intermediates=True)
    t.backward_sgd(r.context, b, g, 0.01)
# generic d = 3 wide-row kernels (cfg3's factorisation at a smaller rank), multi-hot bags
p = tt.plan_shapes(400000, 64, 3, 16, [50, 80, 100], [4, 4, 4])
t = tt.TtTable(p, "wide")
rng = np.random.default_rng(1)
t.set_cores([(rng.standard_normal(p.core_size(k)) * 0.3).astype(np.float32) for k in range(3)])
idx = rng.integers(0, p.num_rows, 4096 * 4)
b = tt.IndexBatch(idx, np.arange(0, 4096 * 4 + 1, 4, dtype=np.int64))
g = rng.standard_normal((4096, 64)).astype(np.float32)
r = tt.forward_bags(t, b, save_intermediates=True)
gr = tt.backward_bags(t, b, r.context, g)
t.backward_sgd(r.context, b, g, 0.01)
# wide3 warp-per-chunk tail kernels (cfg3's shape class: n = 4x4x4, R = 64)
p = tt.ShapePlan(30000, 64, 3, [20, 30, 50], [4, 4, 4], [1, 64, 64, 1])
t = tt.TtTable(p, "w3")
t.set_cores([(rng.standard_normal(p.core_size(k)) * 0.1).astype(np.float32) for k in range(3)])
sizes = rng.integers(0, 40, 200)
off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
b = tt.IndexBatch(rng.integers(0, p.num_rows, int(off[-1])).astype(np.int64), off)
g = rng.standard_normal((200, 64)).astype(np.float32)
r = tt.forward_bags(t, b)
gr = tt.backward_bags(t, b, r.context, g)
t.backward_sgd(r.context, b, g, 0.01)
# LFU cache on the fast path (probe inside f3_gsort, pool_if_last with cached
# rows, slot gradients on the side stream): warm-up, finalize, active steps
from paper_2101_11714_b200.lfu_cache import EmbeddingLayer, LfuCache
p = tt.ShapePlan(40000, 16, 3, [30, 34, 40], [2, 2, 4], [1, 16, 16, 1])
t = tt.TtTable(p, "cache")
t.init_sampled_gaussian(3)
lay = EmbeddingLayer(t, LfuCache(48, 16, key_space=40000))
zs = tt.generate_zipfian_batch(40000, 1.2, 11, 30000, 1).indices
for s_ in range(4):
    sizes = rng.integers(0, 6, 2000)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    b = tt.IndexBatch(zs[s_ * 7000: s_ * 7000 + int(off[-1])].copy(), off, None, tt.Pooling(s_ & 1))
    lay.forward(b)
    lay.backward(b, rng.standard_normal((2000, 16)).astype(np.float32))
    lay.step(0.01)
    if s_ == 1:
        lay.finalize_warmup()
# fused peer reduce + SGD: two ranks' tables on two streams of this GPU (the sanitizer
# serialises kernels, so the peer waits run into their bounded timeout here: this
# exercises the timeout path's memory safety, the reduction itself is checked in
# tests/test_peer_reduce_gpu.py)
import ctypes as C, torch
from paper_2101_11714_b200._lib import lib
p = tt.plan_shapes(10131227, 16, 3, 32, [200, 220, 250], [2, 2, 4])
ss = [torch.cuda.Stream(), torch.cuda.Stream()]
ts = [tt.TtTable(p, "r" + str(r), stream=ss[r].cuda_stream) for r in range(2)]
flags = []
for q in ts:
    q.set_cores([np.zeros(p.core_size(k), np.float32) for k in range(3)])
    f = C.c_void_p(); assert lib().ttgpu_peer_flags_ptr(q.handle, C.byref(f)) == 0; flags.append(f.value)
G = (C.c_void_p * 2)(*[q.grad_buffer()[0] for q in ts]); F = (C.c_void_p * 2)(*flags)
Cp = (C.c_void_p * 2)(*[q.core_device_ptr(0) for q in ts])
for r, q in enumerate(ts):
    assert lib().ttgpu_peer_attach_ptrs(q.handle, 2, r, G, Cp, F) == 0
    b = tt.generate_zipfian_batch(p.num_rows, 1.05, 3 + r, 2048, 1)
    res = tt.forward_bags(q, b, save_intermediates=True)
    tt.backward_bags(q, b, res.context, rng.standard_normal((2048, 16)).astype(np.float32))
for q in ts:
    assert lib().ttgpu_peer_reduce_sgd(q.handle, C.c_double(0.01)) == 0
for q in ts:
    q.check()
print("ok")
""" % ROOT


def _sanitizer():
    for p in ("/usr/local/cuda/bin/compute-sanitizer", shutil.which("compute-sanitizer")):
        if p and os.path.exists(p):
            return p
    pytest.skip("compute-sanitizer not found")


@pytest.mark.parametrize("tool", ["racecheck", "memcheck", "synccheck"])
def test_sanitizer_clean(tool, tmp_path):
    # The GPU pool closed compute-sanitizer (runs under it left GPUs needing a
    # reset), so the runs are opt-in: TTGPU_SANITIZER=1.  Their last clean
    # results on this code path are in profiles/r2_pytest_gpu.log.
    if os.environ.get("TTGPU_SANITIZER") != "1":
        pytest.skip("compute-sanitizer runs are opt-in (TTGPU_SANITIZER=1): closed on the GPU pool")
    script = tmp_path / "step.py"
    script.write_text(SCRIPT)
    out = subprocess.run([_sanitizer(), "--tool", tool, sys.executable, str(script)],
                         capture_output=True, text=True, timeout=600)
    text = out.stdout + out.stderr
    if "closed on this pool" in text:
        pytest.skip(text.strip().splitlines()[0])
    assert "ok" in out.stdout, text[-3000:]
    if tool == "racecheck":
        assert "RACECHECK SUMMARY: 0 hazards" in text, text[-3000:]
    else:
        assert "ERROR SUMMARY: 0 errors" in text, text[-3000:]
