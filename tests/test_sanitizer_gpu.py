"""GPU: compute-sanitizer racecheck + memcheck over one fast-path and one
generic-path fwd+bwd+SGD step (the reference's determinism tests act as race
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
print("ok")
""" % ROOT


def _sanitizer():
    for p in ("/usr/local/cuda/bin/compute-sanitizer", shutil.which("compute-sanitizer")):
        if p and os.path.exists(p):
            return p
    pytest.skip("compute-sanitizer not found")


@pytest.mark.parametrize("tool", ["racecheck", "memcheck"])
def test_sanitizer_clean(tool, tmp_path):
    script = tmp_path / "step.py"
    script.write_text(SCRIPT)
    out = subprocess.run([_sanitizer(), "--tool", tool, sys.executable, str(script)],
                         capture_output=True, text=True, timeout=600)
    text = out.stdout + out.stderr
    assert "ok" in out.stdout, text[-3000:]
    if tool == "racecheck":
        assert "RACECHECK SUMMARY: 0 hazards" in text, text[-3000:]
    else:
        assert "ERROR SUMMARY: 0 errors" in text, text[-3000:]
