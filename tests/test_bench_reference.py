"""bench.py's reference arm (CPU, no GPU needed): the driver's JSON contract --
the reference's own OpenMP step timed on the host cores, K timed steps after
W warm-ups, `impl` / `cpu_baseline` / zero-byte `e2e` keys; under torchrun
only rank 0 prints."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra, *args):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                           *args], capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)


def test_reference_arm_json_line():
    out = _run({}, "--config", "cfg1", "--steps", "3", "--warmup", "3")
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["unit"] == "indices/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 3 and d["warmup"] == 3
    assert d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["cpu_baseline"]["cores"] >= 1 and "3 steps" in d["cpu_baseline"]["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "indices/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["config"]["lookups_per_step"] == 4096


def test_reference_arm_other_ranks_silent():
    out = _run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}, "--config", "cfg1",
               "--gpus", "2", "--steps", "1", "--warmup", "3")
    assert out.returncode == 0, out.stderr[-2000:]
    assert not [l for l in out.stdout.splitlines() if l.startswith("{")]


def test_world_size_must_match_gpus():
    out = _run({"RANK": "0", "WORLD_SIZE": "2", "LOCAL_RANK": "0"}, "--config", "cfg1",
               "--gpus", "1", "--steps", "1", "--warmup", "3")
    assert out.returncode != 0 and "WORLD_SIZE" in (out.stderr + out.stdout)


def test_reference_arm_does_not_load_the_package():
    """The reference arm draws its inputs with the reference's own generators
    and never imports paper_2101_11714_b200 (or maps libttgpu.so)."""
    code = ("import sys, runpy; sys.argv=['bench.py','--impl','reference','--config','cfg1',"
            "'--steps','1','--warmup','3']; runpy.run_path('bench.py', run_name='__main__');"
            "import sys as s2; bad=[m for m in s2.modules if m.startswith('paper_2101_11714_b200')];"
            "maps=open('/proc/self/maps').read();"
            "assert not bad, bad; assert 'libttgpu' not in maps; print('CLEAN')")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0 and "CLEAN" in out.stdout, out.stderr[-2000:]


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_both_arms_same_inputs_and_config(name):
    """Both arms time the same bytes (reference generators vs this package's
    restatement) and print the same `config` object."""
    sys.path.insert(0, ROOT)
    import bench
    import paper_2101_11714_b200 as tt
    from pyoracle import ref_available

    if not ref_available():
        pytest.skip("oracle/_ref not built")
    cfg = dict(bench.CONFIGS[name])
    cfg["bags"] = 2048  # same generator, shorter stream
    a = bench.make_inputs(cfg, 7, tt)
    b = bench.make_inputs_reference(cfg, 7)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    assert bench.workload_config(cfg, 2) == bench.workload_config(dict(cfg), 2)
