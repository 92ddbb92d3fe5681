"""TTRECV01 checkpoint interop against the reference's
Checkpoint (checkpoint.hpp, src/checkpoint.cpp).  tests/golden/ckpt_ref.ttrec
was written by the reference itself (tests/golden/make_golden.py ckpt)."""
import os

import numpy as np
import pytest

from paper_2101_11714_b200 import InvalidArgument, RuntimeFailure, ShapePlan
from paper_2101_11714_b200.checkpoint import Checkpoint
from pyoracle import Oracle, Plan, ref_available

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ckpt_ref.ttrec")


def test_load_resave_reproduces_reference_file_bytes(tmp_path):
    cp = Checkpoint.load(GOLD)
    assert [t.name for t in cp.tables()] == ["emb0", "emb1"]
    assert [t.dtype for t in cp.tables()] == ["f32", "f64"]
    assert cp.tables()[0].plan.ranks == [1, 6, 5, 1]
    assert cp.has_array("dense.w") and cp.get_array("dense.w").shape == (37,)
    out = tmp_path / "again.ttrec"
    cp.save(str(out))
    assert out.read_bytes() == open(GOLD, "rb").read()


def test_rebuilt_from_host_cores_is_byte_identical(tmp_path):
    """put_table order, header JSON (keys, offsets, compact form) and payloads
    match the reference writer exactly when built from scratch."""
    src = Checkpoint.load(GOLD)
    cp = Checkpoint()
    for e in src.tables():
        dt = np.float32 if e.dtype == "f32" else np.float64
        cp.put_cores(e.name, e.plan, src.get_cores(e.name, dt), dt)
    cp.put_array("dense.w", [37], src.get_array("dense.w"))
    out = tmp_path / "rebuilt.ttrec"
    cp.save(str(out))
    assert out.read_bytes() == open(GOLD, "rb").read()
    assert '"layout": "row_digit_major"' in cp.header_json()


def test_errors_follow_reference_contract(tmp_path):
    cp = Checkpoint.load(GOLD)
    with pytest.raises(RuntimeFailure, match="no table named 'nope'"):
        cp.get_cores("nope")
    with pytest.raises(RuntimeFailure, match="stored as f64, requested f32"):
        cp.get_cores("emb1", np.float32)
    with pytest.raises(InvalidArgument, match="duplicate table name 'emb0'"):
        cp.put_cores("emb0", cp.tables()[0].plan, cp.get_cores("emb0"))
    with pytest.raises(InvalidArgument, match="shape holds 6 elements but 5 were given"):
        cp.put_array("x", [2, 3], np.zeros(5, np.float32))
    bad = tmp_path / "bad.ttrec"
    bad.write_bytes(b"NOTACKPT" + bytes(16))
    with pytest.raises(RuntimeFailure, match="is not a TTRECV01 checkpoint"):
        Checkpoint.load(str(bad))
    trunc = tmp_path / "trunc.ttrec"
    trunc.write_bytes(open(GOLD, "rb").read()[:-10])
    with pytest.raises(RuntimeFailure, match="truncated data section"):
        Checkpoint.load(str(trunc))


@pytest.mark.skipif(not ref_available(), reason="reference build (oracle/_ref) not present")
def test_reference_loads_our_file_and_we_load_its(tmp_path):
    from pyoracle import RefImpl

    ref = RefImpl()
    rng = np.random.default_rng(4)
    plan = ShapePlan(20000, 16, 3, [20, 25, 40], [2, 2, 4], [1, 8, 8, 1])
    cores = [rng.standard_normal(plan.core_size(k)).astype(np.float32) for k in range(3)]
    cp = Checkpoint()
    cp.put_cores("trained", plan, cores)
    arr = rng.standard_normal(10).astype(np.float32)
    cp.put_array("mlp.b", [10], arr)
    path = tmp_path / "ours.ttrec"
    cp.save(str(path))
    oplan = Plan(20000, 16, [20, 25, 40], [2, 2, 4], [1, 8, 8, 1])
    t = ref.checkpoint_load_table(str(path), "trained", oplan)
    for a, b in zip(t.get_cores(), cores):
        assert np.array_equal(a, b)
    assert np.array_equal(ref.checkpoint_load_array(str(path), "mlp.b", 10), arr)
    # and the reference's save of the same table reproduces our bytes
    t2 = ref.table(oplan, np.float32, "trained")
    t2.set_cores(cores)
    path2 = tmp_path / "theirs.ttrec"
    ref.checkpoint_save(str(path2), [t2], [("mlp.b", arr)])
    assert path2.read_bytes() == path.read_bytes()


@pytest.mark.gpu
def test_device_tables_round_trip_bit_exactly(tmp_path):
    """get_table uploads the stored cores to the GPU; a GPU-trained table
    saved with put_table reloads to the same bytes; forward on the loaded
    table is bit-identical to the oracle on the stored cores."""
    import paper_2101_11714_b200 as tt

    src = Checkpoint.load(GOLD)
    t = src.get_table("emb0")
    cores = src.get_cores("emb0")
    for k in range(3):
        assert np.array_equal(t.core(k), cores[k])
    rng = np.random.default_rng(0)
    idx = rng.integers(0, 5000, 300)
    b = tt.IndexBatch(idx, np.arange(301, dtype=np.int64))
    res = tt.forward_bags(t, b, save_intermediates=True)
    p = Plan(5000, 16, [10, 20, 25], [2, 2, 4], [1, 6, 5, 1])
    assert np.array_equal(res.output, Oracle().forward(p, cores, idx, b.offsets))
    g = tt.backward_bags(t, b, res.context, rng.standard_normal((300, 16)).astype(np.float32))
    tt.sgd_step(t, g, 0.05)
    out = Checkpoint()
    out.put_table(t)
    out.save(str(tmp_path / "trained.ttrec"))
    back = Checkpoint.load(str(tmp_path / "trained.ttrec")).get_table("emb0")
    for k in range(3):
        assert np.array_equal(back.core(k), t.core(k))
    t64 = src.get_table("emb1", np.float64)
    for a, c in zip([t64.core(k) for k in range(2)], src.get_cores("emb1", np.float64)):
        assert np.array_equal(a, c)
