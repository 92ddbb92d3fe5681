"""CPU: pin the oracle (oracle/tt_oracle.c) before trusting it.

* bit-exact against the committed golden fixtures, which were produced by the
  reference implementation itself (tests/golden/make_golden.py);
* bit-exact against the reference compiled from its own sources
  (oracle/_ref/libttref.so) on fresh random plans, when that build exists;
* the reference's known-answer tests (test_embedding_ops.cpp:231-254,
  test_shape_plan.cpp:100-111).
"""
import numpy as np
import pytest

from helpers import cfg1, load_plans, scaled_max_err, small_cases
from pyoracle import Oracle, Plan, RefImpl, ref_available


@pytest.fixture(scope="module")
def orc():
    return Oracle()


def test_oracle_matches_golden_small_cases(orc):
    for c in small_cases():
        p = c["plan"]
        cores = [x.copy() for x in c["cores"]]
        out = orc.forward(p, cores, c["idx"], c["off"], c["w"], c["pooling"])
        assert out.dtype == c["fwd"].dtype
        assert np.array_equal(out, c["fwd"]), "forward differs from ref::forward_bags"
        grads = orc.backward(p, cores, c["idx"], c["off"], c["grad_out"], c["w"], c["pooling"])
        for g, want in zip(grads, c["grads"]):
            assert np.array_equal(g, want), "backward differs from ref::backward_bags"
        orc.sgd(p, cores, grads, 0.05)
        for a, want in zip(cores, c["after"]):
            assert np.array_equal(a, want), "sgd differs from ttrec::sgd_step"


def test_oracle_matches_golden_cfg1(orc):
    plan, z = cfg1()
    cores = [z[f"core{k}"] for k in range(3)]
    out = orc.forward(plan, cores, z["idx"], z["off"])
    assert np.array_equal(out, z["fwd"])
    grads = orc.backward(plan, cores, z["idx"], z["off"], z["grad_out"])
    for k in range(3):
        # golden grads come from the OpenMP backward_bags (worker-merged); the
        # serial oracle agrees to summation-order rounding only
        assert scaled_max_err(grads[k], z[f"grad{k}"]) <= 1e-5
    for r, want in zip(z["rows"], z["lookup"]):
        assert np.array_equal(orc.lookup_row(plan, cores, int(r)), want)


def test_decode_goldens(orc):
    for e in load_plans()["decode"]:
        assert list(orc.decompose_row(e["flat"], [200, 220, 250])) == e["digits"]
    # test_shape_plan.cpp:102-106
    assert list(orc.decompose_row(10131226, [200, 220, 250])) == [184, 44, 226]
    assert list(orc.decompose_row(250, [200, 220, 250])) == [0, 1, 0]


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_one_param_per_core_exact(orc, dtype):
    # test_embedding_ops.cpp:231-254: fwd 15, grads (5, 3), SGD -> (2.5, 4.7)
    p = Plan(1, 1, [1, 1], [1, 1], [1, 1, 1])
    cores = [np.array([3.0], dtype), np.array([5.0], dtype)]
    out = orc.forward(p, cores, [0], [0, 1])
    assert out[0, 0] == 15.0
    g = orc.backward(p, cores, [0], [0, 1], np.array([[1.0]], dtype))
    assert g[0][0] == 5.0 and g[1][0] == 3.0
    orc.sgd(p, cores, g, 0.1)
    assert cores[0][0] == pytest.approx(2.5) and cores[1][0] == pytest.approx(4.7)


def test_empty_bags_and_batch(orc):
    p = Plan(40, 16, [4, 4, 4], [2, 2, 4], [1, 2, 2, 1])
    rng = np.random.default_rng(0)
    cores = [rng.standard_normal(p.core_size(k)).astype(np.float32) for k in range(3)]
    out = orc.forward(p, cores, np.zeros(0, np.int64), [0])
    assert out.shape == (0, 16)
    out = orc.forward(p, cores, [1, 2, 3], [0, 2, 2, 3], pooling=1)
    assert np.all(out[1] == 0)


def test_oracle_rejects_bad_input(orc):
    p = Plan(40, 16, [4, 4, 4], [2, 2, 4], [1, 2, 2, 1])
    cores = [np.zeros(p.core_size(k), np.float32) for k in range(3)]
    with pytest.raises(ValueError):
        orc.forward(p, cores, [40], [0, 1])
    with pytest.raises(ValueError):
        orc.forward(p, cores, [0, 1], [0, 2, 1])


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_oracle_bit_exact_vs_reference_random_plans(orc):
    ref = RefImpl()
    rng = np.random.default_rng(99)
    for trial in range(24):
        d = int(rng.integers(2, 5))
        rank = int(rng.integers(1, 9))
        rows = int(rng.integers(10, 300))
        p, _ = ref.plan_shapes(rows, 16, d, rank, None, [2, 2, 2, 2] if d == 4 else None)
        for dt in (np.float32, np.float64):
            t = ref.table(p, dt, "pin")
            t.fill_normal(trial)
            cores = t.get_cores()
            idx, off, w = ref.random_batch(trial, rows, 20, 0, 6, trial % 2 == 1)
            pool = int(trial % 3 == 0)
            assert np.array_equal(t.serial_forward(idx, off, w, pool),
                                  orc.forward(p, cores, idx, off, w, pool))
            g = rng.standard_normal((len(off) - 1, 16)).astype(dt)
            for a, b in zip(t.serial_backward(idx, off, g, w, pool),
                            orc.backward(p, cores, idx, off, g, w, pool)):
                assert np.array_equal(a, b)


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_reference_plan_goldens():
    ref = RefImpl()
    for e in load_plans()["table2"]:
        _, info = ref.plan_shapes(e["rows"], 16, 3, e["rank"], e["row_factors"], [2, 2, 4])
        assert info["params"] == e["params"] and info["reduction"] == e["reduction"]
    # acceptance.cpp:72-80 / tests/golden/table2_r32.txt:1
    _, info = ref.plan_shapes(10131227, 16, 3, 32, [200, 220, 250], [2, 2, 4])
    assert info["params"] == 495360 and info["reduction"] == 327


@pytest.mark.skipif(not ref_available(), reason="reference build missing")
def test_reference_model_driver():
    """The reference DlrmModel / SyntheticDataSource wrappers the GPU DLRM test
    checks against (oracle/ref_driver.cpp): parameter shapes follow the config
    and a few training steps give finite, decreasing-ish losses."""
    from pyoracle import RefModel, RefSource

    ref = RefImpl()
    tables = [(5000, True, 8), (300, False, 0)]
    m = RefModel(ref, 3, 16, tables, [16], [8, 1])
    m.init(2)
    assert m.param(0, 0).size == 16 * 3 and m.param(1, 0).size == 16
    assert m.param(2, 0).size == 8 * (16 + 3) and m.param(2, 1).size == 8
    assert m.param(5, 1).size == 300 * 16
    src = RefSource(ref, 3, [t[0] for t in tables], 1.05, 64, 1, 3)
    mb = src.next(0)
    assert mb["dense"].shape == (64, 3) and set(np.unique(mb["labels"])) <= {0.0, 1.0}
    assert all(len(o) == 65 for o in mb["off"])
    losses = [m.step(src.next(i), 0.05)[1] for i in range(6)]
    assert all(np.isfinite(losses))
