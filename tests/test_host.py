"""CPU: the C-ABI library loads and exports include/ttgpu.h; host-side logic
(shape planning, index decode, synthetic streams, batch validation) matches
the reference goldens.  No CUDA compute here."""
import ctypes

import numpy as np
import pytest

import paper_2101_11714_b200 as tt
from helpers import GOLDEN, load_plans
from paper_2101_11714_b200._lib import header_symbols, lib
from pyoracle import RefImpl, ref_available


def test_library_exports_every_header_symbol():
    syms = header_symbols()
    assert len(syms) >= 30
    so = ctypes.CDLL(lib().path)
    missing = [s for s in syms if not hasattr(so, s)]
    assert not missing, f"libttgpu.so lacks {missing}"


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", lib().path], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_table2_plans_match_reference_goldens():
    # acceptance.cpp:72-109 criterion 1 / tests/golden/table2_r{16,32,64}.txt
    for e in load_plans()["table2"]:
        p = tt.plan_shapes(e["rows"], 16, 3, e["rank"], e["row_factors"], [2, 2, 4])
        assert p.row_factors == e["row_factors"]
        assert p.ranks == e["ranks"]
        assert p.parameter_count() == e["params"]
        assert p.memory_reduction() == e["reduction"]
        assert p.padded_rows() == e["padded_rows"]


def test_auto_plans_match_reference():
    for e in load_plans()["auto"]:
        if "error" in e:
            with pytest.raises(tt.InvalidArgument):
                tt.plan_shapes(e["rows"], e["emb"], e["d"], e["rank"])
            continue
        p = tt.plan_shapes(e["rows"], e["emb"], e["d"], e["rank"])
        assert (p.row_factors, p.col_factors, p.ranks) == (
            e["row_factors"], e["col_factors"], e["ranks"])
        assert p.parameter_count() == e["params"]


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_plans_vs_reference_random():
    ref = RefImpl()
    rng = np.random.default_rng(5)
    for _ in range(200):
        d = int(rng.integers(2, 6))
        rows = int(rng.integers(1, 10**7))
        emb = int(rng.choice([8, 12, 16, 24, 32, 48, 64, 128]))
        rank = int(rng.integers(1, 70))
        try:
            want, info = ref.plan_shapes(rows, emb, d, rank)
        except Exception:  # noqa: BLE001
            with pytest.raises(tt.InvalidArgument):
                tt.plan_shapes(rows, emb, d, rank)
            continue
        got = tt.plan_shapes(rows, emb, d, rank)
        assert (got.row_factors, got.col_factors, got.ranks) == (
            want.row_factors, want.col_factors, want.ranks)
        assert got.memory_reduction() == info["reduction"]


def test_decompose_recompose():
    # test_shape_plan.cpp:100-111
    r = [200, 220, 250]
    assert tt.decompose_index(10131226, r) == [184, 44, 226]
    assert tt.decompose_index(0, r) == [0, 0, 0]
    assert tt.decompose_index(249, r) == [0, 0, 249]
    assert tt.decompose_index(250, r) == [0, 1, 0]
    assert tt.recompose_index([184, 44, 226], r) == 10131226
    with pytest.raises(tt.OutOfRange):
        tt.decompose_index(-1, r)
    with pytest.raises(tt.OutOfRange):
        tt.decompose_index(200 * 220 * 250, r)
    with pytest.raises(tt.OutOfRange):
        tt.recompose_index([200, 0, 0], r)
    rng = np.random.default_rng(42)
    for _ in range(200):
        rad = [int(x) for x in rng.integers(2, 40, int(rng.integers(2, 6)))]
        flat = int(rng.integers(0, int(np.prod(rad))))
        assert tt.recompose_index(tt.decompose_index(flat, rad), rad) == flat


def test_plan_validation_errors():
    with pytest.raises(tt.InvalidArgument):
        tt.plan_shapes(100, 16, 1, 4)
    with pytest.raises(tt.InvalidArgument):
        tt.plan_shapes(0, 16, 3, 4)
    with pytest.raises(tt.InvalidArgument):
        tt.plan_shapes(100, 16, 3, 0)
    with pytest.raises(tt.InvalidArgument, match="col factors multiply"):
        tt.plan_shapes(100, 16, 3, 4, None, [2, 2, 2])
    with pytest.raises(tt.InvalidArgument, match="need >= num_rows"):
        tt.plan_shapes(1000, 16, 3, 4, [5, 5, 5], [2, 2, 4])
    with pytest.raises(tt.InvalidArgument, match="factorization"):
        tt.plan_shapes(100, 7, 3, 4)


def test_zipf_stream_matches_reference_bytes():
    z = np.load(f"{GOLDEN}/zipf_stream.npz")
    b = tt.generate_zipfian_batch(10131227, 1.05, 7, 4096, 1)
    assert np.array_equal(b.indices, z["idx"]) and np.array_equal(b.offsets, z["off"])


def test_uniform_stream_matches_reference_bytes():
    z = np.load(f"{GOLDEN}/cfg1.npz")
    assert np.array_equal(tt.uniform_indices(1000000, 3, 4096), z["idx"])


def test_index_batch_validation():
    b = tt.IndexBatch([0, 1], [0, 2, 1])
    with pytest.raises(tt.InvalidArgument, match="non-decreasing"):
        b.validate(10)
    with pytest.raises(tt.InvalidArgument, match="start at 0"):
        tt.IndexBatch([0], [1, 1]).validate(10)
    with pytest.raises(tt.InvalidArgument, match="offsets end"):
        tt.IndexBatch([0, 1], [0, 1]).validate(10)
    with pytest.raises(tt.InvalidArgument, match="weights"):
        tt.IndexBatch([0, 1], [0, 2], np.ones(3)).validate(10)
    s = tt.IndexBatch.singles([3, 4, 5])
    assert s.num_bags() == 3 and s.bag_size(1) == 1 and not s.has_weights()
