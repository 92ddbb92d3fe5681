"""bench_pooling on the GPU (§8(f) f4): the reference's CSV schema and its
acceptance-criterion-7 trend checks (acceptance.cpp:647-688) on GPU numbers."""
import numpy as np
import pytest

from paper_2101_11714_b200.bench_pooling import HEADER, BenchConfig, median_of_means


def test_csv_header_matches_reference_cli():
    # tools/ttrec.cpp:263-265
    assert HEADER == ("pooling,rank,fwd_us_per_sample,bwd_us_per_sample,fwd_us_per_lookup,"
                      "bwd_us_per_lookup,serial_fwd_us_per_lookup,serial_bwd_us_per_lookup,"
                      "fwd_spread_us,bwd_spread_us")


def test_median_of_means_matches_reference_definition():
    v, s = median_of_means([1, 2, 3, 4, 5, 6, 7, 8, 9, 10])  # 5 groups of 2
    assert v == 5.5 and abs(s - np.std([1.5, 3.5, 5.5, 7.5, 9.5])) < 1e-12
    assert median_of_means([]) == (0.0, 0.0)


def test_derived_stream_matches_reference_rng():
    """The sweep's batches are Rng::derive(seed, rank<<20 ^ pooling) draws."""
    from paper_2101_11714_b200 import derived_uniform_indices
    from pyoracle import RefImpl, ref_available

    if not ref_available():
        pytest.skip("reference build absent")
    import ctypes as C

    ref = RefImpl()
    if not hasattr(ref.lib, "ref_derived_uniform_int"):
        pytest.skip("reference driver without ref_derived_uniform_int")
    out = np.zeros(1000, np.int64)
    ref.lib.ref_derived_uniform_int(C.c_uint64(3), C.c_uint64((4 << 20) ^ 10), C.c_int64(50000),
                                    C.c_int64(1000), out.ctypes.data_as(C.c_void_p))
    assert np.array_equal(derived_uniform_indices(50000, 3, (4 << 20) ^ 10, 1000), out)


@pytest.mark.gpu
def test_criterion7_trends_on_gpu():
    from paper_2101_11714_b200.bench_pooling import bench_pooling

    cfg = BenchConfig(rows=50000, emb_dim=16, tt_dim=3, ranks=[4, 64], poolings=[1, 10, 100],
                      bags=8, reps=24, micro_batch=256, seed=3, target_lookups_per_rep=12800)
    rows = {(r.rank, r.pooling): r for r in bench_pooling(cfg)}
    for r in rows.values():
        print(r.csv())
    p1, p10, p100 = (rows[(4, p)].fwd_us_per_lookup for p in (1, 10, 100))
    assert p1 > p10 > p100, (p1, p10, p100)
    q1, q10, q100 = (rows[(64, p)].bwd_us_per_lookup for p in (1, 10, 100))
    assert q1 > q10 > q100, (q1, q10, q100)
