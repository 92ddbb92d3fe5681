"""CPU: pin the LFU-cache oracle (oracle/lfu_oracle.py) against the reference.

The fixtures were produced by the reference's own LfuCache / EmbeddingLayer
(tests/golden/make_golden.py: cache_case, cache_train): hot sets, slot order,
top-k tie-breaks, frequencies, per-step access / hit counters and drift must
match exactly; admitted values come from the oracle's bit-exact lookup_row.
"""
import os

import numpy as np
import pytest

from helpers import GOLDEN, cache_case
from lfu_oracle import LfuOracle, hot_set_drift
from pyoracle import Oracle, Plan, RefImpl, ref_available


def test_lfu_oracle_matches_reference_cache_case():
    z = cache_case()
    emb = z["values"].shape[1]
    plan = Plan(20000, emb, list(z["rf"]), list(z["cf"]), list(z["rk"]))
    cores = [z["core0"], z["core1"]]
    orc = Oracle()
    o = LfuOracle(128, emb)
    for s in range(z["stream_idx"].shape[0]):
        o.record_and_partition(z["stream_idx"][s], z["stream_off"][s])
    o.warmup_finalize(lambda r: orc.lookup_row(plan, cores, r))
    assert np.array_equal(np.array(o.hot_rows()), z["hot"])
    assert [o.slot_of[int(r)] for r in z["hot"]] == list(z["slots"])
    for r, s, v in zip(z["hot"], z["slots"], z["values"]):
        assert np.array_equal(o.store[s], v), "admitted value differs from lookup_row"
    assert o.top_k(128) == list(z["top_k"])
    assert [o.counts[int(r)] for r in z["hot"]] == list(z["freq_hot"])
    part = o.record_and_partition(z["probe_idx"], z["probe_off"], z["probe_w"])
    for key in ("cached_slots", "cached_rows", "cached_offsets", "tt_indices", "tt_offsets"):
        assert np.array_equal(part[key], z["part_" + key]), key
    assert o.hits / max(o.accesses, 1) == pytest.approx(float(z["hit_rate"][0]), abs=0)


@pytest.mark.parametrize("name", ["cache_train3", "cache_train2"])
def test_lfu_oracle_matches_reference_training_trajectory(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    cap, fin, ref_at = 48, 5, 10
    o = LfuOracle(cap, z["out"].shape[2])
    for s in range(z["out"].shape[0]):
        o.record_and_partition(z[f"idx{s}"], z[f"off{s}"])
        assert o.accesses == z["accesses"][s] and o.hits == z["hits"][s], f"step {s}"
        if s == fin:
            o.warmup_finalize()
            assert np.array_equal(np.array(o.slot_rows), z["fin_rows"])
        if s == ref_at:
            d = o.refresh()
            assert d == float(z["drift"][0])
            assert np.array_equal(np.array(o.slot_rows), z["ref_rows"])
    assert np.array_equal(np.array(o.slot_rows), z["end_rows"])
    assert [o.counts[int(r)] for r in z["end_rows"]] == list(z["freq_end_rows"])


def test_hot_set_drift_known_values():
    # test_lfu_cache.cpp:126-134: identical sets 0, disjoint sets 1, half overlap 0.5
    assert hot_set_drift([1, 2], [2, 1], 2) == 0.0
    assert hot_set_drift([1, 2], [3, 4], 2) == 1.0
    assert hot_set_drift([1, 2], [1, 3], 2) == 0.5


@pytest.mark.skipif(not ref_available(), reason="reference build (oracle/_ref) absent")
def test_lfu_oracle_matches_live_reference_random_streams():
    ref = RefImpl()
    from pyoracle import RefCache

    for seed in range(3):
        rows, cap = 5000 + 1000 * seed, 16 + 8 * seed
        c = RefCache(ref, cap, 4)
        o = LfuOracle(cap, 4)
        p, _ = ref.plan_shapes(rows, 4, 2, 2)
        t = ref.table(p, np.float32, "r")
        for s in range(6):
            idx, off = ref.zipf_batch(rows, 1.1, 40 * seed + s, 200, 2)
            want = c.record_and_partition(idx, off)
            got = o.record_and_partition(idx, off)
            for key in want:
                assert np.array_equal(got[key], want[key]), (seed, s, key)
            if s == 2:
                c.warmup_finalize(t)
                o.warmup_finalize()
                assert np.array_equal(np.array(o.hot_rows()), c.hot_rows())
            if s == 4:
                assert o.refresh() == c.refresh(t)
