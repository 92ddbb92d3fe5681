"""GPU: the LFU hot-row cache and the cached EmbeddingLayer against the reference.

* routing / admission: hot sets, slot order, per-step hit counters, drift and
  frequencies bit-exact with the reference's own LfuCache (golden fixtures
  and the LFU oracle);
* values: cached forward of the first active step bit-identical; training
  trajectories (outputs, cores, cached rows) within the fp32 tolerance;
* slot gradients against a float64 restatement, deterministic bitwise;
* the reference's error contract and the zero-chain-rows criterion
  (acceptance.cpp:709-713).
"""
import os

import numpy as np
import pytest

from helpers import GOLDEN, cache_case, scaled_max_err
from lfu_oracle import LfuOracle
from pyoracle import Oracle, Plan

pytestmark = pytest.mark.gpu

FIN, REF_AT, CAP, LR = 5, 10, 48, 0.002


def _tt():
    import paper_2101_11714_b200 as tt
    return tt


def _zipf(rows, s, seed, bags, pf):
    b = _tt().generate_zipfian_batch(rows, s, seed, bags, pf)
    return b.indices, b.offsets


def _layer(z, generic=False):
    tt = _tt()
    from paper_2101_11714_b200.lfu_cache import EmbeddingLayer, LfuCache

    d = len(z["rf"])
    emb = int(np.prod(z["cf"]))
    plan = tt.ShapePlan(20000, emb, d, [int(x) for x in z["rf"]], [int(x) for x in z["cf"]],
                        [int(x) for x in z["rk"]])
    table = tt.TtTable(plan, "cached")
    table.set_cores([z[f"init_core{k}"] for k in range(d)])
    if generic:
        table.set_generic_path(True)
    cache = LfuCache(CAP, emb, key_space=20000)
    return table, cache, EmbeddingLayer(table, cache)


def _batch(z, s):
    tt = _tt()
    w = z[f"w{s}"] if f"w{s}" in z else None
    return tt.IndexBatch(z[f"idx{s}"], z[f"off{s}"], w,
                         tt.Pooling.Mean if s % 3 == 2 else tt.Pooling.Sum)


@pytest.mark.parametrize("name,generic", [("cache_train3", False), ("cache_train3", True),
                                          ("cache_train2", False)])
def test_cached_training_trajectory_matches_reference(name, generic):
    z = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    table, cache, layer = _layer(z, generic)
    if name == "cache_train3" and not generic:
        assert table.fast_path_kind() >= 0
    for s in range(z["out"].shape[0]):
        b = _batch(z, s)
        out = layer.forward(b)
        if s == 0:
            assert np.array_equal(out, z["out"][0]), "first forward not bit-identical"
        if s == FIN + 1:
            # first active step: cached rows were just admitted from lookup_row
            assert scaled_max_err(out, z["out"][s]) < 1e-5
        assert scaled_max_err(out, z["out"][s]) < 1e-4, f"step {s}"
        layer.backward(b, z[f"grad{s}"])
        layer.step(LR)
        assert cache.active_accesses() == z["accesses"][s], f"step {s}"
        assert cache.active_hits() == z["hits"][s], f"step {s}"
        if s == FIN:
            layer.finalize_warmup()
            assert np.array_equal(cache.slot_rows(), z["fin_rows"])
            assert scaled_max_err(cache.all_row_values(), z["fin_values"]) < 1e-5
        if s == REF_AT:
            assert layer.refresh_cache() == float(z["drift"][0])
            assert np.array_equal(cache.slot_rows(), z["ref_rows"])
            assert scaled_max_err(cache.all_row_values(), z["ref_values"]) < 1e-4
    assert np.array_equal(cache.slot_rows(), z["end_rows"])
    assert scaled_max_err(cache.all_row_values(), z["end_values"]) < 1e-4
    f = cache.freq()
    assert [f.count(int(r)) for r in z["end_rows"]] == list(z["freq_end_rows"])
    for k in range(len(z["rf"])):
        assert scaled_max_err(table.core(k), z[f"core{k}"]) < 1e-4, f"core {k}"


def test_admission_values_bit_exact_and_partition_matches_reference():
    tt = _tt()
    from paper_2101_11714_b200.lfu_cache import LfuCache

    z = cache_case()
    emb = z["values"].shape[1]
    plan = tt.ShapePlan(20000, emb, 2, [int(x) for x in z["rf"]], [int(x) for x in z["cf"]],
                        [int(x) for x in z["rk"]])
    table = tt.TtTable(plan, "cache")
    table.set_cores([z["core0"], z["core1"]])
    cache = LfuCache(128, emb, key_space=20000)
    for s in range(z["stream_idx"].shape[0]):
        part = cache.record_and_partition(tt.IndexBatch(z["stream_idx"][s], z["stream_off"][s]))
        assert part.cached.num_lookups() == 0  # WarmUp: everything to the chain
    cache.warmup_finalize(table)
    assert np.array_equal(cache.hot_rows(), z["hot"])
    vals = cache.all_row_values()
    for r, s, v in zip(z["hot"], z["slots"], z["values"]):
        assert cache.slot_of(int(r)) == s
        assert np.array_equal(vals[s], v), "admitted value not bit-identical to lookup_row"
    assert cache.freq().top_k(128) == list(z["top_k"])
    part = cache.record_and_partition(
        tt.IndexBatch(z["probe_idx"], z["probe_off"], z["probe_w"], tt.Pooling.Mean))
    assert np.array_equal(part.cached.indices, z["part_cached_slots"])
    assert np.array_equal(part.cached_rows, z["part_cached_rows"])
    assert np.array_equal(part.cached.offsets, z["part_cached_offsets"])
    assert np.array_equal(part.tt.indices, z["part_tt_indices"])
    assert np.array_equal(part.tt.offsets, z["part_tt_offsets"])
    assert cache.hit_rate() == pytest.approx(float(z["hit_rate"][0]), abs=0)


def test_partition_with_hits_matches_oracle():
    """Zipf stream with many hits, weights and Mean pooling: partition parts
    (order, offsets, weights) identical to the LFU oracle's."""
    tt = _tt()
    from paper_2101_11714_b200.lfu_cache import LfuCache

    rows, cap = 30000, 64
    plan = tt.plan_shapes(rows, 8, 2, 4)
    table = tt.TtTable(plan, "p")
    table.init_sampled_gaussian(3)
    cache = LfuCache(cap, 8, key_space=rows)
    o = LfuOracle(cap, 8)
    rng = np.random.default_rng(0)
    for s in range(8):
        idx, off = _zipf(rows, 1.2, 100 + s, 300, 3)
        w = rng.uniform(0.1, 2.0, len(idx))
        part = cache.record_and_partition(tt.IndexBatch(idx, off, w, tt.Pooling.Mean))
        want = o.record_and_partition(idx, off, w)
        assert np.array_equal(part.cached.indices, want["cached_slots"])
        assert np.array_equal(part.cached_rows, want["cached_rows"])
        assert np.array_equal(part.cached.offsets, want["cached_offsets"])
        assert np.array_equal(part.tt.indices, want["tt_indices"])
        assert np.array_equal(part.tt.offsets, want["tt_offsets"])
        assert np.array_equal(part.cached.weights, want["cached_weights"])
        assert np.array_equal(part.tt.weights, want["tt_weights"])
        if s == 2:
            cache.warmup_finalize(table)
            o.warmup_finalize()
        if s == 5:
            assert cache.refresh(table) == o.refresh()
        assert cache.active_hits() == o.hits and cache.active_accesses() == o.accesses
    assert part.cached.num_lookups() > 0.3 * len(idx)
    assert np.array_equal(cache.slot_rows(), np.array(o.slot_rows))


def _slot_grad_reference(part, grad, pooling, cap, emb):
    """model.hpp:242-261 in float64: grad_eff (Mean: / original bag size), then
    Σ w·grad_eff[bag] per slot."""
    g = grad.astype(np.float64).reshape(-1, emb).copy()
    B = len(part.cached.offsets) - 1
    if pooling == 1:
        for b in range(B):
            sz = part.original_bag_size(b)
            if sz > 1:
                g[b] *= 1.0 / sz
    out = np.zeros((cap, emb))
    touched = np.zeros(cap, bool)
    for b in range(B):
        for t in range(part.cached.offsets[b], part.cached.offsets[b + 1]):
            s = part.cached.indices[t]
            out[s] += part.cached.weight(t) * g[b]
            touched[s] = True
    return out, touched


@pytest.mark.parametrize("pooling", [0, 1])
def test_slot_gradients_and_cached_sgd(pooling):
    tt = _tt()
    from paper_2101_11714_b200.lfu_cache import EmbeddingLayer, LfuCache

    rows, cap, emb = 40000, 32, 16
    plan = tt.ShapePlan(rows, emb, 3, [30, 34, 40], [2, 2, 4], [1, 16, 16, 1])
    table = tt.TtTable(plan, "sg")
    table.init_sampled_gaussian(9)
    cache = LfuCache(cap, emb, key_space=rows)
    layer = EmbeddingLayer(table, cache)
    warm_idx, warm_off = _zipf(rows, 1.3, 5, 4000, 2)
    cache.record(tt.IndexBatch(warm_idx, warm_off))
    layer.finalize_warmup()
    idx, off = _zipf(rows, 1.3, 6, 2000, 4)  # hot slot gets ~thousands of hits
    w = np.random.default_rng(1).uniform(0.5, 1.5, len(idx))
    batch = tt.IndexBatch(idx, off, w, tt.Pooling(pooling))
    grad = np.random.default_rng(2).standard_normal((2000, emb)).astype(np.float32)
    # the partition the layer will see (frequencies bumped once more by forward)
    layer.forward(batch)
    layer.backward(batch, grad)
    g, touched = cache.slot_grads()
    # rebuild the partition on a twin cache to get the reference sums
    twin = LfuCache(cap, emb, key_space=rows)
    twin.record(tt.IndexBatch(warm_idx, warm_off))
    twin.warmup_finalize(table)
    part = twin.record_and_partition(batch)
    want, want_t = _slot_grad_reference(part, grad, pooling, cap, emb)
    assert np.array_equal(touched, want_t)
    assert scaled_max_err(g, want) < 1e-5
    assert part.cached.num_lookups() > 1000
    # deterministic: a second backward gives the same bits
    layer.backward(batch, grad)
    g2, _ = cache.slot_grads()
    assert np.array_equal(g, g2)
    before = cache.all_row_values()
    layer.step(0.1)
    after = cache.all_row_values()
    exp = before.copy()
    exp[touched] = before[touched] - np.float32(0.1) * g[touched]
    assert np.array_equal(after, exp), "cached_sgd_update is row -= T(lr)*g, separately rounded"


def test_fused_cached_step_matches_unfused():
    tt = _tt()
    import torch
    from paper_2101_11714_b200.lfu_cache import LfuCache

    rows, cap, emb = 40000, 32, 16
    plan = tt.ShapePlan(rows, emb, 3, [30, 34, 40], [2, 2, 4], [1, 16, 16, 1])
    tabs, caches = [], []
    for _ in range(2):
        t = tt.TtTable(plan, "f")
        t.init_sampled_gaussian(4)
        c = LfuCache(cap, emb, key_space=rows)
        widx, woff = _zipf(rows, 1.2, 5, 3000, 1)
        c.record(tt.IndexBatch(widx, woff))
        c.warmup_finalize(t)
        tabs.append(t)
        caches.append(c)
    idx, off = _zipf(rows, 1.2, 8, 4096, 1)
    grad = np.random.default_rng(3).standard_normal((4096, emb)).astype(np.float32)
    from paper_2101_11714_b200._lib import lib
    from paper_2101_11714_b200.ttrec import ForwardContext, _raise

    d_idx = torch.from_numpy(idx).cuda()
    d_off = torch.from_numpy(off).cuda()
    d_grad = torch.from_numpy(grad).cuda()
    res = []
    for fused, t, c in zip((False, True), tabs, caches):
        ctx = ForwardContext(t)
        d_out = torch.empty((4096, emb), device="cuda")
        torch.cuda.synchronize()
        _raise(lib().ttgpu_cache_forward_device(c.handle, t.handle, ctx.handle, d_idx.data_ptr(),
                                                len(idx), d_off.data_ptr(), 4096, None, 0, 1,
                                                d_out.data_ptr()))
        if fused:
            _raise(lib().ttgpu_cache_backward_step_device(c.handle, t.handle, ctx.handle,
                                                          d_grad.data_ptr(), 0.05))
        else:
            _raise(lib().ttgpu_cache_backward_device(c.handle, t.handle, ctx.handle,
                                                     d_grad.data_ptr()))
            _raise(lib().ttgpu_cache_step(c.handle, t.handle, 0.05))
        t.sync()
        res.append((d_out.cpu().numpy(), [t.core(k) for k in range(3)], c.all_row_values()))
    assert np.array_equal(res[0][0], res[1][0])
    assert np.array_equal(res[0][2], res[1][2]), "fused slot SGD differs"
    for a, b in zip(res[0][1], res[1][1]):
        assert scaled_max_err(a, b) < 1e-6


def test_all_hit_stream_computes_no_chain_rows():
    """acceptance.cpp:709-713: a 100%-hit stream does no TT-chain work."""
    tt = _tt()
    from paper_2101_11714_b200.lfu_cache import EmbeddingLayer, LfuCache

    plan = tt.plan_shapes(10000, 8, 2, 4)
    table = tt.TtTable(plan, "hit")
    table.init_sampled_gaussian(1)
    cache = LfuCache(16, 8, key_space=10000)
    layer = EmbeddingLayer(table, cache)
    hot = np.arange(16, dtype=np.int64)
    cache.record(tt.IndexBatch.singles(np.repeat(hot, 4)))
    layer.finalize_warmup()
    tt.EmbeddingStats.reset()
    b = tt.IndexBatch(np.tile(hot, 8), np.arange(0, 129, 4, dtype=np.int64))
    out = layer.forward(b)
    assert tt.EmbeddingStats.tt_rows_computed() == 0
    vals = cache.all_row_values()
    want = np.zeros((32, 8), np.float32)
    for bb in range(32):
        for t in range(4 * bb, 4 * bb + 4):
            want[bb] += vals[b.indices[t]]
    assert np.array_equal(out, want)
    assert cache.hit_rate() == 1.0


def test_freq_table_operations():
    tt = _tt()
    from paper_2101_11714_b200.lfu_cache import LfuCache

    cache = LfuCache(4, 4, key_space=1000)
    idx = np.array([5, 7, 7, 3, 5, 7, 999, 0, 0, 3], np.int64)
    cache.record(tt.IndexBatch.singles(idx))
    f = cache.freq()
    assert f.count(7) == 3 and f.count(5) == 2 and f.count(1) == 0 and f.size() == 5
    # (count desc, key asc): test_lfu_cache.cpp:85-100 tie-break
    assert f.top_k(3) == [7, 0, 3]
    assert f.entries_sorted() == [(7, 3), (0, 2), (3, 2), (5, 2), (999, 1)]
    f.decay(0.5)  # floor(count * factor), zeros drop out (lfu_cache.cpp:78-88)
    assert f.entries_sorted() == [(0, 1), (3, 1), (5, 1), (7, 1)]
    f.clear()
    assert f.size() == 0


def test_cache_errors_follow_reference_contract():
    tt = _tt()
    from paper_2101_11714_b200.lfu_cache import EmbeddingLayer, LfuCache

    with pytest.raises(tt.InvalidArgument, match="capacity"):
        LfuCache(0, 4, key_space=10)
    with pytest.raises(tt.InvalidArgument, match="refresh_period"):
        LfuCache(4, 4, 0, key_space=10)
    plan = tt.plan_shapes(1000, 8, 2, 4)
    table = tt.TtTable(plan, "errs")
    cache = LfuCache(4, 8, key_space=1000)
    with pytest.raises(tt.InvalidArgument, match="refresh before warmup_finalize"):
        cache.refresh(table)
    cache.warmup_finalize(table)
    with pytest.raises(tt.InvalidArgument, match="already active"):
        cache.warmup_finalize(table)
    other = tt.TtTable(tt.plan_shapes(1000, 4, 2, 4), "e4")
    with pytest.raises(tt.InvalidArgument, match="emb_dim"):
        LfuCache(4, 8, key_space=1000).warmup_finalize(other)
    layer = EmbeddingLayer(table, cache)
    with pytest.raises(tt.OutOfRange, match="errs"):
        layer.forward(tt.IndexBatch.singles([1, 1000]))
    with pytest.raises(tt.InvalidArgument, match="empty slot"):
        cache.cached_sgd_update([3], np.zeros((1, 8), np.float32), 0.1)  # nothing admitted
    assert tt.lfu_cache.default_capacity(10131227) == 1013  # test_lfu_cache.cpp:323
    assert tt.lfu_cache.default_capacity(100) == 1
