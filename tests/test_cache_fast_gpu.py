"""GPU: the cache fast path (the LFU cache consulted inside the fast-path sort,
f3_gsort key 3) against the partition path (record_and_partition +
forward_bags(part.tt) + combine, lfu_cache.hpp:187-219 / model.hpp:195-284).

Both paths keep the same relative order of the chain lookups and sort the
cached lookups stably by slot, so the fast path reproduces the partition path
BIT FOR BIT in the outputs, the partition itself, the hit counters, the slot
gradients and the cached rows after the SGD step; the chain gradients agree
to fp32 rounding (the backward's CTA ranges follow the chain-part size, which
only the partition path shrinks).  The partition path is itself pinned
to the reference LfuCache / EmbeddingLayer by test_cache_gpu.py and
test_fullsize_gpu.py.  Also: the fused cached step captured in a CUDA graph
(no host sync) replays to the eager results.
"""
import numpy as np
import pytest

from helpers import scaled_max_err

pytestmark = pytest.mark.gpu


def _tt():
    import paper_2101_11714_b200 as tt
    return tt


def _ragged_batch(rng, zipf_idx, bags, pooling, weighted):
    """Bags of 0..5 lookups (empty, single and multi-lookup bags, mixed
    cached / chain members) over a Zipf stream."""
    tt = _tt()
    sizes = rng.integers(0, 6, bags)
    sizes[::7] = 1
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    idx = zipf_idx[: off[-1]].copy()
    w = rng.uniform(0.5, 1.5, len(idx)) if weighted else None
    return tt.IndexBatch(idx, off, w, tt.Pooling(pooling))


def _pair(rows, rf, cf, rk, cap, seed):
    tt = _tt()
    from paper_2101_11714_b200.lfu_cache import EmbeddingLayer, LfuCache

    plan = tt.ShapePlan(rows, int(np.prod(cf)), 3, rf, cf, rk)
    layers = []
    for fast in (True, False):
        t = tt.TtTable(plan, "fast" if fast else "part")
        t.init_sampled_gaussian(seed)
        c = LfuCache(cap, plan.emb_dim, key_space=rows)
        c.set_fast(fast)
        layers.append(EmbeddingLayer(t, c))
    return layers


def _same_partition(a, b):
    assert np.array_equal(a.cached.indices, b.cached.indices)
    assert np.array_equal(a.cached_rows, b.cached_rows)
    assert np.array_equal(a.cached.offsets, b.cached.offsets)
    assert np.array_equal(a.tt.indices, b.tt.indices)
    assert np.array_equal(a.tt.offsets, b.tt.offsets)
    if a.cached.weights is not None or b.cached.weights is not None:
        assert np.array_equal(a.cached.weights, b.cached.weights)
        assert np.array_equal(a.tt.weights, b.tt.weights)


@pytest.mark.parametrize("pooling,weighted", [(0, False), (1, True), (0, True)])
def test_fast_path_bitwise_equals_partition_path(pooling, weighted):
    tt = _tt()
    rows, rf, cf, rk, cap, emb = 40000, [30, 34, 40], [2, 2, 4], [1, 16, 16, 1], 48, 16
    fast, part = _pair(rows, rf, cf, rk, cap, 7)
    rng = np.random.default_rng(pooling * 2 + weighted)
    stream = tt.generate_zipfian_batch(rows, 1.2, 11, 40000, 1).indices
    # warm-up forwards (WarmUp: every lookup on the chain, frequencies recorded)
    for s in range(2):
        b = _ragged_batch(rng, stream[s * 9000:], 2000, pooling, weighted)
        o1, o2 = fast.forward(b), part.forward(b)
        assert np.array_equal(o1, o2), f"warm-up forward {s}"
    fast.finalize_warmup()
    part.finalize_warmup()
    assert np.array_equal(fast.cache.slot_rows(), part.cache.slot_rows())
    for s in range(3):
        b = _ragged_batch(rng, stream[20000 + s * 6000:], 2000, pooling, weighted)
        g = rng.standard_normal((b.num_bags(), emb)).astype(np.float32)
        # the chain part's backward grid depends on its lookup count (the
        # partition path sees only the chain lookups), so its gradients may
        # differ in the last bits: restart both from the same cores each step
        part.tt.set_cores(fast.tt.cores())
        o1, o2 = fast.forward(b), part.forward(b)
        assert np.array_equal(o1, o2), f"step {s}: forward differs"
        p1, p2 = fast.cache.last_partition(), part.cache.last_partition()
        _same_partition(p1, p2)
        assert p1.cached.num_lookups() > 0.3 * b.num_lookups()
        assert fast.cache.last_counts() == (p2.cached.num_lookups(), p2.tt.num_lookups())
        assert fast.cache.active_hits() == part.cache.active_hits()
        assert fast.cache.active_accesses() == part.cache.active_accesses()
        fast.backward(b, g)
        part.backward(b, g)
        g1, t1 = fast.cache.slot_grads()
        g2, t2 = part.cache.slot_grads()
        assert np.array_equal(t1, t2)
        assert np.array_equal(g1, g2), f"step {s}: slot gradients differ"
        for k in range(3):
            assert scaled_max_err(fast.tt.grad(k), part.tt.grad(k)) <= 1e-5, f"step {s}: chain grad {k}"
        fast.step(0.05)
        part.step(0.05)
        for k in range(3):
            assert scaled_max_err(fast.tt.core(k), part.tt.core(k)) <= 1e-5, f"step {s}: core {k}"
        assert np.array_equal(fast.cache.all_row_values(), part.cache.all_row_values())
    assert fast.cache.hit_rate() == part.cache.hit_rate()


def test_fast_cfg4_shape_matches_partition_path():
    """cfg4: 10,131,227 rows, 1,013 slots, Zipf(1.2), 65,536 single-lookup bags."""
    tt = _tt()
    rows, cap = 10131227, 1013
    fast, part = _pair(rows, [200, 220, 250], [2, 2, 4], [1, 32, 32, 1], cap, 1)
    rng = np.random.default_rng(5)
    for s in range(5):
        b = tt.generate_zipfian_batch(rows, 1.2, 900 + s, 65536, 1)
        g = rng.standard_normal((65536, 16)).astype(np.float32)
        o1, o2 = fast.forward(b), part.forward(b)
        assert scaled_max_err(o1, o2) <= 1e-5, s
        fast.backward(b, g)
        part.backward(b, g)
        fast.step(1e-5)
        part.step(1e-5)
        if s == 1:
            fast.finalize_warmup()
            part.finalize_warmup()
        if s >= 2:
            _same_partition(fast.cache.last_partition(), part.cache.last_partition())
    for k in range(3):
        assert scaled_max_err(fast.tt.core(k), part.tt.core(k)) <= 1e-5, k
    assert scaled_max_err(fast.cache.all_row_values(), part.cache.all_row_values()) <= 1e-5
    assert fast.cache.active_hits() == part.cache.active_hits()
    assert fast.cache.active_hits() > 0.7 * fast.cache.active_accesses()


def test_fast_cached_step_replays_from_a_cuda_graph():
    """The fused cached step (forward_device + backward_step_device) has no host
    sync on the fast path: captured once, replayed on new batches copied into
    the same device buffers, it reproduces an eager twin bit for bit."""
    tt = _tt()
    import torch
    from paper_2101_11714_b200._lib import lib
    from paper_2101_11714_b200.lfu_cache import LfuCache
    from paper_2101_11714_b200.ttrec import ForwardContext, _raise

    rows, cap, emb, B = 40000, 48, 16, 4096
    plan = tt.ShapePlan(rows, emb, 3, [30, 34, 40], [2, 2, 4], [1, 16, 16, 1])
    st = torch.cuda.Stream()
    side = []
    for _ in range(2):
        t = tt.TtTable(plan, "g", stream=st.cuda_stream)
        t.init_sampled_gaussian(3)
        c = LfuCache(cap, emb, key_space=rows, stream=st.cuda_stream)
        c.record(tt.generate_zipfian_batch(rows, 1.2, 1, 20000, 1))
        c.warmup_finalize(t)
        side.append((t, c, ForwardContext(t)))
    batches = [tt.generate_zipfian_batch(rows, 1.2, 20 + s, B, 1) for s in range(4)]
    grads = [np.random.default_rng(s).standard_normal((B, emb)).astype(np.float32) for s in range(4)]
    with torch.cuda.stream(st):
        d_idx = torch.empty(B, dtype=torch.int64, device="cuda")
        d_off = torch.empty(B + 1, dtype=torch.int64, device="cuda")
        d_grad = torch.empty((B, emb), dtype=torch.float32, device="cuda")
        d_out = torch.empty((B, emb), dtype=torch.float32, device="cuda")

    def load(s):
        with torch.cuda.stream(st):
            d_idx.copy_(torch.from_numpy(batches[s].indices))
            d_off.copy_(torch.from_numpy(batches[s].offsets))
            d_grad.copy_(torch.from_numpy(grads[s]))

    def step(t, c, ctx):
        _raise(lib().ttgpu_cache_forward_device(c.handle, t.handle, ctx.handle, d_idx.data_ptr(), B,
                                                d_off.data_ptr(), B, None, 0, 1, d_out.data_ptr()))
        _raise(lib().ttgpu_cache_backward_step_device(c.handle, t.handle, ctx.handle,
                                                      d_grad.data_ptr(), 0.05))

    outs = [[], []]
    for which in (0, 1):
        t, c, ctx = side[which]
        load(0)
        step(t, c, ctx)  # sizes every buffer (no allocation under capture)
        st.synchronize()
        outs[which].append(d_out.cpu().numpy())
        if which == 0:
            t.graph_begin()
            step(t, c, ctx)
            t.graph_end()
        for s in range(1, 4):
            load(s)
            if which == 0:
                t.graph_launch()
            else:
                step(t, c, ctx)
            st.synchronize()
            outs[which].append(d_out.cpu().numpy())
    for s in range(4):
        assert np.array_equal(outs[0][s], outs[1][s]), s
    (t0, c0, _), (t1, c1, _) = side
    for k in range(3):
        assert np.array_equal(t0.core(k), t1.core(k)), k
    assert np.array_equal(c0.all_row_values(), c1.all_row_values())
    # the graph's (device-side) access / hit counters advanced with the replays
    assert c0.active_accesses() == c1.active_accesses() == 4 * B
    assert c0.active_hits() == c1.active_hits()
