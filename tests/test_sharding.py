"""Multi-GPU host logic on CPU: bag sharding, the SUM
allreduce of dense core gradients, identical SGD on every replica, and the LFU
frequency sync -- world_size 2 over `gloo`, with the CPU oracle standing in for
the per-rank GPU backward (tests only).  The GPU side of the same helpers is
covered by tests/test_parity_gpu.py::test_data_parallel_world1_nccl."""
import os
import socket

import numpy as np
import pytest

from paper_2101_11714_b200 import IndexBatch, Pooling
from paper_2101_11714_b200.sharding import (equal_bag_bounds, partition_bags, replica_checksum,
                                            shard_batch, shard_rows)
from pyoracle import Oracle, Plan, ref_available


def _ref_partition(offsets, workers):
    """embedding_ops.hpp:50-62 restated with an explicit lower_bound loop."""
    bags, lookups = len(offsets) - 1, int(offsets[-1])
    bounds = [bags] * (workers + 1)
    bounds[0] = 0
    for w in range(1, workers):
        target = lookups * w // workers
        b = 0
        while b < len(offsets) and offsets[b] < target:
            b += 1
        bounds[w] = min(max(b, bounds[w - 1]), bags)
    return bounds


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("workers", [1, 2, 3, 4, 8])
def test_partition_bags_matches_reference(seed, workers):
    rng = np.random.default_rng(seed)
    bags = int(rng.integers(0, 40))
    sizes = rng.integers(0, 6, bags)
    if seed == 0:
        sizes[:] = 0  # all-empty bags
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    got = partition_bags(off, workers)
    assert list(got) == _ref_partition(off, workers)
    assert got[0] == 0 and got[-1] == bags and np.all(np.diff(got) >= 0)


def _random_batch(rng, rows, bags, weighted, pooling):
    sizes = rng.integers(0, 5, bags)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    idx = rng.integers(0, rows, int(off[-1])).astype(np.int64)
    w = rng.uniform(-1, 1, len(idx)) if weighted else None
    return IndexBatch(idx, off, w, pooling)


@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_shards_concatenate_to_batch(world):
    rng = np.random.default_rng(world)
    b = _random_batch(rng, 1000, 37, True, Pooling.Mean)
    for bounds in (partition_bags(b.offsets, world), equal_bag_bounds(b.num_bags(), world)):
        parts = [shard_batch(b, bounds, r) for r in range(world)]
        assert np.array_equal(np.concatenate([p.indices for p in parts]), b.indices)
        assert np.array_equal(np.concatenate([p.weights for p in parts]), b.weights)
        assert sum(p.num_bags() for p in parts) == b.num_bags()
        for r, p in enumerate(parts):
            assert p.offsets[0] == 0 and p.pooling == Pooling.Mean
            sizes = np.diff(b.offsets)[bounds[r]: bounds[r + 1]]
            assert np.array_equal(np.diff(p.offsets), sizes)
        g = rng.standard_normal((b.num_bags(), 4))
        assert np.array_equal(np.concatenate([shard_rows(g, bounds, r) for r in range(world)]), g)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


PLAN = Plan(5000, 16, [10, 20, 25], [2, 2, 4], [1, 6, 5, 1])


def _case(dtype):
    rng = np.random.default_rng(11)
    cores = [rng.standard_normal(PLAN.core_size(k)).astype(dtype) * 0.5 for k in range(3)]
    batch = _random_batch(rng, PLAN.num_rows, 61, True, Pooling.Mean)
    grad = rng.standard_normal((batch.num_bags(), PLAN.emb_dim)).astype(dtype)
    return cores, batch, grad


def _dp_worker(rank, world, port, dtype, q):
    import torch
    import torch.distributed as dist

    from paper_2101_11714_b200.sharding import allreduce_sum_

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = Oracle()
        cores, batch, grad = _case(dtype)
        bounds = partition_bags(batch.offsets, world)
        sb = shard_batch(batch, bounds, rank)
        sg = shard_rows(grad, bounds, rank)
        # this rank's dense gradient (the GPU backward_bags in production)
        g = orc.backward(PLAN, cores, sb.indices, sb.offsets, sg, sb.weights, int(sb.pooling))
        flat = torch.from_numpy(np.concatenate(g).copy())
        allreduce_sum_(flat)  # the one collective
        sizes = [PLAN.core_size(k) for k in range(3)]
        summed = np.split(flat.numpy(), np.cumsum(sizes)[:-1])
        after = [c.copy() for c in cores]
        orc.sgd(PLAN, after, summed, 0.05)
        ck = torch.tensor(replica_checksum(after), dtype=torch.int64)
        all_ck = [torch.zeros_like(ck) for _ in range(world)]
        dist.all_gather(all_ck, ck)
        q.put((rank, [s.copy() for s in summed], [a.copy() for a in after],
               all(torch.equal(all_ck[0], c) for c in all_ck)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dtype,tol", [(np.float64, 1e-12), (np.float32, 1e-4)])
def test_gloo_world2_allreduce_equals_full_batch(dtype, tol):
    import torch.multiprocessing as mp

    from helpers import scaled_max_err

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dp_worker, args=(r, world, port, dtype, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    orc = Oracle()
    cores, batch, grad = _case(dtype)
    full = orc.backward(PLAN, cores, batch.indices, batch.offsets, grad, batch.weights,
                        int(batch.pooling))
    want_after = [c.copy() for c in cores]
    orc.sgd(PLAN, want_after, full, 0.05)
    for _, summed, after, same in res:
        assert same, "replicas diverged"
        for k in range(3):
            assert scaled_max_err(summed[k], full[k]) <= tol
            assert scaled_max_err(after[k], want_after[k]) <= tol
    # both ranks hold bitwise identical replicas
    for k in range(3):
        assert np.array_equal(res[0][2][k], res[1][2][k])


def _freq_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2101_11714_b200.sharding import FrequencySync

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        keys = 500
        counts = torch.zeros(keys, dtype=torch.int64)
        fs = FrequencySync(counts)
        rng = np.random.default_rng(3)
        streams = [rng.zipf(1.3, 4000) % keys for _ in range(3 * world)]
        for phase in range(3):  # record, sync (= an admission point), repeat
            s = streams[phase * world + rank]
            counts += torch.bincount(torch.from_numpy(s.astype(np.int64)), minlength=keys)
            fs.sync()
        q.put((rank, counts.numpy().copy()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_frequency_sync_gives_global_counts():
    import torch.multiprocessing as mp

    from lfu_oracle import LfuOracle

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_freq_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(3)
    streams = [rng.zipf(1.3, 4000) % 500 for _ in range(3 * world)]
    want = np.bincount(np.concatenate(streams).astype(np.int64), minlength=500)
    assert np.array_equal(res[0][1], want) and np.array_equal(res[1][1], want)
    # the same hot set on every replica: top_k by (count desc, row asc), lfu_cache.cpp:98-113
    orc = LfuOracle(20, 4)
    orc.record(np.concatenate(streams).astype(np.int64))
    top = orc.top_k(20)
    order = sorted(range(500), key=lambda r: (-int(res[0][1][r]), r))[:20]
    assert list(top) == order


@pytest.mark.skipif(not ref_available(), reason="reference build (oracle/_ref) not present")
def test_partition_bags_on_reference_batches():
    from pyoracle import RefImpl

    ref = RefImpl()
    for seed in range(4):
        idx, off, w = ref.random_batch(seed, 1000, 50, 0, 7, True)
        for workers in (2, 3, 8):
            assert list(partition_bags(off, workers)) == _ref_partition(list(off), workers)


def _coalesced_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2101_11714_b200.sharding import allreduce_sum_coalesced_

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        bufs = [torch.full((n,), float(rank + 1) * (k + 1)) for k, n in enumerate((7, 3, 11))]
        allreduce_sum_coalesced_(bufs)
        q.put((rank, [b.numpy().copy() for b in bufs]))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_coalesced_allreduce_of_table_gradients():
    """The multi-table step reduces every table's gradient buffer in one group."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_coalesced_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, bufs in res:
        for k, b in enumerate(bufs):
            assert np.all(b == 3.0 * (k + 1))
