"""Fused cross-GPU reduce + SGD over peer memory (ttgpu_peer_reduce_sgd).

One B200 is available, so ranks share it: (1) two or three tables in one
process whose peer pointers are each other's buffers
(ttgpu_peer_attach_ptrs), the kernels running concurrently on separate
streams; (2) two processes exchanging CUDA IPC handles (the production path)
over a gloo group.  Checks: replicas bitwise equal, equal to the oracle's
full-batch SGD within 1e-4, and equal to NCCL-free host arithmetic
(core - lr*(g0+g1+...)) bit for bit."""
import ctypes as C
import os
import socket

import numpy as np
import pytest

import paper_2101_11714_b200 as tt
from helpers import scaled_max_err
from pyoracle import Oracle, Plan

pytestmark = pytest.mark.gpu

PLAN_ARGS = (10131227, 16, 3, 32, [200, 220, 250], [2, 2, 4])


def _case():
    plan = tt.plan_shapes(*PLAN_ARGS)
    rng = np.random.default_rng(21)
    cores = [(rng.standard_normal(plan.core_size(k)) * 0.3).astype(np.float32) for k in range(3)]
    b = tt.generate_zipfian_batch(plan.num_rows, 1.05, 4, 4096, 1)
    g = rng.standard_normal((b.num_bags(), 16)).astype(np.float32)
    return plan, cores, b, g


def _oplan(p):
    return Plan(p.num_rows, p.emb_dim, p.row_factors, p.col_factors, p.ranks)


@pytest.mark.parametrize("world", [2, 3])
def test_ranks_in_one_process_concurrent_streams(world):
    """W tables on W streams of this GPU act as the ranks: every rank reduces
    its 1/W shard (W = 3: uneven shards) and pushes it into every replica."""
    import torch

    from paper_2101_11714_b200._lib import lib
    from paper_2101_11714_b200.sharding import partition_bags, shard_batch, shard_rows

    plan, cores, b, g = _case()
    bounds = partition_bags(b.offsets, world)
    streams = [torch.cuda.Stream() for _ in range(world)]
    tabs = []
    for r in range(world):
        t = tt.TtTable(plan, f"rank{r}", stream=streams[r].cuda_stream)
        t.set_cores(cores)
        tabs.append(t)
    flags = []
    for t in tabs:
        p = C.c_void_p()
        assert lib().ttgpu_peer_flags_ptr(t.handle, C.byref(p)) == 0
        flags.append(p.value)
    G = (C.c_void_p * world)(*[t.grad_buffer()[0] for t in tabs])
    Cp = (C.c_void_p * world)(*[t.core_device_ptr(0) for t in tabs])
    F = (C.c_void_p * world)(*flags)
    for r, t in enumerate(tabs):
        assert lib().ttgpu_peer_attach_ptrs(t.handle, world, r, G, Cp, F) == 0, lib().ttgpu_last_error()
    for step in range(2):
        host_g = []
        for r, t in enumerate(tabs):
            sb = shard_batch(b, bounds, r)
            res = tt.forward_bags(t, sb, save_intermediates=True)
            host_g.append(tt.backward_bags(t, sb, res.context, shard_rows(g, bounds, r)))
        before = [tabs[0].core(k) for k in range(3)]
        for t in tabs:
            assert lib().ttgpu_peer_reduce_sgd(t.handle, C.c_double(0.01)) == 0
        for t in tabs:
            t.check()
            st = C.c_int()
            assert lib().ttgpu_peer_status(t.handle, C.byref(st)) == 0 and st.value == 0
        # replicas bitwise equal, and equal to core - lr*(g0 + g1 + ...) in rank order
        for k in range(3):
            gsum = host_g[0].cores[k].copy()
            for r in range(1, world):
                gsum = (gsum + host_g[r].cores[k]).astype(np.float32)
            want = (before[k] - np.float32(0.01) * gsum).astype(np.float32)
            for t in tabs:
                assert np.array_equal(t.core(k), want), k
        if step == 0:
            full = Oracle().backward(_oplan(plan), cores, b.indices, b.offsets, g)
            ref = [c.copy() for c in cores]
            Oracle().sgd(_oplan(plan), ref, full, 0.01)
            for k in range(3):
                assert scaled_max_err(tabs[0].core(k), ref[k]) <= 1e-4


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ipc_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2101_11714_b200.sharding import (PeerReducer, partition_bags, replica_checksum,
                                                shard_batch, shard_rows)

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        plan, cores, b, g = _case()
        stream = torch.cuda.Stream()
        t = tt.TtTable(plan, "ipc", stream=stream.cuda_stream)
        t.set_cores(cores)
        pr = PeerReducer(t)
        bounds = partition_bags(b.offsets, world)
        sb = shard_batch(b, bounds, rank)
        res = tt.forward_bags(t, sb, save_intermediates=True)
        tt.backward_bags(t, sb, res.context, shard_rows(g, bounds, rank))
        dist.barrier()
        pr.reduce_sgd(0.01)
        t.check()
        to = pr.timed_out()
        ck = torch.tensor(replica_checksum([t.core(k) for k in range(3)]), dtype=torch.int64)
        allc = [torch.zeros_like(ck) for _ in range(world)]
        dist.all_gather(allc, ck)
        q.put((rank, to, all(torch.equal(allc[0], c) for c in allc),
               [t.core(k).copy() for k in range(3)]))
    finally:
        dist.destroy_process_group()


def test_two_processes_cuda_ipc():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(2)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    plan, cores, b, g = _case()
    full = Oracle().backward(_oplan(plan), cores, b.indices, b.offsets, g)
    ref = [c.copy() for c in cores]
    Oracle().sgd(_oplan(plan), ref, full, 0.01)
    for rank, timed_out, same, got in res:
        assert not timed_out and same
        for k in range(3):
            assert scaled_max_err(got[k], ref[k]) <= 1e-4
