"""Batch-sharded data parallelism for TT tables.

One process per GPU, cores replicated on every rank, the batch split into
contiguous bag ranges.  Each rank runs forward_bags + backward_bags on its
shard into the table's dense gradient buffer; the only collective is one
allreduce(SUM) of that buffer (reference semantics sum over all lookups,
embedding_ops.hpp:355-357 -- not a mean), followed by the identical
`core -= lr * g` on every replica (embedding_ops.hpp:361-376), so the replicas
stay bitwise equal.

For the LFU cache (lfu_cache.hpp:187-243) the dense per-row frequency counters
are allreduced (SUM) before `warmup_finalize` / `refresh`, so every replica
admits the same hot set.

The host logic here (bag partitioning, shard extraction, the allreduce
helpers) is backend-agnostic and is exercised with world_size-2 `gloo` tests on
CPU (tests/test_sharding.py); on the GPU box the same helpers run over NCCL on
the device buffers the C ABI exposes (ttgpu_grad_buffer,
ttgpu_cache_counts_device_ptr).
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np

from .ttrec import ForwardContext, IndexBatch, InvalidArgument, TtTable


def partition_bags(offsets: np.ndarray, workers: int) -> np.ndarray:
    """detail::partition_bags (embedding_ops.hpp:50-62): contiguous bag ranges
    with roughly equal lookup counts, `workers + 1` bounds.  bounds[w] is the
    first bag whose offset is >= L*w/workers (lower_bound), clamped to be
    non-decreasing."""
    if workers < 1:
        raise InvalidArgument(f"workers must be positive, got {workers}")
    offsets = np.asarray(offsets, np.int64)
    bags = len(offsets) - 1
    lookups = int(offsets[-1])
    bounds = np.full(workers + 1, bags, np.int64)
    bounds[0] = 0
    for w in range(1, workers):
        target = lookups * w // workers
        b = int(np.searchsorted(offsets, target, side="left"))
        bounds[w] = min(max(b, int(bounds[w - 1])), bags)
    return bounds


def equal_bag_bounds(num_bags: int, workers: int) -> np.ndarray:
    """Equal bag counts per rank (the weak-scaling bench's split: a fixed
    number of bags per GPU, so the pooled-output rows split evenly)."""
    return np.array([num_bags * w // workers for w in range(workers + 1)], np.int64)


def shard_batch(batch: IndexBatch, bounds: np.ndarray, rank: int) -> IndexBatch:
    """The sub-batch of bags [bounds[rank], bounds[rank+1]) with offsets rebased
    to 0; weights sliced alongside, pooling kept (so Mean divides by the same
    bag sizes as on one GPU)."""
    b0, b1 = int(bounds[rank]), int(bounds[rank + 1])
    lo, hi = int(batch.offsets[b0]), int(batch.offsets[b1])
    off = batch.offsets[b0: b1 + 1] - lo
    w = batch.weights[lo:hi] if batch.has_weights() else None
    return IndexBatch(batch.indices[lo:hi], off, w, batch.pooling)


def shard_rows(x: np.ndarray, bounds: np.ndarray, rank: int) -> np.ndarray:
    """Rows of a (num_bags x N) array (pooled output or grad_output) owned by `rank`."""
    return x[int(bounds[rank]): int(bounds[rank + 1])]


def allreduce_sum_(tensor, group=None):
    """In-place SUM allreduce of a core-gradient / frequency buffer (one
    collective; NCCL on the GPU, gloo in the CPU tests)."""
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(tensor, op=dist.ReduceOp.SUM, group=group)
    return tensor


def allreduce_sum_coalesced_(tensors, group=None):
    """SUM-allreduce several buffers as ONE collective group (NCCL coalescing:
    one launch for all of a multi-table step's core gradients); backends
    without coalescing (gloo in the CPU tests) reduce them one by one."""
    import torch.distributed as dist

    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return tensors
    if dist.get_backend(group) == "nccl":
        with dist._coalescing_manager(group=group, device=tensors[0].device):
            for t in tensors:
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    else:
        for t in tensors:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return tensors


def _device_view(ptr: int, n: int, typestr: str, device: int):
    """Zero-copy torch view of a library-owned device buffer."""
    import torch

    class _Arr:
        __cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                    "version": 3, "strides": None}

    return torch.as_tensor(_Arr(), device=torch.device("cuda", device))


class DataParallelTable:
    """A replicated TtTable trained on this rank's bag shard.

    step(): forward_device(save) -> backward_device (dense gradient into the
    table's buffer) -> allreduce(SUM) over the process group on the table's
    stream -> apply_grad(lr).  With world_size 1 the collective is skipped and
    the fused backward+SGD path is used instead."""

    def __init__(self, table: TtTable, group=None, device: int = 0):
        import torch
        import torch.distributed as dist

        self.table = table
        self.group = group
        self.device = device
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.ctx = ForwardContext(table)
        ptr, n = table.grad_buffer()
        self.grad_view = _device_view(ptr, n, "<f8" if table.dtype == np.float64 else "<f4",
                                      device)
        self._torch = torch

    def broadcast_cores(self, src: int = 0):
        """Make every replica start from rank src's cores (one broadcast per core)."""
        import torch.distributed as dist

        if self.world == 1:
            return
        for k in range(self.table.dim()):
            n = self.table.plan().core_size(k)
            v = _device_view(self.table.core_device_ptr(k), n,
                             "<f8" if self.table.dtype == np.float64 else "<f4", self.device)
            self.table.sync()
            dist.broadcast(v, src, group=self.group)
        self._torch.cuda.synchronize(self.device)
        self.table.mark_mutated()

    def forward(self, idx_ptr: int, L: int, off_ptr: int, B: int, out_ptr: int,
                weights_ptr: int = 0, pooling: int = 0):
        self.table.forward_device(self.ctx, idx_ptr, L, off_ptr, B, out_ptr, weights_ptr, pooling,
                                  save=True)

    def backward_step(self, grad_ptr: int, lr: float, stream=None):
        """backward -> allreduce(SUM) -> SGD, all ordered on the table's stream.
        With an explicit `stream` for the collective, events order it after the
        backward and the SGD after it (no race on the gradient buffer)."""
        if self.world == 1:
            self.table.backward_sgd_device(self.ctx, grad_ptr, lr)
            return
        torch = self._torch
        self.table.backward_device(self.ctx, grad_ptr)
        ts = torch.cuda.ExternalStream(self.table.stream, device=self.device) \
            if self.table.stream else torch.cuda.default_stream(self.device)
        s = stream if stream is not None else ts
        if s.cuda_stream != ts.cuda_stream:
            s.wait_stream(ts)  # the collective reads the finished gradient
        with torch.cuda.stream(s):
            allreduce_sum_(self.grad_view, self.group)
        if s.cuda_stream != ts.cuda_stream:
            ts.wait_stream(s)  # the SGD reads the reduced gradient
        self.table.apply_grad(lr)


class PeerReducer:
    """Fused reduce + SGD over peer memory for one replicated table
    (ttgpu_peer_reduce_sgd): a reduce-scatter + all-gather over NVLink in
    one kernel -- each rank sums its 1/W shard of every rank's dense gradient
    in rank order, applies the SGD and stores the result into every replica's
    cores.  The NCCL allreduce and the separate SGD launch disappear.
    Handles (gradients, cores, flags) are exchanged once with an all_gather
    on `group`."""

    def __init__(self, table: TtTable, group=None):
        import ctypes as C

        import torch
        import torch.distributed as dist

        from ._lib import lib
        from .ttrec import _raise

        self.table = table
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        gh = (C.c_char * 64)()
        ch = (C.c_char * 64)()
        fh = (C.c_char * 64)()
        # a failed export still joins the (collective) exchange, flagged, so no
        # rank is left waiting; every rank then raises together
        exported = lib().ttgpu_peer_export(table.handle, gh, ch, fh) == 0
        mine = torch.tensor(list(bytes(gh)) + list(bytes(ch)) + list(bytes(fh)) +
                            [1 if exported else 0], dtype=torch.uint8)
        if world > 1:
            bufs = [torch.zeros_like(mine) for _ in range(world)]
            dist.all_gather_object(bufs, mine, group=group)
        else:
            bufs = [mine]
        if not all(int(b[192]) for b in bufs):
            raise RuntimeError("peer reduce: a rank could not export its buffers")
        allg = b"".join(bytes(b[:64].tolist()) for b in bufs)
        allc = b"".join(bytes(b[64:128].tolist()) for b in bufs)
        allf = b"".join(bytes(b[128:192].tolist()) for b in bufs)
        self._g = C.create_string_buffer(allg, len(allg))
        self._c = C.create_string_buffer(allc, len(allc))
        self._f = C.create_string_buffer(allf, len(allf))
        _raise(lib().ttgpu_peer_attach(table.handle, world, rank, self._g, self._c, self._f))
        self.world, self.rank = world, rank

    def reduce_sgd(self, lr: float):
        from ._lib import lib
        from .ttrec import _raise

        _raise(lib().ttgpu_peer_reduce_sgd(self.table.handle, float(lr)))

    def timed_out(self) -> bool:
        import ctypes as C

        from ._lib import lib
        from .ttrec import _raise

        v = C.c_int()
        _raise(lib().ttgpu_peer_status(self.table.handle, C.byref(v)))
        return bool(v.value)


def replica_checksum(cores: List[np.ndarray]) -> Tuple[int, ...]:
    """Bitwise fingerprint of a replica's cores (for cross-rank equality checks)."""
    import hashlib

    h = hashlib.sha256()
    for c in cores:
        h.update(np.ascontiguousarray(c).tobytes())
    return tuple(h.digest()[:8])


class FrequencySync:
    """LFU cache (lfu_cache.hpp:187-243) under data parallelism: every replica
    must admit the same hot set, so the dense per-row frequency counters are
    made global before `warmup_finalize` / `refresh`.  Counters keep growing
    between admissions, so only the increments since the last sync are summed
    (a plain allreduce of the running counts would re-add earlier totals):
    delta = counts - snapshot; allreduce(delta, SUM); counts = snapshot + delta.
    After sync() every rank holds identical counts, hence identical top_k
    (count desc, row asc)."""

    def __init__(self, counts, group=None):
        self.counts = counts
        self.group = group
        self.snapshot = counts.clone()

    def sync(self):
        delta = self.counts - self.snapshot
        allreduce_sum_(delta, self.group)
        self.counts.copy_(self.snapshot + delta)
        self.snapshot.copy_(self.counts)
        return self.counts


def cache_counts_view(cache, device: int = 0):
    """Device view of an LfuCache's dense uint64 frequency counters (int64 for torch)."""
    import ctypes as C

    from ._lib import lib
    from .ttrec import _raise

    p, n = C.c_void_p(), C.c_int64()
    _raise(lib().ttgpu_cache_counts_device_ptr(cache.handle, C.byref(p), C.byref(n)))
    return _device_view(p.value, n.value, "<i8", device)


__all__ = ["partition_bags", "equal_bag_bounds", "shard_batch", "shard_rows", "allreduce_sum_",
           "allreduce_sum_coalesced_", "PeerReducer",
           "DataParallelTable", "replica_checksum", "FrequencySync", "cache_counts_view"]
