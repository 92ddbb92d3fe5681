"""Multi-table TT embedding step (BASELINE cfg5's TT part).

The 7 largest Criteo-Kaggle tables TT-compressed at rank 32 (paper Table 2,
the reference's kRefTables, tools/ttrec.cpp:30-34), each one TtTable on its
own CUDA stream.  One training step runs every table's forward_bags(save) +
backward_bags + sgd_step; the per-table pipelines are independent, so they
are captured into ONE CUDA graph with a fork/join over the table streams:
each table's kernels are short latency-bound launches that leave most SMs
idle, and the graph lets the 7 pipelines fill the GPU together.

Multi-GPU (`world > 1`): batch-sharded like DataParallelTable; every table's
dense core gradient goes into one coalesced NCCL allreduce(SUM) (a single
collective group for all 7 buffers), then the identical SGD per replica.

The 19 uncompressed DLRM features run as one DenseEmbeddingBags group
(dense.py) on its own stream of the same graph.  Not here: the MLPs and the
interaction (out of scope) -- this is the embedding part
of the cfg5 step.
"""
from __future__ import annotations

from typing import List, Sequence

import numpy as np

from .ttrec import ForwardContext, ShapePlan, TtTable, plan_shapes

# paper Table 2 / the reference's kRefTables (tools/ttrec.cpp:30-34): rows, row factors
KAGGLE_TT_TABLES = [
    (10131227, [200, 220, 250]), (8351593, [200, 200, 209]), (7046547, [200, 200, 200]),
    (5461306, [166, 175, 188]), (2202608, [125, 130, 136]), (286181, [53, 72, 75]),
    (142572, [50, 52, 55]),
]


def kaggle_plans(rank: int = 32, emb_dim: int = 16) -> List[ShapePlan]:
    return [plan_shapes(n, emb_dim, 3, rank, rf, [2, 2, 4]) for n, rf in KAGGLE_TT_TABLES]


class TtEmbeddingCollection:
    """Several TtTables trained in one step; inputs are device pointers."""

    def __init__(self, plans: Sequence[ShapePlan], names: Sequence[str] = (), device: int = 0,
                 seed: int = 1, group=None, dense_rows: Sequence[int] = (), dense_dim: int = 16):
        import torch
        import torch.distributed as dist

        self.torch = torch
        self.device = device
        self.dev = torch.device("cuda", device)
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.streams = [torch.cuda.Stream(device=self.dev) for _ in plans]
        self.main = torch.cuda.Stream(device=self.dev)
        self.tables: List[TtTable] = []
        for i, p in enumerate(plans):
            name = names[i] if i < len(names) else f"tt{i}"
            t = TtTable(p, name, np.float32, device=device, stream=self.streams[i].cuda_stream)
            t.init_sampled_gaussian(seed + i)
            # the one-kernel cooperative sort occupies every SM, so the tables'
            # sorts would serialise across the graph's streams; the three-kernel
            # sort lets them overlap (cfg5: 0.75 -> 0.70 ms)
            t.set_grid_sort(False)
            self.tables.append(t)
        self.ctxs = [ForwardContext(t) for t in self.tables]
        # the uncompressed features (dense.py): one group on its own stream
        self.dense = None
        if dense_rows:
            from .dense import DenseEmbeddingBags

            self.dense_stream = torch.cuda.Stream(device=self.dev)
            self.dense = DenseEmbeddingBags(dense_rows, dense_dim, device=device,
                                            stream=self.dense_stream.cuda_stream)
            self.dense.init_uniform(seed + 1000)
            self._dense_grad = None
            if self.world > 1:
                from .sharding import _device_view

                ptr, n = self.dense.grad_buffer()
                self._dense_grad = _device_view(ptr, n, "<f4", device)
        self.graph = None
        self._grad_views = None
        self.reducers = None
        if self.world > 1:
            from .sharding import PeerReducer, _device_view

            views = []
            for t in self.tables:
                ptr, n = t.grad_buffer()
                views.append(_device_view(ptr, n, "<f4", device))
            self._grad_views = views
            # fused reduce+SGD over peer memory per table when every rank can
            # attach (one kernel per table, graph-capturable); else NCCL
            ok = 1
            reducers = []
            try:
                for t in self.tables:
                    reducers.append(PeerReducer(t, group))
            except Exception:  # noqa: BLE001
                ok = 0
            flag = torch.tensor([ok], device=self.dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
            self.reducers = reducers if int(flag.item()) else None

    @property
    def capturable(self) -> bool:
        """The step can be captured as one CUDA graph (no host-side collective)."""
        if self.world == 1:
            return True
        return self.reducers is not None and self.dense is None

    def _table_step(self, i, idx_ptr, L, off_ptr, B, out_ptr, grad_ptr, lr):
        t, c = self.tables[i], self.ctxs[i]
        t.forward_device(c, idx_ptr, L, off_ptr, B, out_ptr, save=True)
        if self.world == 1:
            t.backward_sgd_device(c, grad_ptr, lr)
        elif self.reducers is not None:
            t.backward_device(c, grad_ptr)
            self.reducers[i].reduce_sgd(lr)
        else:
            t.backward_device(c, grad_ptr)

    def step(self, inputs, lr: float, dense_inputs=None):
        """inputs: per TT table (idx_ptr, L, off_ptr, B, out_ptr, grad_ptr);
        dense_inputs: (idx_ptr [n_dense x L], L, off_ptr, B, out_ptr, grad_ptr) for
        the uncompressed group.  Forks the table streams off `main`, joins them
        back; with world > 1 the gradients are reduced before the SGD."""
        torch = self.torch
        ev0 = torch.cuda.Event()
        ev0.record(self.main)
        for i, s in enumerate(self.streams):
            s.wait_event(ev0)
            self._table_step(i, *inputs[i], lr)
        streams = list(self.streams)
        if self.dense is not None and dense_inputs is not None:
            di, dl, do, db, dout, dg = dense_inputs
            self.dense_stream.wait_event(ev0)
            self.dense.forward_device(di, dl, do, db, dout)
            if self.world == 1:
                self.dense.backward_device(dg, lr, fused=True)
            else:
                self.dense.backward_device(dg, 0.0, fused=False)
                import torch.distributed as dist

                with torch.cuda.stream(self.dense_stream):
                    dist.all_reduce(self._dense_grad, op=dist.ReduceOp.SUM, group=self.group)
                self.dense.apply_grad(lr)
            streams.append(self.dense_stream)
        for s in streams:
            e = torch.cuda.Event()
            e.record(s)
            self.main.wait_event(e)
        if self.world > 1 and self.reducers is None:
            from .sharding import allreduce_sum_coalesced_

            with torch.cuda.stream(self.main):
                allreduce_sum_coalesced_(self._grad_views, self.group)
            ev1 = torch.cuda.Event()
            ev1.record(self.main)
            for i, s in enumerate(self.streams):
                s.wait_event(ev1)
                self.tables[i].apply_grad(lr)
            for s in self.streams:
                e = torch.cuda.Event()
                e.record(s)
                self.main.wait_event(e)

    def capture(self, inputs, lr: float, dense_inputs=None):
        """One CUDA graph of the whole multi-table step (fork/join over the
        table streams).  Workspaces must already exist (run step() once)."""
        torch = self.torch
        g = torch.cuda.CUDAGraph()
        torch.cuda.synchronize(self.dev)
        with torch.cuda.graph(g, stream=self.main):
            self.step(inputs, lr, dense_inputs)
        self.graph = g
        return g

    def replay(self):
        self.graph.replay()

    def synchronize(self):
        self.torch.cuda.synchronize(self.dev)
        for t in self.tables:
            t.check()
        if self.dense is not None:
            self.dense.check()
