"""Data-parallel DLRM step check (run under torchrun; tests/test_dlrm_multirank_gpu.py):
every rank trains its half of each global batch with DlrmModel's single flat
allreduce of all gradients; rank 0 then trains a non-parallel twin on the full
batches and checks that every parameter agrees (fp32 tolerance)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_11714_b200 as tt  # noqa: E402
from paper_2101_11714_b200.dlrm import DlrmModel  # noqa: E402


def scaled_max_err(a, b):
    """max|a-b| / max(1, max|a|, max|b|) (tests/helpers.py, oracle_helpers.hpp:43-53)."""
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(np.max(np.abs(a - b)) / max(1.0, np.max(np.abs(a)), np.max(np.abs(b))))

dist.init_process_group(os.environ.get("DP_BACKEND", "gloo"))
rank, world = dist.get_rank(), dist.get_world_size()
dev = int(os.environ.get("DP_DEVICE", "0"))
torch.cuda.set_device(dev)
tables = [(20000, True, 8), (800, False, 0), (50000, True, 16), (300, False, 0)]
bottom, top, BS, STEPS = [32, 16], [8, 1], 512, 4


def batch(it):
    rng = np.random.default_rng(100 + it)
    return {"dense": rng.standard_normal((BS, 3)).astype(np.float32),
            "labels": rng.integers(0, 2, BS).astype(np.float64),
            "idx": [tt.generate_zipfian_batch(n, 1.05, 1000 * it + t, BS, 1).indices for t, (n, _, _) in
                    enumerate(tables)],
            "off": [np.arange(BS + 1, dtype=np.int64) for _ in tables]}


def shard(mb, r, w):
    lo, hi = r * BS // w, (r + 1) * BS // w
    return {"dense": mb["dense"][lo:hi], "labels": mb["labels"][lo:hi],
            "idx": [i[lo:hi] for i in mb["idx"]], "off": [np.arange(hi - lo + 1, dtype=np.int64)
                                                        for _ in mb["off"]]}


m = DlrmModel(3, 16, tables, bottom, top, device=dev)
m.init(5)
assert m.world == world
losses = []
for it in range(STEPS):
    _, loss = m.train_step(m.to_device(shard(batch(it), rank, world)), 0.05)
    losses.append(float(loss.item()))
if rank == 0:
    ref = DlrmModel(3, 16, tables, bottom, top, device=dev, data_parallel=False)
    ref.init(5)
    for it in range(STEPS):
        _, loss = ref.train_step(ref.to_device(batch(it)), 0.05)
        assert abs(float(loss.item()) - losses[it]) <= 1e-5 * max(1.0, abs(losses[it])), (it, losses[it])
    for which, layers in (("bottom", bottom), ("top", top)):
        for i in range(len(layers)):
            a, b = m.mlp_params(which, i), ref.mlp_params(which, i)
            assert scaled_max_err(a[0], b[0]) <= 1e-4 and scaled_max_err(a[1], b[1]) <= 1e-4, (which, i)
    for t, (_, use_tt, _) in enumerate(tables):
        if use_tt:
            for k in range(3):
                assert scaled_max_err(m.tt_core(t, k), ref.tt_core(t, k)) <= 1e-4, (t, k)
        else:
            assert scaled_max_err(m.dense_table(t), ref.dense_table(t)) <= 1e-4, t
    print("dp ok", losses, flush=True)
dist.barrier()
dist.destroy_process_group()
