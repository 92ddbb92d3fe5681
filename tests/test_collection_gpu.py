"""Multi-table TT step (§8(f) f1): the fork/join CUDA graph over the table
streams must give exactly what each table's own step gives (the pipelines
are independent: same kernels, same inputs, same fixed-order reductions)."""
import numpy as np
import pytest

import paper_2101_11714_b200 as tt

pytestmark = pytest.mark.gpu


def test_collection_graph_equals_independent_tables():
    import torch

    from paper_2101_11714_b200.collection import TtEmbeddingCollection, kaggle_plans

    plans = kaggle_plans(32)[4:] + [tt.plan_shapes(5000, 16, 3, 4)]  # 3 fast-path + 1 generic
    col = TtEmbeddingCollection(plans, device=0, seed=5)
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(0)
    host, inputs, keep = [], [], []
    for p in plans:
        b = tt.generate_zipfian_batch(p.num_rows, 1.05, int(rng.integers(1 << 30)), 2048, 2)
        g = rng.standard_normal((b.num_bags(), 16)).astype(np.float32)
        d_idx = torch.from_numpy(b.indices).to(dev)
        d_off = torch.from_numpy(b.offsets).to(dev)
        d_g = torch.from_numpy(g).to(dev)
        d_out = torch.empty((b.num_bags(), 16), device=dev)
        keep += [d_idx, d_off, d_g, d_out]
        host.append((b, g))
        inputs.append((d_idx.data_ptr(), b.num_lookups(), d_off.data_ptr(), b.num_bags(),
                       d_out.data_ptr(), d_g.data_ptr()))
    torch.cuda.synchronize()
    # independent twins on the default path
    twins = []
    for i, p in enumerate(plans):
        t = tt.TtTable(p, f"twin{i}")
        t.set_cores([col.tables[i].core(k) for k in range(3)])
        twins.append(t)
    col.step(inputs, 0.02)                  # eager (allocates workspaces)
    col.synchronize()
    col.capture(inputs, 0.02)
    col.replay()
    col.replay()
    col.synchronize()
    for i, ((b, g), t) in enumerate(zip(host, twins)):
        for _ in range(3):
            res = tt.forward_bags(t, b, save_intermediates=True)
            t.backward_sgd(res.context, b, g, 0.02)
        t.sync()
        for k in range(3):
            assert np.array_equal(col.tables[i].core(k), t.core(k)), (i, k)
