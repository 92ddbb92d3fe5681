import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle'); sys.path.insert(0, 'tests')
import paper_2101_11714_b200 as tt
from pyoracle import Oracle, Plan
from helpers import scaled_max_err
orc = Oracle()
for rank, L, expo in [(32, 16384, 0.0), (32, 4096, 0.0), (32, 16384, 1.05), (16, 16384, 0.0), (8, 4096, 0.0)]:
    p = tt.plan_shapes(10131227, 16, 3, rank, [200, 220, 250], [2, 2, 4])
    t = tt.TtTable(p, "dbg")
    rng = np.random.default_rng(0)
    cores = [(rng.standard_normal(p.core_size(k)) * 0.3).astype(np.float32) for k in range(3)]
    t.set_cores(cores)
    b = tt.generate_zipfian_batch(p.num_rows, expo, 5, L, 1)
    g = rng.standard_normal((L, 16)).astype(np.float32)
    op = Plan(p.num_rows, p.emb_dim, p.row_factors, p.col_factors, p.ranks)
    want = orc.backward(op, cores, b.indices, b.offsets, g)
    r = tt.forward_bags(t, b)
    got = tt.backward_bags(t, b, r.context, g)
    errs = [scaled_max_err(got.cores[k], want[k]) for k in range(3)]
    # which slices are wrong in each core
    bad = []
    for k in range(3):
        d = np.abs(got.cores[k] - want[k]).reshape(p.row_factors[k], -1).max(1)
        bad.append(list(np.nonzero(d > 1e-3 * max(1, np.abs(want[k]).max()))[0][:10]))
    print(rank, L, expo, "kind", t.fast_path_kind(), "errs", ["%.2e" % e for e in errs], "bad", bad, flush=True)
