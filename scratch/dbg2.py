import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle'); sys.path.insert(0, 'tests')
import paper_2101_11714_b200 as tt
from pyoracle import Oracle, Plan
from helpers import scaled_max_err
orc = Oracle()
p = tt.plan_shapes(10131227, 16, 3, 32, [200, 220, 250], [2, 2, 4])
op = Plan(p.num_rows, p.emb_dim, p.row_factors, p.col_factors, p.ranks)
rng = np.random.default_rng(0)
cores = [(rng.standard_normal(p.core_size(k)) * 0.3).astype(np.float32) for k in range(3)]
for L in [8192, 10000, 12000, 14000, 16384, 24000, 32768, 65536]:
    t = tt.TtTable(p, "dbg"); t.set_cores(cores)
    b = tt.generate_zipfian_batch(p.num_rows, 0.0, 5, L, 1)
    g = rng.standard_normal((L, 16)).astype(np.float32)
    want = orc.backward(op, cores, b.indices, b.offsets, g)
    r = tt.forward_bags(t, b); got = tt.backward_bags(t, b, r.context, g)
    r = tt.forward_bags(t, b); got2 = tt.backward_bags(t, b, r.context, g)
    print(L, ["%.1e" % scaled_max_err(got.cores[k], want[k]) for k in range(3)],
          "repeat-equal", all(np.array_equal(got.cores[k], got2.cores[k]) for k in range(3)), flush=True)
