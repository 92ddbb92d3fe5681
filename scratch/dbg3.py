import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle'); sys.path.insert(0, 'tests')
import paper_2101_11714_b200 as tt
p = tt.plan_shapes(10131227, 16, 3, 32, [200, 220, 250], [2, 2, 4])
rng = np.random.default_rng(0)
cores = [(rng.standard_normal(p.core_size(k)) * 0.3).astype(np.float32) for k in range(3)]
t = tt.TtTable(p, "dbg"); t.set_cores(cores)
L = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
b = tt.generate_zipfian_batch(p.num_rows, 0.0, 5, L, 1)
g = rng.standard_normal((L, 16)).astype(np.float32)
r = tt.forward_bags(t, b); got = tt.backward_bags(t, b, r.context, g)
print("done", float(np.abs(got.cores[0]).sum()))
