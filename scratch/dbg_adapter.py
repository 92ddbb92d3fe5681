import sys; sys.path.insert(0,'.'); sys.path.insert(0,'oracle')
import numpy as np
import paper_2101_11714_b200 as tt
from pyoracle import RefImpl
ref = RefImpl()
plan = tt.plan_shapes(127, 16, 4, 1)
print(plan.row_factors, plan.col_factors, plan.ranks)
idx, off, w = ref.random_batch(7, 127, 37, 0, 6, False)
print(len(idx), idx.max(), off[-1])
t = tt.TtTable(plan, "rand0")
rng = np.random.default_rng(0)
t.set_cores([rng.standard_normal(plan.core_size(k)).astype(np.float32) for k in range(4)])
b = tt.IndexBatch(idx, off)
try:
    r = tt.forward_bags(t, b, save_intermediates=True)
    print("ok", r.output.shape)
except Exception as e:
    print("ERR", type(e), e)
