import sys
import numpy as np
sys.path.insert(0, '.')
import paper_2101_11714_b200 as tt
from paper_2101_11714_b200.lfu_cache import EmbeddingLayer, LfuCache
rows, rf, cf, rk = 40000, [30, 34, 40], [2, 2, 4], [1, 16, 16, 1]
plan = tt.ShapePlan(rows, 16, 3, rf, cf, rk)
t = tt.TtTable(plan, "x"); t.init_sampled_gaussian(7)
c = LfuCache(48, 16, key_space=rows)
lay = EmbeddingLayer(t, c)
rng = np.random.default_rng(0)
stream = tt.generate_zipfian_batch(rows, 1.2, 11, 40000, 1).indices
sizes = rng.integers(0, 6, 2000); sizes[::7] = 1
off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
b = tt.IndexBatch(stream[: off[-1]].copy(), off)
o1 = lay.forward(b)
o2 = tt.forward_bags(t, b).output
print("equal", np.array_equal(o1, o2))
