import sys, time
import numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests'); sys.path.insert(0, 'oracle')
import paper_2101_11714_b200 as tt
from paper_2101_11714_b200.lfu_cache import EmbeddingLayer, LfuCache
rows, rf, cf, rk = 40000, [30, 34, 40], [2, 2, 4], [1, 16, 16, 1]
plan = tt.ShapePlan(rows, 16, 3, rf, cf, rk)
t = tt.TtTable(plan, "x"); t.init_sampled_gaussian(7)
c = LfuCache(48, 16, key_space=rows)
lay = EmbeddingLayer(t, c)
idx = tt.generate_zipfian_batch(rows, 1.2, 11, 4000, 1).indices
off = np.arange(4001, dtype=np.int64)
b = tt.IndexBatch(idx, off)
o1 = lay.forward(b)
r = tt.forward_bags(t, b)
o2 = r.output
print("fast nonzero rows", int((np.abs(o1).sum(1) > 0).sum()), "ref nonzero", int((np.abs(o2).sum(1) > 0).sum()), "equal", np.array_equal(o1, o2))
print("kind", t.fast_path_kind())
c2 = LfuCache(48, 16, key_space=rows); c2.set_fast(False)
lay2 = EmbeddingLayer(t, c2)
o3 = lay2.forward(b)
print("partition equal ref", np.array_equal(o3, o2))
t0 = time.time()
rows4 = 10131227
p4 = tt.plan_shapes(rows4, 16, 3, 32, [200, 220, 250], [2, 2, 4])
t4 = tt.TtTable(p4, "cfg4"); t4.init_sampled_gaussian(1)
l4 = EmbeddingLayer(t4, LfuCache(1013, 16, key_space=rows4))
for s in range(4):
    bb = tt.generate_zipfian_batch(rows4, 1.2, 500 + s, 65536, 1)
    t1 = time.time(); o = l4.forward(bb); t2 = time.time()
    g = np.ones((65536, 16), np.float32)
    l4.backward(bb, g); l4.step(1e-5); t3 = time.time()
    print("cfg4 step", s, round(t2 - t1, 3), round(t3 - t2, 3), flush=True)
    if s == 1:
        l4.finalize_warmup(); print("finalized", round(time.time() - t3, 3), flush=True)
