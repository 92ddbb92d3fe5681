"""GPU: the warp-per-chunk wide-row tail kernels (wide3.cuh; cfg3's shape
class: fp32, n0·n1 = 16, R2 = 64, n2 = 4) against the oracle and against the
shared-memory staged kernels they replace (set_wide3(False)).

* forward: bit-identical to the oracle (reference order) and to the old path,
  on ragged weighted batches in Sum and Mean pooling, and on a skewed batch
  whose pair runs span many chunks;
* backward: gradients within 1e-4 of the oracle, and within fp32 rounding of
  the old path (same per-element chains; dG2 slab order differs);
* fused SGD: cores within tolerance of the oracle's SGD of its gradients;
* repeated runs are bitwise equal (deterministic).
"""
import numpy as np
import pytest

import paper_2101_11714_b200 as tt
from helpers import scaled_max_err
from pyoracle import Oracle, Plan

pytestmark = pytest.mark.gpu
GRAD_TOL = 1e-4


def _plan():
    return tt.ShapePlan(20 * 30 * 50, 64, 3, [20, 30, 50], [4, 4, 4], [1, 64, 64, 1])


def _oplan(p):
    return Plan(p.num_rows, p.emb_dim, list(p.row_factors), list(p.col_factors), list(p.ranks))


def _table(p, seed, wide3):
    t = tt.TtTable(p, "w3")
    rng = np.random.default_rng(seed)
    cores = [(rng.standard_normal(p.core_size(k)) * 0.1).astype(np.float32) for k in range(3)]
    t.set_cores(cores)
    t.set_wide3(wide3)
    return t, cores


def _batches(p):
    rng = np.random.default_rng(3)
    out = []
    for pooling, weighted in ((tt.Pooling.Sum, False), (tt.Pooling.Mean, True)):
        sizes = rng.integers(0, 40, 300)
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        idx = rng.integers(0, p.num_rows, int(off[-1])).astype(np.int64)
        w = rng.uniform(-2, 2, len(idx)) if weighted else None
        out.append(tt.IndexBatch(idx, off, w, pooling))
    # skew: a few rows repeated -> pair runs spanning many 32-lookup chunks
    idx = np.concatenate([np.zeros(3000, np.int64), rng.integers(0, 2000, 2000),
                          np.full(1000, p.num_rows - 1, np.int64)])
    rng.shuffle(idx)
    out.append(tt.IndexBatch(idx, np.arange(0, len(idx) + 1, 8, dtype=np.int64)))
    return out


@pytest.mark.parametrize("case", [0, 1, 2])
def test_wide3_forward_backward_vs_oracle_and_staged_path(case):
    p = _plan()
    b = _batches(p)[case]
    orc = Oracle()
    op = _oplan(p)
    tw, cores = _table(p, 1, True)
    to, _ = _table(p, 1, False)
    g = np.random.default_rng(9).standard_normal((b.num_bags(), 64)).astype(np.float32)
    w = b.weights if b.has_weights() else None
    want_y = orc.forward(op, cores, b.indices, b.offsets, w, int(b.pooling))
    rw = tt.forward_bags(tw, b)
    ro = tt.forward_bags(to, b)
    assert np.array_equal(rw.output, want_y), "wide3 forward not bit-identical to the oracle"
    assert np.array_equal(rw.output, ro.output)
    gw = tt.backward_bags(tw, b, rw.context, g)
    go = tt.backward_bags(to, b, ro.context, g)
    want = orc.backward(op, cores, b.indices, b.offsets, g, w, int(b.pooling))
    for k in range(3):
        assert scaled_max_err(gw.cores[k], want[k]) <= GRAD_TOL, k
        assert scaled_max_err(gw.cores[k], go.cores[k]) <= 1e-5, k
    # deterministic
    gw2 = tt.backward_bags(tw, b, rw.context, g)
    for k in range(3):
        assert np.array_equal(gw.cores[k], gw2.cores[k]), k


def test_wide3_fused_step_vs_oracle_sgd():
    p = _plan()
    b = _batches(p)[0]
    orc = Oracle()
    op = _oplan(p)
    t, cores = _table(p, 2, True)
    g = np.random.default_rng(5).standard_normal((b.num_bags(), 64)).astype(np.float32)
    want = orc.backward(op, cores, b.indices, b.offsets, g)
    res = tt.forward_bags(t, b)
    t.backward_sgd(res.context, b, g, 0.01)
    for k in range(3):
        exp = cores[k] - np.float32(0.01) * want[k]
        assert scaled_max_err(t.core(k), exp) <= GRAD_TOL, k
