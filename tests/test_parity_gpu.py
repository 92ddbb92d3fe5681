"""GPU parity: the CUDA path through the C ABI vs the CPU oracle on identical
inputs.  Mirrors the reference's kernel tests (test_embedding_ops.cpp:44-353,
acceptance.cpp criteria 2/3) plus the BASELINE configs.

Tolerances (BASELINE.json north_star): forward rel 1e-5, gradients rel 1e-4
(scaled_max_err, oracle_helpers.hpp:43-53).  With exact forward (the default)
forward_bags and lookup_row are additionally required to be BIT-identical to
the oracle, which is itself bit-identical to the reference.
"""
import numpy as np
import pytest

import paper_2101_11714_b200 as tt
from helpers import CFG2, CFG3, cfg1, scaled_max_err, small_cases
from pyoracle import Oracle, Plan, RefImpl, ref_available

pytestmark = pytest.mark.gpu

FWD_TOL = 1e-5
GRAD_TOL = 1e-4


@pytest.fixture(scope="module")
def orc():
    return Oracle()


def as_oplan(p: tt.ShapePlan) -> Plan:
    return Plan(p.num_rows, p.emb_dim, p.row_factors, p.col_factors, p.ranks)


def to_tt(p: Plan) -> tt.ShapePlan:
    return tt.ShapePlan(p.num_rows, p.emb_dim, p.tt_dim, list(p.row_factors), list(p.col_factors),
                        list(p.ranks))


def make_table(plan, dtype, seed, name="t", scale=1.0):
    t = tt.TtTable(plan, name, dtype)
    rng = np.random.default_rng(seed)
    cores = [(rng.standard_normal(plan.core_size(k)) * scale).astype(dtype)
             for k in range(plan.tt_dim)]
    t.set_cores(cores)
    return t, cores


def random_batch(rng, rows, bags, lo, hi, weighted, pooling):
    sizes = rng.integers(lo, hi + 1, bags)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    idx = rng.integers(0, rows, int(off[-1])).astype(np.int64)
    w = rng.uniform(-2, 2, len(idx)) if weighted else None
    return tt.IndexBatch(idx, off, w, pooling)


def small_plan(rng):
    d = int(rng.integers(2, 5))
    rank = int(rng.integers(1, 9))
    rows = int(rng.integers(10, 300))
    return tt.plan_shapes(rows, 16, d, rank, None, [2, 2, 2, 2] if d == 4 else None), rows


# ------------------------------------------------------------ goldens ----
def test_golden_small_cases():
    """Reference-generated cases: forward bit-exact, grads within tolerance,
    sgd_step with the reference's gradients bit-exact."""
    for c in small_cases():
        p = to_tt(c["plan"])
        t = tt.TtTable(p, "golden", c["dtype"])
        t.set_cores(c["cores"])
        b = tt.IndexBatch(c["idx"], c["off"], c["w"], tt.Pooling(c["pooling"]))
        res = tt.forward_bags(t, b)
        assert np.array_equal(res.output, c["fwd"])
        g = tt.backward_bags(t, b, res.context, c["grad_out"])
        tol = 1e-12 if c["dtype"] == np.float64 else GRAD_TOL
        for k in range(p.tt_dim):
            assert scaled_max_err(g.cores[k], c["grads"][k]) <= tol
        tt.sgd_step(t, tt.CoreGradients(c["grads"]), 0.05)
        for k in range(p.tt_dim):
            assert np.array_equal(t.core(k), c["after"][k])


def test_golden_cfg1():
    """BASELINE configs[0] (1M rows, R=16, 4096 uniform) from the reference."""
    plan, z = cfg1()
    p = to_tt(plan)
    t = tt.TtTable(p, "cfg1")
    t.set_cores([z[f"core{k}"] for k in range(3)])
    b = tt.IndexBatch(z["idx"], z["off"])
    res = tt.forward_bags(t, b, save_intermediates=True)
    assert np.array_equal(res.output, z["fwd"])
    g = tt.backward_bags(t, b, res.context, z["grad_out"])
    for k in range(3):
        assert scaled_max_err(g.cores[k], z[f"grad{k}"]) <= GRAD_TOL
    for r, want in zip(z["rows"], z["lookup"]):
        assert np.array_equal(tt.lookup_row(t, int(r)), want)


# ------------------------------------------- test_embedding_ops.cpp ports --
def test_lookup_row_matches_oracle_and_bounds(orc):
    rng = np.random.default_rng(101)
    for trial in range(10):
        p, rows = small_plan(rng)
        for dt in (np.float32, np.float64):
            t, cores = make_table(p, dt, 500 + trial, "lk")
            for r in rng.integers(0, rows, 20):
                assert np.array_equal(tt.lookup_row(t, int(r)),
                                      orc.lookup_row(as_oplan(p), cores, int(r)))
    t = tt.TtTable(tt.plan_shapes(50, 16, 3, 2), "bounds")
    with pytest.raises(tt.OutOfRange, match="bounds"):
        tt.lookup_row(t, 50)
    with pytest.raises(tt.OutOfRange):
        tt.lookup_row(t, -1)


@pytest.mark.parametrize("exact", [True, False])
def test_forward_random_plans(orc, exact):
    rng = np.random.default_rng(202)
    for trial in range(30):
        p, rows = small_plan(rng)
        pooling = tt.Pooling.Mean if trial % 3 == 0 else tt.Pooling.Sum
        b = random_batch(rng, rows, int(rng.integers(1, 24)), 0, 8, trial % 2 == 1, pooling)
        for dt in (np.float32, np.float64):
            t, cores = make_table(p, dt, 900 + trial, "fw")
            t.set_exact_forward(exact)
            got = tt.forward_bags(t, b, int(rng.integers(1, 64))).output
            want = orc.forward(as_oplan(p), cores, b.indices, b.offsets, b.weights, int(pooling))
            if exact:
                assert np.array_equal(got, want)
            else:
                tol = 1e-12 if dt == np.float64 else FWD_TOL
                assert scaled_max_err(got, want) <= tol


def test_forward_independent_of_micro_batch():
    rng = np.random.default_rng(303)
    p = tt.plan_shapes(500, 16, 3, 8)
    t, _ = make_table(p, np.float32, 3)
    b = random_batch(rng, 500, 64, 0, 12, True, tt.Pooling.Mean)
    base = tt.forward_bags(t, b, tt.kDefaultMicroBatch).output
    for mb in (1, 2, 3, 7, 61, 4096):
        assert np.array_equal(base, tt.forward_bags(t, b, mb).output)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_backward_random_plans(orc, dtype):
    rng = np.random.default_rng(404)
    for trial in range(24):
        p, rows = small_plan(rng)
        pooling = tt.Pooling.Mean if trial % 2 else tt.Pooling.Sum
        t, cores = make_table(p, dtype, 40 + trial)
        b = random_batch(rng, rows, 16, 0, 6, trial % 3 == 0, pooling)
        g = rng.standard_normal((b.num_bags(), 16)).astype(dtype)
        res = tt.forward_bags(t, b, 7, trial % 2 == 0)
        got = tt.backward_bags(t, b, res.context, g)
        want = orc.backward(as_oplan(p), cores, b.indices, b.offsets, g, b.weights, int(pooling))
        tol = 1e-11 if dtype == np.float64 else GRAD_TOL
        for k in range(p.tt_dim):
            assert scaled_max_err(got.cores[k], want[k]) <= tol, (trial, k)


def test_saved_and_recomputed_backward_bitwise():
    rng = np.random.default_rng(404)
    for trial in range(6):
        p, rows = small_plan(rng)
        t, _ = make_table(p, np.float32, 40 + trial)
        b = random_batch(rng, rows, 16, 0, 6, trial % 2 == 0, tt.Pooling.Sum)
        g = rng.standard_normal((b.num_bags(), 16)).astype(np.float32)
        saved = tt.forward_bags(t, b, 7, True)
        recomputed = tt.forward_bags(t, b, 7, False)
        assert np.array_equal(saved.output, recomputed.output)
        gs = tt.backward_bags(t, b, saved.context, g)
        gr = tt.backward_bags(t, b, recomputed.context, g)
        for k in range(p.tt_dim):
            assert np.array_equal(gs.cores[k], gr.cores[k])


def test_backward_deterministic():
    rng = np.random.default_rng(7)
    p = tt.plan_shapes(10131227, 16, 3, 32, [200, 220, 250], [2, 2, 4])
    t, _ = make_table(p, np.float32, 1, scale=0.2)
    b = tt.generate_zipfian_batch(p.num_rows, 1.05, 11, 8192, 1)
    g = rng.standard_normal((8192, 16)).astype(np.float32)
    r1 = tt.forward_bags(t, b)
    a = tt.backward_bags(t, b, r1.context, g)
    r2 = tt.forward_bags(t, b)
    c = tt.backward_bags(t, b, r2.context, g)
    assert np.array_equal(r1.output, r2.output)
    for k in range(3):
        assert np.array_equal(a.cores[k], c.cores[k])


def test_backward_finite_differences():
    # test_embedding_ops.cpp:169-205 in f64 on the GPU
    rng = np.random.default_rng(606)
    for trial in range(8):
        d = int(rng.integers(2, 5))
        cols = [2, 2, 2, 1] if d == 4 else None
        p = tt.plan_shapes(int(rng.integers(8, 60)), 8, d, int(rng.integers(1, 5)), None, cols)
        t, cores = make_table(p, np.float64, 60 + trial)
        pooling = tt.Pooling.Sum if trial % 2 == 0 else tt.Pooling.Mean
        b = random_batch(rng, p.num_rows, 6, 0, 4, trial % 3 == 0, pooling)
        g = rng.standard_normal((b.num_bags(), p.emb_dim))
        res = tt.forward_bags(t, b, 5, trial % 2 == 0)
        grads = tt.backward_bags(t, b, res.context, g)

        def loss(cs):
            t.set_cores(cs)
            return float((tt.forward_bags(t, b).output * g).sum())

        h = 1e-6
        for _ in range(12):
            k = int(rng.integers(0, d))
            i = int(rng.integers(0, cores[k].size))
            up = [c.copy() for c in cores]
            dn = [c.copy() for c in cores]
            up[k][i] += h
            dn[k][i] -= h
            fd = (loss(up) - loss(dn)) / (2 * h)
            an = grads.cores[k][i]
            assert abs(fd - an) <= 1e-6 * max(1.0, abs(fd), abs(an))
        t.set_cores(cores)


def test_gradients_linear_in_upstream():
    rng = np.random.default_rng(707)
    p = tt.plan_shapes(80, 16, 3, 4)
    t, _ = make_table(p, np.float64, 12)
    b = random_batch(rng, 80, 10, 1, 4, False, tt.Pooling.Sum)
    g1 = rng.standard_normal((10, 16))
    g2 = rng.standard_normal((10, 16))
    ctx = tt.forward_bags(t, b).context
    b1 = tt.backward_bags(t, b, ctx, g1)
    b2 = tt.backward_bags(t, b, ctx, g2)
    bs = tt.backward_bags(t, b, ctx, g1 + g2)
    for k in range(3):
        assert scaled_max_err(b1.cores[k] + b2.cores[k], bs.cores[k]) <= 1e-12


def test_one_param_per_core_exact_sgd_and_stale():
    p = tt.plan_shapes(1, 1, 2, 1, [1, 1], [1, 1])
    t = tt.TtTable(p, "one", np.float64)
    t.set_core(0, [3.0])
    t.set_core(1, [5.0])
    b = tt.IndexBatch.singles([0])
    fwd = tt.forward_bags(t, b)
    assert fwd.output[0, 0] == 15.0
    g = tt.backward_bags(t, b, fwd.context, [1.0])
    assert g.cores[0][0] == 5.0 and g.cores[1][0] == 3.0
    tt.sgd_step(t, g, 0.1)
    assert t.core(0)[0] == pytest.approx(2.5) and t.core(1)[0] == pytest.approx(4.7)
    with pytest.raises(tt.InvalidArgument, match="stale"):
        tt.backward_bags(t, b, fwd.context, [1.0])


def test_empty_bags_and_batches(orc):
    p = tt.plan_shapes(40, 16, 3, 2)
    t, cores = make_table(p, np.float32, 9)
    empty = tt.IndexBatch(pooling=tt.Pooling.Mean)
    r = tt.forward_bags(t, empty)
    assert r.output.shape == (0, 16)
    g = tt.backward_bags(t, empty, r.context, np.zeros(0, np.float32))
    assert g.total_elements() == p.parameter_count()
    assert all(np.all(c == 0) for c in g.cores)
    mixed = tt.IndexBatch([1, 2, 3], [0, 2, 2, 3], None, tt.Pooling.Mean)
    out = tt.forward_bags(t, mixed).output
    assert np.all(out[1] == 0)
    assert np.array_equal(out, orc.forward(as_oplan(p), cores, [1, 2, 3], [0, 2, 2, 3], None, 1))
    # all bags empty, lookups zero
    allempty = tt.IndexBatch(np.zeros(0, np.int64), [0, 0, 0], None, tt.Pooling.Mean)
    r = tt.forward_bags(t, allempty)
    assert np.all(r.output == 0)
    g = tt.backward_bags(t, allempty, r.context, np.ones((2, 16), np.float32))
    assert all(np.all(c == 0) for c in g.cores)


def test_invalid_inputs_rejected():
    p = tt.plan_shapes(40, 16, 3, 2)
    a, _ = make_table(p, np.float32, 1, "alpha")
    bt, _ = make_table(p, np.float32, 2, "beta")
    batch = tt.IndexBatch.singles([0, 1, 2])
    fwd = tt.forward_bags(a, batch)
    grad = np.ones((3, 16), np.float32)
    with pytest.raises(tt.InvalidArgument):
        tt.backward_bags(bt, batch, fwd.context, grad)
    with pytest.raises(tt.InvalidArgument):
        tt.backward_bags(a, tt.IndexBatch.singles([0, 1]), fwd.context, grad)
    with pytest.raises(tt.InvalidArgument):
        tt.backward_bags(a, batch, fwd.context, np.ones(3, np.float32))
    with pytest.raises(tt.InvalidArgument):
        tt.forward_bags(a, batch, 0)
    with pytest.raises(tt.OutOfRange, match="alpha"):
        tt.forward_bags(a, tt.IndexBatch.singles([40]))
    with pytest.raises(tt.OutOfRange, match="alpha"):
        tt.forward_bags(a, tt.IndexBatch.singles([0, 5, -3]))
    with pytest.raises(tt.InvalidArgument):
        tt.forward_bags(a, tt.IndexBatch([0, 1], [0, 2, 1]))
    # the table keeps working after a rejected batch
    assert np.array_equal(tt.forward_bags(a, batch).output, fwd.output)


def test_row_counter():
    p = tt.plan_shapes(300, 16, 3, 8)
    t, _ = make_table(p, np.float32, 21)
    rng = np.random.default_rng(909)
    b = random_batch(rng, 300, 128, 2, 6, False, tt.Pooling.Sum)
    tt.EmbeddingStats.reset()
    fwd = tt.forward_bags(t, b, 32)
    assert tt.EmbeddingStats.tt_rows_computed() == b.num_lookups()
    tt.backward_bags(t, b, fwd.context, np.ones((128, 16), np.float32))
    assert tt.EmbeddingStats.tt_rows_computed() == b.num_lookups()
    tt.lookup_row(t, 5)
    assert tt.EmbeddingStats.tt_rows_computed() == b.num_lookups() + 1
    assert tt.EmbeddingStats.peak_workspace_bytes() > 0


# ----------------------------------------------------- BASELINE configs --
def test_cfg2_full_batch(orc):
    """configs[1]: 10,131,227 x 16, R=32, 65,536 x 1 Zipf(1.05), fwd+bwd+SGD."""
    p = tt.plan_shapes(10131227, 16, 3, 32, [200, 220, 250], [2, 2, 4])
    t = tt.TtTable(p, "cfg2")
    t.init_sampled_gaussian(1)
    cores = t.cores()
    b = tt.generate_zipfian_batch(p.num_rows, 1.05, 7, 65536, 1)
    rng = np.random.default_rng(2)
    g = rng.standard_normal((65536, 16)).astype(np.float32)
    res = tt.forward_bags(t, b, save_intermediates=True)
    op = as_oplan(p)
    assert np.array_equal(res.output, orc.forward(op, cores, b.indices, b.offsets))
    grads = tt.backward_bags(t, b, res.context, g)
    want = orc.backward(op, cores, b.indices, b.offsets, g)
    for k in range(3):
        assert scaled_max_err(grads.cores[k], want[k]) <= GRAD_TOL
    tt.sgd_step(t, grads, 0.01)
    orc.sgd(op, cores, grads.cores, 0.01)
    for k in range(3):
        assert np.array_equal(t.core(k), cores[k])


@pytest.mark.parametrize("exponent", [0.0, 1.05, 1.2])
def test_fused_device_step_matches_oracle(orc, exponent):
    """The bench path: device API, fused backward+SGD, vs oracle fwd+bwd+sgd."""
    import torch

    p = tt.plan_shapes(10131227, 16, 3, 32, [200, 220, 250], [2, 2, 4])
    t = tt.TtTable(p, "cfg2dev")
    t.init_sampled_gaussian(1)
    cores = t.cores()
    b = tt.generate_zipfian_batch(p.num_rows, exponent, 5, 16384, 1)
    g = np.random.default_rng(3).standard_normal((16384, 16)).astype(np.float32)
    dev = torch.device("cuda:0")
    idx = torch.from_numpy(b.indices).to(dev)
    off = torch.from_numpy(b.offsets).to(dev)
    gd = torch.from_numpy(g).to(dev)
    out = torch.empty((16384, 16), dtype=torch.float32, device=dev)
    ctx = tt.ForwardContext(t)
    t.set_exact_forward(False)
    t.forward_device(ctx, idx.data_ptr(), 16384, off.data_ptr(), 16384, out.data_ptr())
    t.backward_sgd_device(ctx, gd.data_ptr(), 0.01)
    t.check()
    op = as_oplan(p)
    want_out = orc.forward(op, cores, b.indices, b.offsets)
    assert scaled_max_err(out.cpu().numpy(), want_out) <= FWD_TOL
    want_g = orc.backward(op, cores, b.indices, b.offsets, g)
    for k in range(3):
        # the gradient implied by the fused in-place update (core - lr*g)
        implied = (cores[k].astype(np.float64) - t.core(k).astype(np.float64)) / 0.01
        ulp_slack = np.abs(cores[k]).max() * 2.0 ** -23 / 0.01  # f32 rounding of the update
        err = np.abs(implied - want_g[k]).max() / max(1.0, np.abs(want_g[k]).max())
        assert err <= GRAD_TOL + ulp_slack / max(1.0, np.abs(want_g[k]).max())


@pytest.mark.parametrize("tensor", [True, False])
def test_cfg3_subsample(orc, tensor):
    """configs[2] shape (40M rows, dim 64 = 4x4x4, R=64, P=32) on 256 bags;
    head backward on the tcgen05 3xTF32 path and on the FFMA path."""
    p = tt.plan_shapes(40000000, 64, 3, 64, [200, 200, 1000], [4, 4, 4])
    t, cores = make_table(p, np.float32, 5, "cfg3", scale=0.1)
    t.set_tensor_path(tensor)
    rng = np.random.default_rng(8)
    idx = rng.integers(0, p.num_rows, 256 * 32).astype(np.int64)
    off = np.arange(0, 256 * 32 + 1, 32, dtype=np.int64)
    b = tt.IndexBatch(idx, off)
    g = rng.standard_normal((256, 64)).astype(np.float32)
    res = tt.forward_bags(t, b)
    op = as_oplan(p)
    assert np.array_equal(res.output, orc.forward(op, cores, idx, off))
    grads = tt.backward_bags(t, b, res.context, g)
    want = orc.backward(op, cores, idx, off, g)
    for k in range(3):
        assert scaled_max_err(grads.cores[k], want[k]) <= GRAD_TOL


def test_skewed_segments_large_runs(orc):
    """Every lookup on one row (a single huge pair / i2 segment) and a mix."""
    p = tt.plan_shapes(10131227, 16, 3, 32, [200, 220, 250], [2, 2, 4])
    t, cores = make_table(p, np.float32, 6, scale=0.2)
    rng = np.random.default_rng(4)
    for idx in (np.zeros(20000, np.int64), np.full(5000, 10131226, np.int64),
                np.concatenate([np.zeros(7000, np.int64), rng.integers(0, 300, 3000)])):
        off = np.arange(len(idx) + 1, dtype=np.int64)
        g = rng.standard_normal((len(idx), 16)).astype(np.float32)
        b = tt.IndexBatch(idx, off)
        res = tt.forward_bags(t, b)
        grads = tt.backward_bags(t, b, res.context, g)
        want = orc.backward(as_oplan(p), cores, idx, off, g)
        for k in range(3):
            assert scaled_max_err(grads.cores[k], want[k]) <= GRAD_TOL


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_init_matches_reference_initializer():
    ref = RefImpl()
    p = tt.plan_shapes(10131227, 16, 3, 32, [200, 220, 250], [2, 2, 4])
    t = tt.TtTable(p, "init")
    t.init_sampled_gaussian(1)
    r = ref.table(as_oplan(p), np.float32, "init")
    r.init_sampled_gaussian(1)
    for a, b in zip(t.cores(), r.get_cores()):
        assert np.array_equal(a, b)


# ------------------------------------------------ specialised 3-core path --
@pytest.mark.parametrize("rank", [4, 8, 16, 32, 64])
@pytest.mark.parametrize("exponent", [0.0, 1.2])
def test_fast_path_vs_oracle_and_generic(orc, rank, exponent):
    """The compiled-shape fast path (tile counting sort, smem partials) against
    the oracle and against the generic pipeline on the same inputs; multi-hot,
    weighted, Mean-pooled bags with empties."""
    p = tt.plan_shapes(10131227, 16, 3, rank, [200, 220, 250], [2, 2, 4])
    t, cores = make_table(p, np.float32, rank, "fast", scale=0.3)
    assert t.fast_path_kind() >= 0
    rng = np.random.default_rng(rank)
    base = tt.generate_zipfian_batch(p.num_rows, exponent, 3, 3000, 3)
    sizes = rng.integers(0, 6, 3000)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    idx = np.resize(base.indices, int(off[-1])).astype(np.int64)
    w = rng.uniform(-2, 2, len(idx))
    b = tt.IndexBatch(idx, off, w, tt.Pooling.Mean)
    g = rng.standard_normal((3000, 16)).astype(np.float32)
    op = as_oplan(p)
    res = tt.forward_bags(t, b)
    assert np.array_equal(res.output, orc.forward(op, cores, idx, off, w, 1))
    got = tt.backward_bags(t, b, res.context, g)
    want = orc.backward(op, cores, idx, off, g, w, 1)
    for k in range(3):
        assert scaled_max_err(got.cores[k], want[k]) <= GRAD_TOL
    t.set_generic_path(True)
    assert t.fast_path_kind() == -1
    res2 = tt.forward_bags(t, b)
    assert np.array_equal(res2.output, res.output)
    got2 = tt.backward_bags(t, b, res2.context, g)
    for k in range(3):
        assert scaled_max_err(got.cores[k], got2.cores[k]) <= GRAD_TOL


@pytest.mark.parametrize("nlook", [1, 2, 31, 32, 33, 65, 100])
def test_fast_path_tiny_batches(orc, nlook):
    """Batches with fewer tiles than CTAs (pipeline prologue only, ragged last
    tile, one bucket, repeated rows) through the fast path against the oracle."""
    p = tt.plan_shapes(10131227, 16, 3, 32, [200, 220, 250], [2, 2, 4])
    t, cores = make_table(p, np.float32, 32, "tiny", scale=0.3)
    assert t.fast_path_kind() >= 0
    rng = np.random.default_rng(nlook)
    # half the lookups share bucket i1 = 0 (rows < 250), the rest anywhere
    idx = np.where(rng.random(nlook) < 0.5, rng.integers(0, 250, nlook),
                   rng.integers(0, p.num_rows, nlook)).astype(np.int64)
    nb = max(1, nlook // 2)
    cuts = np.sort(rng.integers(0, nlook + 1, nb - 1))
    off = np.concatenate([[0], cuts, [nlook]]).astype(np.int64)
    b = tt.IndexBatch(idx, off)
    g = rng.standard_normal((nb, 16)).astype(np.float32)
    op = as_oplan(p)
    res = tt.forward_bags(t, b)
    assert np.array_equal(res.output, orc.forward(op, cores, idx, off))
    got = tt.backward_bags(t, b, res.context, g)
    want = orc.backward(op, cores, idx, off, g)
    for k in range(3):
        assert scaled_max_err(got.cores[k], want[k]) <= GRAD_TOL


def test_fast_path_fused_sgd_equals_dense_then_sgd():
    p = tt.plan_shapes(10131227, 16, 3, 32, [200, 220, 250], [2, 2, 4])
    a, cores = make_table(p, np.float32, 9, "a", scale=0.3)
    b_, _ = make_table(p, np.float32, 9, "b", scale=0.3)
    batch = tt.generate_zipfian_batch(p.num_rows, 1.05, 9, 20000, 1)
    g = np.random.default_rng(9).standard_normal((20000, 16)).astype(np.float32)
    ra = tt.forward_bags(a, batch)
    grads = tt.backward_bags(a, batch, ra.context, g)
    tt.sgd_step(a, grads, 0.01)
    rb = tt.forward_bags(b_, batch)
    b_.backward_sgd(rb.context, batch, g, 0.01)
    for k in range(3):
        assert np.array_equal(a.core(k), b_.core(k))
    with pytest.raises(tt.InvalidArgument, match="stale"):
        b_.backward_sgd(rb.context, batch, g, 0.01)


@pytest.mark.parametrize("d", [3, 4, 5])
def test_generic_fused_sgd_multistep_equals_dense_then_sgd(d):
    """Several fused backward+SGD steps on DIFFERENT batches equal
    backward_bags + sgd_step each step (generic path, d >= 4 included: the
    tail cores' untouched slices must not re-apply an earlier step's gradient)."""
    rows = 3000
    emb = 32 if d == 5 else 16
    p = tt.plan_shapes(rows, emb, d, 4, None, {4: [2, 2, 2, 2], 5: [2, 2, 2, 2, 2]}.get(d))
    a, _ = make_table(p, np.float32, 21, "a", scale=0.5)
    b_, _ = make_table(p, np.float32, 21, "b", scale=0.5)
    a.set_generic_path(True)
    b_.set_generic_path(True)
    rng = np.random.default_rng(22)
    for step in range(4):
        # small batches over a few rows: most tail slices are untouched each step
        batch = random_batch(rng, min(rows, 40 + 30 * step), 24, 1, 3, False, tt.Pooling.Sum)
        g = rng.standard_normal((24, emb)).astype(np.float32)
        ra = tt.forward_bags(a, batch)
        tt.sgd_step(a, tt.backward_bags(a, batch, ra.context, g), 0.05)
        rb = tt.forward_bags(b_, batch)
        b_.backward_sgd(rb.context, batch, g, 0.05)
        for k in range(d):
            assert np.array_equal(a.core(k), b_.core(k)), f"step {step} core {k}"


def test_data_parallel_shards_sum_to_full_batch(orc):
    """§8(e) on one GPU: the dense gradients of two bag shards (what two ranks
    produce before the allreduce) sum to the full-batch gradient, and the
    DataParallelTable step through a world-1 NCCL group equals the fused step."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    from paper_2101_11714_b200.sharding import DataParallelTable, partition_bags, shard_batch, shard_rows

    plan = tt.plan_shapes(CFG2.num_rows, 16, 3, 32, CFG2.row_factors, CFG2.col_factors)
    rng = np.random.default_rng(5)
    table, cores = make_table(plan, np.float32, 3, scale=0.3)
    b = tt.generate_zipfian_batch(plan.num_rows, 1.05, 9, 4096, 2)
    g = rng.standard_normal((b.num_bags(), 16)).astype(np.float32)
    full = orc.backward(as_oplan(plan), cores, b.indices, b.offsets, g)
    bounds = partition_bags(b.offsets, 2)
    acc = [np.zeros_like(c) for c in cores]
    for r in range(2):
        sb = shard_batch(b, bounds, r)
        res = tt.forward_bags(table, sb)
        gr = tt.backward_bags(table, sb, res.context, shard_rows(g, bounds, r))
        for k in range(3):
            acc[k] += gr.cores[k]
    for k in range(3):
        assert scaled_max_err(acc[k], full[k]) <= GRAD_TOL

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        stream = torch.cuda.Stream()
        t2 = tt.TtTable(plan, "dp", np.float32, stream=stream.cuda_stream)
        t2.set_cores(cores)
        dp = DataParallelTable(t2)
        dp.broadcast_cores()
        d_idx = torch.from_numpy(b.indices).to(dev)
        d_off = torch.from_numpy(b.offsets).to(dev)
        d_g = torch.from_numpy(g).to(dev)
        d_out = torch.empty((b.num_bags(), 16), device=dev)
        torch.cuda.synchronize()
        dp.forward(d_idx.data_ptr(), b.num_lookups(), d_off.data_ptr(), b.num_bags(),
                   d_out.data_ptr())
        dp.backward_step(d_g.data_ptr(), 0.01, stream=stream)
        t2.check()
        want = [c.copy() for c in cores]
        orc.sgd(as_oplan(plan), want, full, 0.01)
        for k in range(3):
            assert scaled_max_err(t2.core(k), want[k]) <= GRAD_TOL
        assert np.array_equal(d_out.cpu().numpy(),
                              orc.forward(as_oplan(plan), cores, b.indices, b.offsets))
    finally:
        dist.destroy_process_group()


def test_host_api_graph_replay_matches_eager(orc):
    """Host C-ABI calls replay a cached graph of their kernels from the third
    call with the same shape on; results must equal the eager calls (and the
    oracle) through shape changes, weights and workspace growth."""
    import torch

    p = tt.plan_shapes(CFG2.num_rows, 16, 3, 32, CFG2.row_factors, CFG2.col_factors)
    stream = torch.cuda.Stream()
    t = tt.TtTable(p, "replay", stream=stream.cuda_stream)
    rng = np.random.default_rng(17)
    cores = [(rng.standard_normal(p.core_size(k)) * 0.3).astype(np.float32) for k in range(3)]
    t.set_cores(cores)
    ctx = tt.ForwardContext(t)
    shapes = [(2048, False), (2048, False), (2048, False), (2048, False), (512, True), (2048, False),
              (2048, False), (4096, True), (2048, False), (2048, False)]
    import ctypes as C

    from paper_2101_11714_b200._lib import lib

    cur = [c.copy() for c in cores]
    for n, weighted in shapes:
        b = tt.generate_zipfian_batch(p.num_rows, 1.05, int(rng.integers(1 << 20)), n, 2)
        w = rng.uniform(-1, 1, b.num_lookups()) if weighted else None
        out = np.zeros((n, 16), np.float32)
        st = lib().ttgpu_forward(t.handle, b.indices.ctypes.data_as(C.c_void_p), b.num_lookups(),
                                 b.offsets.ctypes.data_as(C.c_void_p), n,
                                 None if w is None else w.ctypes.data_as(C.c_void_p), 0, 2048, 1,
                                 out.ctypes.data_as(C.c_void_p), ctx.handle)
        assert st == 0, lib().ttgpu_last_error()
        want = orc.forward(as_oplan(p), cur, b.indices, b.offsets, w)
        assert np.array_equal(out, want)
        g = rng.standard_normal((n, 16)).astype(np.float32)
        ctx._fill(t, b.num_lookups(), n, True)
        t.backward_sgd(ctx, b, g, 1e-4)
        full = orc.backward(as_oplan(p), cur, b.indices, b.offsets, g, w)
        orc.sgd(as_oplan(p), cur, full, 1e-4)
        for k in range(3):
            assert np.all(np.isfinite(t.core(k)))
            assert scaled_max_err(t.core(k), cur[k]) <= GRAD_TOL
        cur = [t.core(k).copy() for k in range(3)]  # track the device state exactly


@pytest.mark.parametrize("nbags", [1, 3, 40, 700])
def test_tensor_head_ragged_runs(orc, nbags):
    """tcgen05 head backward with runs of 1..32 pairs (padded operand rows),
    many i1 values, Mean pooling and weights: gradients within 1e-4 of the
    oracle and of the FFMA path."""
    p = tt.plan_shapes(40000000, 64, 3, 64, [200, 200, 1000], [4, 4, 4])
    rng = np.random.default_rng(nbags)
    # few i0 per i1 for small batches, every i0 for the large one
    rows = rng.integers(0, p.num_rows, nbags * 5).astype(np.int64)
    off = np.arange(0, nbags * 5 + 1, 5, dtype=np.int64)
    w = rng.uniform(0.5, 1.5, len(rows))
    b = tt.IndexBatch(rows, off, w, tt.Pooling.Mean)
    g = rng.standard_normal((nbags, 64)).astype(np.float32)
    op = as_oplan(p)
    got = {}
    for tensor in (True, False):
        t, cores = make_table(p, np.float32, 77, "tc", scale=0.1)
        t.set_tensor_path(tensor)
        res = tt.forward_bags(t, b)
        got[tensor] = tt.backward_bags(t, b, res.context, g)
    want = orc.backward(op, cores, rows, off, g, w, int(tt.Pooling.Mean))
    for k in range(3):
        assert scaled_max_err(got[True].cores[k], want[k]) <= GRAD_TOL
        assert scaled_max_err(got[True].cores[k], got[False].cores[k]) <= GRAD_TOL


@pytest.mark.parametrize("nlook", [1, 45, 4096, 65536, 131072, 131073])
def test_grid_sort_equals_three_kernel_sort(orc, nlook):
    """The one-kernel cooperative sort (gsort.cuh) produces the same permutations, tiles and
    bag data as f3_hist + f3_scan + f3_scatter, so forward outputs and gradients
    are BITWISE equal between the two paths (131,073 lookups exceeds one
    cluster: both runs take the three-kernel sort).  Multi-hot weighted Mean
    bags with empties; checked against the oracle too."""
    p = tt.plan_shapes(10131227, 16, 3, 32, [200, 220, 250], [2, 2, 4])
    t, cores = make_table(p, np.float32, 5, "csort", scale=0.3)
    rng = np.random.default_rng(nlook)
    base = tt.generate_zipfian_batch(p.num_rows, 1.05, 11, nlook, 1)
    idx = base.indices.astype(np.int64)
    nb = max(1, nlook // 3)
    cuts = np.sort(rng.integers(0, nlook + 1, nb - 1))
    off = np.concatenate([[0], cuts, [nlook]]).astype(np.int64)
    w = rng.uniform(-2, 2, nlook)
    b = tt.IndexBatch(idx, off, w, tt.Pooling.Mean)
    g = rng.standard_normal((nb, 16)).astype(np.float32)
    outs, grads = [], []
    for on in (True, False):
        t.set_grid_sort(on)
        res = tt.forward_bags(t, b)
        outs.append(res.output)
        grads.append(tt.backward_bags(t, b, res.context, g).cores)
    assert np.array_equal(outs[0], outs[1])
    for k in range(3):
        assert np.array_equal(grads[0][k], grads[1][k])
    op = as_oplan(p)
    assert np.array_equal(outs[0], orc.forward(op, cores, idx, off, w, 1))
    if nlook <= 4096:
        want = orc.backward(op, cores, idx, off, g, w, 1)
        for k in range(3):
            assert scaled_max_err(grads[0][k], want[k]) <= GRAD_TOL


@pytest.mark.parametrize("rank", [8, 32, 64])
@pytest.mark.parametrize("exponent", [0.0, 1.05])
def test_chunked_vs_tile_kernels(orc, rank, exponent):
    """The chunked kernels (fastc.cuh: 64-lookup bucket chunks, CTA-wide i0
    dedup, fused S/dG1/D0 backward) against the 32-lookup tile kernels and the
    oracle: forward bit-identical, gradients within tolerance, fused SGD
    deterministic across repeats."""
    p = tt.plan_shapes(10131227, 16, 3, rank, [200, 220, 250], [2, 2, 4])
    t, cores = make_table(p, np.float32, rank + 1, "chunk", scale=0.3)
    rng = np.random.default_rng(rank)
    nb = 5000
    base = tt.generate_zipfian_batch(p.num_rows, exponent, 5, nb, 2)
    sizes = rng.integers(0, 4, nb)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    idx = np.resize(base.indices, int(off[-1])).astype(np.int64)
    w = rng.uniform(-2, 2, len(idx))
    b = tt.IndexBatch(idx, off, w, tt.Pooling.Mean)
    g = rng.standard_normal((nb, 16)).astype(np.float32)
    op = as_oplan(p)
    want_out = orc.forward(op, cores, idx, off, w, 1)
    want = orc.backward(op, cores, idx, off, g, w, 1)
    got = {}
    for on in (True, False):
        t.set_chunked(on)
        res = tt.forward_bags(t, b)
        assert np.array_equal(res.output, want_out)
        got[on] = tt.backward_bags(t, b, res.context, g).cores
        for k in range(3):
            assert scaled_max_err(got[on][k], want[k]) <= GRAD_TOL
    t.set_chunked(True)
    res = tt.forward_bags(t, b)
    again = tt.backward_bags(t, b, res.context, g).cores
    for k in range(3):
        assert np.array_equal(again[k], got[True][k])


@pytest.mark.parametrize("rank,nlook", [(32, 1), (32, 45), (32, 4096), (32, 65536), (8, 4096), (64, 4096)])
def test_bwd1_planned_ranges_bitwise(orc, monkeypatch, rank, nlook):
    """f3_bwd1's tile ranges planned once by f3_srows_bwd2's first CTA
    (plan_bwd1) are the ranges every bwd1 CTA derives itself
    (TTGPU_PLAN_BWD1=0): same partition, so the gradients are BITWISE equal;
    tiny, multi-hot weighted Mean batches with empty bags."""
    p = tt.plan_shapes(10131227, 16, 3, rank, [200, 220, 250], [2, 2, 4])
    rng = np.random.default_rng(nlook + rank)
    base = tt.generate_zipfian_batch(p.num_rows, 1.05, 3, nlook, 1)
    nb = max(1, nlook // 3)
    cuts = np.sort(rng.integers(0, nlook + 1, nb - 1))
    off = np.concatenate([[0], cuts, [nlook]]).astype(np.int64)
    b = tt.IndexBatch(base.indices.astype(np.int64), off, rng.uniform(-2, 2, nlook), tt.Pooling.Mean)
    g = rng.standard_normal((nb, 16)).astype(np.float32)
    outs, grads = [], []
    # merge units off: the planned ranges alone must reproduce the in-kernel
    # planning bit for bit
    monkeypatch.setenv("TTGPU_MERGE1", "0")
    for plan in ("1", "0"):
        monkeypatch.setenv("TTGPU_PLAN_BWD1", plan)
        t, cores = make_table(p, np.float32, 9, "plan" + plan, scale=0.3)
        res = tt.forward_bags(t, b)
        outs.append(res.output)
        grads.append(tt.backward_bags(t, b, res.context, g).cores)
    assert np.array_equal(outs[0], outs[1])
    for k in range(3):
        assert np.array_equal(grads[0][k], grads[1][k]), k
    if nlook <= 4096:
        want = orc.backward(as_oplan(p), cores, b.indices, b.offsets, g, b.weights, 1)
        for k in range(3):
            assert scaled_max_err(grads[0][k], want[k]) <= GRAD_TOL


@pytest.mark.parametrize("rank,nlook,s", [(32, 1, 1.05), (32, 45, 1.05), (32, 4096, 1.05), (32, 4096, 1.2),
                                          (32, 65536, 1.05), (8, 4096, 1.2), (64, 4096, 1.05),
                                          (16, 20000, 1.5)])
def test_bwd1_merge_units(orc, monkeypatch, rank, nlook, s):
    """Planned f3_bwd1 merge units (runs of one-slot tiles of one (i1, i0) pair
    whose GEMMs run once on the summed S rows; the default): gradients within
    the tolerance of the unmerged path and of the oracle, deterministic
    (two tables, bitwise equal), and the post-SGD cores of the fused step
    within tolerance; Zipf 1.05 / 1.2 / 1.5 (long runs of hot-pair tiles)."""
    p = tt.plan_shapes(10131227, 16, 3, rank, [200, 220, 250], [2, 2, 4])
    rng = np.random.default_rng(nlook + rank + int(10 * s))
    base = tt.generate_zipfian_batch(p.num_rows, s, 5, nlook, 1)
    nb = max(1, nlook // 2)
    cuts = np.sort(rng.integers(0, nlook + 1, nb - 1))
    off = np.concatenate([[0], cuts, [nlook]]).astype(np.int64)
    b = tt.IndexBatch(base.indices.astype(np.int64), off, rng.uniform(-2, 2, nlook), tt.Pooling.Sum)
    g = rng.standard_normal((nb, 16)).astype(np.float32)
    grads = []
    for merge, name in (("1", "m1a"), ("1", "m1b"), ("0", "m0")):
        monkeypatch.setenv("TTGPU_MERGE1", merge)
        t, cores = make_table(p, np.float32, 9, name, scale=0.3)
        res = tt.forward_bags(t, b)
        grads.append(tt.backward_bags(t, b, res.context, g).cores)
    for k in range(3):
        assert np.array_equal(grads[0][k], grads[1][k]), k
        assert scaled_max_err(grads[0][k], grads[2][k]) <= GRAD_TOL, k
    if nlook <= 4096:
        want = orc.backward(as_oplan(p), cores, b.indices, b.offsets, g, b.weights, 0)
        for k in range(3):
            assert scaled_max_err(grads[0][k], want[k]) <= GRAD_TOL
    # the fused backward + SGD step through the same units equals
    # backward_bags + sgd_step bit for bit
    monkeypatch.setenv("TTGPU_MERGE1", "1")
    a, _ = make_table(p, np.float32, 9, "m1s", scale=0.3)
    c, _ = make_table(p, np.float32, 9, "m1t", scale=0.3)
    tt.sgd_step(a, tt.backward_bags(a, b, tt.forward_bags(a, b).context, g), 0.05)
    c.backward_sgd(tt.forward_bags(c, b).context, b, g, 0.05)
    for k in range(3):
        assert np.array_equal(a.core(k), c.core(k)), k
