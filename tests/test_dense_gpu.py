"""Uncompressed embedding-bag tables (csrc/dense_host.inl): forward bit-equal
to sequential float sums in lookup order, backward+SGD equal to the host sum
of per-row gradients (fixed but different order: 1e-6), deterministic, dense
gradient mode + apply equal to the fused mode, range errors reported."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _setup(rows, L_per_bag, B, dim, seed):
    import torch

    from paper_2101_11714_b200.dense import DenseEmbeddingBags

    rng = np.random.default_rng(seed)
    d = DenseEmbeddingBags(rows, dim)
    tabs = [rng.standard_normal((n, dim)).astype(np.float32) for n in rows]
    for t, v in enumerate(tabs):
        d.set_table(t, v)
    sizes = rng.integers(0, L_per_bag + 1, B)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    L = int(off[-1])
    # skewed indices so some rows are hot (long segments)
    idx = np.stack([np.minimum(rng.zipf(1.3, L) - 1, n - 1) for n in rows]).astype(np.int64)
    g = rng.standard_normal((len(rows), B, dim)).astype(np.float32)
    dev = torch.device("cuda")
    t_idx, t_off, t_g = (torch.from_numpy(x).to(dev) for x in (idx, off, g))
    out = torch.empty((len(rows), B, dim), device=dev)
    return d, tabs, idx, off, g, (t_idx, t_off, t_g, out)


def _host_forward(tabs, idx, off):
    T, B, dim = len(tabs), len(off) - 1, tabs[0].shape[1]
    out = np.zeros((T, B, dim), np.float32)
    for t in range(T):
        for b in range(B):
            acc = np.zeros(dim, np.float32)
            for l in range(off[b], off[b + 1]):
                acc = (acc + tabs[t][idx[t, l]]).astype(np.float32)
            out[t, b] = acc
    return out


def _host_grads(tabs, idx, off, g):
    grads = [np.zeros_like(v, dtype=np.float64) for v in tabs]
    for t in range(len(tabs)):
        for b in range(len(off) - 1):
            for l in range(off[b], off[b + 1]):
                grads[t][idx[t, l]] += g[t, b]
    return grads


def test_forward_bitwise_and_fused_sgd():
    import torch

    rows = [7, 300, 3, 1000]
    d, tabs, idx, off, g, (t_idx, t_off, t_g, out) = _setup(rows, 4, 200, 16, 0)
    L, B = idx.shape[1], len(off) - 1
    d.forward_device(t_idx.data_ptr(), L, t_off.data_ptr(), B, out.data_ptr())
    d.check()
    assert np.array_equal(out.cpu().numpy(), _host_forward(tabs, idx, off))
    d.backward_device(t_g.data_ptr(), 0.05, fused=True)
    torch.cuda.synchronize()
    grads = _host_grads(tabs, idx, off, g)
    for t in range(len(rows)):
        want = (tabs[t] - 0.05 * grads[t]).astype(np.float32)
        got = d.table(t)
        assert np.max(np.abs(got - want)) / max(1.0, np.abs(want).max()) < 1e-5


def test_dense_gradient_mode_equals_fused_and_is_deterministic():
    import torch

    rows = [50, 2, 400]
    outs = []
    for mode in ("fused", "dense", "fused"):
        d, tabs, idx, off, g, (t_idx, t_off, t_g, out) = _setup(rows, 6, 300, 16, 5)
        L, B = idx.shape[1], len(off) - 1
        d.forward_device(t_idx.data_ptr(), L, t_off.data_ptr(), B, out.data_ptr())
        if mode == "fused":
            d.backward_device(t_g.data_ptr(), 0.1, fused=True)
        else:
            d.backward_device(t_g.data_ptr(), 0.0, fused=False)
            d.apply_grad(0.1)
        torch.cuda.synchronize()
        outs.append([d.table(t) for t in range(len(rows))])
    for a, b in zip(outs[0], outs[2]):
        assert np.array_equal(a, b)  # run-to-run bitwise
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)  # same fixed-order sum, applied in place or after


def test_out_of_range_index_is_reported():
    import torch

    from paper_2101_11714_b200 import OutOfRange
    from paper_2101_11714_b200.dense import DenseEmbeddingBags

    d = DenseEmbeddingBags([10, 20], 8)
    idx = torch.tensor([[1, 2, 3], [4, 20, 5]], dtype=torch.int64, device="cuda")
    off = torch.tensor([0, 1, 3], dtype=torch.int64, device="cuda")
    out = torch.empty((2, 2, 8), device="cuda")
    d.forward_device(idx.data_ptr(), 3, off.data_ptr(), 2, out.data_ptr())
    with pytest.raises(OutOfRange, match=r"index 20 out of range \[0, 20\) for dense table 1"):
        d.check()
