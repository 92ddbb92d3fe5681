"""Device index streams (§8(f) f3): range, determinism, counter composition,
and the distribution against the reference ZipfianSampler's probabilities
(the host CDF loop of data.cpp:8-20, which tests/test_host.py pins against
the reference stream byte for byte)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _draw(s, seed, counter, n):
    import torch

    out = torch.empty(n, dtype=torch.int64, device="cuda")
    s.draw_device(seed, counter, n, out.data_ptr())
    torch.cuda.synchronize()
    return out.cpu().numpy()


def _zipf_probs(pop, e):
    w = np.arange(1, pop + 1, dtype=np.float64) ** -e
    return w / w.sum()


@pytest.mark.parametrize("pop,e", [(1000, 1.05), (1000, 1.2), (997, 0.0), (10131227, 1.05)])
def test_range_determinism_and_counter_composition(pop, e):
    from paper_2101_11714_b200.streams import DeviceZipfSampler

    s = DeviceZipfSampler(pop, e)
    a = _draw(s, 7, 0, 20000)
    assert a.min() >= 0 and a.max() < pop
    assert np.array_equal(a, _draw(s, 7, 0, 20000))
    assert np.array_equal(a, np.concatenate([_draw(s, 7, 0, 5000), _draw(s, 7, 5000, 15000)]))
    assert not np.array_equal(a, _draw(s, 8, 0, 20000))


@pytest.mark.parametrize("pop,e", [(1000, 1.05), (200, 1.2), (500, 0.0)])
def test_distribution_matches_reference_sampler(pop, e):
    from paper_2101_11714_b200.streams import DeviceZipfSampler

    n = 2_000_000
    s = DeviceZipfSampler(pop, e)
    x = _draw(s, 3, 0, n)
    f = np.bincount(x, minlength=pop) / n
    p = _zipf_probs(pop, e)
    sigma = np.sqrt(p * (1 - p) / n)
    assert np.all(np.abs(f - p) <= 6 * sigma + 1e-12), float(np.max(np.abs(f - p) / sigma))
    chi2 = float(np.sum((f - p) ** 2 / p) * n)
    assert chi2 < pop + 6 * np.sqrt(2 * pop)


def test_cfg2_head_frequencies():
    """Zipf(1.05) over 10,131,227 rows: the head mass matches the reference's
    CDF (rank 0 carries ~6% of the draws)."""
    from paper_2101_11714_b200.streams import DeviceZipfSampler

    pop, e, n = 10131227, 1.05, 1_000_000
    x = _draw(DeviceZipfSampler(pop, e), 11, 0, n)
    w0 = 1.0
    hsum = np.sum(np.arange(1, pop + 1, dtype=np.float64) ** -e)
    for r in range(5):
        p = (r + 1) ** -e / hsum
        f = np.mean(x == r)
        assert abs(f - p) <= 6 * np.sqrt(p * (1 - p) / n)
    del w0


def test_bag_offsets():
    import torch

    from paper_2101_11714_b200.streams import bag_offsets_device

    off = torch.empty(65537, dtype=torch.int64, device="cuda")
    bag_offsets_device(65536, 32, off.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(off.cpu().numpy(), np.arange(65537, dtype=np.int64) * 32)
