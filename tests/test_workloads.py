"""The seeded input recipes reproduce SURVEY.md Appendix A's
numbers, and the numpy and torch value generators agree bit for bit."""
import numpy as np

from workloads import cfg1_case, cfg4_case, fcn220m
from workloads.values import fill_values_torch, tensor_scales, values_np


def test_fcn220m_totals():
    f = fcn220m()
    assert f.T == 68 and f.G == 10
    assert int(f.numel[0::2].sum()) == 225_100_032 and int(f.numel[1::2].sum()) == 15_105
    assert abs(f.extra["ops_fwd_total"] / 1.7269e13 - 1) < 1e-4   # PAPER.md:211 anchor 1.717e13 (+0.6%)
    assert abs(f.bwd_delay_s.sum() * 1e3 - 35.20) < 0.01
    mb = [round(float(f.numel[f.group_of == g].sum()) * 2 / 1e6, 1) for g in range(10)]
    assert mb == [6.5, 18.9, 51.9, 18.9, 89.7, 75.5, 122.7, 44.9, 18.1, 3.2]
    # release order is reverse-layer, and groups appear in release order
    first_group = [int(f.group_of[2 * l]) for l in f.release_order]
    assert first_group == sorted(first_group)


def test_cfg1_shape():
    c = cfg1_case(3)
    assert c.N == 2 and c.T == 8 and c.G == 3
    assert c.numel.min() >= 1 and c.numel.max() <= 4096
    assert (c.mark_cycle >= 0).all()
    # each rank marks every tensor exactly once, at most 2 per cycle
    for r in range(2):
        assert np.bincount(c.mark_cycle[r]).max() <= 2


def test_cfg4_rotation():
    c = cfg4_case(256, 4)
    assert c.G == 32
    assert (np.bincount(c.mark_cycle[0]) == 16).all()
    assert c.mark_cycle[1, 255 - 64] == 0  # rank 1 starts a quarter of the way round


def test_values_numpy_torch_identical():
    import torch
    s = tensor_scales(5, 4)
    for kind in ("uniform", "int"):
        for t in range(4):
            a = values_np(5, 2, t, np.arange(70000), float(s[t]), kind)
            b = torch.empty(70000, dtype=torch.float32)
            fill_values_torch(b, 5, 2, t, float(s[t]), kind, chunk=30000)
            assert np.array_equal(a.view(np.uint32), b.numpy().view(np.uint32))
    # sampled indices equal the dense fill
    idx = np.array([0, 5, 69999, 123])
    assert np.array_equal(values_np(5, 2, 1, idx, float(s[1])), values_np(5, 2, 1, np.arange(70000), float(s[1]))[idx])


def test_contiguous_groups():
    from paper_1909_11150_b200.torch_reducer import contiguous_groups
    rng = np.random.default_rng(0)
    for _ in range(200):
        T = int(rng.integers(1, 40))
        G = int(rng.integers(1, 10))
        numel = rng.integers(1, 1000, size=T).tolist()
        g = contiguous_groups(numel, G)
        assert sorted(set(g)) == list(range(max(g) + 1)) and max(g) < min(G, T)
        rev = list(reversed(g))  # production (reverse) order: non-decreasing group ids
        assert rev == sorted(rev)


def test_tiny_fcdensenet_cpu():
    import torch
    from harness.fcdensenet import batch, make_model
    m = make_model(0, "cpu")
    x, y = batch(0, 0, "cpu")
    assert m(x).shape == y.shape
