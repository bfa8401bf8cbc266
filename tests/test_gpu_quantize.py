"""GPU quantize (tensor.cpp:87-142) against the
reference's own test_tensor.cpp cases and the compiled reference on random
point clouds: coordinates bit-exact in first-appearance order, features
exact for DedupRule::first and within 1e-12 (f64 sums vs running mean) for
DedupRule::mean."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sk():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2311_12862_b200 import sparse
    return sparse


def f64(t):
    import torch
    return t.to(torch.float64).cpu().numpy()


def test_floors_toward_negative_infinity(sk):  # test_tensor.cpp:12-20
    cs, _ = sk.quantize([-0.5, 0.5, 0.0, -1.0, 2.9, 0.0])
    assert cs.numpy().tolist() == [[0, -1, 0, 0], [0, -1, 2, 0]]


def test_scales_by_voxel_size_per_axis(sk):  # test_tensor.cpp:22-28
    cs, _ = sk.quantize([1.0, 1.0, 1.0], voxel=(0.5, 1.0, 2.0))
    assert cs.numpy().tolist() == [[0, 2, 1, 0]]


def test_dedup_first_or_mean(sk):  # test_tensor.cpp:30-41
    import torch
    raw = [0.1, 0.1, 0.1, 0.2, 0.2, 0.2, 5.0, 5.0, 5.0]
    feats = np.array([[1.0], [3.0], [10.0]])
    cs, f = sk.quantize(raw, feats=feats, rule="first", dtype=torch.float64)
    assert cs.n == 2 and f64(f).ravel().tolist() == [1.0, 10.0]
    cs, f = sk.quantize(raw, feats=feats, rule="mean", dtype=torch.float64)
    assert f64(f).ravel().tolist() == [2.0, 10.0]


def test_no_features_one_occupancy_channel(sk):  # test_tensor.cpp:43-49
    cs, f = sk.quantize([0, 0, 0, 3, 3, 3])
    assert tuple(f.shape) == (2, 1) and f64(f).ravel().tolist() == [1.0, 1.0]


def test_identity_on_integer_input(sk):  # test_tensor.cpp:51-69
    import torch
    rng = np.random.default_rng(11)
    pts = rng.integers(-20, 21, size=(200, 3))
    _, first = np.unique(pts, axis=0, return_index=True)
    pts = pts[np.sort(first)]
    feats = (np.arange(len(pts)) * 0.5)[:, None]
    cs, f = sk.quantize(pts.astype(np.float64), feats=feats, dtype=torch.float64)
    assert np.array_equal(cs.numpy()[:, 1:], pts)
    assert np.array_equal(f64(f), feats)


def test_rejects_non_finite_and_out_of_range(sk):  # test_tensor.cpp:71-76
    with pytest.raises(sk.ValidationError):
        sk.quantize([0.0, 0.0, float("nan")])
    with pytest.raises(sk.ValidationError):
        sk.quantize([1e7, 0.0, 0.0])
    with pytest.raises(sk.ValidationError):
        sk.quantize([1.0, 1.0, 1.0], voxel=(0.0, 1.0, 1.0))


def test_keeps_batches_separate(sk):  # test_tensor.cpp:78-86
    cs, _ = sk.quantize([0, 0, 0, 0, 0, 0], batch=[0, 1])
    assert cs.numpy()[:, 0].tolist() == [0, 1]


def test_empty(sk):
    cs, f = sk.quantize(np.zeros((0, 3)))
    assert cs.n == 0 and tuple(f.shape) == (0, 1)


@pytest.mark.parametrize("seed,m,voxel,dims,batches", [
    (1, 50_000, (0.05, 0.05, 0.05), 3, 1), (2, 20_000, (0.1, 0.1, 0.15), 3, 3),
    (3, 5_000, (0.3, 0.2, 1.0), 2, 2)])
def test_matches_reference(sk, reference, seed, m, voxel, dims, batches):
    import torch
    from paper_2311_12862_b200.synth import planar_patches
    rng = np.random.default_rng(seed)
    pts = planar_patches(m, seed, 4.0)[:, :dims] - 2.0  # negative coordinates too
    feats = rng.standard_normal((len(pts), 3))
    batch = rng.integers(0, batches, len(pts)).astype(np.int32) if batches > 1 else None
    for rule, code in (("first", 0), ("mean", 1)):
        rc, rf = reference.quantize(pts.ravel(), dims, feats, voxel[:dims], rule=code, batch=batch)
        cs, f = sk.quantize(pts, dims=dims, feats=feats, voxel=voxel, rule=rule, batch=batch,
                            dtype=torch.float64)
        assert np.array_equal(cs.numpy(), rc)
        if rule == "first":
            assert np.array_equal(f64(f), rf)
        else:
            assert np.max(np.abs(f64(f) - rf) / np.maximum(np.abs(rf), 1.0)) <= 1e-12
    # quantized sets feed the map pipeline directly
    m_ = sk.build_kmap(cs, cs, 3, 1)
    assert m_.n_out == cs.n
