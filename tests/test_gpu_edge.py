"""Edge cases the reference's tests exercise (test_kmap.cpp / test_exec.cpp):
empty coordinate sets through every map kind, dataflow and the network
runner; coordinates on the packable boundary (maps must match the reference,
neighbours beyond the range are simply absent); a single voxel."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2311_12862_b200 import sparse
    return torch, sparse


def test_empty_inputs_everywhere(env):
    torch, sk = env
    from paper_2311_12862_b200.models import minkunet18
    from paper_2311_12862_b200.network import NetworkRunner
    c = sk.CoordSet.create(np.zeros((0, 4), np.int32))
    assert c.n == 0
    o = sk.build_out_coords(c, 2)
    assert o.n == 0
    m = sk.build_kmap(c, c, 3, 1)
    assert m.total_pairs() == 0
    x = torch.zeros(0, 32, device="cuda").half()
    w = torch.randn(27, 32, 64, device="cuda").half()
    dy = torch.zeros(0, 64, device="cuda").half()
    for cfg in [sk.DataflowConfig(sk.IMPLICIT_GEMM, 1), sk.DataflowConfig(sk.IMPLICIT_GEMM, 3),
                sk.DataflowConfig(sk.FETCH_ON_DEMAND), sk.DataflowConfig(sk.GATHER_GEMM_SCATTER)]:
        assert tuple(sk.conv_forward(m, x, w, cfg).shape) == (0, 64)
        assert tuple(sk.conv_dgrad(m, dy, w, cfg).shape) == (0, 32)
    dw = sk.conv_wgrad(m, x, dy)
    assert tuple(dw.shape) == (27, 32, 64) and float(dw.abs().sum()) == 0.0
    assert sk.build_kmap(c, o, 3, 2).total_pairs() == 0
    assert sk.build_kmap(o, c, 3, 2, transposed=True).total_pairs() == 0
    net = NetworkRunner(minkunet18(), dtype=torch.float16)
    y, _ = net.forward(c, torch.zeros(0, 4, device="cuda").half())
    torch.cuda.synchronize()
    assert tuple(y.shape) == (0, 96)


def test_packable_boundary_matches_reference(env, reference):
    torch, sk = env
    rng = np.random.default_rng(5)
    lo, hi = -65536, 65535
    pts = []
    for corner in [(lo, lo, lo), (hi, hi, hi), (lo, hi, 0), (hi, 0, lo)]:
        base = np.array(corner)
        d = rng.integers(0, 3, size=(60, 3)) * np.sign(-base + 0.5).astype(int)
        pts.append(base + d)
    xyz = np.clip(np.concatenate(pts), lo, hi)
    c_np = np.concatenate([np.zeros((len(xyz), 1), np.int64), xyz], 1).astype(np.int32)
    _, first = np.unique(c_np, axis=0, return_index=True)
    c_np = c_np[np.sort(first)]
    c = sk.CoordSet.create(c_np)
    for k in (3, 5):
        m = sk.build_kmap(c, c, k, 1)
        rm = reference.kmap(3, k, c_np, c_np, [1, 1, 1])
        assert np.array_equal(m.os()[0], rm.os()[0])
        assert np.array_equal(m.os()[1], rm.os()[1])
    o = sk.build_out_coords(c, 2)
    assert np.array_equal(o.numpy(), reference.out_coords(3, c_np, [2, 2, 2]))
    m = sk.build_kmap(c, o, 3, 2)
    rm = reference.kmap(3, 3, c_np, o.numpy(), [2, 2, 2])
    assert np.array_equal(m.os()[0], rm.os()[0])


def test_single_voxel_conv(env, restatement):
    torch, sk = env
    c_np = np.array([[0, 3, -4, 7]], np.int32)
    c = sk.CoordSet.create(c_np)
    m = sk.build_kmap(c, c, 3, 1)
    ent, _ = m.os()
    x = torch.randn(1, 64).half()
    w = (torch.randn(27, 64, 64) / 8).half()
    ref = restatement.conv(ent, x.double().numpy(), w.double().numpy())
    for cfg in [sk.DataflowConfig(sk.IMPLICIT_GEMM, 1), sk.DataflowConfig(sk.FETCH_ON_DEMAND)]:
        y = sk.conv_forward(m, x.cuda(), w.cuda(), cfg).double().cpu().numpy()
        assert np.max(np.abs(y - ref) / np.maximum(np.abs(ref), 1.0)) <= 1e-2
