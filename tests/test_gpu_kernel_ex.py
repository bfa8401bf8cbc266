"""Generalized kernels (an EXTENSION beyond the reference:
per-axis / even kernel sizes and dilation), bit-exact against the plain-C
restatement sko_kmap_os_ex, with the reduction to the reference for standard
shapes, and the dataflows running on the resulting maps (MinkUNet's k=2
down/up convs, SECOND's (3,1,1) conv_out, dilated submanifold convs)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sk():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2311_12862_b200 import sparse
    return sparse


CASES = [  # kernel, dilation, stride, transposed
    ((2, 2, 2), (1, 1, 1), 2, False), ((2, 2, 2), (1, 1, 1), 2, True),
    ((3, 1, 1), (1, 1, 1), (2, 1, 1), False), ((3, 3, 3), (2, 2, 2), 1, False),
    ((3, 3, 3), (1, 2, 3), 1, False), ((4, 4, 4), (1, 1, 1), 1, False),
    ((5, 3, 1), (2, 1, 1), 1, False), ((3, 3, 3), (2, 2, 2), 2, True), ((1, 1, 3), (1, 1, 4), 1, False)]


@pytest.mark.parametrize("kernel,dil,stride,transposed", CASES)
def test_maps_match_restatement(sk, restatement, kernel, dil, stride, transposed):
    from paper_2311_12862_b200.synth import random_instance_coords
    c_np = random_instance_coords(7, 4000, -25, 25, 2)
    st = list(stride) if isinstance(stride, tuple) else [stride] * 3
    c = sk.CoordSet.create(c_np)
    o = sk.build_out_coords(c, st)
    a, b = (o, c) if transposed else (c, o)
    m = sk.build_kmap(a, b, kernel, st, transposed, dilation=dil)
    ref = restatement.kmap_os_ex(3, list(kernel), list(dil), a.numpy(), b.numpy(), st, transposed)
    ent, masks = m.os()
    assert np.array_equal(ent, ref)
    assert np.array_equal(masks, restatement.masks(ref))
    assert m.num_offsets == int(np.prod(kernel))


def test_standard_shape_is_the_reference_map(sk, reference):
    from paper_2311_12862_b200.synth import random_instance_coords
    c_np = random_instance_coords(9, 3000, -20, 20)
    c = sk.CoordSet.create(c_np)
    a = sk.build_kmap(c, c, 3, 1)
    b = sk.build_kmap(c, c, (3, 3, 3), 1, dilation=1)
    assert a.ptr.value == b.ptr.value  # same cached map
    rm = reference.kmap(3, 3, c_np, c_np, [1, 1, 1])
    assert np.array_equal(b.os()[0], rm.os()[0])


@pytest.mark.parametrize("kernel,dil,stride", [((2, 2, 2), (1, 1, 1), 2), ((3, 1, 1), (1, 1, 1), 1),
                                               ((3, 3, 3), (2, 2, 2), 1)])
def test_dataflows_on_generalized_maps(sk, restatement, kernel, dil, stride):
    import torch
    from paper_2311_12862_b200.synth import random_instance_coords
    c_np = random_instance_coords(5, 5000, -30, 30)
    c = sk.CoordSet.create(c_np)
    o = sk.build_out_coords(c, stride)
    m = sk.build_kmap(c, o, kernel, stride, dilation=dil)
    ent, _ = m.os()
    kd = int(np.prod(kernel))
    g = torch.Generator().manual_seed(3)
    x = torch.randn(m.n_in, 32, generator=g).half()
    w = (torch.randn(kd, 32, 64, generator=g) / 16).half()
    dy = torch.randn(m.n_out, 64, generator=g).half()
    y_ref = restatement.conv(ent, x.double().numpy(), w.double().numpy())
    t = restatement.transpose_os(ent, m.n_in)
    dx_ref = restatement.dgrad(t, dy.double().numpy(), w.double().numpy())
    dw_ref = restatement.wgrad(ent, x.double().numpy(), dy.double().numpy())
    for cfg in [sk.DataflowConfig(sk.IMPLICIT_GEMM, 1), sk.DataflowConfig(sk.FETCH_ON_DEMAND),
                sk.DataflowConfig(sk.GATHER_GEMM_SCATTER)]:
        y = sk.conv_forward(m, x.cuda(), w.cuda(), cfg).double().cpu().numpy()
        dx = sk.conv_dgrad(m, dy.cuda(), w.cuda(), cfg).double().cpu().numpy()
        assert np.max(np.abs(y - y_ref) / np.maximum(np.abs(y_ref), 1.0)) <= 1e-2, cfg.name()
        assert np.max(np.abs(dx - dx_ref) / np.maximum(np.abs(dx_ref), 1.0)) <= 1e-2, cfg.name()
    dw = sk.conv_wgrad(m, x.cuda(), dy.cuda()).double().cpu().numpy()
    assert np.abs(dw - dw_ref).max() / max(1.0, np.abs(dw_ref).max()) <= 1e-2


def test_validation(sk):
    c = sk.CoordSet.create(np.array([[0, 0, 0, 0]], np.int32))
    with pytest.raises(sk.ValidationError):
        sk.build_kmap(c, c, (9, 1, 1), 1)
    with pytest.raises(sk.ValidationError):
        sk.build_kmap(c, c, (3, 3, 3), 1, dilation=0)
    with pytest.raises(sk.ValidationError):
        sk.build_kmap(c, c, (6, 6, 6), 1)  # volume 216 > 128
