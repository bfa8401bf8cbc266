"""Graph (R-GCN) maps (kmap_from_edges, kmap.cpp:317-336)
through the pair-list dataflows: WS lists equal to the reference's (stable by
dst per relation), forward and wgrad within tolerance of the compiled
reference (dgrad / transpose raise ContractError, as in the reference), including the reference's own test_exec.cpp:292-306 instance and
duplicate (dst, relation) pairs that have no OS form."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2311_12862_b200 import sparse
    return torch, sparse


def rel_err(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1.0))) if np.size(a) else 0.0


def check_graph(torch, sk, reference, edges, R, n_in, n_out, c_in, c_out, seed):
    g = sk.kmap_from_edges(edges, R, n_in, n_out)
    rg = reference.graph_map(edges, R, n_in, n_out)
    ptr, inn, out = g.ws()
    for k in range(R):
        ri, ro = rg.pairs(k)
        assert np.array_equal(inn[ptr[k]:ptr[k + 1]], ri)
        assert np.array_equal(out[ptr[k]:ptr[k + 1]], ro)
    rng = np.random.default_rng(seed)
    for dt, tol in ((torch.float32, 1e-5), (torch.float16, 1e-2)):
        x = torch.from_numpy(rng.standard_normal((n_in, c_in))).to(dt)
        w = torch.from_numpy(rng.standard_normal((R, c_in, c_out)) / np.sqrt(c_in)).to(dt)
        dy = torch.from_numpy(rng.standard_normal((n_out, c_out))).to(dt)
        xd, wd, dyd = x.double().numpy(), w.double().numpy(), dy.double().numpy()
        y_ref = reference.conv_forward(rg, xd, wd, kind=1)
        dw_ref = reference.conv_wgrad(rg, xd, dyd)
        for kind in (sk.GATHER_GEMM_SCATTER, sk.FETCH_ON_DEMAND):
            cfg = sk.DataflowConfig(kind)
            y = sk.conv_forward(g, x.cuda(), w.cuda(), cfg)
            torch.cuda.synchronize()
            assert rel_err(y.double().cpu().numpy(), y_ref) <= tol, (kind, dt)
            with pytest.raises(sk.ContractError):
                sk.conv_dgrad(g, dy.cuda(), w.cuda(), cfg)
        dw = sk.conv_wgrad(g, x.cuda(), dy.cuda())
        torch.cuda.synchronize()
        scale = max(1.0, float(np.abs(dw_ref).max()))
        assert float(np.abs(dw.double().cpu().numpy() - dw_ref).max()) / scale <= tol
    return g


def test_reference_instance(env, reference):  # test_exec.cpp:292-306
    torch, sk = env
    edges = [[0, 0, 0], [1, 0, 0], [2, 0, 1], [0, 1, 1], [1, 1, 1], [2, 1, 0], [0, 1, 0]]
    g = check_graph(torch, sk, reference, edges, 2, 3, 2, 2, 1, 1)
    x = torch.tensor([[1, 2], [3, 4], [5, 6]], dtype=torch.float32).cuda()
    w = torch.tensor([[[1.0], [-1.0]], [[0.5], [2.0]]]).cuda()
    ref = reference.conv_ref(reference.graph_map(edges, 2, 3, 2), x.double().cpu().numpy(),
                             w.double().cpu().numpy())
    y = sk.conv_forward(g, x, w, sk.DataflowConfig(sk.FETCH_ON_DEMAND))
    assert np.allclose(y.double().cpu().numpy(), ref, rtol=0, atol=1e-6)


@pytest.mark.parametrize("seed,E,R,n_in,n_out,c_in,c_out", [
    (1, 5000, 4, 800, 700, 16, 32), (2, 40000, 8, 3000, 2000, 64, 64), (3, 100, 3, 50, 40, 8, 16)])
def test_random_graphs(env, reference, seed, E, R, n_in, n_out, c_in, c_out):
    torch, sk = env
    rng = np.random.default_rng(seed)
    edges = np.stack([rng.integers(0, n_in, E), rng.integers(0, n_out, E),
                      rng.integers(0, R, E)], 1).astype(np.int32)
    check_graph(torch, sk, reference, edges, R, n_in, n_out, c_in, c_out, seed)


def test_graph_contracts(env):
    torch, sk = env
    g = sk.kmap_from_edges([[0, 0, 0], [1, 0, 0]], 1, 2, 1)
    x = torch.zeros(2, 16, device="cuda").half()
    w = torch.zeros(1, 16, 16, device="cuda").half()
    with pytest.raises(sk.ContractError):
        sk.conv_forward(g, x, w, sk.DataflowConfig(sk.IMPLICIT_GEMM, 1))
    with pytest.raises(sk.ContractError):
        g.os()
    with pytest.raises(sk.ValidationError):
        sk.kmap_from_edges([[0, 0, 5]], 2, 2, 2)  # relation id out of range
    with pytest.raises(sk.ValidationError):
        sk.kmap_from_edges([[9, 0, 0]], 1, 2, 2)  # node id out of range
    e = sk.kmap_from_edges(np.zeros((0, 3), np.int32), 2, 4, 3)
    assert e.total_pairs() == 0
    y = sk.conv_forward(e, torch.zeros(4, 16, device="cuda").half(),
                        torch.zeros(2, 16, 16, device="cuda").half(),
                        sk.DataflowConfig(sk.FETCH_ON_DEMAND))
    assert tuple(y.shape) == (3, 16) and float(y.abs().sum()) == 0.0
