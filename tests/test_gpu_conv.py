"""GPU dataflow numerics (hot path (2)) against the CPU oracle.

Tolerances (BASELINE.json north_star), metric = golden::max_rel_err
(golden.hpp:127-136: |a-b| / max(|b|, 1)):
  * fp16 / bf16 inputs, fp32 accumulate (tcgen05 path): <= 1e-2, oracle run
    in f64 on the SAME half-rounded inputs;
  * fp32 path (SIMT FFMA): <= 1e-5 against the f64 oracle.
Every dataflow (gather-GEMM-scatter, fetch-on-demand, implicit GEMM with
splits 0..4) for forward, dgrad and wgrad, over channel shapes that exercise
each smem swizzle (K-chunk 16/32/64), N tiling and the SIMT fallback.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL_HALF = 1e-2
TOL_F32 = 1e-5


def max_rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1.0))) if a.size else 0.0


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2311_12862_b200 import sparse
    return torch, sparse


def make(sk, torch, seed, n, stride, k=3, rng=20):
    from paper_2311_12862_b200.synth import random_instance_coords
    c_np = random_instance_coords(seed, n, -rng, rng)
    c = sk.CoordSet.create(c_np)
    o = sk.build_out_coords(c, stride)
    m = sk.build_kmap(c, o, k, stride)
    return c, o, m


def configs(sk):
    """The tuner's whole space: the reference's 12 entries (tuner.cpp:9-26)
    plus the B200 kernel variants (one CTA per SM, TMA gather4 producers,
    single-slab 32-channel stages), so every variant the tuner may pick is
    checked against the oracle."""
    from paper_2311_12862_b200.network import default_space
    out = default_space()
    ref = [sk.DataflowConfig(sk.GATHER_GEMM_SCATTER), sk.DataflowConfig(sk.FETCH_ON_DEMAND)]
    for s in range(5):
        for t in (sk.tile_small(), sk.tile_large()):
            ref.append(sk.DataflowConfig(sk.IMPLICIT_GEMM, s, t))
    assert out[:12] == ref and len(out) > 12
    return out


SHAPES = [(16, 16), (32, 32), (64, 64), (64, 128), (96, 96), (128, 256), (256, 64), (48, 80),
          (4, 32), (3, 5)]


@pytest.mark.parametrize("dtype", ["float16", "bfloat16", "float32"])
@pytest.mark.parametrize("cin,cout", SHAPES)
def test_forward_all_dataflows(env, restatement, dtype, cin, cout):
    torch, sk = env
    dt = getattr(torch, dtype)
    c, o, m = make(sk, torch, 100 + cin + cout, 3000, 1 if cin % 2 else 2)
    ent, _ = m.os()
    g = torch.Generator().manual_seed(cin * 1000 + cout)
    x = torch.randn(m.n_in, cin, generator=g).to(dt)
    w = (torch.randn(m.num_offsets, cin, cout, generator=g) / np.sqrt(cin * 27)).to(dt)
    y_ref = restatement.conv(ent, x.double().numpy(), w.double().numpy())
    tol = TOL_F32 if dtype == "float32" else TOL_HALF
    for cfg in configs(sk):
        y = sk.conv_forward(m, x.cuda(), w.cuda(), cfg)
        torch.cuda.synchronize()
        err = max_rel_err(y.double().cpu().numpy(), y_ref)
        assert err <= tol, (cfg.name(), dtype, cin, cout, err)


@pytest.mark.parametrize("dtype", ["float16", "float32"])
@pytest.mark.parametrize("cin,cout", [(32, 64), (64, 64), (128, 96), (4, 16), (256, 128),
                                      (96, 256), (16, 8), (4, 32), (3, 48), (1, 32), (8, 40)])
@pytest.mark.parametrize("stride", [1, 2])
def test_dgrad_wgrad(env, restatement, dtype, cin, cout, stride):
    torch, sk = env
    dt = getattr(torch, dtype)
    c, o, m = make(sk, torch, 7 + cin + stride, 4000, stride)
    ent, _ = m.os()
    g = torch.Generator().manual_seed(cin + 31 * cout + stride)
    x = torch.randn(m.n_in, cin, generator=g).to(dt)
    w = (torch.randn(m.num_offsets, cin, cout, generator=g) / np.sqrt(cin * 27)).to(dt)
    dy = torch.randn(m.n_out, cout, generator=g).to(dt)
    t = restatement.transpose_os(ent, m.n_in)
    dx_ref = restatement.dgrad(t, dy.double().numpy(), w.double().numpy())
    dw_ref = restatement.wgrad(ent, x.double().numpy(), dy.double().numpy())
    tol = TOL_F32 if dtype == "float32" else TOL_HALF
    for cfg in configs(sk):
        dx = sk.conv_dgrad(m, dy.cuda(), w.cuda(), cfg)
        torch.cuda.synchronize()
        assert max_rel_err(dx.double().cpu().numpy(), dx_ref) <= tol, cfg.name()
    dw = sk.conv_wgrad(m, x.cuda(), dy.cuda())
    torch.cuda.synchronize()
    # wgrad sums up to n_out products per cell: compare relative to the cell scale
    scale = max(1.0, float(np.abs(dw_ref).max()))
    assert float(np.abs(dw.double().cpu().numpy() - dw_ref).max()) / scale <= tol


def test_transposed_layer_forward(env, restatement):
    """conv_transposed uses the transposed map of its encoder (network.cpp:243-252)."""
    torch, sk = env
    c, o, m = make(sk, torch, 55, 5000, 2)
    t = m.transpose()
    ent_t, _ = t.os()
    x = torch.randn(t.n_in, 64).half()
    w = (torch.randn(27, 64, 32) / 40).half()
    y_ref = restatement.conv(ent_t, x.double().numpy(), w.double().numpy())
    for cfg in configs(sk):
        y = sk.conv_forward(t, x.cuda(), w.cuda(), cfg)
        assert max_rel_err(y.double().cpu().numpy(), y_ref) <= TOL_HALF, cfg.name()


def test_deterministic_mode_is_bitwise_repeatable(env):
    torch, sk = env
    c, o, m = make(sk, torch, 77, 6000, 1)
    x = torch.randn(m.n_in, 64, device="cuda").half()
    w = (torch.randn(27, 64, 64, device="cuda") / 40).half()
    ctx = sk.Context.get()
    ctx.deterministic = True
    try:
        for cfg in configs(sk):
            a = sk.conv_forward(m, x, w, cfg)
            b = sk.conv_forward(m, x, w, cfg)
            assert torch.equal(a, b), cfg.name()
        dw1 = sk.conv_wgrad(m, x, x)
        dw2 = sk.conv_wgrad(m, x, x)
        assert torch.equal(dw1, dw2)
    finally:
        ctx.deterministic = False


def test_golden_conv_values(env):
    """test_exec.cpp:57-86 golden outputs through every GPU dataflow (fp32)."""
    import json, os
    torch, sk = env
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fig2.json")))
    cin = sk.CoordSet.create(np.array(g["in_coords"], np.int32), dims=2)
    cout = sk.CoordSet.create(np.array(g["out_coords"], np.int32), dims=2)
    m = sk.build_kmap(cin, cout, 3, 1)
    x = torch.arange(1, 6, dtype=torch.float32).reshape(5, 1).cuda()
    w = torch.arange(1, 10, dtype=torch.float32).reshape(9, 1, 1).cuda()
    x2 = torch.tensor([[j + 1.0, 2.0 * j] for j in range(5)]).cuda()
    w2 = torch.tensor([[[k + 1.0, 0.5], [-1.0, k]] for k in range(9)]).cuda()
    for cfg in configs(sk):
        assert sk.conv_forward(m, x, w, cfg)[:, 0].tolist() == g["conv_c1"], cfg.name()
        assert sk.conv_forward(m, x2, w2, cfg).tolist() == g["conv_c2"], cfg.name()


def test_contract_errors(env):
    torch, sk = env
    c, o, m = make(sk, torch, 3, 500, 1)
    x = torch.randn(m.n_in + 1, 16, device="cuda").half()
    w = torch.randn(27, 16, 16, device="cuda").half()
    with pytest.raises(sk.ContractError):
        sk.conv_forward(m, x, w)
    x = torch.randn(m.n_in, 16, device="cuda").half()
    with pytest.raises(sk.ContractError):
        sk.conv_forward(m, x, w.float())
    with pytest.raises(sk.ValidationError):
        sk.conv_forward(m, x, w, sk.DataflowConfig(sk.IMPLICIT_GEMM, 99))


@pytest.mark.parametrize("dtype", ["float16", "bfloat16"])
@pytest.mark.parametrize("cin,cout", [(32, 96), (96, 96), (128, 256), (256, 256), (4, 32)])
def test_identity_k1_dense_path(env, restatement, cin, cout, dtype):
    """K=1 stride-1 layers on one coordinate set run as a dense GEMM (the map
    is the identity); every dataflow config must agree with the oracle."""
    torch, sk = env
    from paper_2311_12862_b200.synth import random_instance_coords
    c_np = random_instance_coords(5, 9000, -20, 20)
    c = sk.CoordSet.create(c_np)
    m = sk.build_kmap(c, c, 1, 1)
    ent, _ = m.os()
    assert (ent[:, 0] == np.arange(len(c_np))).all()
    dt = getattr(torch, dtype)
    x = torch.randn(m.n_in, cin).to(dt)
    w = (torch.randn(1, cin, cout) / np.sqrt(cin)).to(dt)
    y_ref = restatement.conv(ent, x.double().numpy(), w.double().numpy())
    dy = torch.randn(m.n_out, cout).to(dt)
    dx_ref = restatement.dgrad(restatement.transpose_os(ent, m.n_in), dy.double().numpy(),
                               w.double().numpy())
    for cfg in configs(sk)[:4]:
        y = sk.conv_forward(m, x.cuda(), w.cuda(), cfg)
        assert max_rel_err(y.double().cpu().numpy(), y_ref) <= TOL_HALF, cfg.name()
        dx = sk.conv_dgrad(m, dy.cuda(), w.cuda(), cfg)
        assert max_rel_err(dx.double().cpu().numpy(), dx_ref) <= TOL_HALF, cfg.name()


def test_stem_paths_and_misaligned_features(env, restatement):
    """The 4-channel stem runs as a neighbour gather + one dense tcgen05 GEMM
    (8 B row loads); a feature base that is not 8 B aligned takes the general
    path. Both match the oracle."""
    torch, sk = env
    c, o, m = make(sk, torch, 91, 4000, 1)
    ent, _ = m.os()
    g = torch.Generator().manual_seed(5)
    x = torch.randn(m.n_in, 4, generator=g).half()
    w = (torch.randn(27, 4, 64, generator=g) / 10).half()
    y_ref = restatement.conv(ent, x.double().numpy(), w.double().numpy())
    cfg = sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large())
    y = sk.conv_forward(m, x.cuda(), w.cuda(), cfg)
    buf = torch.empty(m.n_in * 4 + 1, dtype=torch.float16, device="cuda")
    xm = buf[1:].view(m.n_in, 4)  # base 2 B past an 8 B boundary
    xm.copy_(x.cuda())
    assert xm.data_ptr() % 8 != 0
    y2 = sk.conv_forward(m, xm, w.cuda(), cfg)
    torch.cuda.synchronize()
    assert max_rel_err(y.double().cpu().numpy(), y_ref) <= TOL_HALF
    assert max_rel_err(y2.double().cpu().numpy(), y_ref) <= TOL_HALF


def test_dynamic_item_queue_slots_wrap(env, restatement):
    """Every tensor-core conv launch takes one of the context's 16384 dynamic
    item-queue counters and its last CTA re-zeroes it: more launches than
    slots (the ring wraps) still give the oracle's result every time."""
    torch, sk = env
    c, o, m = make(sk, torch, 123, 600, 1)
    ent, _ = m.os()
    g = torch.Generator().manual_seed(9)
    x = torch.randn(m.n_in, 16, generator=g).half()
    w = (torch.randn(27, 16, 16, generator=g) / 20).half()
    y_ref = restatement.conv(ent, x.double().numpy(), w.double().numpy())
    xd, wd = x.cuda(), w.cuda()
    cfg = sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large())
    y = torch.empty(m.n_out, 16, device="cuda", dtype=torch.float16)
    for i in range(17000):
        sk.conv_forward(m, xd, wd, cfg, out=y)
        if i % 4250 == 0 or i == 16999:
            torch.cuda.synchronize()
            assert max_rel_err(y.double().cpu().numpy(), y_ref) <= TOL_HALF, i
