"""Parity on the BASELINE.json configurations themselves, at their stated
sizes (north_star: "bit-exact kernel maps and in-tolerance outputs vs the CPU
oracle on all five configs").

Inputs come from synth.py's exact restatement of the reference's generators
(bit-equal to the compiled gen_cloud / quantize, tests/test_synth.py), so the
voxel counts are SURVEY.md §8(d)'s: C1 100,642; C2 124,756; C3 149,357; C5
1,040,205 (10 tiles of n=160k) and 279,846 (n=480k).

Checks, all against the compiled, unmodified reference (oracle/_ref):
  * kernel maps bit-exact: output coordinates in first-appearance order, the
    OS matrix (-1 sentinels) and the big-endian masks, for every map group of
    the network configs (submanifold per level, strided, transposed, K=1);
  * features with golden::max_rel_err (golden.hpp:127-136, per element
    |a - b| / max(|b|, 1)): <= 1e-5 for the fp32 path, <= 1e-2 for fp16 inputs
    with fp32 accumulation (the reference runs f64 on the SAME half-rounded
    inputs), per conv, per network and per training step.

Reference protocol: test_exec.cpp:88-116 (every config vs conv_ref),
acceptance_main.cpp:63-99; the reference's f64 executors run on all host
cores (GGS, ExecContext.threads = nproc) so the suite stays within minutes.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL_HALF = 1e-2
TOL_F32 = 1e-5
THREADS = os.cpu_count() or 1
F64 = 1  # reference Precision::f64


def scaled_err(a, b):
    """golden::max_rel_err's mixed metric with the TENSOR's scale as the
    denominator: max |a - b| / max(1, max |b|). Weight gradients sum 10^5-10^6
    products per cell (|dW| up to ~10^3 at C2 size), so a near-zero cell's
    error is set by the scale of its terms, not by its own value: measured
    fp32 errors are ~5e-8 of the scale (per-cell ~1e-4), fp16 ~8e-4."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b))))) if a.size else 0.0


def max_rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1.0))) if a.size else 0.0


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2311_12862_b200 import models, network, sparse, synth
    return torch, sparse, network, models, synth


def all_configs(sk):
    """The tuner's space: the 12 default_space entries plus the B200 variants."""
    from paper_2311_12862_b200.network import default_space
    return default_space()


def assert_map_equal(gpu_map, ref_map, what):
    ent, masks = gpu_map.os()
    rent, rmasks = ref_map.os()
    assert ent.shape == rent.shape, what
    assert np.array_equal(ent, rent), f"{what}: OS entries differ"
    assert np.array_equal(masks, rmasks), f"{what}: masks differ"


def network_maps_equal(sk, reference, layers, coords):
    """Every layer's execution map of `layers` on `coords`, GPU vs reference:
    strided output coordinates (values and order), forward maps, transposed
    maps (NetworkRunner orient, network.cpp:243-252). Returns pairs per layer."""
    cs = sk.CoordSet.create(coords)
    gsets, rsets = {"": cs}, {"": coords}
    gmaps, rmaps, pairs = {}, {}, []
    names = [l.name for l in layers]
    for l in layers:
        src = l.inputs[0] if l.inputs else ""
        if l.kind == "conv":
            g_out = sk.build_out_coords(gsets[src], l.stride)
            r_out = reference.out_coords(3, rsets[src], [l.stride] * 3)
            assert np.array_equal(g_out.numpy(), r_out), f"{l.name}: output coordinates"
            key = (src, l.kernel, l.stride)
            if key not in gmaps:
                gmaps[key] = sk.build_kmap(gsets[src], g_out, l.kernel, l.stride)
                rmaps[key] = reference.kmap(3, l.kernel, rsets[src], r_out, [l.stride] * 3)
                assert_map_equal(gmaps[key], rmaps[key], l.name)
            gsets[l.name], rsets[l.name] = g_out, r_out
            pairs.append(gmaps[key].total_pairs())
        else:
            j = layers[names.index(l.transpose_of)]
            jsrc = j.inputs[0] if j.inputs else ""
            key = ("T", jsrc, j.kernel, j.stride)
            if key not in gmaps:
                fkey = (jsrc, j.kernel, j.stride)
                gmaps[key] = gmaps[fkey].transpose()
                rmaps[key] = rmaps[fkey].transpose()
                assert_map_equal(gmaps[key], rmaps[key], l.name + " (transposed)")
            gsets[l.name], rsets[l.name] = gsets[jsrc], rsets[jsrc]
            pairs.append(gmaps[key].total_pairs())
    return pairs


# --------------------------------------------------------------------------- C1
def test_c1_single_conv_all_configs(env, reference):
    """C1: 100,642 uniform voxels (mt19937_64(1), 127,000 draws in [0,64)^3),
    1,072,298 pairs, K=3 s=1, C_in = C_out = 64. All 12 default_space
    configs, forward and dgrad, fp32 (<= 1e-5) and fp16 (<= 1e-2); wgrad in
    both precisions."""
    torch, sk, N, M, S = env
    coords = S.uniform_voxels(127_000, 64, 1)
    assert len(coords) == 100_642
    cs = sk.CoordSet.create(coords)
    m = sk.build_kmap(cs, cs, 3, 1)
    rm = reference.kmap(3, 3, coords, coords, [1, 1, 1])
    assert_map_equal(m, rm, "C1")
    assert m.total_pairs() == 1_072_298
    ptr, a, b = m.ws()
    for k in range(27):  # WS lists: ascending out row per offset (kmap.cpp:113-134)
        ra, rb = rm.pairs(k)
        assert np.array_equal(a[ptr[k]:ptr[k + 1]], ra) and np.array_equal(b[ptr[k]:ptr[k + 1]], rb)

    rng = np.random.default_rng(2)
    n, C = len(coords), 64
    x = rng.standard_normal((n, C))
    w = rng.standard_normal((27, C, C)) / np.sqrt(27 * C)
    dy = rng.standard_normal((n, C))
    bad = []
    for dtype, tol in (("float32", TOL_F32), ("float16", TOL_HALF)):
        dt = getattr(torch, dtype)
        xt, wt, dyt = (torch.from_numpy(v).to(dt) for v in (x, w, dy))
        xr, wr, dyr = (v.double().numpy() for v in (xt, wt, dyt))  # the rounded inputs
        y_ref = reference.conv_forward(rm, xr, wr, kind=0, prec=F64, deterministic=False,
                                       threads=THREADS)
        dx_ref = reference.conv_dgrad(rm, dyr, wr, kind=0, prec=F64, deterministic=False,
                                      threads=THREADS)
        dw_ref = reference.conv_wgrad(rm, xr, dyr, prec=F64, threads=THREADS)
        xg, wg, dyg = xt.cuda(), wt.cuda(), dyt.cuda()
        for cfg in all_configs(sk):
            y = sk.conv_forward(m, xg, wg, cfg)
            dx = sk.conv_dgrad(m, dyg, wg, cfg)
            dw = sk.conv_wgrad(m, xg, dyg, cfg)
            torch.cuda.synchronize()
            for what, got, want in (("forward", y, y_ref), ("dgrad", dx, dx_ref),
                                    ("wgrad", dw, dw_ref)):
                e = max_rel_err(got.double().cpu().numpy(), want)
                if e > tol:
                    bad.append((what, dtype, cfg.name(), e))
    assert not bad, bad


# --------------------------------------------------------------------------- C2/C3
def half_weights(torch, net, seed):
    """Weights N(0, 1/sqrt(K^D c_in)) rounded to fp16 (so the fp32 and fp16
    runners and the f64 reference all see the same values)."""
    rng = np.random.default_rng(seed)
    ws = []
    for i in range(net.num_layers):
        kd, ci, co, _ = net.layer_shapes[i]
        ws.append(torch.from_numpy(rng.standard_normal((kd, ci, co)) / np.sqrt(kd * ci)).half())
    return ws


def network_parity(env, reference, layers, coords, configs):
    torch, sk, N, M, S = env
    network_maps_equal(sk, reference, layers, coords)
    probe = N.NetworkRunner(layers, dtype=torch.float32)
    ws = half_weights(torch, probe, 5)
    del probe
    x = torch.from_numpy(np.random.default_rng(6).standard_normal((len(coords), layers[0].c_in))).half()
    rn = reference.network(3, M.spec_text(layers), prec=F64, threads=0,
                           weights=[w.double().numpy() for w in ws])
    rn.set_input(coords, x.double().numpy(), prec=F64)
    y_ref = rn.output()
    errs = {}
    for dtype, tol in (("float32", TOL_F32), ("float16", TOL_HALF)):
        dt = getattr(torch, dtype)
        net = N.NetworkRunner(layers, dtype=dt)
        for i, w in enumerate(ws):
            net.set_weight(i, w.to(dt).cuda())
        net.weights_updated()
        cs = sk.CoordSet.create(coords)
        for cfg in configs(sk):
            net.set_all(cfg)
            y, _ = net.forward(cs, x.to(dt).cuda())
            torch.cuda.synchronize()
            assert y.shape == y_ref.shape
            errs[(dtype, cfg.name())] = (max_rel_err(y.double().cpu().numpy(), y_ref), tol)
    print("network max_rel_err:", errs)
    assert all(e <= tol for e, tol in errs.values()), errs


def net_configs(sk):
    return [sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large()),
            sk.DataflowConfig(sk.IMPLICIT_GEMM, 3, sk.tile_small()),
            sk.DataflowConfig(sk.FETCH_ON_DEMAND), sk.DataflowConfig(sk.GATHER_GEMM_SCATTER)]


def test_c2_minkunet_scan(env, reference):
    """C2: MinkUNet-18 (SURVEY App. B, 77 convs, 14 groups) on the 124,756-voxel
    SemanticKITTI-shaped scan: all maps bit-exact, network output vs the
    reference NetworkRunner in f64 (fp32 <= 1e-5, fp16 <= 1e-2)."""
    torch, sk, N, M, S = env
    coords = S.lidar_scan()
    assert len(coords) == 124_756
    network_parity(env, reference, M.minkunet18(), coords, net_configs)


def test_c3_second_scan(env, reference):
    """C3: SECOND/CenterPoint encoder on the 149,357-voxel Waymo-shaped scan
    (kernel maps reused across each stride level)."""
    torch, sk, N, M, S = env
    coords = S.waymo_scan()
    assert len(coords) == 149_357
    network_parity(env, reference, M.second_encoder(), coords, net_configs)


# --------------------------------------------------------------------------- C4
def test_c4_training_step_gradients(env):
    """C4: one MinkUNet training step (forward + chained dgrad + wgrad) on a
    C2 scan: every layer's weight gradient vs fp64 autograd over the exported
    (reference-pinned) maps on the same half-rounded weights and inputs,
    the output per element (golden metric) and each layer's dW against its
    own scale (scaled_err), fp16 <= 1e-2 and fp32 <= 1e-5."""
    torch, sk, N, M, S = env
    layers = M.minkunet18()
    coords = S.lidar_scan(seed=2)
    cs = sk.CoordSet.create(coords)
    probe = N.NetworkRunner(layers, dtype=torch.float32)
    ws = half_weights(torch, probe, 7)
    shapes = probe.layer_shapes
    del probe
    x = torch.from_numpy(np.random.default_rng(8).standard_normal((len(coords), 4))).half()

    # execution-orientation maps of every layer (network_maps_equal pins them
    # to the reference on the C2 scan; these are the same kernels)
    names = [l.name for l in layers]
    sets, fwd, maps = {"": cs}, {}, []
    for l in layers:
        src = l.inputs[0] if l.inputs else ""
        if l.kind == "conv":
            o = sk.build_out_coords(sets[src], l.stride)
            key = (src, l.kernel, l.stride)
            if key not in fwd:
                fwd[key] = sk.build_kmap(sets[src], o, l.kernel, l.stride)
            sets[l.name] = o
            maps.append(torch.from_numpy(fwd[key].os()[0]).long().cuda())
        else:
            j = layers[names.index(l.transpose_of)]
            jsrc = j.inputs[0] if j.inputs else ""
            maps.append(torch.from_numpy(fwd[(jsrc, j.kernel, j.stride)].transpose().os()[0])
                        .long().cuda())
            sets[l.name] = sets[jsrc]
    wr = [w.double().cuda().requires_grad_(True) for w in ws]
    outs = {}
    for i, l in enumerate(layers):
        xi = (x.double().cuda() if not l.inputs else
              outs[l.inputs[0]] if len(l.inputs) == 1 else outs[l.inputs[0]] + outs[l.inputs[1]])
        ent = maps[i]
        y = torch.zeros(ent.shape[0], l.c_out, dtype=torch.float64, device="cuda")
        for k in range(ent.shape[1]):
            idx = ent[:, k]
            rows = torch.nonzero(idx >= 0).flatten()
            if rows.numel():
                y = y.index_add(0, rows, xi[idx[rows]] @ wr[i][k])
        outs[l.name] = y
    y_ref = outs[layers[-1].name]
    r = torch.from_numpy(np.random.default_rng(9).standard_normal(tuple(y_ref.shape))).half()
    (y_ref * r.double().cuda()).sum().backward()

    bad = []
    for dtype, tol in (("float32", TOL_F32), ("float16", TOL_HALF)):
        dt = getattr(torch, dtype)
        net = N.NetworkRunner(layers, dtype=dt)
        for i, w in enumerate(ws):
            net.set_weight(i, w.to(dt).cuda())
        net.weights_updated()
        net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large()))
        y, _ = net.forward(cs, x.to(dt).cuda())
        g = torch.zeros(net.num_params, device="cuda")
        net.backward(r.to(dt).cuda(), g)
        torch.cuda.synchronize()
        e_y = max_rel_err(y.double().cpu().numpy(), y_ref.detach().cpu().numpy())
        errs = [scaled_err(net.weight_grad(g, i).double().cpu().numpy(), wr[i].grad.cpu().numpy())
                for i in range(len(layers))]
        worst = int(np.argmax(errs))
        print(f"C4 {dtype}: output {e_y:.3g}; worst weight-gradient max_rel_err {errs[worst]:.3g} "
              f"({layers[worst].name}) over {len(layers)} layers")
        bad += [(dtype, "output", e_y)] if e_y > tol else []
        bad += [(dtype, layers[i].name, e) for i, e in enumerate(errs) if e > tol]
    assert not bad, bad


# --------------------------------------------------------------------------- C5
def test_c5_sweep_1m_k3_c64(env, reference):
    """C5: the 1,040,205-voxel point (10 disjoint tiles of the n=160k planar
    recipe), K=3 s=1, C=64: map bit-exact; fp16 implicit GEMM (s1) and FOD
    forward <= 1e-2 and the fp32 path <= 1e-5 vs the reference in f64."""
    torch, sk, N, M, S = env
    coords = S.sweep_cloud(160_000, seed=1, tiles=10)
    assert len(coords) == 1_040_205  # exact gen_cloud restatement (SURVEY: ~1M)
    cs = sk.CoordSet.create(coords)
    m = sk.build_kmap(cs, cs, 3, 1)
    rm = reference.kmap(3, 3, coords, coords, [1, 1, 1])
    assert_map_equal(m, rm, "C5 1M")
    rng = np.random.default_rng(11)
    x = rng.standard_normal((len(coords), 64))
    w = rng.standard_normal((27, 64, 64)) / np.sqrt(27 * 64)
    for dtype, tol, cfgs in (("float16", TOL_HALF,
                              [sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large()),
                               sk.DataflowConfig(sk.FETCH_ON_DEMAND)]),
                             ("float32", TOL_F32,
                              [sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large())])):
        dt = getattr(torch, dtype)
        xt, wt = torch.from_numpy(x).to(dt), torch.from_numpy(w).to(dt)
        y_ref = reference.conv_forward(rm, xt.double().numpy(), wt.double().numpy(), kind=0,
                                       prec=F64, deterministic=False, threads=THREADS)
        for cfg in cfgs:
            y = sk.conv_forward(m, xt.cuda(), wt.cuda(), cfg)
            torch.cuda.synchronize()
            e = max_rel_err(y.double().cpu().numpy(), y_ref)
            assert e <= tol, (dtype, cfg.name(), e)


def test_c5_sweep_280k_k5_c256(env, reference):
    """C5: the 279,846-voxel point (n=480k), K=5 (125 offsets, two-word masks)
    s=1, C_in = C_out = 256: map bit-exact vs the reference; fp16 forward on
    a 4096-row sample of output rows vs an f64 restatement of conv_ref over
    the (pinned) map, <= 1e-2 (the full f64 CPU conv is ~0.5 TMAC)."""
    torch, sk, N, M, S = env
    coords = S.sweep_cloud(480_000, seed=1)
    assert len(coords) == 279_846
    cs = sk.CoordSet.create(coords)
    m = sk.build_kmap(cs, cs, 5, 1)
    rm = reference.kmap(3, 5, coords, coords, [1, 1, 1])
    assert_map_equal(m, rm, "C5 K=5")
    ent = rm.os()[0]
    rng = np.random.default_rng(12)
    xt = torch.from_numpy(rng.standard_normal((len(coords), 256))).half()
    wt = torch.from_numpy(rng.standard_normal((125, 256, 256)) / np.sqrt(125 * 256)).half()
    xr, wr = xt.double().numpy(), wt.double().numpy()
    rows = np.sort(rng.choice(len(coords), 4096, replace=False))
    y_ref = np.zeros((len(rows), 256))
    for k in range(125):  # conv_ref order: offset-major (exec.cpp:101-115)
        idx = ent[rows, k]
        live = idx >= 0
        y_ref[live] += xr[idx[live]] @ wr[k]
    for cfg in (sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large()),
                sk.DataflowConfig(sk.IMPLICIT_GEMM, 2, sk.tile_small()),
                sk.DataflowConfig(sk.FETCH_ON_DEMAND)):
        y = sk.conv_forward(m, xt.cuda(), wt.cuda(), cfg)
        torch.cuda.synchronize()
        e = max_rel_err(y[torch.from_numpy(rows).cuda()].double().cpu().numpy(), y_ref)
        assert e <= TOL_HALF, (cfg.name(), e)
