"""GPU NetworkRunner / tuner parity (network.cpp, tuner.cpp) against the
compiled reference and a PyTorch fp64 autograd reference of the same op.

* group partition == the reference's (test_net_io.cpp:85-119);
* toy U-Net and MinkUNet-18 skeleton forward: fp32 GPU vs reference f64 with
  identical weights (golden metric <= 1e-5 through the network);
* outputs independent of the group assignment (test_net_io.cpp:142-171),
  cached maps reused, mapping vs kernel timing split (:173-195);
* chained backward vs torch autograd over the exported maps;
* tuner: |log| = G x |space|, winners are the per-group argmin (test_tuner.cpp).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2311_12862_b200 import models, network, sparse
    return torch, sparse, network, models


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1.0))) if a.size else 0.0


def scan(n_points=20000, seed=4, extent=1.0, voxel=0.05):
    from paper_2311_12862_b200.synth import planar_patches, quantize
    return quantize(planar_patches(n_points, seed, extent), [voxel] * 3)


def test_groups_match_reference(env, reference):
    torch, sk, N, M = env
    for layers in (M.toy_unet(), M.minkunet18(), M.second_encoder()):
        net = N.NetworkRunner(layers, dtype=torch.float32)
        rn = reference.network(3, M.spec_text(layers))
        assert net.num_groups == rn.num_groups
        assert [net.group_of_layer(i) for i in range(net.num_layers)] == \
            [rn.group_of_layer(i) for i in range(net.num_layers)]
    net = N.NetworkRunner(M.toy_unet(), dtype=torch.float32)
    assert net.groups() == [[0, 1, 5], [2, 4], [3]]
    assert N.NetworkRunner(M.minkunet18(), dtype=torch.float32).num_groups == 14


@pytest.mark.parametrize("which", ["toy", "minkunet", "second"])
def test_forward_matches_reference(env, reference, which):
    torch, sk, N, M = env
    layers = {"toy": M.toy_unet, "minkunet": M.minkunet18, "second": M.second_encoder}[which]()
    coords = scan(6000 if which != "second" else 20000, seed=5,
                  extent=1.0 if which != "second" else 3.0,
                  voxel=0.05 if which != "second" else 0.08)
    net = N.NetworkRunner(layers, dtype=torch.float32, weight_seed=11)
    ws = [net.weight(i).double().cpu().numpy() for i in range(net.num_layers)]
    rn = reference.network(3, M.spec_text(layers), prec=1, weights=ws)
    c_in = layers[0].c_in
    g = torch.Generator().manual_seed(1)
    x = torch.randn(len(coords), c_in, generator=g)
    rn.set_input(coords, x.double().numpy(), prec=1)
    y_ref = rn.output()
    cs = sk.CoordSet.create(coords)
    for cfg in (sk.DataflowConfig(sk.IMPLICIT_GEMM, 1), sk.DataflowConfig(sk.FETCH_ON_DEMAND),
                sk.DataflowConfig(sk.GATHER_GEMM_SCATTER), sk.DataflowConfig(sk.IMPLICIT_GEMM, 3)):
        net.set_all(cfg)
        y, _ = net.forward(cs, x.cuda())
        torch.cuda.synchronize()
        assert y.shape == y_ref.shape
        assert rel(y.double().cpu().numpy(), y_ref) <= 1e-5, cfg.name()


def test_half_network_close_to_reference(env, reference):
    """fp16 tensor-core path through the 77-layer MinkUNet stays close to the
    f64 reference on the same (half-rounded) weights and inputs."""
    torch, sk, N, M = env
    layers = M.minkunet18()
    coords = scan(8000, seed=6)
    net = N.NetworkRunner(layers, dtype=torch.float16, weight_seed=12)
    ws = [net.weight(i).double().cpu().numpy() for i in range(net.num_layers)]
    rn = reference.network(3, M.spec_text(layers), prec=1, weights=ws)
    x = torch.randn(len(coords), 4, generator=torch.Generator().manual_seed(2)).half()
    rn.set_input(coords, x.double().numpy(), prec=1)
    y_ref = rn.output()
    net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, 1))
    y, _ = net.forward(sk.CoordSet.create(coords), x.cuda())
    torch.cuda.synchronize()
    err = rel(y.double().cpu().numpy(), y_ref)  # golden metric per element
    assert err <= 1e-2, err


def test_map_cache_and_timing_split(env):
    torch, sk, N, M = env
    net = N.NetworkRunner(M.toy_unet(), dtype=torch.float16)
    cs = sk.CoordSet.create(scan(3000, seed=7))
    x = torch.randn(cs.n, 1, device="cuda").half()
    _, st1 = net.forward(cs, x, stats=True)
    builds = net.map_build_count()
    _, st2 = net.forward(cs, x, stats=True)
    assert net.map_build_count() == builds  # cached maps reused (network.cpp:207)
    assert st1["mapping_ms"].sum() > 0 and st1["kernel_ms"].sum() > 0
    assert st2["mapping_ms"].sum() < st1["mapping_ms"].sum() * 0.5
    assert net.measure_ms(cs, x, True, True, True) > 0
    for g in range(net.num_groups):
        assert net.modeled_group_traffic(g, sk.DataflowConfig(sk.IMPLICIT_GEMM, 1)) > 0


def _torch_reference(torch, layers, net, cs_maps, x, ws):
    """fp64 autograd restatement of run_forward over the GPU's exported maps."""
    outs = {}
    name_idx = {l.name: i for i, l in enumerate(layers)}
    for i, l in enumerate(layers):
        if not l.inputs:
            xi = x
        elif len(l.inputs) == 1:
            xi = outs[l.inputs[0]]
        else:
            xi = outs[l.inputs[0]] + outs[l.inputs[1]]
        ent = cs_maps[i]
        y = torch.zeros(ent.shape[0], l.c_out, dtype=torch.float64)
        for k in range(ent.shape[1]):
            idx = ent[:, k]
            m = idx >= 0
            if m.any():
                y = y.index_add(0, torch.nonzero(m).flatten(),
                                xi[idx[m]] @ ws[i][k])
        outs[l.name] = y
    return outs[layers[-1].name]


def test_backward_matches_torch_autograd(env):
    torch, sk, N, M = env
    layers = M.toy_unet()
    coords = scan(2500, seed=8)
    net = N.NetworkRunner(layers, dtype=torch.float32, weight_seed=13)
    cs = sk.CoordSet.create(coords)
    x = torch.randn(cs.n, 1, generator=torch.Generator().manual_seed(3))
    net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, 1))
    y, _ = net.forward(cs, x.cuda())
    r = torch.randn(y.shape, generator=torch.Generator().manual_seed(4))
    wgrad = torch.zeros(net.num_params, device="cuda")
    net.backward(r.cuda(), wgrad)
    torch.cuda.synchronize()
    # exported execution-orientation maps of every layer
    ins = {}
    maps = []
    down = sk.build_out_coords(cs, 2)
    for l in layers:
        if l.name == "down":
            maps.append(sk.build_kmap(cs, down, 3, 2).os()[0])
        elif l.name == "up":
            maps.append(sk.build_kmap(cs, down, 3, 2).transpose().os()[0])
        elif l.name == "mid":
            maps.append(sk.build_kmap(down, down, 3, 1).os()[0])
        else:
            maps.append(sk.build_kmap(cs, cs, 3, 1).os()[0])
    maps = [torch.from_numpy(m).long() for m in maps]
    ws = [net.weight(i).double().cpu().requires_grad_(True) for i in range(net.num_layers)]
    yr = _torch_reference(torch, layers, net, maps, x.double(), ws)
    assert rel(y.double().cpu().numpy(), yr.detach().numpy()) <= 1e-4
    (yr * r.double()).sum().backward()
    for i in range(net.num_layers):
        got = net.weight_grad(wgrad, i).double().cpu().numpy()
        want = ws[i].grad.numpy()
        scale = max(1.0, float(np.abs(want).max()))
        assert float(np.abs(got - want).max()) / scale <= 1e-4, layers[i].name


def test_tuner_contracts(env):
    torch, sk, N, M = env
    net = N.NetworkRunner(M.toy_unet(), dtype=torch.float16)
    cs = sk.CoordSet.create(scan(3000, seed=9))
    x = torch.randn(cs.n, 1, device="cuda").half()
    space = N.default_space()
    # the reference's 12 entries (tuner.cpp:9-26) first, then the B200
    # kernel variants (sk_tile: one CTA per SM, TMA gather4, 32-channel
    # slabs, one-tile work items)
    assert len(space) == 21
    assert all(c.kind == sk.IMPLICIT_GEMM and c.splits in (1, 2, 3) for c in space[12:])
    assert len({(c.kind, c.splits, c.tile) for c in space}) == len(space)
    lat, log = net.tune(cs, x, training=0, warmup=1, runs=3)
    G = net.num_groups
    assert len(log) == G * len(space)  # tuner.cpp:86-119 call count
    for g in range(G):
        rows = log[log[:, 1] == g]
        best = int(rows[np.argmin(rows[:, 3]), 2])
        assert net.config(g) == space[best]
    lat2, log2 = net.tune(cs, x, training=2, warmup=0, runs=1)
    assert len(log2) == 2 * G * len(space)


def test_cold_map_tuning(env):
    """sk_net_set_tune_cold: every probe builds the maps of a fresh copy of the
    tuning set (map preparation timed with each candidate); same call counts
    and argmin contract, the tuning set's own maps untouched, and the tuned
    runner's output equals the same configs installed by hand."""
    torch, sk, N, M = env
    net = N.NetworkRunner(M.toy_unet(), dtype=torch.float16, weight_seed=5)
    cs = sk.CoordSet.create(scan(3000, seed=19))
    x = torch.randn(cs.n, 1, device="cuda").half()
    space = N.default_space()
    net.set_tune_cold(True)
    builds0 = net.map_build_count()
    lat, log = net.tune(cs, x, training=0, warmup=1, runs=2)
    net.set_tune_cold(False)
    G = net.num_groups
    assert len(log) == G * len(space) and lat > 0
    for g in range(G):
        rows = log[log[:, 1] == g]
        assert net.config(g) == space[int(rows[np.argmin(rows[:, 3]), 2])]
    assert net.map_build_count() > builds0  # maps were rebuilt per probe
    y, _ = net.forward(cs, x)
    ref = N.NetworkRunner(M.toy_unet(), dtype=torch.float16, weight_seed=5)
    for g in range(G):
        ref.set_config(g, net.config(g))
    y2, _ = ref.forward(sk.CoordSet.create(scan(3000, seed=19)), x)
    assert torch.allclose(y.float(), y2.float(), atol=1e-2, rtol=1e-2)


def test_tune_result_and_tspw_weights_roundtrip(env, tmp_path):
    """A tuned assignment and the weights leave one runner as reference-format
    files (TuneResult JSON, TSPW) and reproduce the same network in another."""
    torch, sk, N, M = env
    from paper_2311_12862_b200 import io
    cs = sk.CoordSet.create(scan(3000, seed=13))
    x = torch.randn(cs.n, 1, device="cuda").half()
    net = N.NetworkRunner(M.toy_unet(), dtype=torch.float16)
    net.init_weights(5)
    lat, log = net.tune(cs, x, training=0, warmup=0, runs=1)
    text = io.tune_result_to_json(io.tune_result_of(net, lat, log))
    p = str(tmp_path / "w.tspw")
    io.write_tspw(p, [net.weight(i).float().cpu().numpy() for i in range(net.num_layers)])
    net2 = N.NetworkRunner(M.toy_unet(), dtype=torch.float16)
    io.apply_tune_result(net2, io.tune_result_from_json(text))
    for i, w in enumerate(io.read_tspw(p)):
        net2.set_weight(i, torch.from_numpy(w).half().cuda())
    net2.weights_updated()
    for g in range(net.num_groups):
        assert net2.config(g) == net.config(g)
    y1, _ = net.forward(cs, x)
    y2, _ = net2.forward(cs, x)
    torch.cuda.synchronize()
    # tuned split-K dataflows flush partials with fp32 atomics (order-dependent
    # last bits), so the two runners agree to fp16 rounding, not bitwise
    assert torch.allclose(y1.float(), y2.float(), rtol=2e-3, atol=2e-3)


def test_scan_pipeline_matches_serial_forward(env):
    """pipeline.ScanPipeline (copy-in / compute / copy-out streams, 1-3 worker
    threads with replicated runners) returns, scan by scan, exactly what a
    serial H2D -> forward -> D2H returns, including a smaller scan after a
    larger one and depth 3."""
    torch, sk, N, M = env
    from paper_2311_12862_b200.pipeline import ScanPipeline
    net = N.NetworkRunner(M.minkunet18(), dtype=torch.float16, weight_seed=2)
    net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large()))  # no red.add: bitwise stable
    rng = np.random.default_rng(0)
    scans = []
    for s, n_pts in enumerate([20000, 8000, 20000, 12000, 5000]):
        c = scan(n_pts, seed=10 + s)
        f = rng.standard_normal((len(c), 4)).astype(np.float16)
        scans.append((torch.from_numpy(c).pin_memory(), torch.from_numpy(f).pin_memory()))
    want = []
    for c, f in scans:
        y, _ = net.forward(sk.CoordSet.create(c.cuda()), f.cuda())
        want.append(y.cpu().numpy())
    from paper_2311_12862_b200.pipeline import replicate
    for depth, workers in ((2, 1), (3, 1), (2, 2), (2, 3)):
        pipe = ScanPipeline(replicate(net, workers), max(len(c) for c, _ in scans), 4,
                            depth=depth)
        got = {}
        pipe.run(scans, on_result=lambda i, h: got.__setitem__(i, h.numpy().copy()))
        assert sorted(got) == list(range(len(scans)))
        for i in range(len(scans)):
            assert got[i].shape == want[i].shape
            assert np.array_equal(got[i], want[i]), i
        assert pipe.d2h_bytes == sum(w.nbytes for w in want)
    with pytest.raises(sk.ValidationError):
        ScanPipeline(net, 10, 4).run(scans[:1])


def test_overlapped_map_build_matches_serial(env):
    """The overlapped map build (helper thread + map stream, sk_net_set_overlap)
    returns exactly the serial build's outputs, scan after scan, and its maps
    serve the chained backward (SGD on the same runner)."""
    torch, sk, N, M = env
    net = N.NetworkRunner(M.minkunet18(), dtype=torch.float16, weight_seed=4)
    net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large()))  # no red.add: bitwise
    rng = np.random.default_rng(3)
    for s, n_pts in enumerate([20000, 9000, 20000]):
        c = scan(n_pts, seed=40 + s)
        f = torch.from_numpy(rng.standard_normal((len(c), 4)).astype(np.float16)).cuda()
        builds = net.map_build_count()
        net.set_overlap(True)
        y_on, _ = net.forward(sk.CoordSet.create(c), f)
        assert net.map_build_count() == builds + 1
        g_on = torch.zeros(net.num_params, device="cuda")
        net.backward(torch.ones_like(y_on), g_on)
        net.set_overlap(False)
        y_off, _ = net.forward(sk.CoordSet.create(c), f)
        g_off = torch.zeros(net.num_params, device="cuda")
        net.backward(torch.ones_like(y_off), g_off)
        torch.cuda.synchronize()
        assert torch.equal(y_on, y_off), s
        # wgrad flushes with fp32 atomics (order-dependent): compare to the scale
        err = float((g_on - g_off).abs().max() / g_off.abs().max().clamp_min(1.0))
        assert err <= 1e-4, (s, err)


@pytest.mark.parametrize("overlap", [True, False])
def test_forward_error_inside_map_build_propagates(env, overlap):
    """A map-build failure (here an unsupported kernel volume, K=7 -> 343
    offsets, at the third layer) surfaces from forward as the reference's
    ValidationError with both the overlapped (helper thread) and the serial
    map build, and the runner keeps working on a valid network afterwards."""
    torch, sk, N, M = env
    from paper_2311_12862_b200.models import Layer
    layers = M.toy_unet()
    bad = [Layer(l.name, l.kind, l.c_in, l.c_out, 7 if l.name == "mid" else l.kernel, l.stride,
                 list(l.inputs), l.transpose_of) for l in layers]
    c = scan(3000, seed=21)
    x = torch.randn(len(c), 1, device="cuda").half()
    net = N.NetworkRunner(bad, dtype=torch.float16, weight_seed=1)
    net.set_overlap(overlap)
    with pytest.raises(sk.ValidationError):
        net.forward(sk.CoordSet.create(c), x)
    good = N.NetworkRunner(layers, dtype=torch.float16, weight_seed=1)
    good.set_overlap(overlap)
    y, _ = good.forward(sk.CoordSet.create(c), x)
    assert y.shape == (len(c), 2) and bool(torch.isfinite(y.float()).all())


@pytest.mark.parametrize("which", ["toy", "minkunet"])
def test_traffic_model_matches_reference(env, reference, which):
    """modeled_group_traffic (network.cpp:453-471) = traffic_model
    (cost.cpp:47-93) summed over a group's layers: byte-for-byte equal to the
    compiled reference for every group and every default_space config (the
    reference presets' cta_m 32 / 64 as the pad multiple), fp32 runners
    (elem_bytes 4 on both sides)."""
    torch, sk, N, M = env
    layers = {"toy": M.toy_unet, "minkunet": M.minkunet18}[which]()
    coords = scan(5000, seed=17)
    net = N.NetworkRunner(layers, dtype=torch.float32, weight_seed=3)
    x = torch.randn(len(coords), layers[0].c_in, generator=torch.Generator().manual_seed(5))
    net.forward(sk.CoordSet.create(coords), x.cuda())
    rn = reference.network(3, M.spec_text(layers), prec=0, threads=0)
    rn.set_input(coords, x.double().numpy(), prec=0)
    rn.forward()
    presets = {False: sk.TilePreset(32, 16, 16, 8, 4), True: sk.TilePreset(64, 32, 32, 8, 8)}
    space = [(sk.GATHER_GEMM_SCATTER, 0, False), (sk.FETCH_ON_DEMAND, 0, False)]
    space += [(sk.IMPLICIT_GEMM, s, t) for s in range(5) for t in (False, True)]
    checked = 0
    for g in range(net.num_groups):
        for kind, s, large in space:
            try:
                want = rn.group_traffic(g, kind, s, large)
            except ValueError:  # the reference rejects splits > K^D (K=1 groups)
                continue
            got = net.modeled_group_traffic(g, sk.DataflowConfig(kind, s, presets[large]))
            assert got == want, (g, kind, s, large, got, want)
            checked += 1
    assert checked >= net.num_groups * 4


def test_pdl_and_overlap_settings_do_not_change_results(env):
    """Programmatic dependent launch (sk_net_set_pdl) and the overlapped map
    build (sk_net_set_overlap) only change when kernels may start: a forward
    and a chained backward are bitwise identical with each on or off
    (store-only dataflow, no float atomics)."""
    torch, sk, N, M = env
    net = N.NetworkRunner(M.minkunet18(), dtype=torch.float16, weight_seed=4)
    net.set_all(sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large()))
    c = torch.from_numpy(scan(20000, seed=31)).cuda()
    x = torch.randn(c.shape[0], 4, device="cuda", generator=torch.Generator("cuda").manual_seed(1)).half()
    outs = []
    for pdl, overlap in ((True, True), (False, True), (True, False), (False, False)):
        net.set_pdl(pdl)
        net.set_overlap(overlap)
        y, _ = net.forward(sk.CoordSet.create(c), x)
        torch.cuda.synchronize()
        outs.append(y.cpu())
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
