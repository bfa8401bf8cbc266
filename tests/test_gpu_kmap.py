"""GPU kernel-map parity (hot path (1)): bit-exact against the compiled
reference (oracle/_ref) and the frozen golden vectors.

Checked per instance: output coordinates (values AND first-appearance order),
OS matrix, per-row big-endian masks, WS pair lists (ascending out row per
offset), split_and_sort + pad_map row orders/entries/masks for several split
counts and pad multiples, transposed maps, MAC counts.
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def sk():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2311_12862_b200 import sparse
    return sparse


def ws_lists(ptr, inn, out):
    return [[[int(inn[i]), int(out[i])] for i in range(ptr[k], ptr[k + 1])]
            for k in range(len(ptr) - 1)]


def test_golden_fig2(sk):
    g = json.load(open(os.path.join(GOLD, "fig2.json")))
    cin = sk.CoordSet.create(np.array(g["in_coords"], np.int32), dims=2)
    cout = sk.CoordSet.create(np.array(g["out_coords"], np.int32), dims=2)
    m = sk.build_kmap(cin, cout, 3, 1)
    ent, masks = m.os()
    assert ent.tolist() == g["os_matrix"]
    assert masks[:, 0].tolist() == g["masks"]
    assert ws_lists(*m.ws()) == g["ws_pairs"]
    assert m.total_pairs() == g["effective_macs"]
    assert m.split(1)[0][3].tolist() == g["sorted_order_s1"]
    assert [s[3].tolist() for s in m.split(3)] == g["sorted_order_s3"]
    assert [s[1] - s[0] for s in m.split(2)] == [5, 4]
    for splits, want in ((0, g["redundant_unsorted"]), (1, g["redundant_s1"]),
                         (3, g["redundant_s3"])):
        assert m.count_macs(splits, 4, 4, 1, 1) == (g["effective_macs"], want)
    with pytest.raises(sk.ValidationError):
        m.prepare(10)


def test_random_fixture(sk):
    d = json.load(open(os.path.join(GOLD, "random.json")))
    for case in d["cases"]:
        c = sk.CoordSet.create(np.array(case["in_coords"], np.int32))
        o = sk.build_out_coords(c, case["stride"])
        assert o.numpy().tolist() == case["out_coords"]
        m = sk.build_kmap(c, o, case["kernel"], case["stride"])
        ent, masks = m.os()
        assert ent.tolist() == case["os"]
        assert [[int(v) for v in r] for r in masks] == case["masks"]
        for got, want in zip(m.split(2, 8), case["split2_pad8"]):
            assert got[3].tolist() == want["out_row"]
            assert got[2].tolist() == want["entries"]


CASES = [
    # seed, n, stride, K, batches, coordinate range
    (1, 300, 1, 3, 1, 12), (2, 400, 2, 3, 1, 12), (3, 350, 3, 3, 2, 12), (4, 200, 1, 5, 1, 12),
    (5, 5000, 2, 3, 3, 40), (6, 1, 1, 3, 1, 12), (7, 3000, (2, 1, 1), 3, 1, 30),
    (8, 20000, 1, 3, 1, 60), (9, 20000, 2, 5, 2, 60), (10, 4000, 1, 1, 1, 20),
]


@pytest.mark.parametrize("seed,n,stride,k,batches,rng", CASES)
def test_maps_match_reference(sk, reference, seed, n, stride, k, batches, rng):
    from paper_2311_12862_b200.synth import random_instance_coords
    c_np = random_instance_coords(seed, n, -rng, rng, batches)
    st = list(stride) if isinstance(stride, tuple) else [stride] * 3
    c = sk.CoordSet.create(c_np)
    o = sk.build_out_coords(c, st)
    out_ref = reference.out_coords(3, c_np, st)
    assert np.array_equal(o.numpy(), out_ref)  # values and first-appearance order
    if st != [1, 1, 1]:
        assert o.stride_tag == tuple(st)
    for transposed in (False, True):
        a, b = (o, c) if transposed else (c, o)
        a_np, b_np = (out_ref, c_np) if transposed else (c_np, out_ref)
        m = sk.build_kmap(a, b, k, st, transposed)
        rm = reference.kmap(3, k, a_np, b_np, st, transposed)
        ent, masks = m.os()
        ent_r, masks_r = rm.os()
        assert np.array_equal(ent, ent_r)
        assert np.array_equal(masks, masks_r)
        ptr, inn, out = m.ws()
        for kk in range(rm.kd):
            ri, ro = rm.pairs(kk)
            assert np.array_equal(inn[ptr[kk]:ptr[kk + 1]], ri)
            assert np.array_equal(out[ptr[kk]:ptr[kk + 1]], ro)
        kd = rm.kd
        for splits in sorted({0, 1, 2, 5, min(kd, 27)} & set(range(kd + 1))):
            for pad in (1, 8, 128):
                got, want = m.split(splits, pad), rm.prepare(splits, pad)
                assert len(got) == len(want)
                for g_, w_ in zip(got, want):
                    assert (g_[0], g_[1]) == (w_[0], w_[1])
                    assert np.array_equal(g_[2], w_[2]), (splits, pad)
                    assert np.array_equal(g_[3], w_[3]), (splits, pad)
                    assert np.array_equal(g_[4], w_[4]), (splits, pad)
                assert m.count_macs(splits, pad, 32, 4, 8) == rm.count_macs(32, 4, 8)
    # transpose_map (kmap.cpp:290-315) == reference transpose == direct build
    m = sk.build_kmap(c, o, k, st)
    t = m.transpose()
    rt = reference.kmap(3, k, c_np, out_ref, st).transpose()
    assert np.array_equal(t.os()[0], rt.os()[0])
    assert np.array_equal(t.os()[1], rt.os()[1])
    direct = sk.build_kmap(o, c, k, st, transposed=True)
    assert np.array_equal(direct.os()[0], t.os()[0])


def test_map_cache_builds_once(sk):
    from paper_2311_12862_b200.synth import random_instance_coords
    c = sk.CoordSet.create(random_instance_coords(3, 500))
    a = sk.build_kmap(c, c, 3, 1)
    b = sk.build_kmap(c, c, 3, 1)
    assert a.ptr.value == b.ptr.value  # same object per MapKey (kmap.cpp:359-391)
    t = sk.build_kmap(c, c, 3, 1, transposed=True)
    assert t.ptr.value != a.ptr.value
    o1 = sk.build_out_coords(c, 2)
    o2 = sk.build_out_coords(c, 2)
    assert o1.id == o2.id
    assert sk.build_out_coords(c, 1).id == c.id  # submanifold keeps the set


def test_map_cache_threads_and_streams(sk):
    """MapCache once-per-key under an 8-thread race (test_kmap.cpp:227-264),
    with every thread on its own CUDA stream: all threads get the same cached
    map / down-sampled set / prepared map, and the convs they launch right
    after the cache hit on their own stream see the complete structures
    (stream_after: the cached object's build stream is waited for)."""
    import threading
    import torch
    from paper_2311_12862_b200.synth import lidar_scan
    coords = torch.from_numpy(lidar_scan(120_000, seed=9)).cuda()
    x = torch.randn(coords.shape[0], 32, device="cuda").half()
    w = (torch.randn(27, 32, 32, device="cuda") / 30).half()
    cfg = sk.DataflowConfig(sk.IMPLICIT_GEMM, 2, sk.tile_large())
    det = sk.DataflowConfig(sk.IMPLICIT_GEMM, 1, sk.tile_large())  # no red.add: bitwise stable
    c0 = sk.CoordSet.create(coords)
    m0 = sk.build_kmap(c0, c0, 3, 1)
    d0 = sk.build_out_coords(c0, 2)
    md0 = sk.build_kmap(c0, d0, 3, 2)
    want = [sk.conv_forward(m0, x, w, det).cpu(), sk.conv_forward(md0, x, w, det).cpu(),
            sk.conv_forward(m0, x, w, cfg).float().cpu()]
    shared = sk.CoordSet.create(coords)
    torch.cuda.synchronize()
    T = 8
    barrier = threading.Barrier(T)
    out = [None] * T

    def work(t):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                barrier.wait()
                m = sk.build_kmap(shared, shared, 3, 1)
                d = sk.build_out_coords(shared, 2)
                md = sk.build_kmap(shared, d, 3, 2)
                ys = [sk.conv_forward(m, x, w, det), sk.conv_forward(md, x, w, det),
                      sk.conv_forward(m, x, w, cfg).float()]
                s.synchronize()
                out[t] = (m.ptr.value, d.id, md.ptr.value, [y.cpu() for y in ys])
        except BaseException as e:
            out[t] = e
    th = [threading.Thread(target=work, args=(t,)) for t in range(T)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for r in out:
        assert not isinstance(r, BaseException), r
    assert len({r[0] for r in out}) == 1 and len({r[1] for r in out}) == 1
    assert len({r[2] for r in out}) == 1
    for r in out:
        assert torch.equal(r[3][0], want[0]) and torch.equal(r[3][1], want[1])
        assert torch.allclose(r[3][2], want[2], rtol=1e-2, atol=1e-2)


def test_validation_errors(sk):
    with pytest.raises(sk.ValidationError):
        sk.CoordSet.create(np.array([[0, 70000, 0, 0]], np.int32))  # outside packable range
    with pytest.raises(sk.ValidationError):
        sk.CoordSet.create(np.array([[5000, 0, 0, 0]], np.int32))
    c = sk.CoordSet.create(np.array([[0, 0, 0, 0], [0, 1, 0, 0]], np.int32))
    with pytest.raises(sk.ValidationError):
        sk.build_kmap(c, c, 2, 1)  # even kernel (kmap.cpp:60-61)
    with pytest.raises(sk.ValidationError):
        sk.build_out_coords(c, 0)


def test_large_scan_matches_reference(sk, reference):
    """C1-sized submanifold map (~100k uniform voxels) and a strided level."""
    from paper_2311_12862_b200.synth import uniform_voxels
    c_np = uniform_voxels(127_000, 64, seed=1)
    c = sk.CoordSet.create(c_np)
    m = sk.build_kmap(c, c, 3, 1)
    rm = reference.kmap(3, 3, c_np, c_np, [1, 1, 1])
    ent, masks = m.os()
    ent_r, masks_r = rm.os()
    assert np.array_equal(ent, ent_r) and np.array_equal(masks, masks_r)
    got, want = m.split(1, 128), rm.prepare(1, 128)
    assert np.array_equal(got[0][3], want[0][3]) and np.array_equal(got[0][2], want[0][2])
    o = sk.build_out_coords(c, 2)
    assert np.array_equal(o.numpy(), reference.out_coords(3, c_np, [2, 2, 2]))


BLOCK_CHECK = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from oracle.oracle import Reference
from paper_2311_12862_b200 import sparse as sk
from paper_2311_12862_b200.synth import random_instance_coords, lidar_scan
ref = Reference()
sk.Context.get().set_kmap_block_rows(int(sys.argv[2]))
cases = [(1, 300, 3, 1, 12), (4, 200, 5, 1, 12), (8, 20000, 3, 1, 60), (11, 6000, 5, 3, 25),
         (12, 3000, 3, 2, 400)]
for seed, n, k, batches, rng in cases:
    c_np = random_instance_coords(seed, n, -rng, rng, batches)
    c = sk.CoordSet.create(c_np)
    o = sk.build_out_coords(c, 2)  # a different output set, still stride 1
    o_np = o.numpy()
    for out, out_np in ((c, c_np), (o, o_np)):
        m = sk.build_kmap(c, out, k, 1)
        rm = ref.kmap(3, k, c_np, out_np, [1, 1, 1])
        assert np.array_equal(m.os()[0], rm.os()[0]), (seed, k)
        assert np.array_equal(m.os()[1], rm.os()[1]), (seed, k)
        ptr, inn, outs = m.ws()
        for kk in range(rm.kd):
            ri, ro = rm.pairs(kk)
            assert np.array_equal(inn[ptr[kk]:ptr[kk + 1]], ri)
            assert np.array_equal(outs[ptr[kk]:ptr[kk + 1]], ro)
    for k in (3, 5):  # strided / transposed maps on the same sets (hash query)
        m = sk.build_kmap(c, o, k, 2)
        rm = ref.kmap(3, k, c_np, o_np, [2, 2, 2])
        assert np.array_equal(m.os()[0], rm.os()[0]) and np.array_equal(m.os()[1], rm.os()[1])
        mt = sk.build_kmap(o, c, k, 2, transposed=True)
        rmt = ref.kmap(3, k, o_np, c_np, [2, 2, 2], transposed=True)
        assert np.array_equal(mt.os()[0], rmt.os()[0]), (seed, k, "transposed")
for dims, k in ((2, 3), (2, 5)):  # 2-D sets: z == 0, one block layer
    c_np = random_instance_coords(21, 3000, -40, 40, 2, dims=2)
    c = sk.CoordSet.create(c_np, dims=2)
    m, rm = sk.build_kmap(c, c, k, 1), ref.kmap(2, k, c_np, c_np, [1, 1, 1])
    assert np.array_equal(m.os()[0], rm.os()[0]) and np.array_equal(m.os()[1], rm.os()[1])
s_np = lidar_scan(60_000, seed=5)
s = sk.CoordSet.create(s_np)
m, rm = sk.build_kmap(s, s, 3, 1), ref.kmap(3, 3, s_np, s_np, [1, 1, 1])
assert np.array_equal(m.os()[0], rm.os()[0]) and np.array_equal(m.os()[1], rm.os()[1])
print("blocks ok")
'''


@pytest.mark.parametrize("min_rows", [1, 100])
def test_block_query_matches_reference(reference, min_rows):
    """The 4x4x4 block-index query (stride-1 3-D maps on >= 2^19-voxel input
    sets) forced on small instances (every set, or sets >= 100 voxels): K=3/5,
    batches, negative coordinates, output set != input set, a LiDAR scan, and
    the hash-query maps (strided, transposed, 2-D sets) next to it; OS, masks
    and the WS lists bit-exact vs the reference."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", BLOCK_CHECK, root, str(min_rows)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "blocks ok" in r.stdout, r.stdout + r.stderr


def test_large_set_lazy_table(sk, reference):
    """Sets of >= 2^19 voxels are range-checked by a check kernel at creation
    and get their hash table on first use (strided maps, down-sampling): the
    packable-range error still comes from CoordSet.create, and maps that read
    the lazily built table (strided, transposed) plus the block-index
    submanifold map are bit-exact against the reference."""
    from paper_2311_12862_b200.synth import uniform_voxels
    c_np = uniform_voxels(620_000, 160, seed=4)
    assert len(c_np) >= 1 << 19
    bad = c_np.copy()
    bad[len(bad) // 2, 1] = 70000
    with pytest.raises(sk.ValidationError):
        sk.CoordSet.create(bad)
    c = sk.CoordSet.create(c_np)
    m = sk.build_kmap(c, c, 3, 1)  # block index only
    rm = reference.kmap(3, 3, c_np, c_np, [1, 1, 1])
    assert np.array_equal(m.os()[0], rm.os()[0]) and np.array_equal(m.os()[1], rm.os()[1])
    o = sk.build_out_coords(c, 2)
    o_np = o.numpy()
    assert np.array_equal(o_np, reference.out_coords(3, c_np, [2, 2, 2]))
    ms = sk.build_kmap(c, o, 3, 2)  # first hash query on c: builds its table
    rms = reference.kmap(3, 3, c_np, o_np, [2, 2, 2])
    assert np.array_equal(ms.os()[0], rms.os()[0]) and np.array_equal(ms.os()[1], rms.os()[1])
    mt = sk.build_kmap(o, c, 3, 2, transposed=True)
    rmt = reference.kmap(3, 3, o_np, c_np, [2, 2, 2], transposed=True)
    assert np.array_equal(mt.os()[0], rmt.os()[0]) and np.array_equal(mt.os()[1], rmt.os()[1])
