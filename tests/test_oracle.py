"""Pin the CPU oracle before trusting it (CPU-only, no GPU).

1. The plain-C restatement (oracle/sk_oracle.c) reproduces every frozen golden
   vector of the reference's own tests (proj/tests/golden.hpp via
   tests/golden/fig2.json; test_kmap.cpp:37-90, test_exec.cpp:57-86,
   test_cost.cpp:42-57).
2. Restatement == compiled reference (oracle/_ref) bit-for-bit on seeded random
   instances: out coords, OS maps, masks, split orders, transposes, f64 conv,
   dgrad, wgrad.
3. The compiled reference reproduces tests/golden/random.json.
"""
import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def fig2():
    return json.load(open(os.path.join(GOLD, "fig2.json")))


def rand_coords(seed, n, lo=-12, hi=12, batches=1):
    rng = np.random.default_rng(seed)
    raw = rng.integers(lo, hi + 1, size=(n, 3))
    b = rng.integers(0, batches, size=(n, 1))
    c = np.concatenate([b, raw], 1).astype(np.int32)
    _, first = np.unique(c, axis=0, return_index=True)
    return c[np.sort(first)]


# --- 1. golden vectors --------------------------------------------------------

def test_offsets_lexicographic_mirror(restatement):
    o2 = restatement.offsets(2, 3)
    assert o2.tolist()[0] == [-1, -1, 0] and o2.tolist()[4] == [0, 0, 0]
    o3 = restatement.offsets(3, 3)
    assert len(o3) == 27 and o3[13].tolist() == [0, 0, 0]
    assert (o3[::-1] == -o3).all()  # mirror(i) = size-1-i (kmap.hpp:24)
    assert len(restatement.offsets(3, 5)) == 125
    with pytest.raises(ValueError):
        restatement.offsets(3, 2)


def test_golden_os_ws_masks(restatement, fig2):
    ent = restatement.kmap_os(2, 3, fig2["in_coords"], fig2["out_coords"], [1, 1, 1])
    assert ent.tolist() == fig2["os_matrix"]
    ptr, inn, out = restatement.ws(ent)
    got = [[[int(inn[i]), int(out[i])] for i in range(ptr[k], ptr[k + 1])] for k in range(9)]
    assert got == fig2["ws_pairs"]
    assert int(ptr[-1]) == fig2["effective_macs"]
    assert restatement.masks(ent)[:, 0].tolist() == fig2["masks"]


def test_golden_sort_orders(restatement, fig2):
    ent = restatement.kmap_os(2, 3, fig2["in_coords"], fig2["out_coords"], [1, 1, 1])
    s1 = restatement.split_sort(ent, 1)
    assert s1[0][3].tolist() == fig2["sorted_order_s1"]
    s3 = restatement.split_sort(ent, 3)
    assert [s[3].tolist() for s in s3] == fig2["sorted_order_s3"]
    s2 = restatement.split_sort(ent, 2)
    assert [s[1] - s[0] for s in s2] == [5, 4]  # test_kmap.cpp:101-102
    with pytest.raises(ValueError):
        restatement.split_sort(ent, 10)


def test_golden_mac_counts(restatement, fig2):
    ent = restatement.kmap_os(2, 3, fig2["in_coords"], fig2["out_coords"], [1, 1, 1])
    for splits, want in ((0, fig2["redundant_unsorted"]), (1, fig2["redundant_s1"]),
                         (3, fig2["redundant_s3"])):
        eff, red = restatement.count_macs(restatement.split_sort(ent, splits, 4), 4, 1, 1)
        assert (eff, red) == (fig2["effective_macs"], want)


def test_golden_conv(restatement, fig2):
    ent = restatement.kmap_os(2, 3, fig2["in_coords"], fig2["out_coords"], [1, 1, 1])
    x = np.arange(1, 6, dtype=np.float64)[:, None]
    w = np.arange(1, 10, dtype=np.float64).reshape(9, 1, 1)
    assert restatement.conv(ent, x, w)[:, 0].tolist() == fig2["conv_c1"]
    x2 = np.array([[j + 1.0, 2.0 * j] for j in range(5)])
    w2 = np.array([[[k + 1.0, 0.5], [-1.0, k]] for k in range(9)])
    assert restatement.conv(ent, x2, w2).tolist() == fig2["conv_c2"]


def test_golden_pad(restatement, fig2):
    ent = restatement.kmap_os(2, 3, fig2["in_coords"], fig2["out_coords"], [1, 1, 1])
    for (b, e, en, orow, m) in restatement.split_sort(ent, 2, 4):
        assert en.shape[0] == 8 and orow[6:].tolist() == [-1, -1]
        assert (en[6:] == -1).all() and (m[6:] == 0).all()


def test_two_word_masks(restatement):
    # test_kmap.cpp:208-225: K=5 needs 2 words, offset-0 row outranks offset-124 row
    ent = restatement.kmap_os(3, 5, [[0, 0, 0, 0]], [[0, -2, -2, -2], [0, 2, 2, 2]], [1, 1, 1])
    assert restatement.masks(ent).shape[1] == 2
    assert restatement.split_sort(ent, 1)[0][3].tolist() == [1, 0]


# --- 2. restatement == compiled reference ------------------------------------

CASES = [(1, 300, 1, 3, 1), (2, 400, 2, 3, 1), (3, 350, 3, 3, 2), (4, 200, 1, 5, 1),
         (5, 500, 2, 3, 3), (6, 1, 1, 3, 1), (7, 300, (2, 1, 1), 3, 1)]


@pytest.mark.parametrize("seed,n,stride,k,batches", CASES)
def test_restatement_matches_reference_maps(restatement, reference, seed, n, stride, k, batches):
    c = rand_coords(seed, n, batches=batches)
    st = list(stride) if isinstance(stride, tuple) else [stride] * 3
    out_r = reference.out_coords(3, c, st)
    assert np.array_equal(restatement.out_coords(3, c, st), out_r)
    for transposed in (False, True):
        a, b = (out_r, c) if transposed else (c, out_r)
        m = reference.kmap(3, k, a, b, st, transposed)
        ent_r, masks_r = m.os()
        ent = restatement.kmap_os(3, k, a, b, st, transposed)
        assert np.array_equal(ent, ent_r)
        assert np.array_equal(restatement.masks(ent), masks_r)
        for splits in (0, 1, 2, 5):
            for pad in (1, 8, 128):
                got = restatement.split_sort(ent, splits, pad)
                want = m.prepare(splits, pad)
                assert len(got) == len(want)
                for g, w in zip(got, want):
                    assert g[0] == w[0] and g[1] == w[1]
                    assert np.array_equal(g[2], w[2]) and np.array_equal(g[3], w[3])
                    assert np.array_equal(g[4], w[4])
                assert restatement.count_macs(got, 32, 4, 8) == m.count_macs(32, 4, 8)
    # transpose_map (kmap.cpp:290-315)
    m = reference.kmap(3, k, c, out_r, st)
    ent_t_r, _ = m.transpose().os()
    assert np.array_equal(restatement.transpose_os(m.os()[0], len(c)), ent_t_r)


@pytest.mark.parametrize("seed,stride", [(11, 1), (12, 2)])
def test_restatement_matches_reference_numerics(restatement, reference, seed, stride):
    rng = np.random.default_rng(seed)
    c = rand_coords(seed, 400)
    st = [stride] * 3
    out = reference.out_coords(3, c, st)
    m = reference.kmap(3, 3, c, out, st)
    ent, _ = m.os()
    cin, cout = 5, 7
    x = rng.standard_normal((len(c), cin))
    w = rng.standard_normal((27, cin, cout))
    dy = rng.standard_normal((len(out), cout))
    # f64 deterministic reference is bit-exact with the canonical order
    assert np.array_equal(restatement.conv(ent, x, w), reference.conv_ref(m, x, w))
    t = restatement.transpose_os(ent, len(c))
    assert np.array_equal(restatement.dgrad(t, dy, w), reference.conv_dgrad(m, dy, w))
    assert np.array_equal(restatement.wgrad(ent, x, dy), reference.conv_wgrad(m, x, dy))
    # every reference dataflow agrees (exec.hpp:79-83)
    for kind, splits in ((0, 0), (1, 0), (2, 0), (2, 1), (2, 3)):
        y = reference.conv_forward(m, x, w, kind=kind, splits=splits)
        assert np.array_equal(y, reference.conv_ref(m, x, w))


# --- 3. committed reference-made fixtures --------------------------------------

def test_reference_reproduces_random_fixture(reference):
    d = json.load(open(os.path.join(GOLD, "random.json")))
    for case in d["cases"]:
        c = np.array(case["in_coords"], np.int32)
        out = reference.out_coords(3, c, case["stride"])
        assert out.tolist() == case["out_coords"]
        m = reference.kmap(3, case["kernel"], c, out, case["stride"])
        ent, masks = m.os()
        assert ent.tolist() == case["os"]
        y = reference.conv_ref(m, np.array(case["x"]), np.array(case["w"]))
        assert np.allclose(y, np.array(case["y"]), rtol=0, atol=1e-12)


def test_restatement_reproduces_random_fixture(restatement):
    d = json.load(open(os.path.join(GOLD, "random.json")))
    for case in d["cases"]:
        c = np.array(case["in_coords"], np.int32)
        out = restatement.out_coords(3, c, case["stride"])
        assert out.tolist() == case["out_coords"]
        ent = restatement.kmap_os(3, case["kernel"], c, out, case["stride"])
        assert ent.tolist() == case["os"]
        sp = restatement.split_sort(ent, 2, 8)
        for g, w in zip(sp, case["split2_pad8"]):
            assert g[3].tolist() == w["out_row"] and g[2].tolist() == w["entries"]
