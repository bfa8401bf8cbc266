"""The bench / parity input generators (paper_2311_12862_b200/synth.py) are an
exact restatement of the reference's gen_cloud + quantize (gen.cpp:32-85,
tensor.cpp:87-142): bit-equal point clouds and voxel lists against the
compiled reference, and the SURVEY.md §8(d) voxel counts."""
import numpy as np
import pytest

from paper_2311_12862_b200 import synth as S


def test_mt19937_64_standard_value():
    # C++ [rand.predef]: the 10000th output of a default-constructed
    # mt19937_64 (seed 5489) is 9981545732273789042
    assert int(S.MT19937_64(5489).raw(10000)[-1]) == 9981545732273789042


@pytest.mark.parametrize("kind", ["uniform", "planar_patches", "gaussian_clusters"])
@pytest.mark.parametrize("n,seed,extent", [(7, 3, 1.0), (12345, 1, 4.0), (40000, 9, 8.0)])
def test_gen_cloud_bit_equal_reference(reference, kind, n, seed, extent):
    want = reference.gen_cloud(S.CLOUD_KINDS[kind], n, seed, extent)
    got = S.gen_cloud(kind, n, seed, extent)
    assert got.shape == want.shape
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("n,seed,extent,voxel", [(200_000, 1, 4.0, (0.05, 0.05, 0.05)),
                                                 (60_000, 5, 8.0, (0.1, 0.1, 0.15))])
def test_quantized_scans_equal_reference(reference, n, seed, extent, voxel):
    want = reference.gen_voxels(1, n, seed, extent, voxel)
    got = S.quantize(S.gen_cloud("planar_patches", n, seed, extent), voxel)
    assert np.array_equal(got, want)


def test_survey_voxel_counts():
    # C1 100,642; C2 124,756; C3 149,357 (137,141 at
    # n=250k); C5 sweep n=16k/48k/160k -> 10,711 / 32,608 / 102,817
    assert len(S.uniform_voxels(127_000, 64, 1)) == 100_642
    assert len(S.lidar_scan()) == 124_756
    assert len(S.waymo_scan()) == 149_357
    assert len(S.waymo_scan(250_000)) == 137_141
    assert [len(S.sweep_cloud(n)) for n in (16_000, 48_000, 160_000)] == [10_711, 32_608,
                                                                          102_817]


def test_uniform_int_matches_libstdcxx_reduction():
    # Lemire reduction: draw = (x * range) >> 64
    e1, e2 = S.MT19937_64(7), S.MT19937_64(7)
    got = S.uniform_int(e1, -12, 12, 1000)
    x = [int(v) for v in e2.raw(1000)]
    assert got.tolist() == [((v * 25) >> 64) - 12 for v in x]
