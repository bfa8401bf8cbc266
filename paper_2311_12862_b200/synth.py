"""Synthetic scans for tests and benchmarks (numpy, seeded).

The shapes follow the reference's generator (gen.cpp:32-85: uniform,
planar_patches = n/2500 random planar squares, the LiDAR stand-in) and
quantize (tensor.cpp:87-142: floor(p / voxel), first-appearance dedup). The
random streams are numpy's, not libstdc++'s, so voxel counts are close to but
not identical with SURVEY.md §8(d); both bench arms consume the same arrays.
"""
from __future__ import annotations

import numpy as np


def first_unique(coords: np.ndarray) -> np.ndarray:
    """Rows of `coords` deduplicated keeping first appearance order."""
    _, first = np.unique(coords, axis=0, return_index=True)
    return coords[np.sort(first)]


def uniform_voxels(draws: int, hi: int, seed: int, batch: int = 0) -> np.ndarray:
    """`draws` integer points in [0, hi)^3, first-appearance dedup -> int32 [n, 4]."""
    rng = np.random.default_rng(seed)
    p = rng.integers(0, hi, size=(draws, 3), dtype=np.int32)
    c = np.concatenate([np.full((draws, 1), batch, np.int32), p], 1)
    return first_unique(c).astype(np.int32)


def planar_patches(n: int, seed: int, extent: float) -> np.ndarray:
    """gen_cloud(planar_patches) shape (gen.cpp:44-61): n/2500 squares with
    random centre, normal and radius (0.2..0.5)*extent; float64 [n, 3]."""
    rng = np.random.default_rng(seed)
    n_p = max(1, n // 2500)
    per = n // n_p
    out = []
    for p in range(n_p):
        c = rng.random(3) * extent
        nrm = rng.standard_normal(3)
        nrm /= max(np.linalg.norm(nrm), 1e-12)
        ref = np.array([1.0, 0, 0]) if abs(nrm[0]) < 0.9 else np.array([0, 1.0, 0])
        u = np.cross(nrm, ref)
        u /= np.linalg.norm(u)
        v = np.cross(nrm, u)
        radius = (0.2 + 0.3 * rng.random()) * extent
        m = n - per * (n_p - 1) if p == n_p - 1 else per
        ab = (2 * rng.random((m, 2)) - 1) * radius
        out.append(c + ab[:, :1] * u + ab[:, 1:] * v)
    return np.concatenate(out, 0)


def quantize(points: np.ndarray, voxel, batch: int = 0) -> np.ndarray:
    """floor(p / voxel) + first-appearance dedup (tensor.cpp:87-142) -> int32 [n, 4]."""
    q = np.floor(points / np.asarray(voxel, np.float64)).astype(np.int32)
    c = np.concatenate([np.full((len(q), 1), batch, np.int32), q], 1)
    return first_unique(c).astype(np.int32)


def lidar_scan(n_points: int = 200_000, seed: int = 1, extent: float = 4.0,
               voxel=(0.05, 0.05, 0.05), batch: int = 0) -> np.ndarray:
    """C2 recipe: planar_patches n=200k, extent 4, 5 cm voxels
    -> ~125k voxels."""
    return quantize(planar_patches(n_points, seed, extent), voxel, batch)


def waymo_scan(n_points: int = 275_000, seed: int = 1, extent: float = 8.0,
               voxel=(0.1, 0.1, 0.15), batch: int = 0) -> np.ndarray:
    """C3 recipe: planar_patches n=275k, extent 8, voxel (0.1, 0.1, 0.15)."""
    return quantize(planar_patches(n_points, seed, extent), voxel, batch)


def random_instance_coords(seed: int, n: int, lo: int = -12, hi: int = 12, batches: int = 1,
                           dims: int = 3) -> np.ndarray:
    """make_random_instance coordinates (golden.hpp:95-106) with numpy RNG."""
    rng = np.random.default_rng(seed)
    raw = rng.integers(lo, hi + 1, size=(n, 3))
    if dims == 2:
        raw[:, 2] = 0
    b = rng.integers(0, batches, size=(n, 1))
    return first_unique(np.concatenate([b, raw], 1).astype(np.int32)).astype(np.int32)
