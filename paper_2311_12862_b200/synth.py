"""Synthetic scans for tests and benchmarks (seeded, host side).

Exact restatement of the reference's generators so both bench arms and the
parity tests see the survey's voxel counts:

* ``MT19937_64`` — std::mt19937_64 (vectorised twist, checked against the
  standard's 10000th-output value);
* ``_Canonical`` — libstdc++ generate_canonical<double, 53> (one 64-bit draw,
  x / 2^64), uniform_real_distribution(0, 1) and the Marsaglia-polar
  normal_distribution with its cached second value;
* ``gen_cloud`` (gen.cpp:32-85: uniform / planar_patches /
  gaussian_clusters) and ``quantize`` (tensor.cpp:87-142: floor(p / voxel),
  first-appearance dedup);
* ``uniform_int`` = uniform_int_distribution<int32_t> on a 64-bit engine
  (Lemire's nearly-divisionless reduction, libstdc++ 13) for the C1 cloud and
  make_random_instance (golden.hpp:95-106).

Pinned against the compiled reference's gen_cloud / quantize in
tests/test_synth.py. This module is input generation only: no product code
path reads it.
"""
from __future__ import annotations

import math

import numpy as np

_U64 = np.uint64
_M64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (the C++ standard's parameters)."""

    NN, MM = 312, 156
    _A = _U64(0xB5026F5AA96619E9)
    _UM = _U64(0xFFFFFFFF80000000)
    _LM = _U64(0x7FFFFFFF)

    def __init__(self, seed: int):
        mt = [seed & _M64]
        for i in range(1, self.NN):
            prev = mt[-1]
            mt.append((6364136223846793005 * (prev ^ (prev >> 62)) + i) & _M64)
        self.mt = np.array(mt, dtype=_U64)
        self.buf = np.empty(0, _U64)
        self.pos = 0

    def _mix(self, a, b):
        x = (a & self._UM) | (b & self._LM)
        return (x >> _U64(1)) ^ np.where((x & _U64(1)) != 0, self._A, _U64(0))

    def _twist(self):
        mt, NN, MM = self.mt, self.NN, self.MM
        # each slice reads only values the sequential recurrence would see
        mt[:NN - MM] = mt[MM:] ^ self._mix(mt[:NN - MM], mt[1:NN - MM + 1])
        mt[NN - MM:NN - 1] = mt[:MM - 1] ^ self._mix(mt[NN - MM:NN - 1], mt[NN - MM + 1:NN])
        mt[NN - 1] = mt[MM - 1] ^ self._mix(mt[NN - 1:NN], mt[0:1])[0]
        y = mt.copy()
        y ^= (y >> _U64(29)) & _U64(0x5555555555555555)
        y ^= (y << _U64(17)) & _U64(0x71D67FFFEDA60000)
        y ^= (y << _U64(37)) & _U64(0xFFF7EEE000000000)
        y ^= y >> _U64(43)
        return y

    def raw(self, n: int) -> np.ndarray:
        out = []
        while n > 0:
            if self.pos >= len(self.buf):
                self.buf, self.pos = self._twist(), 0
            take = min(n, len(self.buf) - self.pos)
            out.append(self.buf[self.pos:self.pos + take])
            self.pos += take
            n -= take
        return np.concatenate(out) if out else np.empty(0, _U64)


class _Canonical:
    """uniform_real_distribution<double>(0, 1) and normal_distribution<double>
    (0, 1) sharing one engine, as gen.cpp uses them."""

    def __init__(self, seed: int):
        self.eng = MT19937_64(seed)
        self.saved = None

    def uni(self, n: int) -> np.ndarray:
        # generate_canonical<double, 53>: double(x) / 2^64, clamped below 1
        u = self.eng.raw(n).astype(np.float64) / 18446744073709551616.0
        return np.where(u >= 1.0, np.nextafter(1.0, 0.0), u)

    def gauss(self) -> float:
        if self.saved is not None:
            v, self.saved = self.saved, None
            return v
        while True:
            x = 2.0 * float(self.uni(1)[0]) - 1.0
            y = 2.0 * float(self.uni(1)[0]) - 1.0
            r2 = x * x + y * y
            if not (r2 > 1.0 or r2 == 0.0):
                break
        mult = math.sqrt(-2 * math.log(r2) / r2)  # libm, like std::log / std::sqrt
        self.saved = x * mult
        return y * mult


def _normalize(v):
    n = math.sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2])
    if n < 1e-12:
        return (1.0, 0.0, 0.0)
    return (v[0] / n, v[1] / n, v[2] / n)


def _cross(a, b):
    return (a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0])


CLOUD_KINDS = {"uniform": 0, "planar_patches": 1, "gaussian_clusters": 2}


def gen_cloud(kind, n: int, seed: int, extent: float) -> np.ndarray:
    """gen_cloud (gen.cpp:32-85) bit for bit -> float64 [n, 3]."""
    kind = CLOUD_KINDS.get(kind, kind)
    if n < 0:
        raise ValueError("point count must be >= 0")
    if not extent > 0:
        raise ValueError("extent must be positive")
    r = _Canonical(seed)
    if kind == 0:
        return (r.uni(3 * n) * extent).reshape(n, 3)
    out = []
    if kind == 1:
        n_p = max(1, n // 2500)
        per = n // n_p
        for p in range(n_p):
            c = [float(x) * extent for x in r.uni(3)]
            nrm = _normalize((r.gauss(), r.gauss(), r.gauss()))
            ref = (1.0, 0.0, 0.0) if abs(nrm[0]) < 0.9 else (0.0, 1.0, 0.0)
            u = _normalize(_cross(nrm, ref))
            v = _cross(nrm, u)
            radius = (0.2 + 0.3 * float(r.uni(1)[0])) * extent
            m = n - per * (n_p - 1) if p == n_p - 1 else per
            ab = r.uni(2 * m).reshape(m, 2)
            a = (2 * ab[:, 0] - 1) * radius
            b = (2 * ab[:, 1] - 1) * radius
            out.append(np.stack([(c[d] + a * u[d]) + b * v[d] for d in range(3)], 1))
    elif kind == 2:
        n_c = max(1, n // 4000)
        per = n // n_c
        for p in range(n_c):
            c = [float(x) * extent for x in r.uni(3)]
            sigma = (0.05 + 0.1 * float(r.uni(1)[0])) * extent
            m = n - per * (n_c - 1) if p == n_c - 1 else per
            g = np.array([r.gauss() for _ in range(3 * m)]).reshape(m, 3)
            out.append(np.asarray(c)[None, :] + sigma * g)
    else:
        raise ValueError(f"unknown cloud kind {kind}")
    return np.concatenate(out, 0) if out else np.zeros((0, 3))


def uniform_int(eng: MT19937_64, lo: int, hi: int, n: int) -> np.ndarray:
    """n draws of uniform_int_distribution<int32_t>(lo, hi) on a 64-bit engine
    (libstdc++ 13, Lemire: product = x * range; the high 64 bits are the draw,
    a low half below (2^64 - range) % range means redraw)."""
    rng = hi - lo + 1
    assert 0 < rng < (1 << 32)
    thr = ((1 << 64) - rng) % rng
    x = eng.raw(n)
    lo_part = (x & _U64(0xFFFFFFFF)) * _U64(rng)
    hi64 = ((x >> _U64(32)) * _U64(rng) + (lo_part >> _U64(32))) >> _U64(32)
    if thr and bool(np.any(x * _U64(rng) < _U64(thr))):
        # p < 2^-32 per draw for these ranges; an exact redraw would shift
        # the rest of the stream, so refuse rather than diverge silently
        raise RuntimeError("uniform_int: rejection sample hit; sequence not restated")
    return hi64.astype(np.int64) + lo


def first_unique(coords: np.ndarray) -> np.ndarray:
    """Rows of `coords` deduplicated keeping first appearance order."""
    _, first = np.unique(coords, axis=0, return_index=True)
    return coords[np.sort(first)]


def uniform_voxels(draws: int, hi: int, seed: int, batch: int = 0) -> np.ndarray:
    """`draws` points of uniform_int_distribution<int32_t>(0, hi-1)^3 on
    mt19937_64(seed) (x, y, z per point), first-appearance dedup -> int32
    [n, 4]. C1: draws=127000, hi=64, seed=1 -> 100,642 voxels."""
    p = uniform_int(MT19937_64(seed), 0, hi - 1, 3 * draws).reshape(draws, 3).astype(np.int32)
    c = np.concatenate([np.full((draws, 1), batch, np.int32), p], 1)
    return first_unique(c).astype(np.int32)


def planar_patches(n: int, seed: int, extent: float) -> np.ndarray:
    """Quick numpy-RNG cloud of the planar_patches SHAPE (gen.cpp:44-61) for
    small test scans; gen_cloud is the exact restatement."""
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
    """C2 recipe: gen_cloud(planar_patches, n=200k, seed,
    extent 4), 5 cm voxels -> 124,756 voxels at seed 1."""
    return quantize(gen_cloud("planar_patches", n_points, seed, extent), voxel, batch)


def waymo_scan(n_points: int = 275_000, seed: int = 1, extent: float = 8.0,
               voxel=(0.1, 0.1, 0.15), batch: int = 0) -> np.ndarray:
    """C3 recipe: gen_cloud(planar_patches, n=275k, extent 8), voxel
    (0.1, 0.1, 0.15) -> 149,357 voxels at seed 1."""
    return quantize(gen_cloud("planar_patches", n_points, seed, extent), voxel, batch)


def sweep_cloud(n_points: int, seed: int = 1, extent: float = 2.0, voxel=0.025,
                tiles: int = 1, batch: int = 0) -> np.ndarray:
    """C5 recipe: gen_cloud(planar_patches, n, seed, extent 2) at voxel 0.025;
    tiles > 1 concatenates `tiles` disjoint copies (seeds seed..seed+tiles-1,
    tile t shifted +200 t voxels in x), e.g. 1M voxels = 10 tiles of n=160k."""
    out = []
    for t in range(tiles):
        c = quantize(gen_cloud("planar_patches", n_points, seed + t, extent), [voxel] * 3, batch)
        c[:, 1] += 200 * t
        out.append(c)
    return np.concatenate(out, 0)


def random_instance_coords(seed: int, n: int, lo: int = -12, hi: int = 12, batches: int = 1,
                           dims: int = 3) -> np.ndarray:
    """make_random_instance coordinates (golden.hpp:95-106) with numpy RNG."""
    rng = np.random.default_rng(seed)
    raw = rng.integers(lo, hi + 1, size=(n, 3))
    if dims == 2:
        raw[:, 2] = 0
    b = rng.integers(0, batches, size=(n, 1))
    return first_unique(np.concatenate([b, raw], 1).astype(np.int32)).astype(np.int32)
