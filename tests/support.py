"""Test helpers mirroring the reference's tests/support/oracles.hpp.

``MT64`` is std::mt19937_64 with the libstdc++-13 ``uniform_real_distribution``
/ ``uniform_int_distribution`` draws (random.tcc:3349-3381,
uniform_int_dist.h:256-319), so scenes built here match the reference's
seeded fixtures value for value.
"""
from __future__ import annotations

import math

import numpy as np

from paper_2504_12905_b200.types import Camera, GaussianSet

_M64 = (1 << 64) - 1


class MT64:
    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & _M64
        for i in range(1, 312):
            prev = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & _M64
        self.idx = 312

    def __call__(self) -> int:
        if self.idx >= 312:
            mt = self.mt
            for i in range(312):
                y = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
                mt[i] = mt[(i + 156) % 312] ^ (y >> 1) ^ (0xB5026F5AA96619E9 if y & 1 else 0)
            self.idx = 0
        z = self.mt[self.idx]
        self.idx += 1
        z ^= (z >> 29) & 0x5555555555555555
        z ^= (z << 17) & 0x71D67FFFEDA60000 & _M64
        z ^= (z << 37) & 0xFFF7EEE000000000 & _M64
        z ^= z >> 43
        return z & _M64

    def canonical(self) -> float:
        r = float(self()) / 18446744073709551616.0
        return math.nextafter(1.0, 0.0) if r >= 1.0 else r

    def uniform_real(self, a: float, b: float) -> float:
        return self.canonical() * (b - a) + a

    def uniform_int(self, a: int, b: int) -> int:
        rng = (b - a) + 1
        prod = self() * rng
        low = prod & _M64
        if low < rng:
            thr = ((-rng) & _M64) % rng
            while low < thr:
                prod = self() * rng
                low = prod & _M64
        return (prod >> 64) + a


def random_scene(count: int, rng: MT64) -> GaussianSet:
    """oracles::random_scene (tests/support/oracles.hpp:66-84)."""
    g = GaussianSet.zeros(count)
    lo_s, hi_s = math.log(0.15), math.log(0.45)
    for i in range(count):
        for c in range(3):
            g.means[3 * i + c] = rng.uniform_real(-0.7, 0.7)
            g.log_scales[3 * i + c] = rng.uniform_real(lo_s, hi_s)
            g.colors[3 * i + c] = rng.uniform_real(-1.1, 1.1)
        for c in range(4):
            g.rotations[4 * i + c] = rng.uniform_real(-1.0, 1.0)
        g.opacity_logits[i] = rng.uniform_real(-0.8, 1.2)
    g.renormalize_rotations()
    return g


def test_camera(size: int = 32, dist: float = 3.0) -> Camera:
    """oracles::test_camera (oracles.hpp:86-94): identity rotation, f = size."""
    return Camera(np.eye(3).reshape(9), np.array([0.0, 0.0, dist]), float(size), float(size),
                  0.5 * size, 0.5 * size, size, size)


def random_image(w: int, h: int, rng: MT64) -> np.ndarray:
    """oracles::random_image (oracles.hpp:96-101)."""
    img = np.zeros((h, w, 3))
    flat = img.reshape(-1)
    for i in range(flat.size):
        flat[i] = rng.uniform_real(0.0, 1.0)
    return img


def random_vector(n: int, rng: np.random.Generator, scale: float = 1.0) -> np.ndarray:
    return rng.uniform(-scale, scale, n)


def rel_error(got: float, want: float) -> float:
    """oracles::rel_error (oracles.hpp:113-116)."""
    return abs(got - want) / max(abs(got), abs(want), 1e-300)


def norm_rel(got: np.ndarray, want: np.ndarray) -> float:
    """Norm-relative error, the north-star parity measure for vectors."""
    d = float(np.linalg.norm(np.asarray(got, np.float64) - np.asarray(want, np.float64)))
    n = float(np.linalg.norm(np.asarray(want, np.float64)))
    return d / max(n, 1e-300)


# ---- golden fixture loaders (tests/golden/*.npz, made by make_golden.py) ----
import os as _os

from paper_2504_12905_b200.types import SamplePlan

GOLDEN = _os.path.join(_os.path.dirname(_os.path.abspath(__file__)), "golden")
_golden_cache: dict = {}


def golden(name: str):
    if name not in _golden_cache:
        _golden_cache[name] = dict(np.load(_os.path.join(GOLDEN, f"{name}.npz")))
    return _golden_cache[name]


def g_cams(arr) -> list:
    cams = []
    for row in np.atleast_2d(arr):
        cams.append(Camera(row[0:9].copy(), row[9:12].copy(), row[12], row[13], row[14], row[15],
                           int(row[17]), int(row[18]), row[16]))
    return cams


def g_set(d, prefix) -> GaussianSet:
    g = GaussianSet(d[f"{prefix}_opacity_logits"].size)
    for k in ("means", "log_scales", "rotations", "opacity_logits", "colors"):
        setattr(g, k, d[f"{prefix}_{k}"].astype(np.float64).copy())
    return g


def g_plan(d, prefix, samples_per_tile=32) -> SamplePlan:
    return SamplePlan(d[f"{prefix}_view_camera"].astype(np.int32),
                      d[f"{prefix}_view_offset"].astype(np.int64),
                      d[f"{prefix}_px"].astype(np.int32), d[f"{prefix}_py"].astype(np.int32),
                      d[f"{prefix}_tile"].astype(np.int32), d[f"{prefix}_weight"].astype(np.float64),
                      samples_per_tile)
