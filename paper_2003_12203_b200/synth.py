"""Seeded synthetic inputs and fault samplers for the BASELINE.json configs.

No dataset is used: ImageNet and the paper's pretrained models are
replaced by seeded tensors with the configs' shapes and value distributions.  The
same arrays feed the GPU path and the CPU oracle, so any seeded generator works;
numpy's PCG64 is used (fast, portable).
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def relu_like(shape, seed: int) -> np.ndarray:
    """Config 1 input: each element 0 with p=0.5, else U(0,1)."""
    g = np.random.default_rng(seed)
    zero = g.random(shape) < 0.5
    v = g.random(shape)
    return np.where(zero, 0.0, v).astype(np.float32)


def normal(shape, sigma: float, seed: int) -> np.ndarray:
    g = np.random.default_rng(seed)
    return (g.standard_normal(shape) * sigma).astype(np.float32)


def uniform(shape, lo: float, hi: float, seed: int) -> np.ndarray:
    g = np.random.default_rng(seed)
    return g.uniform(lo, hi, shape).astype(np.float32)


def he_normal(M: int, Ckw: int, R: int, seed: int) -> np.ndarray:
    """He-normal kernels N(0, sqrt(2/(Ckw*R*R)))."""
    return normal((M, Ckw, R, R), float(np.sqrt(2.0 / (Ckw * R * R))), seed)


def config1(seed: int = 12345):
    """BASELINE config 1: N=16, Cin=64, H=56, Cout=64, 3x3, s1, p1."""
    D = relu_like((16, 64, 56, 56), seed)
    W = he_normal(64, 64, 3, seed + 1)
    return D, W


def flip_sample(base: int, r: int, N: int, M: int, E: int, bit_lo: int = 20, bit_hi: int = 30):
    """Run r of a seeded single-flip campaign: seed_r = splitmix64(base ^ r) ->
    (n, m, x, y, bit) with bit in [bit_lo, bit_hi]."""
    s = splitmix64((base ^ r) & MASK64)
    g = np.random.default_rng(s)
    n = int(g.integers(0, N))
    m = int(g.integers(0, M))
    x = int(g.integers(0, E))
    y = int(g.integers(0, E))
    bit = int(g.integers(bit_lo, bit_hi + 1))
    return n, m, x, y, bit


def flip32(v, bit: int) -> np.float32:
    """fault.hpp:82-87 on an FP32 word (sign bit excluded)."""
    u = np.array([v], np.float32).view(np.uint32)
    u ^= np.uint32(1 << (bit % 31))
    return u.view(np.float32)[0]
