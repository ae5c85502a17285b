"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This module draws random numbers only; it holds none of the method's arithmetic (no
encoding, no NTT, no packing). Every quantity the method itself draws (the server's output
mask r, §7) is generated here and passed in as an input to both sides.

Distributions:
* ciphertext residues: uniform in [0, q_j) per limb -- a fresh RLWE ciphertext is
  computationally indistinguishable from uniform (App. C);
* secret shares x0, x1 and masks r: uniform in [0, 2^t_bits) (§2.1);
* kernels: round(2^12 * N(0, 2/fan_in)) mod 2^37, the 37-bit / scale-12 fixed point of
  PAPER.md:441 (§8) with He-normal weights;
* client key material (test harness only): ternary secret, rounded Gaussian error
  (sigma = 3.2, |e| <= 19) as in PAPER.md:657 (App. C) / SPEC.md:551.
"""
from __future__ import annotations

from typing import Sequence

import numpy as np


def rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(np.random.PCG64(seed))


def uniform_below(g: np.random.Generator, shape, bound: int) -> np.ndarray:
    """uint64 array, i.i.d. uniform in [0, bound)."""
    return g.integers(0, bound, size=shape, dtype=np.uint64)


def uniform_residues(g: np.random.Generator, lead_shape, primes: Sequence[int], n: int) -> np.ndarray:
    """uint64 array of shape (*lead_shape, L, n); limb j uniform in [0, primes[j])."""
    lead_shape = tuple(lead_shape)
    out = np.empty(lead_shape + (len(primes), n), dtype=np.uint64)
    for j, q in enumerate(primes):
        out[..., j, :] = g.integers(0, q, size=lead_shape + (n,), dtype=np.uint64)
    return out


def quantized_kernel(g: np.random.Generator, M: int, C: int, kh: int, kw: int, t_bits: int = 37,
                     scale_bits: int = 12) -> np.ndarray:
    """uint64 (M, C, kh, kw) fixed-point weights in [0, 2^t_bits) (two's complement mod 2^t)."""
    fan_in = C * kh * kw
    w = np.rint(g.normal(0.0, np.sqrt(2.0 / fan_in), size=(M, C, kh, kw)) * (1 << scale_bits)).astype(np.int64)
    return (w.astype(np.uint64)) & np.uint64((1 << t_bits) - 1)


def full_range_kernel(g: np.random.Generator, M: int, C: int, kh: int, kw: int, t_bits: int = 37) -> np.ndarray:
    """Worst-case kernels: uniform in [0, 2^t_bits) (stresses the centred lift and the noise bound)."""
    return uniform_below(g, (M, C, kh, kw), 1 << t_bits)


def ternary(g: np.random.Generator, n: int) -> np.ndarray:
    """int64 array in {-1, 0, 1}, uniform."""
    return g.integers(-1, 2, size=n, dtype=np.int64)


def rounded_gaussian(g: np.random.Generator, n: int, sigma: float = 3.2, bound: int = 19) -> np.ndarray:
    """int64 array: round(N(0, sigma^2)) clipped to [-bound, bound]."""
    return np.clip(np.rint(g.normal(0.0, sigma, size=n)), -bound, bound).astype(np.int64)
