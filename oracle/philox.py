"""Philox4x32-10 and the server's mask drawn from it -- oracle side (test infrastructure only).

The paper's server "applies a random mask for security" (§7) without saying how r
is drawn. Reading R17: the library can draw r itself on the device from the
counter-based generator Philox4x32-10 (Salmon, Moraes, Dror, Shaw, "Parallel Random Numbers: As
Easy as 1, 2, 3", SC'11), so the server's mask never crosses PCIe. This module is the plain
definition of that draw, written from the generator's specification:

    round:  (c0, c1, c2, c3) -> (hi(M1 c2) ^ c1 ^ k0, lo(M1 c2), hi(M0 c0) ^ c3 ^ k1, lo(M0 c0))
            with M0 = 0xD2511F53, M1 = 0xCD9E8D57 (32 x 32 -> 64-bit products)
    key schedule: (k0, k1) += (0x9E3779B9, 0xBB67AE85) between rounds; 10 rounds.

The mask word of output ciphertext c (the layer's output index m*S + s, plus the call's first
index ct0 for a rank slice), coefficient e, for the 64-bit seed and the 32-bit stream id u:

    (w0, w1, w2, w3) = Philox4x32-10(counter = (e >> 1, c, u, 0), key = (seed mod 2^32, seed >> 32))
    r[c][e] = (w1 * 2^32 + w0) mod 2^t   if e is even,   (w3 * 2^32 + w2) mod 2^t   if e is odd.

2^t divides 2^64, so r is uniform on [0, 2^t). Pinned by the generator's published known-answer
vectors (tests/golden/philox4x32_10_kat.txt) and by NVIDIA's independent implementation
(curand_Philox4x32_10, compiled for the host in tests/test_oracle_philox.py).
"""
from __future__ import annotations

import numpy as np

M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
_MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr, key):
    """ctr: 4 arrays (or ints) of 32-bit counter words; key: 2 of 32-bit key words (broadcast).
    Returns the 4 output words as uint64 arrays holding 32-bit values."""
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint64) & _MASK32 for x in ctr)
    k0, k1 = (np.asarray(x, dtype=np.uint64) & _MASK32 for x in key)
    m0, m1 = np.uint64(M0), np.uint64(M1)
    for rnd in range(10):
        if rnd:
            k0 = (k0 + np.uint64(W0)) & _MASK32
            k1 = (k1 + np.uint64(W1)) & _MASK32
        p0 = m0 * c0  # < 2^64: exact in uint64
        p1 = m1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK32
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return c0, c1, c2, c3


def philox4x32_10_int(ctr, key):
    """The same generator on Python integers (one counter), for the known-answer tests."""
    c = [int(x) & 0xFFFFFFFF for x in ctr]
    k = [int(x) & 0xFFFFFFFF for x in key]
    for rnd in range(10):
        if rnd:
            k = [(k[0] + W0) & 0xFFFFFFFF, (k[1] + W1) & 0xFFFFFFFF]
        p0, p1 = M0 * c[0], M1 * c[2]
        c = [(p1 >> 32) ^ c[1] ^ k[0], p1 & 0xFFFFFFFF, (p0 >> 32) ^ c[3] ^ k[1], p0 & 0xFFFFFFFF]
    return c


def mask(seed: int, stream: int, n_ct: int, n: int, t_bits: int, ct0: int = 0) -> np.ndarray:
    """r [n_ct][n] (uint64 < 2^t_bits) for output ciphertexts ct0 .. ct0 + n_ct - 1 (reading R17)."""
    e = np.arange(n // 2, dtype=np.uint64)
    out = np.empty((n_ct, n), dtype=np.uint64)
    key = (seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    tm = np.uint64((1 << t_bits) - 1)
    for i in range(n_ct):
        w0, w1, w2, w3 = philox4x32_10((e, np.full_like(e, ct0 + i), np.full_like(e, stream), np.zeros_like(e)), key)
        out[i, 0::2] = ((w1 << np.uint64(32)) | w0) & tm
        out[i, 1::2] = ((w3 << np.uint64(32)) | w2) & tm
    return out
