"""Plain integer 2-D convolution mod 2^t (test infrastructure only).

SecONNds' linear layers are exact over Z_{2^b} (§8, §6.1), so the
reconstructed secure output must equal this plaintext convolution mod 2^37 bit for bit.
uint64 wrap-around arithmetic is exact mod 2^t because 2^t divides 2^64.
"""
from __future__ import annotations

import numpy as np


def conv2d_mod(x: np.ndarray, K: np.ndarray, stride: int, pad: int, t_bits: int) -> np.ndarray:
    """x (C,H,W), K (M,C,kh,kw), both uint64 -> y (M,OH,OW) uint64 in [0, 2^t):
    y[m,oy,ox] = sum_{c,l,l'} x[c, oy*stride + l - pad, ox*stride + l' - pad] K[m,c,l,l'] (0 outside)."""
    C, H, W = x.shape
    M, C2, kh, kw = K.shape
    assert C == C2
    OH = (H + 2 * pad - kh) // stride + 1
    OW = (W + 2 * pad - kw) // stride + 1
    xp = np.zeros((C, H + 2 * pad, W + 2 * pad), dtype=np.uint64)
    xp[:, pad:pad + H, pad:pad + W] = x
    y = np.zeros((M, OH, OW), dtype=np.uint64)
    with np.errstate(over="ignore"):
        for c in range(C):
            for l in range(kh):
                for l2 in range(kw):
                    patch = xp[c, l:l + (OH - 1) * stride + 1:stride, l2:l2 + (OW - 1) * stride + 1:stride]
                    y += K[:, c, l, l2][:, None, None] * patch[None]
    return y & np.uint64((1 << t_bits) - 1)
