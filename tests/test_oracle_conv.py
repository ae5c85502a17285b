"""Pins for oracle/conv.py (plain integer convolution mod 2^t), not gpu."""
import numpy as np
import pytest
import torch

from oracle import conv


def _brute(x, K, stride, pad, t_bits):
    C, H, W = x.shape
    M, _, kh, kw = K.shape
    OH, OW = (H + 2 * pad - kh) // stride + 1, (W + 2 * pad - kw) // stride + 1
    y = np.zeros((M, OH, OW), dtype=object)
    for m in range(M):
        for oy in range(OH):
            for ox in range(OW):
                s = 0
                for c in range(C):
                    for l in range(kh):
                        for l2 in range(kw):
                            iy, ix = oy * stride + l - pad, ox * stride + l2 - pad
                            if 0 <= iy < H and 0 <= ix < W:
                                s += int(x[c, iy, ix]) * int(K[m, c, l, l2])
                y[m, oy, ox] = s % (1 << t_bits)
    return y.astype(np.uint64)


@pytest.mark.parametrize("shape,stride,pad", [((2, 5, 5, 3, 2), 1, 0), ((3, 7, 6, 2, 3), 2, 1), ((1, 4, 4, 2, 1), 2, 0)])
def test_conv_matches_bruteforce_bigint(shape, stride, pad):
    C, H, W, M, k = shape
    rng = np.random.default_rng(1)
    x = rng.integers(0, 1 << 37, (C, H, W), dtype=np.uint64)
    K = rng.integers(0, 1 << 37, (M, C, k, k), dtype=np.uint64)
    assert (conv.conv2d_mod(x, K, stride, pad, 37) == _brute(x, K, stride, pad, 37)).all()


def test_conv_matches_torch_float64_small_values():
    rng = np.random.default_rng(2)
    x = rng.integers(0, 1000, (4, 16, 16), dtype=np.uint64)
    K = rng.integers(0, 1000, (8, 4, 3, 3), dtype=np.uint64)
    ref = torch.nn.functional.conv2d(torch.tensor(x.astype(np.float64))[None], torch.tensor(K.astype(np.float64)),
                                     stride=1, padding=1)[0].numpy().astype(np.uint64)
    assert (conv.conv2d_mod(x, K, 1, 1, 37) == ref).all()
