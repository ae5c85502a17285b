"""HE fully-connected layer (matrix-vector product) -- oracle side (test infrastructure only).

SURVEY.md §8f row 3. The paper: "The typical linear layers in CNNs consist of the convolution
layers, fully-connected/matrix multiplication layers ... matrix multiplications that appear only
at the very end of the CNN" (§6); SPEC.md:612-619 (`fc_secure`: "same protocol
shape as conv2d_secure with a dot-product packing; exact mod 2^b").

The server's computation is the one of ``he.server_mac`` (share add, sum over input blocks of
ct (*) plaintext, mask); only the packing differs. Reading R15 (paper silent; Cheetah's
matrix-vector packing [outside]): with block sizes nib (inputs per poly) and nob (output rows
per poly), nib * nob <= N,

    input poly g:        coeff[i]                      = x[g*nib + i]                 (i < nib)
    weight poly (m, g):  coeff[j*nib + nib - 1 - i]    = W[m*nob + j, g*nib + i]      (j < nob, i < nib)
    output poly m, designated coefficient j*nib + nib - 1
                       = sum_g sum_i x[g*nib + i] W[m*nob + j, g*nib + i]  = y[m*nob + j]

(the product term x_a w_b lands at a + b; for the designated index the bounds force a = i and
b inside row j's segment, and a + b < nib + nob*nib <= N + nib - 1 never wraps onto it). The
block sizes minimise the algorithmic bytes of the layer as reading R6 does for convolutions:
    8*L*N*(2*G + M*G + 2*M) + 8*N*M,   G = ceil(n_i/nib), M = ceil(n_o/nob),  nob = min(n_o, N // nib)
tie-breaking on fewer M*G products, then larger nib. Pinned by tests/test_oracle_fc.py
(decrypt(server_fc(Enc(x1), x0, W, r)) + (t - r) = W (x0 + x1) mod 2^t, and brute force).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import he
from .params import Params


@dataclass(frozen=True)
class FcPlan:
    n_i: int
    n_o: int
    nib: int  # input values per input poly
    nob: int  # output rows per output poly
    G: int    # input polys (input blocks)
    M: int    # output polys (output blocks)


def plan_fc(n_i: int, n_o: int, n: int = 4096, L: int = 2, nib: Optional[int] = None) -> FcPlan:
    """Reading R15 (module docstring). An explicit nib is validated and used instead."""
    if n_i < 1 or n_o < 1:
        raise ValueError("empty matrix")
    cands = [nib] if nib is not None else range(1, min(n_i, n) + 1)
    best = None
    for a in cands:
        if a < 1 or a > min(n_i, n):
            continue
        b = min(n_o, n // a)
        G, M = -(-n_i // a), -(-n_o // b)
        cost = 8 * L * n * (2 * G + M * G + 2 * M) + 8 * n * M
        key = (cost, M * G, -a)
        if best is None or key < best[0]:
            best = (key, a, b, G, M)
    if best is None:
        raise ValueError("invalid nib")
    _, a, b, G, M = best
    return FcPlan(n_i, n_o, a, b, G, M)


def pack_fc_input(x: np.ndarray, p: FcPlan, n: int) -> np.ndarray:
    """Input share x [n_i] -> polys [G][N]."""
    out = np.zeros((p.G, n), dtype=np.uint64)
    for g in range(p.G):
        seg = x[g * p.nib:(g + 1) * p.nib]
        out[g, :seg.size] = seg
    return out


def fc_weight_polys(Wm: np.ndarray, p: FcPlan, n: int) -> np.ndarray:
    """W [n_o][n_i] (values < 2^t) -> raw mirrored plaintext polys [M][G][N] (not lifted)."""
    out = np.zeros((p.M, p.G, n), dtype=np.uint64)
    for m in range(p.M):
        for g in range(p.G):
            for j in range(p.nob):
                o = m * p.nob + j
                if o >= p.n_o:
                    break
                for i in range(p.nib):
                    c = g * p.nib + i
                    if c >= p.n_i:
                        break
                    out[m, g, j * p.nib + p.nib - 1 - i] = Wm[o, c]
    return out


def fc_designated(p: FcPlan):
    """(poly index, coefficient index) of every output y[o], o < n_o."""
    o = np.arange(p.n_o)
    return o // p.nob, (o % p.nob) * p.nib + p.nib - 1


def fc_extract(polys: np.ndarray, p: FcPlan) -> np.ndarray:
    """polys [M][N] (values mod t) -> y [n_o] at the designated coefficients."""
    m, coef = fc_designated(p)
    return polys[m, coef]


def server_fc(ct_in: np.ndarray, x0: Optional[np.ndarray], Wm: np.ndarray, r: Optional[np.ndarray], p: FcPlan,
              P: Params, sel: Optional[np.ndarray] = None) -> np.ndarray:
    """ct_in [G][2][L][N], x0 [G][N] or None, W [n_o][n_i] < 2^t, r [M][N] or None -> [M][2][L][N]."""
    return he.server_mac(ct_in, x0, fc_weight_polys(Wm, p, P.n), r, p.G, 1, p.M, P, sel)


def matvec_mod(Wm: np.ndarray, x: np.ndarray, t_bits: int) -> np.ndarray:
    """Plain y = W x mod 2^t_bits in uint64 wrap-around arithmetic (exact: 2^t | 2^64)."""
    Wu = np.ascontiguousarray(Wm, dtype=np.uint64)
    xu = np.ascontiguousarray(x, dtype=np.uint64)
    y = np.zeros(Wu.shape[0], dtype=np.uint64)
    with np.errstate(over="ignore"):
        for c in range(Wu.shape[1]):
            y += Wu[:, c] * xu[c]
    return y & np.uint64((1 << t_bits) - 1)
