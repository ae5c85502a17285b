"""Pins for oracle/extract.py (not gpu): modulus switching and coefficient extraction of the
server's output ciphertexts (reading R16).

* exact rounding: round(c Q'/Q) against Python's exact rational arithmetic (fractions) on
  random, edge and near-half values;
* the error property |c' P - c| < P/2 (P = Q/Q') checked with plain integers;
* end to end: the server's conv output, switched to L' limbs and extracted, decrypts (as LWE
  ciphertexts at the designated coefficients) with the server share to conv(x0 + x1, K) mod 2^37
  (PAPER.md:441 exactness; PAPER.md:131 sparse output).
"""
from fractions import Fraction
import math

import numpy as np
import pytest

from oracle import conv, extract, he, packing, params
from oracle.params import Params
from workloads import inputs, layers


def _residues(P, vals):
    return np.array([[v % q for v in vals] for q in P.primes], dtype=np.uint64)


@pytest.mark.parametrize("primes,keep", [(params.PRIMES32, 2), (params.PRIMES32, 3), (params.PRIMES32, 1),
                                         (params.DEFAULT_PRIMES, 1)])
def test_modswitch_exact_rounding_and_error_bound(primes, keep):
    P = Params(logn=4, primes=primes)
    Ps = extract.switched_params(P, keep)
    Q, Qp = P.Q, Ps.Q
    Pd = Q // Qp
    g = np.random.default_rng(keep)
    vals = [0, 1, Q - 1, Pd, 5 * Pd, Pd // 2, Pd // 2 + 1, Q - Pd // 2, Q // 2]
    vals += [int(x) % Q for x in g.integers(0, 2**62, 7)]
    got = extract.modswitch(_residues(P, vals)[None], keep, P)[0]
    for k, c in enumerate(vals):
        exact = math.floor(Fraction(c * Qp, Q) + Fraction(1, 2)) % Qp
        assert [int(got[i, k]) for i in range(keep)] == [exact % q for q in Ps.primes], (k, c)
        # error property with plain integers: c' P - c is within P/2 of a multiple of Q
        d = (exact * Pd - c) % Q
        assert min(d, Q - d) <= Pd // 2
    assert [int(got[i, 3]) for i in range(keep)] == [1 % q for q in Ps.primes]  # c = P -> 1
    assert all(int(got[i, 2]) == 0 for i in range(keep))                       # c = Q - 1 -> Q' = 0


def _e2e(layer, P, keep, seed):
    pl = packing.plan_conv(layer.C, layer.H, layer.W, layer.M, layer.k, layer.k, layer.stride, layer.pad, P.n, P.L)
    g = inputs.rng(seed)
    x1 = inputs.uniform_below(g, (layer.C, layer.H, layer.W), P.t)
    x0 = inputs.uniform_below(g, (layer.C, layer.H, layer.W), P.t)
    K = inputs.quantized_kernel(g, layer.M, layer.C, layer.k, layer.k)
    sk = inputs.ternary(g, P.n)
    xin = packing.pack_input(x1, pl, P.n)
    ct = np.stack([he.encrypt(xin[i], sk, inputs.uniform_residues(g, (), P.primes, P.n),
                              inputs.rounded_gaussian(g, P.n), P) for i in range(pl.G * pl.S)])
    r = inputs.uniform_below(g, (pl.M * pl.S, P.n), P.t)
    out = he.server_conv(ct, packing.pack_input(x0, pl, P.n), K, r, pl, P)
    s_idx, coef = packing.designated_map(pl)
    a, b = extract.server_lwe_outputs(out, keep, P, s_idx, coef, pl.M, pl.S)
    Ps = extract.switched_params(P, keep)
    y = np.zeros((pl.M, pl.OH, pl.OW), np.uint64)
    for m in range(pl.M):
        for s in range(pl.S):
            sel = s_idx == s
            if sel.any():
                dec = extract.decrypt_lwe(a[m * pl.S + s], b[m][sel], coef[sel], sk, Ps)
                y[m][sel] = (dec + (P.t - r[m * pl.S + s, coef[sel]]) % P.t) % np.uint64(P.t)
    ref = conv.conv2d_mod((x0 + x1) & np.uint64(P.t - 1), K, layer.stride, layer.pad, P.t_bits)
    return y, ref


@pytest.mark.parametrize("primes,keep", [(params.DEFAULT_PRIMES, 1), (params.PRIMES32, 2)], ids=["q60_49->q60", "q27x4->x2"])
def test_e2e_switched_extracted_outputs_decrypt_to_conv(primes, keep):
    y, ref = _e2e(layers.tiny()[0], Params(primes=primes), keep, 51)
    assert (y == ref).all()


@pytest.mark.parametrize("lay,seed", [(layers.ConvLayer("s2", 3, 20, 20, 4, 3, 2, 0), 52),
                                      (layers.ConvLayer("multi", 9, 9, 9, 3, 3, 1, 1), 53)])
def test_e2e_switched_small_ring(lay, seed):
    y, ref = _e2e(lay, Params(logn=8, primes=params.PRIMES32), 2, seed)
    assert (y == ref).all()
