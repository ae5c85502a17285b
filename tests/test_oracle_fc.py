"""Pins for oracle/fc.py (not gpu): the HE fully-connected layer.

The end-to-end pin is the paper's exactness of linear layers over Z_{2^b} (
SPEC.md:612-619 `fc_secure`: "exact mod 2^b"): Dec(server_fc(Enc(x1), x0, W, r)) + (t - r)
= W (x0 + x1) mod 2^37 at every designated coefficient. A brute-force pin checks the packing
alone: the negacyclic product of the packed input and weight polys, computed with Python
integers, holds every dot product at its designated coefficient.
"""
import numpy as np
import pytest

from oracle import fc, he, params
from oracle.params import Params
from workloads import inputs


def _matrix(g, n_o, n_i, t, full=False):
    if full:
        return inputs.uniform_below(g, (n_o, n_i), t)
    return inputs.quantized_kernel(g, n_o, n_i, 1, 1).reshape(n_o, n_i)


@pytest.mark.parametrize("n_i,n_o,n", [(64, 16, 4096), (2048, 1000, 4096), (512, 1000, 4096), (5, 3, 64),
                                       (100, 37, 256), (4096, 1, 4096), (1, 4096, 4096)])
def test_plan_invariants(n_i, n_o, n):
    p = fc.plan_fc(n_i, n_o, n)
    assert p.nib * p.nob <= n
    assert p.G * p.nib >= n_i > (p.G - 1) * p.nib
    assert p.M * p.nob >= n_o > (p.M - 1) * p.nob
    assert p.nob == min(n_o, n // p.nib)


def _negacyclic(a, b, n):
    c = [0] * n
    for i, x in enumerate(a):
        if x:
            for j, y in enumerate(b):
                if y:
                    k = i + j
                    if k < n:
                        c[k] += x * y
                    else:
                        c[k - n] -= x * y
    return c


@pytest.mark.parametrize("n_i,n_o,n,nib", [(5, 3, 16, None), (7, 9, 32, 3), (12, 4, 64, None), (3, 40, 64, 1)])
def test_packing_brute_force(n_i, n_o, n, nib):
    """Plain integers, no encryption: sum_g x_g (*) w_{m,g} holds y[m*nob + j] at j*nib + nib - 1."""
    p = fc.plan_fc(n_i, n_o, n, nib=nib)
    g = np.random.default_rng(3)
    x = g.integers(0, 100, n_i)
    Wm = g.integers(0, 100, (n_o, n_i))
    X = fc.pack_fc_input(x.astype(np.uint64), p, n)
    Wp = fc.fc_weight_polys(Wm.astype(np.uint64), p, n)
    y = Wm @ x
    for m in range(p.M):
        acc = [0] * n
        for gg in range(p.G):
            prod = _negacyclic([int(v) for v in X[gg]], [int(v) for v in Wp[m, gg]], n)
            acc = [a + b for a, b in zip(acc, prod)]
        for j in range(p.nob):
            o = m * p.nob + j
            if o < n_o:
                assert acc[j * p.nib + p.nib - 1] == y[o], (m, j)


def _e2e(n_i, n_o, P, seed, full=False, with_x0=True, sel_blocks=None, Wm=None):
    p = fc.plan_fc(n_i, n_o, P.n, P.L)
    g = inputs.rng(seed)
    x1 = inputs.uniform_below(g, n_i, P.t)
    x0 = inputs.uniform_below(g, n_i, P.t) if with_x0 else np.zeros_like(x1)
    if Wm is None:
        Wm = _matrix(g, n_o, n_i, P.t, full)
    sk = inputs.ternary(g, P.n)
    xin = fc.pack_fc_input(x1, p, P.n)
    ct = np.stack([he.encrypt(xin[i], sk, inputs.uniform_residues(g, (), P.primes, P.n),
                              inputs.rounded_gaussian(g, P.n), P) for i in range(p.G)])
    r = inputs.uniform_below(g, (p.M, P.n), P.t)
    sel = None
    if sel_blocks is not None:
        sel = np.zeros(p.M, np.uint8)
        sel[list(sel_blocks)] = 1
    out = fc.server_fc(ct, fc.pack_fc_input(x0, p, P.n) if with_x0 else None, Wm, r, p, P, sel=sel)
    m_idx, coef = fc.fc_designated(p)
    y = np.zeros(n_o, np.uint64)
    done = np.zeros(n_o, bool)
    for m in range(p.M):
        if sel is not None and not sel[m]:
            continue
        pick = m_idx == m
        dec = he.decrypt(out[m], sk, P, coef[pick])
        y[pick] = (dec + (P.t - r[m, coef[pick]]) % P.t) % np.uint64(P.t)
        done[pick] = True
    ref = fc.matvec_mod(Wm, (x0 + x1) & np.uint64(P.t - 1), P.t_bits)
    return p, y[done], ref[done]


@pytest.mark.parametrize("primes", [params.DEFAULT_PRIMES, params.PRIMES32], ids=["q60_49", "q27x4"])
def test_e2e_spec_16x64_exact(primes):
    """SPEC.md:618 example: a random 16 x 64 matvec matches the plaintext result exactly."""
    p, y, ref = _e2e(64, 16, Params(primes=primes), 31)
    assert y.size == 16 and (y == ref).all()


@pytest.mark.parametrize("n_i,n_o,seed,full", [(100, 37, 32, False), (300, 50, 33, True), (17, 200, 34, True),
                                               (257, 5, 35, False)])
def test_e2e_small_ring_exact(n_i, n_o, seed, full):
    P = Params(logn=8, primes=params.PRIMES32 if seed % 2 else params.DEFAULT_PRIMES)
    p, y, ref = _e2e(n_i, n_o, P, seed, full=full)
    assert p.G > 1 or p.M > 1
    assert (y == ref).all()


def test_e2e_1000x512_tiled_sampled_blocks():
    """SPEC.md:619 example: a 1000 x 512 tiled matvec (two output blocks decrypted)."""
    P = Params()
    p = fc.plan_fc(512, 1000, P.n, P.L)
    _, y, ref = _e2e(512, 1000, P, 36, sel_blocks=(0, p.M - 1))
    assert y.size > 0 and (y == ref).all()


def test_identity_weights_reconstruct_input():
    """an identity-like weight reconstructs the input share sum."""
    P = Params(logn=8)
    n = 40
    Wm = np.eye(n, dtype=np.uint64)
    p, y, ref = _e2e(n, n, P, 37, Wm=Wm)
    assert (y == ref).all()


def test_no_server_share():
    P = Params(logn=8)
    _, y, ref = _e2e(50, 20, P, 38, with_x0=False)
    assert (y == ref).all()
