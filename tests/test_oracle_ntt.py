"""Pins for the oracle's schoolbook product and direct-evaluation NTT/INTT (not gpu).

What pins them (other than themselves): the hand-checked N=8/q=17 worked example
(tests/golden/ntt_n8_q17.txt), a pure-Python big-integer polynomial product reduced mod
X^N+1, closed forms (constants, monomials, X^N = -1), the ring-isomorphism property
NTT(a*b) = NTT(a).NTT(b) (App. C.1) and INTT o NTT = id.
"""
from pathlib import Path

import numpy as np
import pytest

from oracle import he, params
from oracle.params import Params

GOLDEN = Path(__file__).parent / "golden"


def _small_params(logn, q):
    P = Params.__new__(Params)
    P.logn, P.primes, P.t_bits = logn, (q,), 2
    P.psi = [params.minimal_psi(q, 1 << logn)]
    return P


def _golden():
    d = {}
    for line in (GOLDEN / "ntt_n8_q17.txt").read_text().splitlines():
        if line.startswith("#") or ":" not in line:
            continue
        k, v = line.split(":")
        d[k.strip()] = np.array([int(x) for x in v.split()], dtype=np.uint64)
    return d


def _py_negacyclic(a, b, q):
    """Independent big-int product: full polynomial product, then fold X^(N+i) -> -X^i."""
    n = len(a)
    full = [0] * (2 * n)
    for i, x in enumerate(a):
        for j, y in enumerate(b):
            full[i + j] += int(x) * int(y)
    return np.array([(full[i] - full[i + n]) % q for i in range(n)], dtype=np.uint64)


def test_worked_example_n8_q17():
    g = _golden()
    P = _small_params(3, 17)
    assert P.psi[0] == 3
    assert (he.ntt(g["a"], P, 0) == g["ntt_a"]).all()
    assert (he.ntt(g["x"], P, 0) == g["ntt_x"]).all()
    assert (he.ntt(g["d"], P, 0) == g["ntt_d"]).all()
    assert (he.negacyclic_mul(g["a"], g["x"], 17) == g["a_times_x"]).all()
    assert (he.negacyclic_mul(g["a"], g["d"], 17) == g["a_times_d"]).all()
    prod = (g["ntt_a"] * g["ntt_d"]) % 17
    assert (he.intt(prod, P, 0) == g["a_times_d"]).all()


@pytest.mark.parametrize("logn,q", [(3, 17), (4, 97), (6, 0x1FFFFFFFCE001), (5, 0x0FFFFFFFFFFFC001)])
def test_schoolbook_matches_python_bigint(logn, q):
    rng = np.random.default_rng(logn)
    n = 1 << logn
    for _ in range(5):
        a = rng.integers(0, q, n, dtype=np.uint64)
        b = rng.integers(0, q, n, dtype=np.uint64)
        assert (he.negacyclic_mul(a, b, q) == _py_negacyclic(a, b, q)).all()


def test_exhaustive_n8_q17_ntt_product_equals_schoolbook():
    P = _small_params(3, 17)
    rng = np.random.default_rng(0)
    # all monomial pairs + random pairs
    for i in range(8):
        for j in range(8):
            a = np.zeros(8, np.uint64); a[i] = 1
            b = np.zeros(8, np.uint64); b[j] = rng.integers(1, 17)
            lhs = he.intt((he.ntt(a, P, 0) * he.ntt(b, P, 0)) % 17, P, 0)
            assert (lhs == he.negacyclic_mul(a, b, 17)).all()
    for _ in range(300):
        a = rng.integers(0, 17, 8, dtype=np.uint64)
        b = rng.integers(0, 17, 8, dtype=np.uint64)
        lhs = he.intt((he.ntt(a, P, 0) * he.ntt(b, P, 0)) % 17, P, 0)
        assert (lhs == he.negacyclic_mul(a, b, 17)).all()


@pytest.mark.parametrize("j", [0, 1])
def test_ntt_isomorphism_and_roundtrip_default_primes_n1024(j):
    P = Params(logn=10)
    q = P.primes[j]
    rng = np.random.default_rng(10 + j)
    a = rng.integers(0, q, P.n, dtype=np.uint64)
    b = rng.integers(0, q, P.n, dtype=np.uint64)
    A, B = he.ntt(a, P, j), he.ntt(b, P, j)
    assert (he.intt(A, P, j) == a).all()
    AB = np.array([int(x) * int(y) % q for x, y in zip(A, B)], dtype=np.uint64)
    assert (he.intt(AB, P, j) == he.negacyclic_mul(a, b, q)).all()


def test_ntt_closed_forms_n4096():
    P = Params()
    for j, q in enumerate(P.primes):
        c = np.zeros(P.n, np.uint64); c[0] = 123456789
        assert (he.ntt(c, P, j) == 123456789).all()           # constant -> constant vector
        x = np.zeros(P.n, np.uint64); x[1] = 1
        X = he.ntt(x, P, j)                                    # X -> the evaluation points
        assert len(set(X.tolist())) == P.n                     # N distinct points
        ks = [0, 1, 2, 3, 1000, 4095]
        assert all(pow(int(X[k]), P.n, q) == q - 1 for k in ks)  # each a root of X^N + 1
        assert int(X[0]) == P.psi[j]                           # entry 0 = psi (brv(0) = 0)
        # X^(N-1) * X = X^N = -1
        xn1 = np.zeros(P.n, np.uint64); xn1[P.n - 1] = 1
        r = he.negacyclic_mul(xn1, x, q)
        assert r[0] == q - 1 and not r[1:].any()


def test_ntt_sampled_matches_full_and_bigint_n4096():
    P = Params()
    rng = np.random.default_rng(3)
    a = rng.integers(0, P.primes[1], P.n, dtype=np.uint64)
    A = he.ntt(a, P, 1)
    ks = np.array([0, 7, 2048, 4095], dtype=np.uint32)
    assert (he.ntt_sampled(a, ks, P, 1) == A[ks]).all()
    # entry k is a(psi^(2 brv(k)+1)) -- Horner evaluation with Python integers
    q = P.primes[1]
    for k in ks:
        z = pow(P.psi[1], 2 * params.brv(int(k), P.logn) + 1, q)
        acc = 0
        for coef in a[::-1]:
            acc = (acc * z + int(coef)) % q
        assert acc == int(A[k])
