"""Pins for oracle/params.py: primes, roots, bit reversal, CRT (not gpu)."""
from pathlib import Path

import pytest

from oracle import params
from oracle.params import Params

GOLDEN = Path(__file__).parent / "golden"


def _trial_division_prime(n):
    if n < 2:
        return False
    d = 2
    while d * d <= n:
        if n % d == 0:
            return False
        d += 1
    return True


def test_is_prime_matches_trial_division():
    for n in range(0, 5000):
        assert params.is_prime(n) == _trial_division_prime(n), n


@pytest.mark.parametrize("q", params.DEFAULT_PRIMES + params.ALT54_PRIMES + params.SWEEP_PRIMES)
def test_parameter_primes_fermat_and_ntt_friendly(q):
    # Fermat witnesses independent of the Miller-Rabin code path, and q = 1 mod 2N (N = 4096)
    for a in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47):
        assert pow(a, q - 1, q) == 1
    assert (q - 1) % 8192 == 0


def test_seal_style_prime_search_reproduces_default_primes():
    # largest primes = 1 mod 2N below 2^60 and 2^49
    assert params.find_primes(60, 4096) == [0x0FFFFFFFFFFFC001]
    assert params.find_primes(49, 4096) == [0x1FFFFFFFCE001]
    assert params.find_primes(54, 4096, 2) == [0x3FFFFFFFFD6001, 0x3FFFFFFFFD2001]


def test_minimal_psi_brute_force_small_primes():
    for q, n in [(17, 8), (97, 16), (7681, 256), (12289, 1024), (257, 64)]:
        psi = params.minimal_psi(q, n)
        assert pow(psi, n, q) == q - 1
        assert all(pow(x, n, q) != q - 1 for x in range(2, psi))


def test_minimal_psi_golden():
    for line in (GOLDEN / "psi_minimal.txt").read_text().splitlines():
        if not line.strip() or line.startswith("#"):
            continue
        n, q, psi = map(int, line.split())
        assert params.minimal_psi(q, n) == psi
        assert pow(psi, n, q) == q - 1


def test_brv_is_involution_and_permutation():
    for bits in range(1, 11):
        vals = [params.brv(i, bits) for i in range(1 << bits)]
        assert sorted(vals) == list(range(1 << bits))
        assert all(params.brv(v, bits) == i for i, v in enumerate(vals))
    assert params.brv(1, 3) == 4 and params.brv(3, 3) == 6 and params.brv(6, 12) == 0b011000000000


def test_crt_roundtrip_and_constants():
    P = Params()
    import random

    rnd = random.Random(5)
    for _ in range(200):
        v = rnd.randrange(P.Q)
        assert P.crt([v % q for q in P.primes]) == v
    assert P.Q.bit_length() == 109
    assert P.q_mod_t == 3355222017
    assert (P.Q // P.t).bit_length() == 72
