"""Ring parameters for the oracle, computed with Python big integers (test infrastructure only).

* Ring R_Q = Z_Q[X]/(X^N+1), Q = prod q_j, each q_j prime with q_j = 1 (mod 2N) so that a
  primitive 2N-th root psi_j exists (§2.1; App. C.1 "primitive
  root of unity").
* The paper never states N or Q (reading R1). Default: N = 4096,
  q0 = 0x0FFFFFFFFFFFC001 (60 bit), q1 = 0x1FFFFFFFCE001 (49 bit), t = 2^37.
  The primes are found by the SEAL-style search: the largest primes below 2^bits that are
  = 1 (mod 2N).
* psi_j is the smallest primitive 2N-th root of unity mod q_j (reading R4).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Sequence


def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin for n < 3.3e24 (bases = first 13 primes)."""
    if n < 2:
        return False
    small = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41]
    for p in small:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in small:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def find_primes(bits: int, n: int, count: int = 1, modulus: int | None = None) -> List[int]:
    """The `count` largest primes q < 2^bits with q = 1 (mod modulus), modulus defaults to 2N."""
    m = modulus or 2 * n
    out, q = [], (1 << bits) - m + 1
    while len(out) < count and q > m:
        if is_prime(q):
            out.append(q)
        q -= m
    return out


def brv(x: int, bits: int) -> int:
    """Bit reversal of x over `bits` bits."""
    r = 0
    for _ in range(bits):
        r = (r << 1) | (x & 1)
        x >>= 1
    return r


def minimal_psi(q: int, n: int) -> int:
    """Smallest primitive 2N-th root of unity modulo the prime q.

    psi is a primitive 2N-th root iff psi^N = -1 (mod q) (2N is a power of two). The
    primitive 2N-th roots are exactly the odd powers of any one of them."""
    assert (q - 1) % (2 * n) == 0
    for x in range(2, q):
        y = pow(x, (q - 1) // (2 * n), q)
        if pow(y, n, q) == q - 1:
            return min(pow(y, k, q) for k in range(1, 2 * n, 2))
    raise ValueError("no primitive root")


DEFAULT_PRIMES = (0x0FFFFFFFFFFFC001, 0x1FFFFFFFCE001)
ALT54_PRIMES = (0x3FFFFFFFFD6001, 0x3FFFFFFFFD2001)
SWEEP_PRIMES = (0xFFFFFFFFFFC0001, 0xFFFFFFFFF840001, 0xFFFFFFFFF6A0001, 0xFFFFFFFFF5A0001)
# Reading R1b: 32-bit RNS limbs -- the four largest 27-bit primes = 1 (mod 2^16); Q = 108 bits.
PRIMES32 = (0x7E90001, 0x7E00001, 0x7DD0001, 0x7D70001)


@dataclass
class Params:
    logn: int = 12
    primes: Sequence[int] = DEFAULT_PRIMES
    t_bits: int = 37
    psi: List[int] = field(init=False)

    def __post_init__(self):
        self.primes = tuple(int(q) for q in self.primes)
        for q in self.primes:
            assert is_prime(q) and (q - 1) % (2 * self.n) == 0, hex(q)
        self.psi = [minimal_psi(q, self.n) for q in self.primes]

    @property
    def n(self) -> int:
        return 1 << self.logn

    @property
    def L(self) -> int:
        return len(self.primes)

    @property
    def t(self) -> int:
        return 1 << self.t_bits

    @property
    def Q(self) -> int:
        Q = 1
        for q in self.primes:
            Q *= q
        return Q

    @property
    def delta_mod_q(self) -> List[int]:
        """floor(Q/t) mod q_j."""
        return [(self.Q // self.t) % q for q in self.primes]

    @property
    def q_mod_t(self) -> int:
        return self.Q % self.t

    def crt(self, residues: Sequence[int]) -> int:
        """The unique v in [0, Q) with v = residues[j] (mod q_j)."""
        Q, v = self.Q, 0
        for r, q in zip(residues, self.primes):
            Mj = Q // q
            v += int(r) * Mj * pow(Mj, -1, q)
        return v % Q
