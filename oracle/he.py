"""RLWE/BFV pieces of the oracle (test infrastructure only; see oracle/__init__.py).

Encryption (App. C): ct = (a, b), b = a*sk + delta*m + eps*e with sk
ternary, e a small Gaussian error. Reading R2: delta*m is the BFV encoding
enc(m) = round(Q*m/t) (coefficient-wise, round-half-up), eps = 1. Decryption returns
round(t*(b - a*sk)/Q) mod t (reading R11).

The server side of one convolution (§7): "adds its own shares to these
ciphertexts, performs linear operations using the NTT-preprocessed weights, applies a random
mask for security, and returns the encrypted result". Its plain definition in the coefficient
domain is ``server_conv`` (calls csrc/oracle.c's schoolbook).
"""
from __future__ import annotations

from typing import Optional

import numpy as np

from . import _c
from .packing import Plan, kernel_polys, sparse
from .params import Params


# ---------------------------------------------------------------------------------------------
# plain definitions (big integers)

def enc_bigint(v: int, P: Params, j: int) -> int:
    """enc_j(v) = round(Q v / t) mod q_j, round half up, exact big-integer arithmetic."""
    return ((P.Q * int(v) + P.t // 2) // P.t) % P.primes[j]


def enc(v: np.ndarray, P: Params, j: int) -> np.ndarray:
    """Vectorised enc_j through csrc/oracle.c (pinned against enc_bigint)."""
    v = np.ascontiguousarray(v, dtype=np.uint64).ravel()
    out = np.empty_like(v)
    _c.lib().orc_enc(v, out, v.size, P.primes[j], P.delta_mod_q[j], P.q_mod_t, P.t_bits)
    return out


def negacyclic_mul(a: np.ndarray, b: np.ndarray, q: int) -> np.ndarray:
    """Schoolbook product in Z_q[X]/(X^N+1)."""
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    c = np.empty_like(a)
    _c.lib().orc_negacyclic_mul(a, b, c, a.size, q)
    return c


def ntt(a: np.ndarray, P: Params, j: int) -> np.ndarray:
    """Direct-evaluation negacyclic NTT of one limb poly, bit-reversed order (reading R4)."""
    a = np.ascontiguousarray(a, dtype=np.uint64)
    out = np.empty_like(a)
    _c.lib().orc_ntt_direct(a, out, P.logn, P.primes[j], P.psi[j])
    return out


def ntt_sampled(a: np.ndarray, ks: np.ndarray, P: Params, j: int) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.uint64)
    ks = np.ascontiguousarray(ks, dtype=np.uint32)
    out = np.empty(ks.size, dtype=np.uint64)
    _c.lib().orc_ntt_direct_sampled(a, ks, out, ks.size, P.logn, P.primes[j], P.psi[j])
    return out


def intt(A: np.ndarray, P: Params, j: int) -> np.ndarray:
    A = np.ascontiguousarray(A, dtype=np.uint64)
    out = np.empty_like(A)
    _c.lib().orc_intt_direct(A, out, P.logn, P.primes[j], P.psi[j])
    return out


def to_mod(x_signed: np.ndarray, q: int) -> np.ndarray:
    """Signed small integers -> residues in [0, q)."""
    return np.array([int(v) % q for v in x_signed], dtype=np.uint64)


# ---------------------------------------------------------------------------------------------
# client side (harness): keygen, encrypt, decrypt

def encrypt(m: np.ndarray, sk: np.ndarray, a: np.ndarray, e: np.ndarray, P: Params) -> np.ndarray:
    """m: [N] plaintext < t; sk ternary int64 [N]; a: [L][N] uniform residues; e: int64 [N].
    Returns ct [2][L][N] = (a, a*sk + enc(m) + e)."""
    ct = np.empty((2, P.L, P.n), dtype=np.uint64)
    for j, q in enumerate(P.primes):
        ct[0, j] = a[j]
        ask = negacyclic_mul(to_mod(sk, q), a[j], q)
        em = enc(m, P, j)
        ee = to_mod(e, q)
        ct[1, j] = np.array([(int(x) + int(y) + int(z)) % q for x, y, z in zip(ask, em, ee)], dtype=np.uint64)
    return ct


def decrypt(ct: np.ndarray, sk: np.ndarray, P: Params, coeffs: Optional[np.ndarray] = None) -> np.ndarray:
    """round(t * CRT(b - a*sk) / Q) mod t at all (or the selected) coefficients."""
    idx = np.arange(P.n) if coeffs is None else np.asarray(coeffs, dtype=np.int64).ravel()
    Q = P.Q
    x = np.zeros(idx.size, dtype=object)
    for j, q in enumerate(P.primes):
        ask = negacyclic_mul(to_mod(sk, q), ct[0, j], q)
        vj = (ct[1, j].astype(object) - ask.astype(object)) % q          # b - a*sk mod q_j
        Mj = Q // q
        x = x + vj[idx] * (Mj * pow(Mj, -1, q))                          # CRT
    x = x % Q
    return ((2 * P.t * x + Q) // (2 * Q) % P.t).astype(np.uint64)


# ---------------------------------------------------------------------------------------------
# server side: the hot path's plain definition

def server_conv(ct_in: np.ndarray, x0: Optional[np.ndarray], K: np.ndarray, r: Optional[np.ndarray],
                plan: Plan, P: Params, sel: Optional[np.ndarray] = None,
                out: Optional[np.ndarray] = None) -> np.ndarray:
    """out[m,s] = sum_g (in[g,s] + enc(x0[g,s]) on b) (*) lift(w[m,g])  (+ enc(r[m,s]) on b).

    ct_in [G*S][2][L][N], x0 [G*S][N] or None, K (M,C,kh,kw) < 2^t, r [M*S][N] or None.
    Returns [M*S][2][L][N]; with `sel` ([M*S] bool) only the selected outputs are computed."""
    return server_mac(ct_in, x0, kernel_polys(K, plan, P.n), r, plan.G, plan.S, plan.M, P, sel, out)


def server_mac(ct_in: np.ndarray, x0: Optional[np.ndarray], kp: np.ndarray, r: Optional[np.ndarray],
               G: int, S: int, M: int, P: Params, sel: Optional[np.ndarray] = None,
               out: Optional[np.ndarray] = None) -> np.ndarray:
    """The server's linear-layer computation for any packing:
    out[m,s] = sum_{g<G} (in[g,s] + enc(x0[g,s]) on b) (*) lift(kp[m,g])  (+ enc(r[m,s]) on b),
    with kp [M][G][N] the raw plaintext polys (values < 2^t, centred-lifted per limb)."""
    return server_mac_sparse(ct_in, x0, sparse(kp), r, G, S, M, P, sel, out)


def server_mac_sparse(ct_in: np.ndarray, x0: Optional[np.ndarray], kp_sparse, r: Optional[np.ndarray],
                      G: int, S: int, M: int, P: Params, sel: Optional[np.ndarray] = None,
                      out: Optional[np.ndarray] = None) -> np.ndarray:
    """server_mac with the plaintext polys already in sparse form (koff, kidx, kval) =
    packing.sparse(kp): the weights are packed once per layer (the server's offline setup,
    PAPER.md:427 §7 step 1) and every online call reuses them."""
    koff, kidx, kval = kp_sparse
    ct_in = np.ascontiguousarray(ct_in, dtype=np.uint64)
    assert ct_in.shape == (G * S, 2, P.L, P.n), ct_in.shape
    if out is None:
        out = np.zeros((M * S, 2, P.L, P.n), dtype=np.uint64)
    x0c = None if x0 is None else np.ascontiguousarray(x0, dtype=np.uint64)
    rc = None if r is None else np.ascontiguousarray(r, dtype=np.uint64)
    selc = None if sel is None else np.ascontiguousarray(sel, dtype=np.uint8)
    _c.lib().orc_he_conv_server(P.logn, P.L, np.array(P.primes, dtype=np.uint64), P.t_bits,
                                np.array(P.delta_mod_q, dtype=np.uint64), P.q_mod_t,
                                G, S, M, ct_in, _c.ptr_or_null(x0c), koff, kidx, kval,
                                _c.ptr_or_null(rc), _c.ptr_or_null(selc), out)
    return out


def mask_add(ct: np.ndarray, r: np.ndarray, P: Params) -> np.ndarray:
    """b_j += enc_j(r) for a batch ct [n][2][L][N], r [n][N] (§7)."""
    out = ct.copy()
    for i in range(ct.shape[0]):
        for j, q in enumerate(P.primes):
            e = enc(r[i], P, j)
            out[i, 1, j] = ((ct[i, 1, j].astype(object) + e.astype(object)) % q).astype(np.uint64)
    return out
