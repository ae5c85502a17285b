"""Coefficient extraction with modulus switching of the server's output ciphertexts -- oracle side
(test infrastructure only). SURVEY.md §8f row 2.

The paper: Cheetah "results in a sparse output with very few coefficients containing the actual
result" (§2.3), the server "returns the encrypted result to the client for
decryption into output shares" (§7); Cheetah's server drops the unused output
coefficients and switches the ciphertext to a smaller modulus before sending it [outside:
Cheetah]. Reading R16:

  * modulus switch to the first L' limbs, Q' = q_0 ... q_{L'-1}:  for every coefficient c of both
    components (c in [0, Q) by CRT),  c' = round(c * Q' / Q) mod Q'  (no ties: Q / Q' is odd);
  * extraction: the a component is kept whole, a' [L'][N] (every designated coefficient of the
    ciphertext shares it); the b component only at the designated coefficients, b'[k] [L'];
  * the client decrypts coefficient k as  m_k = round(t (b'_k - (a' * sk)_k) / Q') mod t,
    (a' * sk)_k the k-th coefficient of the negacyclic product (an LWE decryption).

Pinned by tests/test_oracle_extract.py (exact-rational rounding, the |c' P - c| <= P/2 property,
and end to end: decrypt_lwe of the switched, extracted server output + the server share
= conv(x0 + x1, K) mod 2^37).
"""
from __future__ import annotations

import numpy as np

from . import he
from .params import Params


def switched_params(P: Params, keep: int) -> Params:
    """Parameters of the switched ciphertexts: the first `keep` primes, same N and t."""
    return Params(logn=P.logn, primes=P.primes[:keep], t_bits=P.t_bits)


def _crt_vec(res: np.ndarray, P: Params) -> np.ndarray:
    """residues [L][N] -> object array [N] of the CRT values in [0, Q)."""
    Q = P.Q
    x = np.zeros(res.shape[-1], dtype=object)
    for j, q in enumerate(P.primes):
        Mj = Q // q
        x = x + res[j].astype(object) * (Mj * pow(Mj, -1, q))
    return x % Q


def modswitch(ct: np.ndarray, keep: int, P: Params) -> np.ndarray:
    """ct [..., L, N] residues mod q_j -> [..., keep, N]: round(c Q'/Q) mod q_i for c = CRT(c_0..c_{L-1})
    in [0, Q), Q' = q_0 ... q_{keep-1}; round half up (never a tie: Q/Q' is odd)."""
    Ps = switched_params(P, keep)
    Q, Qp = P.Q, Ps.Q
    lead = ct.shape[:-2]
    flat = np.ascontiguousarray(ct).reshape(-1, P.L, P.n)
    out = np.zeros((flat.shape[0], keep, P.n), dtype=np.uint64)
    for b in range(flat.shape[0]):
        c = _crt_vec(flat[b], P)
        v = (c * Qp + Q // 2) // Q % Qp
        for i, q in enumerate(Ps.primes):
            out[b, i] = (v % q).astype(np.uint64)
    return out.reshape(*lead, keep, P.n)


def extract_lwe(ct_ms: np.ndarray, coef: np.ndarray):
    """A switched ct [2][L'][N] -> (a' [L'][N], b' [len(coef)][L']) at the given coefficients."""
    coef = np.asarray(coef).ravel()
    return ct_ms[0].copy(), np.ascontiguousarray(ct_ms[1][:, coef].T)


def decrypt_lwe(a: np.ndarray, b: np.ndarray, coef: np.ndarray, sk: np.ndarray, Ps: Params) -> np.ndarray:
    """m_k = round(t (b'_k - (a' * sk)_k) / Q') mod t for the extracted coefficients `coef`
    (b' [len(coef)][L']), with the schoolbook a' * sk mod X^N + 1 and the exact CRT of Ps."""
    coef = np.asarray(coef).ravel()
    res = np.zeros((Ps.L, coef.size), dtype=np.uint64)
    for i, q in enumerate(Ps.primes):
        ask = he.negacyclic_mul(he.to_mod(sk, q), a[i], q)[coef]
        res[i] = ((b[:, i].astype(object) - ask.astype(object)) % q).astype(np.uint64)
    v = _crt_vec(res, Ps)
    return ((2 * Ps.t * v + Ps.Q) // (2 * Ps.Q) % Ps.t).astype(np.uint64)


def server_lwe_outputs(out: np.ndarray, keep: int, P: Params, s_idx: np.ndarray, coef: np.ndarray, M: int, S: int):
    """The switched + extracted form of a layer's output cts [M*S][2][L][N] for a conv plan's
    designated map (s_idx, coef, both (OH, OW)): a' [M*S][L'][N], b' [M][OH][OW][L']."""
    ms = modswitch(out, keep, P)
    a = np.ascontiguousarray(ms[:, 0])
    b = np.zeros((M,) + s_idx.shape + (keep,), dtype=np.uint64)
    for m in range(M):
        for i in range(keep):
            b[m, ..., i] = ms[m * S + s_idx, 1, i, coef]
    return a, b
