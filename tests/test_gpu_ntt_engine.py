"""GPU parity of the TMA-staged NTT engine (k_ntt_tma, the plain secn_ntt_fwd / secn_ntt_inv
calls and the weight preprocessing): sampled outputs against the oracle's direct evaluation
(App. C.1; reading R4 for the output order), round trips, and word-for-word
equality with the one-CTA-per-poly kernels (SECN_NTT_TMA=0) on batches with odd poly counts
(the last item of a two-poly item is half empty), several items per persistent CTA and every
limb count."""
import numpy as np
import pytest

from oracle import he, params
from oracle.params import Params
from test_gpu_parity import Dev, secn  # noqa: F401  (fixture)
from workloads import inputs

pytestmark = pytest.mark.gpu


def _ctx(secn, monkeypatch, tma, **kw):
    monkeypatch.setenv("SECN_NTT_TMA", "2" if tma else "0")
    return secn.Context(0, **kw)  # knobs are read at context creation


CASES = [(32, 12, 1, 1), (32, 12, 4, 7), (32, 12, 3, 301), (32, 12, 4, 1777), (32, 12, 2, 2),
         (32, 13, 4, 5), (32, 13, 1, 600), (32, 14, 2, 3), (32, 14, 4, 300),
         (64, 12, 2, 301), (64, 12, 1, 9), (64, 13, 2, 7), (64, 13, 3, 400)]


@pytest.mark.parametrize("wb,logn,L,n", CASES)
def test_tma_engine_matches_direct_evaluation_and_old_kernels(secn, monkeypatch, wb, logn, L, n):
    primes = (params.SWEEP_PRIMES if wb == 64 else params.PRIMES32)[:L]
    kw = dict(log_n=logn, primes=primes, word_bits=wb)
    c_new, c_old = _ctx(secn, monkeypatch, True, **kw), _ctx(secn, monkeypatch, False, **kw)
    D = Dev(c_new)
    P = Params(logn=logn, primes=primes)
    g = inputs.rng(9000 + wb + logn * 7 + L * 3 + n)
    x = inputs.uniform_residues(g, (n,), primes, P.n)
    if n > 2:
        x[1] = np.array([q - 1 for q in primes], np.uint64)[:, None]  # every residue at its maximum
    fwd_new = D.U(c_new.ntt_fwd(D.R(x)))
    fwd_old = D.U(c_old.ntt_fwd(D.R(x)))
    assert (fwd_new == fwd_old).all()
    ks = np.concatenate([[0, 1, P.n // 2, P.n - 1], g.integers(0, P.n, 12)]).astype(np.uint32)
    for i in sorted({0, n // 2, n - 1}):
        j = i % L
        assert (fwd_new[i, j, ks] == he.ntt_sampled(x[i, j], ks, P, j)).all(), (i, j)
    inv_new = D.U(c_new.ntt_inv(D.R(fwd_new)))
    inv_old = D.U(c_old.ntt_inv(D.R(fwd_new)))
    assert (inv_new == x).all()
    assert (inv_old == inv_new).all()
    y = inputs.uniform_residues(g, (min(n, 3),), primes, P.n)  # the inverse on arbitrary inputs too
    a, b = D.U(c_new.ntt_inv(D.R(y))), D.U(c_old.ntt_inv(D.R(y)))
    assert (a == b).all()
    assert (a[0, 0] == he.intt(y[0, 0], P, 0)).all() if logn == 12 else True
    c_new.close()
    c_old.close()


def test_tma_engine_threshold_knob(secn, monkeypatch):
    """Below SECN_NTT_TMA_MIN limb-polys the plain calls keep the one-CTA-per-poly kernels: both
    choices give the same words."""
    primes = params.PRIMES32
    monkeypatch.setenv("SECN_NTT_TMA", "2")
    monkeypatch.setenv("SECN_NTT_TMA_MIN", "100000")
    c_small = secn.Context(0, word_bits=32)
    monkeypatch.delenv("SECN_NTT_TMA_MIN")
    c_tma = secn.Context(0, word_bits=32)
    D = Dev(c_tma)
    x = inputs.uniform_residues(inputs.rng(9100), (33,), primes, 4096)
    assert (D.U(c_small.ntt_fwd(D.R(x))) == D.U(c_tma.ntt_fwd(D.R(x)))).all()
    c_small.close()
    c_tma.close()
