"""Pins for oracle/he.py and oracle/packing.py (not gpu).

The end-to-end pin is the paper's correctness statement: linear layers are exact over
Z_{2^b}, so Dec(server(Enc(<x>_1))) + <y>_0 = conv(x, K) mod 2^37 at
every designated coefficient, where <y>_0 = -r (§7). That equality exercises
enc, encrypt, the share add, the packing, the centred lift, the schoolbook product, the
mask and decrypt together, and fails for a dropped term, a wrong sign (X^N = -1), a
transposed kernel or an index slip.
"""
from fractions import Fraction

import numpy as np
import pytest

from oracle import conv, he, packing, params
from oracle.params import Params
from workloads import inputs, layers


@pytest.fixture(scope="module")
def P():
    return Params()


def test_enc_matches_exact_rational_rounding(P):
    g = inputs.rng(7)
    vals = list(inputs.uniform_below(g, 300, P.t)) + [0, 1, P.t - 1, P.t // 2, P.t // 2 - 1]
    # the exact ties Q v = t/2 (mod t): round half up
    tie = (P.t // 2) * pow(P.Q, -1, P.t) % P.t
    vals.append(tie)
    assert (P.Q * tie) % P.t == P.t // 2
    v = np.array(vals, dtype=np.uint64)
    for j, q in enumerate(P.primes):
        got = he.enc(v, P, j)
        for x, y in zip(vals, got):
            exact = Fraction(P.Q * int(x), P.t)
            rounded = int(exact + Fraction(1, 2)) if exact >= 0 else None  # floor(x + 1/2)
            assert int(y) == rounded % q
            assert int(y) == he.enc_bigint(x, P, j)


def test_encrypt_decrypt_roundtrip_and_additivity():
    P = Params(logn=10)
    g = inputs.rng(11)
    sk = inputs.ternary(g, P.n)

    def E(m):
        return he.encrypt(m, sk, inputs.uniform_residues(g, (), P.primes, P.n), inputs.rounded_gaussian(g, P.n), P)

    m1 = inputs.uniform_below(g, P.n, P.t)
    m2 = inputs.uniform_below(g, P.n, P.t)
    c1, c2 = E(m1), E(m2)
    assert (he.decrypt(c1, sk, P) == m1).all()
    assert (he.decrypt(E(np.zeros(P.n, np.uint64)), sk, P) == 0).all()
    csum = np.empty_like(c1)
    for j, q in enumerate(P.primes):
        csum[:, j] = (c1[:, j].astype(object) + c2[:, j].astype(object)) % q
    assert (he.decrypt(csum, sk, P) == (m1 + m2) % np.uint64(P.t)).all()


def _ct_times_pt(ct, w_signed, P):
    out = np.empty_like(ct)
    for j, q in enumerate(P.primes):
        wj = he.to_mod(w_signed, q)
        for c in range(2):
            out[c, j] = he.negacyclic_mul(ct[c, j], wj, q)
    return out


def test_pt_identity_monomial_and_mac_chain():
    """SPEC.md:532-535 example ideas: pt=1 identity, pt=X negacyclic shift, 8-step MAC chain."""
    P = Params(logn=8)
    g = inputs.rng(12)
    sk = inputs.ternary(g, P.n)

    def E(m):
        return he.encrypt(m, sk, inputs.uniform_residues(g, (), P.primes, P.n), inputs.rounded_gaussian(g, P.n), P)

    m = inputs.uniform_below(g, P.n, P.t)
    ct = E(m)
    one = np.zeros(P.n, np.int64); one[0] = 1
    assert (he.decrypt(_ct_times_pt(ct, one, P), sk, P) == m).all()
    X = np.zeros(P.n, np.int64); X[1] = 1
    shifted = np.concatenate([[(P.t - int(m[-1])) % P.t], m[:-1]]).astype(np.uint64)
    assert (he.decrypt(_ct_times_pt(ct, X, P), sk, P) == shifted).all()
    # MAC chain: sum_i m_i * w_i with small signed plaintexts w_i
    acc = np.zeros_like(ct)
    expect = np.zeros(P.n, dtype=object)
    for _ in range(8):
        mi = inputs.uniform_below(g, P.n, P.t)
        wi = g.integers(-(1 << 12), 1 << 12, P.n, dtype=np.int64)
        prod = _ct_times_pt(E(mi), wi, P)
        for j, q in enumerate(P.primes):
            acc[:, j] = (acc[:, j].astype(object) + prod[:, j].astype(object)) % q
        full = [0] * (2 * P.n)
        for a_i, x in enumerate(mi):
            for b_i, y in enumerate(wi):
                full[a_i + b_i] += int(x) * int(y)
        expect = expect + np.array([full[i] - full[i + P.n] for i in range(P.n)], dtype=object)
    assert (he.decrypt(acc, sk, P) == (expect % P.t).astype(np.uint64)).all()


def test_mask_zero_and_unmask():
    P = Params(logn=8)
    g = inputs.rng(13)
    sk = inputs.ternary(g, P.n)
    m = inputs.uniform_below(g, P.n, P.t)
    ct = he.encrypt(m, sk, inputs.uniform_residues(g, (), P.primes, P.n), inputs.rounded_gaussian(g, P.n), P)
    assert (he.mask_add(ct[None], np.zeros((1, P.n), np.uint64), P)[0] == ct).all()
    r = inputs.uniform_below(g, (1, P.n), P.t)
    dec = he.decrypt(he.mask_add(ct[None], r, P)[0], sk, P)
    assert ((dec - r[0]) % np.uint64(P.t) == m).all()


def _e2e(layer, P, seed, full_range=False, with_x0=True, poly=False, Hw=None, Ww=None):
    pl = packing.plan_conv(layer.C, layer.H, layer.W, layer.M, layer.k, layer.k, layer.stride, layer.pad, P.n, P.L,
                           Hw=Hw, Ww=Ww, poly=poly)
    g = inputs.rng(seed)
    x1 = inputs.uniform_below(g, (layer.C, layer.H, layer.W), P.t)
    x0 = inputs.uniform_below(g, (layer.C, layer.H, layer.W), P.t) if with_x0 else np.zeros_like(x1)
    K = (inputs.full_range_kernel if full_range else inputs.quantized_kernel)(g, layer.M, layer.C, layer.k, layer.k)
    sk = inputs.ternary(g, P.n)
    xin = packing.pack_input(x1, pl, P.n)
    ct = np.stack([he.encrypt(xin[i], sk, inputs.uniform_residues(g, (), P.primes, P.n),
                              inputs.rounded_gaussian(g, P.n), P) for i in range(pl.G * pl.S)])
    r = inputs.uniform_below(g, (pl.M * pl.S, P.n), P.t)
    out = he.server_conv(ct, packing.pack_input(x0, pl, P.n) if with_x0 else None, K, r, pl, P)
    s_idx, coef = packing.designated_map(pl)
    y = np.zeros((pl.M, pl.OH, pl.OW), np.uint64)
    for m in range(pl.M):
        for s in range(pl.S):
            sel = s_idx == s
            if not sel.any():
                continue
            dec = he.decrypt(out[m * pl.S + s], sk, P, coef[sel])
            y[m][sel] = (dec + (P.t - r[m * pl.S + s, coef[sel]]) % P.t) % np.uint64(P.t)
    ref = conv.conv2d_mod((x0 + x1) & np.uint64(P.t - 1), K, layer.stride, layer.pad, P.t_bits)
    return pl, y, ref


@pytest.mark.parametrize("primes", [params.DEFAULT_PRIMES, params.PRIMES32], ids=["q60_49", "q27x4"])
def test_e2e_tiny_config_exact(primes):
    """BASELINE.json configs[0] at the paper parameters: N=4096, t = 2^37, Q = q0 q1 (109 bits) and
    the 32-bit-limb reading R1b (four 27-bit primes, 108 bits)."""
    P = Params(primes=primes)
    pl, y, ref = _e2e(layers.tiny()[0], P, 1)
    assert (pl.Cw, pl.Hw, pl.Ww, pl.G, pl.S, pl.O) == (4, 18, 18, 1, 1, 1010)
    assert (y == ref).all()


L = layers.ConvLayer


@pytest.mark.parametrize("layer,seed,full", [
    (L("multi_tile", 8, 16, 16, 3, 3, 1, 1), 21, False),      # SPEC.md:592 8x16x16 multi-tile
    (L("stride2", 3, 23, 19, 4, 3, 2, 0), 22, False),          # strided 3x3 (conv1-like)
    (L("ds_1x1_s2", 6, 14, 14, 5, 1, 2, 0), 23, False),        # decimated 1x1 / stride 2
    (L("k7s2p3", 2, 20, 20, 3, 7, 2, 3), 24, False),           # ResNet conv1-like
    (L("worstcase", 5, 9, 9, 4, 3, 1, 1), 25, True),           # full-range 37-bit weights
    (L("pointwise", 40, 6, 6, 6, 1, 1, 0), 26, False),         # many channel groups
])
def test_e2e_small_shapes_exact_n256(layer, seed, full):
    P = Params(logn=8, primes=params.PRIMES32 if seed % 2 else params.DEFAULT_PRIMES)
    pl, y, ref = _e2e(layer, P, seed, full_range=full)
    assert pl.G * pl.S > 1
    assert (y == ref).all()


@pytest.mark.parametrize("layer,seed,win", [
    (L("poly_s2k3", 3, 23, 19, 4, 3, 2, 0), 31, None),          # conv1-like, odd extents
    (L("poly_s2k3p1", 4, 16, 16, 3, 3, 2, 1), 32, (5, 6)),      # padded, several blocks
    (L("poly_k7s2p3", 2, 20, 20, 3, 7, 2, 3), 33, None),        # 7x7 / 2 (ResNet conv1-like)
    (L("poly_s3k5", 2, 17, 17, 2, 5, 3, 1), 34, (4, 4)),        # stride 3: 9 phases
])
def test_e2e_polyphase_exact_n256(layer, seed, win):
    """Reading R7b: the polyphase packing of a strided kernel (Ce = C s^2 phase channels,
    ceil(k/s)-sized kernel, every window position an output) decrypts to conv(x, K) mod 2^t."""
    P = Params(logn=8, primes=params.PRIMES32 if seed % 2 else params.DEFAULT_PRIMES)
    Hw, Ww = win if win else (None, None)
    pl, y, ref = _e2e(layer, P, seed, poly=True, Hw=Hw, Ww=Ww)
    assert pl.decim == 2 and pl.Ce == layer.C * layer.stride ** 2 and pl.khe == -(-layer.k // layer.stride)
    assert (y == ref).all()


def test_polyphase_split_reassembles():
    """The polyphase split of input and kernel is a permutation (with zero fill) of the padded
    input and the kernel: the phase correlation equals the strided correlation by brute force."""
    g = inputs.rng(35)
    C, H, W, M, k, s, pad = 2, 11, 9, 3, 3, 2, 1
    pl = packing.plan_conv(C, H, W, M, k, k, s, pad, 256, 2, poly=True)
    x = g.integers(0, 100, (C, H, W)).astype(np.uint64)
    K = g.integers(0, 100, (M, C, k, k)).astype(np.uint64)
    Xe, Ke = packing.effective_input(x, pl), packing.effective_kernel(K, pl)
    xp = np.zeros((C, H + 2 * pad, W + 2 * pad), np.uint64)
    xp[:, pad:pad + H, pad:pad + W] = x
    for m in range(M):
        for oy in range(pl.OH):
            for ox in range(pl.OW):
                a = sum(int(xp[c, oy * s + l, ox * s + l2]) * int(K[m, c, l, l2])
                        for c in range(C) for l in range(k) for l2 in range(k))
                b = sum(int(Xe[c2, oy + i, ox + j]) * int(Ke[m, c2, i, j])
                        for c2 in range(pl.Ce) for i in range(pl.khe) for j in range(pl.kwe))
                assert a == b


def test_e2e_no_server_share():
    P = Params(logn=8)
    pl, y, ref = _e2e(L("noshare", 2, 5, 5, 3, 2, 1, 0), P, 27, with_x0=False)
    assert (y == ref).all()


def test_zero_kernel_gives_mask_only(P):
    pl = packing.plan_conv(4, 16, 16, 8, 3, 3, 1, 1, P.n, P.L)
    g = inputs.rng(9)
    ct = inputs.uniform_residues(g, (pl.G * pl.S, 2), P.primes, P.n)
    out = he.server_conv(ct, None, np.zeros((8, 4, 3, 3), np.uint64), None, pl, P)
    assert not out.any()


SQ11_PLAN = {  # SURVEY.md App. A.5 (survey's independent script): name -> (Cw, Hw, Ww, G, S)
    "conv1": (1, 224, 18, 3, 14), "fire2.sq": (5, 55, 14, 13, 4), "fire2.e3": (2, 57, 35, 8, 2),
    "fire3.sq": (9, 55, 8, 15, 7), "fire4.sq": (16, 27, 9, 8, 3), "fire5.sq": (32, 14, 9, 8, 6),
    "fire6.e1": (24, 13, 13, 2, 1), "fire6.e3": (18, 15, 15, 3, 1), "fire9.sq": (63, 13, 5, 9, 3),
    "conv10": (63, 13, 5, 9, 3),
}


def test_plan_rule_reproduces_survey_table():
    for l in layers.squeezenet11():
        p = packing.plan_conv(l.C, l.H, l.W, l.M, l.k, l.k, l.stride, l.pad, 4096, 2)
        assert p.Cw * p.Hw * p.Ww <= 4096 and p.Hw >= p.kh and p.Ww >= p.kw and p.O < 4096
        if l.name in SQ11_PLAN:
            assert (p.Cw, p.Hw, p.Ww, p.G, p.S) == SQ11_PLAN[l.name], l.name
    tot = [0, 0, 0, 0]
    for l in layers.squeezenet11():
        p = packing.plan_conv(l.C, l.H, l.W, l.M, l.k, l.k, l.stride, l.pad, 4096, 2)
        tot[0] += p.G * p.S; tot[1] += p.M * p.S; tot[2] += p.M * p.G; tot[3] += p.M * p.G * p.S
    assert tot == [493, 8200, 21624, 52520]  # SURVEY.md §8d C3 totals
