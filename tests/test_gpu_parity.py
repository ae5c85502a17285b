"""GPU parity: libsecn (through its C ABI, via the ctypes binding) against the oracle,
element by element on identical seeded inputs. Integer work => bit-exact (every uint64 word).

Run on a B200 with: python -m pytest tests -m gpu
"""
import zlib

import numpy as np
import pytest
import torch

import __graft_entry__
from oracle import conv, he, packing, params
from oracle.params import Params
from workloads import inputs, layers

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda:0")


def T(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(DEV)


def U(t: torch.Tensor) -> np.ndarray:
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint64)


@pytest.fixture(scope="module")
def secn():
    __graft_entry__.build()
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_11586_b200 import secn as m

    return m


@pytest.fixture(scope="module")
def ctx(secn):
    return secn.Context(0)


@pytest.fixture(scope="module")
def P():
    return Params()


# ---------------------------------------------------------------------------------------------
# context tables

@pytest.mark.parametrize("logn,primes", [(12, params.DEFAULT_PRIMES), (12, params.ALT54_PRIMES),
                                         (12, params.SWEEP_PRIMES), (13, params.SWEEP_PRIMES),
                                         (14, params.SWEEP_PRIMES[:2])])
def test_ctx_psi_matches_oracle(secn, logn, primes):
    c = secn.Context(0, log_n=logn, primes=primes)
    assert c.psi == tuple(Params(logn=logn, primes=primes).psi)
    c.close()


# ---------------------------------------------------------------------------------------------
# A1 / A2: NTT and inverse

def _edge_polys(P, g):
    n = P.n
    polys = [inputs.uniform_residues(g, (), P.primes, n)]
    z = np.zeros((P.L, n), np.uint64)
    polys.append(z.copy())                                           # zero
    c = z.copy(); c[:, 0] = 123456789; polys.append(c)                # constant
    top = np.stack([np.full(n, q - 1, np.uint64) for q in P.primes]); polys.append(top)  # all q-1
    mono = z.copy(); mono[:, n - 1] = 1; polys.append(mono)           # X^(N-1)
    return np.stack(polys)


def test_ntt_fwd_matches_direct_evaluation(ctx, P):
    g = inputs.rng(100)
    polys = _edge_polys(P, g)
    got = U(ctx.ntt_fwd(T(polys)))
    for i in range(polys.shape[0]):
        for j in range(P.L):
            if i >= 2 and j == 0:
                continue  # closed-form edge polys: limb 1 suffices, keeps the test fast
            assert (got[i, j] == he.ntt(polys[i, j], P, j)).all(), (i, j)
    # constant -> constant vector, on every limb
    assert (got[2] == 123456789).all()


def test_ntt_inv_matches_direct_and_roundtrips(ctx, P):
    g = inputs.rng(101)
    A = inputs.uniform_residues(g, (2,), P.primes, P.n)
    got = U(ctx.ntt_inv(T(A)))
    assert (got[0, 0] == he.intt(A[0, 0], P, 0)).all()
    assert (got[1, 1] == he.intt(A[1, 1], P, 1)).all()
    big = inputs.uniform_residues(g, (3001,), P.primes, P.n)         # multi-wave batch
    t = T(big)
    ctx.ntt_fwd(t)
    ctx.ntt_inv(t)
    assert (U(t) == big).all()


def test_ntt_pointwise_product_is_negacyclic_product(ctx, P):
    g = inputs.rng(102)
    a = inputs.uniform_residues(g, (), P.primes, P.n)
    b = inputs.uniform_residues(g, (), P.primes, P.n)
    A, B = U(ctx.ntt_fwd(T(a[None]))), U(ctx.ntt_fwd(T(b[None])))
    prod = np.stack([np.array([int(x) * int(y) % q for x, y in zip(A[0, j], B[0, j])], np.uint64)
                     for j, q in enumerate(P.primes)])
    c = U(ctx.ntt_inv(T(prod[None])))[0]
    for j, q in enumerate(P.primes):
        assert (c[j] == he.negacyclic_mul(a[j], b[j], q)).all()


@pytest.mark.parametrize("logn,L", [(12, 4), (13, 1), (13, 3), (14, 2), (14, 4)])
def test_ntt_sweep_sampled(secn, logn, L):
    primes = params.SWEEP_PRIMES[:L]
    c = secn.Context(0, log_n=logn, primes=primes)
    P = Params(logn=logn, primes=primes)
    g = inputs.rng(103 + logn * 10 + L)
    x = inputs.uniform_residues(g, (7,), primes, P.n)
    got = U(c.ntt_fwd(T(x)))
    ks = np.concatenate([[0, 1, P.n // 2, P.n - 1], g.integers(0, P.n, 28)]).astype(np.uint32)
    for i in (0, 6):
        for j in range(L):
            assert (got[i, j, ks] == he.ntt_sampled(x[i, j], ks, P, j)).all(), (i, j)
    back = U(c.ntt_inv(T(got)))
    assert (back == x).all()
    c.close()


def test_empty_batch_is_noop(ctx):
    t = torch.zeros(0, dtype=torch.int64, device=DEV)
    ctx.ntt_fwd(t)
    ctx.ntt_inv(t)
    torch.cuda.synchronize()


# ---------------------------------------------------------------------------------------------
# A6 / A7: server-share add and output mask

def test_mask_and_share_add_match_oracle_enc(ctx, P):
    g = inputs.rng(104)
    n = 5
    ct = inputs.uniform_residues(g, (n, 2), P.primes, P.n)
    r = inputs.uniform_below(g, (n, P.n), P.t)
    r[0, :4] = [0, 1, P.t - 1, P.t // 2]
    got = U(ctx.mask_add(T(ct), T(r)))
    assert (got == he.mask_add(ct, r, P)).all()
    got2 = U(ctx.share_add(T(ct), T(r)))
    assert (got2 == got).all()


# ---------------------------------------------------------------------------------------------
# A3: weight preprocessing

@pytest.mark.parametrize("shape", [(4, 16, 16, 8, 3, 1, 1), (40, 6, 6, 6, 1, 1, 0), (3, 30, 30, 5, 7, 2, 3)])
def test_preprocess_weights_matches_oracle(ctx, P, shape):
    C, H, W, M, k, st, pad = shape
    plan = ctx.plan(C, H, W, M, k, stride=st, pad=pad)
    opl = packing.plan_conv(C, H, W, M, k, k, st, pad, P.n, P.L)
    g = inputs.rng(105)
    K = inputs.full_range_kernel(g, M, C, k, k)
    w = ctx.preprocess_weights(plan, T(K))
    wn = U(w)
    # lifted coefficient-domain polys (oracle packing + centred lift) ...
    kp = packing.kernel_polys(K, opl, P.n)
    lifted = np.zeros((M, opl.G, P.L, P.n), np.uint64)
    for j, q in enumerate(P.primes):
        for m in range(M):
            for gg in range(opl.G):
                v = kp[m, gg].astype(object)
                lifted[m, gg, j] = np.array([(int(x) - P.t) % q if x >= P.t // 2 else int(x) for x in v], np.uint64)
    # ... equal the GPU output brought back by the (separately pinned) GPU inverse NTT
    assert (U(ctx.ntt_inv(w.clone())) == lifted).all()
    # and a sample of NTT-domain words equals direct evaluation of the oracle's lifted polys
    ks = g.integers(0, P.n, 16).astype(np.uint32)
    for j in range(P.L):
        assert (wn[0, 0, j, ks] == he.ntt_sampled(lifted[0, 0, j], ks, P, j)).all()
    # idempotent
    assert (U(ctx.preprocess_weights(plan, T(K))) == wn).all()


def test_zero_kernel_gives_zero_weights(ctx, P):
    plan = ctx.plan(4, 16, 16, 8, 3, pad=1)
    w = ctx.preprocess_weights(plan, torch.zeros((8, 4, 3, 3), dtype=torch.int64, device=DEV))
    assert not U(w).any()


# ---------------------------------------------------------------------------------------------
# the hot path: secn_he_conv2d

def _layer_inputs(P, lay, seed, opl):
    g = inputs.rng(seed)
    G, S, M = opl.G, opl.S, opl.M
    ct = inputs.uniform_residues(g, (G * S, 2), P.primes, P.n)
    x0 = inputs.uniform_below(g, (G * S, P.n), P.t)
    K = inputs.quantized_kernel(g, M, lay.C, lay.k, lay.k)
    r = inputs.uniform_below(g, (M * S, P.n), P.t)
    return ct, x0, K, r


def _run_layer(ctx, lay, ct, x0, K, r, use_x0=True, use_r=True):
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    w = ctx.preprocess_weights(plan, T(K))
    out = ctx.he_conv2d(plan, T(ct), w, x0=T(x0) if use_x0 else None, r=T(r) if use_r else None)
    return plan, U(out)


@pytest.mark.parametrize("use_x0,use_r", [(True, True), (False, False), (True, False), (False, True)])
def test_he_conv2d_tiny_exact(ctx, P, use_x0, use_r):
    lay = layers.tiny()[0]
    opl = packing.plan_conv(lay.C, lay.H, lay.W, lay.M, lay.k, lay.k, lay.stride, lay.pad, P.n, P.L)
    ct, x0, K, r = _layer_inputs(P, lay, 1, opl)
    _, got = _run_layer(ctx, lay, ct, x0, K, r, use_x0, use_r)
    ref = he.server_conv(ct, x0 if use_x0 else None, K, r if use_r else None, opl, P)
    assert (got == ref).all()


L_ = layers.ConvLayer


@pytest.mark.parametrize("lay", [
    L_("multi_g", 40, 12, 12, 7, 3, 1, 1),       # G > 1
    L_("multi_s", 2, 70, 70, 3, 3, 1, 0),        # S > 4 -> several s-groups
    L_("stride2", 3, 40, 40, 5, 3, 2, 0),        # strided 3x3
    L_("ds", 24, 28, 28, 9, 1, 2, 0),            # decimated 1x1 / stride 2
    L_("k7", 3, 64, 64, 4, 7, 2, 3),             # 7x7 / stride 2 / pad 3
    L_("mtile", 8, 8, 8, 37, 1, 1, 0),           # M not a multiple of the m-tile
    L_("scalar", 1, 1, 1, 1, 1, 1, 0),           # 1x1 input, 1x1 kernel
])
def test_he_conv2d_shapes_exact(ctx, P, lay):
    opl = packing.plan_conv(lay.C, lay.H, lay.W, lay.M, lay.k, lay.k, lay.stride, lay.pad, P.n, P.L)
    ct, x0, K, r = _layer_inputs(P, lay, 2, opl)
    _, got = _run_layer(ctx, lay, ct, x0, K, r)
    ref = he.server_conv(ct, x0, K, r, opl, P)
    assert (got == ref).all()


def _sampled_check(ctx, P, lay, seed, n_samples=3):
    opl = packing.plan_conv(lay.C, lay.H, lay.W, lay.M, lay.k, lay.k, lay.stride, lay.pad, P.n, P.L)
    ct, x0, K, r = _layer_inputs(P, lay, seed, opl)
    _, got = _run_layer(ctx, lay, ct, x0, K, r)
    g = inputs.rng(seed + 1)
    n_out = opl.M * opl.S
    pick = np.unique(np.concatenate([[0, n_out - 1], g.integers(0, n_out, n_samples)]))
    sel = np.zeros(n_out, np.uint8)
    sel[pick] = 1
    ref = he.server_conv(ct, x0, K, r, opl, P, sel=sel)
    assert (got[pick] == ref[pick]).all(), lay.name


@pytest.mark.parametrize("lay", layers.squeezenet11(), ids=lambda l: l.name)
def test_he_conv2d_squeezenet11_full_size_sampled(ctx, P, lay):
    """Every SqueezeNet-1.1 layer at full size, in the launch configuration bench.py times."""
    _sampled_check(ctx, P, lay, 300 + zlib.crc32(lay.name.encode()) % 1000)


@pytest.mark.parametrize("name", ["conv1", "l1.b0.c2", "l2.b0.ds", "l4.b0.c2", "l4.b2.c3"])
def test_he_conv2d_resnet50_layers_sampled(ctx, P, name):
    lay = next(l for l in layers.resnet50() if l.name == name)
    _sampled_check(ctx, P, lay, 400, n_samples=2)


def test_extract_share_matches_oracle(ctx, P):
    for lay in [layers.tiny()[0], L_("s2", 3, 40, 40, 5, 3, 2, 0), L_("ds", 24, 28, 28, 9, 1, 2, 0)]:
        plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
        opl = packing.plan_conv(lay.C, lay.H, lay.W, lay.M, lay.k, lay.k, lay.stride, lay.pad, P.n, P.L)
        r = inputs.uniform_below(inputs.rng(5), (opl.M * opl.S, P.n), P.t)
        got = U(ctx.extract_share(plan, T(r)))
        assert (got == packing.extract((P.t - r) % P.t, opl)).all()


def test_end_to_end_decrypts_to_plain_conv(ctx, P):
    """Client (oracle harness) encrypts its share; the GPU server path runs; decrypt + the
    GPU-extracted server share reconstruct conv(x0 + x1, K) mod 2^37 exactly."""
    lay = L_("e2e", 6, 20, 20, 4, 3, 2, 1)
    opl = packing.plan_conv(lay.C, lay.H, lay.W, lay.M, lay.k, lay.k, lay.stride, lay.pad, P.n, P.L)
    g = inputs.rng(77)
    x1 = inputs.uniform_below(g, (lay.C, lay.H, lay.W), P.t)
    x0 = inputs.uniform_below(g, (lay.C, lay.H, lay.W), P.t)
    K = inputs.quantized_kernel(g, lay.M, lay.C, lay.k, lay.k)
    sk = inputs.ternary(g, P.n)
    xin = packing.pack_input(x1, opl, P.n)
    ct = np.stack([he.encrypt(xin[i], sk, inputs.uniform_residues(g, (), P.primes, P.n),
                              inputs.rounded_gaussian(g, P.n), P) for i in range(opl.G * opl.S)])
    r = inputs.uniform_below(g, (opl.M * opl.S, P.n), P.t)
    plan, out = _run_layer(ctx, lay, ct, packing.pack_input(x0, opl, P.n), K, r)
    y0 = U(ctx.extract_share(plan, T(r)))
    s_idx, coef = packing.designated_map(opl)
    y1 = np.zeros_like(y0)
    for m in range(opl.M):
        for s in range(opl.S):
            sel = s_idx == s
            if sel.any():
                y1[m][sel] = he.decrypt(out[m * opl.S + s], sk, P, coef[sel])
    y = (y0 + y1) & np.uint64(P.t - 1)
    assert (y == conv.conv2d_mod((x0 + x1) & np.uint64(P.t - 1), K, lay.stride, lay.pad, P.t_bits)).all()
