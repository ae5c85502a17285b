"""GPU parity: libsecn (through its C ABI, via the ctypes binding) against the oracle,
element by element on identical seeded inputs. Integer work => bit-exact (every word).

Both residue word sizes are covered: 64-bit limbs at the paper parameters (reading R1:
q0 = 60 bit, q1 = 49 bit) and 32-bit limbs (reading R1b: four 27-bit primes).

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
PRIMES = {64: params.DEFAULT_PRIMES, 32: params.PRIMES32}


def TP(a: np.ndarray) -> torch.Tensor:
    """plaintext-side uint64 array -> int64 CUDA tensor"""
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint64).view(np.int64)).to(DEV)


def UP(t: torch.Tensor) -> np.ndarray:
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint64)


class Dev:
    """Residue conversions for one context word size."""

    def __init__(self, ctx):
        self.ctx = ctx
        self.wb = ctx.word_bits

    def R(self, a: np.ndarray) -> torch.Tensor:
        a = np.ascontiguousarray(a, dtype=np.uint64)
        if self.wb == 64:
            return torch.from_numpy(a.view(np.int64)).to(DEV)
        assert (a >> np.uint64(32)).max(initial=0) == 0
        return torch.from_numpy(a.astype(np.uint32).view(np.int32)).to(DEV)

    def U(self, t: torch.Tensor) -> np.ndarray:
        torch.cuda.synchronize()
        x = t.cpu().numpy()
        return x.view(np.uint64) if self.wb == 64 else x.view(np.uint32).astype(np.uint64)


@pytest.fixture(scope="module")
def secn():
    __graft_entry__.build()
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_11586_b200 import secn as m

    return m


@pytest.fixture(scope="module", params=[64, 32], ids=["w64", "w32"])
def env(request, secn):
    wb = request.param
    ctx = secn.Context(0, word_bits=wb)
    P = Params(primes=PRIMES[wb])
    yield ctx, P, Dev(ctx)
    ctx.close()


PLAN_FIELDS = ("OH", "OW", "decim", "Hp", "Wp", "Cw", "Hw", "Ww", "G", "S", "nbh", "nbw", "O")


def same_plan(opl, plan):
    """The oracle's plan and the library's agree field by field (the window is a performance
    choice; the oracle's packing is exact for any valid window, so this is a plan-rule check)."""
    assert tuple(getattr(opl, f) for f in PLAN_FIELDS) == tuple(getattr(plan, f) for f in PLAN_FIELDS), (opl, plan)


def oplan(P, ctx, lay, rule="time"):
    """The oracle's own plan (reading R6b time rule by default, or R6 byte-min), computed without
    the product library and asserted equal to the window the library picks for this layer."""
    opl = packing.plan_conv(lay.C, lay.H, lay.W, lay.M, lay.k, lay.k, lay.stride, lay.pad, P.n, ctx.coef_words64,
                            rule=rule)
    c = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad,
                 rule=secn_mod().PLAN_TIME if rule == "time" else secn_mod().PLAN_BYTES)
    same_plan(opl, c)
    return opl


# ---------------------------------------------------------------------------------------------
# context tables

@pytest.mark.parametrize("logn,primes,wb", [(12, params.DEFAULT_PRIMES, 64), (12, params.ALT54_PRIMES, 64),
                                            (12, params.SWEEP_PRIMES, 64), (13, params.SWEEP_PRIMES, 64),
                                            (14, params.SWEEP_PRIMES[:2], 64), (12, params.PRIMES32, 32),
                                            (14, params.PRIMES32, 32), (15, params.SWEEP_PRIMES, 64),
                                            (15, params.PRIMES32, 32)])
def test_ctx_psi_matches_oracle(secn, logn, primes, wb):
    c = secn.Context(0, log_n=logn, primes=primes, word_bits=wb)
    assert c.psi == tuple(Params(logn=logn, primes=primes).psi)
    c.close()


def test_ctx_rejects_wrong_word_size_calls(secn):
    c32 = secn.Context(0, word_bits=32)
    lib = secn.lib()
    import ctypes

    assert lib.secn_ntt_fwd(c32._h, None, 0, None) == -6
    c64 = secn.Context(0)
    assert lib.secn32_ntt_fwd(c64._h, None, 0, None) == -6
    big = (ctypes.c_uint32 * 1)(0x1FFF0001)  # 29-bit prime > 2^28 bound of 32-bit limbs
    h = ctypes.c_void_p()
    assert lib.secn32_ctx_create(ctypes.byref(h), 0, 12, 1, big, 37) == -2


# ---------------------------------------------------------------------------------------------
# A1 / A2: NTT and inverse

def _edge_polys(P, g):
    n = P.n
    polys = [inputs.uniform_residues(g, (), P.primes, n)]
    z = np.zeros((P.L, n), np.uint64)
    polys.append(z.copy())                                           # zero
    c = z.copy(); c[:, 0] = 1234567; polys.append(c)                  # constant
    top = np.stack([np.full(n, q - 1, np.uint64) for q in P.primes]); polys.append(top)  # all q-1
    mono = z.copy(); mono[:, n - 1] = 1; polys.append(mono)           # X^(N-1)
    return np.stack(polys)


def test_ntt_fwd_matches_direct_evaluation(env):
    ctx, P, D = env
    g = inputs.rng(100)
    polys = _edge_polys(P, g)
    got = D.U(ctx.ntt_fwd(D.R(polys)))
    for i in range(polys.shape[0]):
        for j in range(P.L):
            if (i >= 2 and j != P.L - 1) or (i == 0 and j >= 2):
                continue  # keeps the O(N^2) oracle calls few
            assert (got[i, j] == he.ntt(polys[i, j], P, j)).all(), (i, j)
    assert (got[2] == 1234567).all()  # constant -> constant vector, on every limb


def test_ntt_inv_matches_direct_and_roundtrips(env):
    ctx, P, D = env
    g = inputs.rng(101)
    A = inputs.uniform_residues(g, (2,), P.primes, P.n)
    got = D.U(ctx.ntt_inv(D.R(A)))
    assert (got[0, 0] == he.intt(A[0, 0], P, 0)).all()
    assert (got[1, 1] == he.intt(A[1, 1], P, 1)).all()
    big = inputs.uniform_residues(g, (3001,), P.primes, P.n)         # multi-wave batch
    t = D.R(big)
    ctx.ntt_fwd(t)
    ctx.ntt_inv(t)
    assert (D.U(t) == big).all()


def test_ntt_pointwise_product_is_negacyclic_product(env):
    ctx, P, D = env
    g = inputs.rng(102)
    a = inputs.uniform_residues(g, (), P.primes, P.n)
    b = inputs.uniform_residues(g, (), P.primes, P.n)
    A, B = D.U(ctx.ntt_fwd(D.R(a[None]))), D.U(ctx.ntt_fwd(D.R(b[None])))
    prod = np.stack([np.array([int(x) * int(y) % q for x, y in zip(A[0, j], B[0, j])], np.uint64)
                     for j, q in enumerate(P.primes)])
    c = D.U(ctx.ntt_inv(D.R(prod[None])))[0]
    for j, q in enumerate(P.primes):
        assert (c[j] == he.negacyclic_mul(a[j], b[j], q)).all()


@pytest.mark.parametrize("logn,L,wb", [(12, 4, 64), (13, 1, 64), (13, 3, 64), (14, 2, 64), (14, 4, 64),
                                       (13, 4, 32), (14, 2, 32),
                                       (15, 1, 64), (15, 4, 64), (15, 1, 32), (15, 4, 32)])  # 15: cluster NTT
def test_ntt_sweep_sampled(secn, logn, L, wb):
    primes = (params.SWEEP_PRIMES if wb == 64 else params.PRIMES32)[:L]
    c = secn.Context(0, log_n=logn, primes=primes, word_bits=wb)
    D = Dev(c)
    P = Params(logn=logn, primes=primes)
    g = inputs.rng(103 + logn * 10 + L)
    x = inputs.uniform_residues(g, (7,), primes, P.n)
    got = D.U(c.ntt_fwd(D.R(x)))
    ks = np.concatenate([[0, 1, P.n // 2, P.n - 1], g.integers(0, P.n, 28)]).astype(np.uint32)
    for i in (0, 6):
        for j in range(L):
            assert (got[i, j, ks] == he.ntt_sampled(x[i, j], ks, P, j)).all(), (i, j)
    back = D.U(c.ntt_inv(D.R(got)))
    assert (back == x).all()
    c.close()


@pytest.mark.parametrize("wb", [64, 32])
def test_cluster_ntt_in_place_multi_wave_roundtrip(secn, wb):
    """N = 2^15 (two-CTA clusters, DSMEM exchange in the inverse): a batch of several waves
    transformed in place round-trips, and sampled outputs equal direct evaluation."""
    primes = (params.SWEEP_PRIMES if wb == 64 else params.PRIMES32)[:2]
    c = secn.Context(0, log_n=15, primes=primes, word_bits=wb)
    D = Dev(c)
    P = Params(logn=15, primes=primes)
    g = inputs.rng(777 + wb)
    x = inputs.uniform_residues(g, (301,), primes, P.n)
    t = D.R(x)
    c.ntt_fwd(t)
    got = D.U(t)
    ks = np.concatenate([[0, P.n // 2 - 1, P.n // 2, P.n - 1], g.integers(0, P.n, 12)]).astype(np.uint32)
    for i in (0, 150, 300):
        assert (got[i, 1, ks] == he.ntt_sampled(x[i, 1], ks, P, 1)).all(), i
    c.ntt_inv(t)
    assert (D.U(t) == x).all()
    c.close()


@pytest.mark.parametrize("logn", [13, 14])
@pytest.mark.parametrize("wb", [64, 32])
def test_he_conv2d_other_ring_degrees(secn, logn, wb):
    """The hot path at N = 2^13 and 2^14 (64-bit words at 2^14 use the cluster forward NTT)."""
    primes = (params.SWEEP_PRIMES[:2] if wb == 64 else params.PRIMES32)
    ctx = secn.Context(0, log_n=logn, primes=primes, word_bits=wb)
    P = Params(logn=logn, primes=primes)
    D = Dev(ctx)
    lay = L_("n", 20, 30, 30, 6, 3, 1, 1)
    opl = oplan(P, ctx, lay)
    ct, x0, K, r = _layer_inputs(P, lay, 21, opl)
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    w = ctx.preprocess_weights(plan, TP(K))
    y0 = torch.empty((plan.M, plan.OH, plan.OW), dtype=torch.int64, device=DEV)
    got = D.U(ctx.he_conv2d(plan, D.R(ct), w, x0=TP(x0), r=TP(r), y0=y0))
    assert (got == he.server_conv(ct, x0, K, r, opl, P)).all()
    assert (UP(y0) == packing.extract((P.t - r) % P.t, opl)).all()
    ctx.close()


def test_conv_rejects_n32768(secn):
    c = secn.Context(0, log_n=15, primes=params.PRIMES32, word_bits=32)
    plan = c.plan(4, 16, 16, 8, 3, stride=1, pad=1)
    K = torch.zeros((8, 4, 3, 3), dtype=torch.int64, device=DEV)
    with pytest.raises(secn.SecnError):
        c.preprocess_weights(plan, K)
    c.close()


def test_empty_batch_is_noop(env):
    ctx, P, D = env
    t = torch.zeros(0, dtype=ctx.rdtype, device=DEV)
    ctx.ntt_fwd(t)
    ctx.ntt_inv(t)
    torch.cuda.synchronize()


# ---------------------------------------------------------------------------------------------
# A6 / A7: server-share add and output mask

def test_mask_and_share_add_match_oracle_enc(env):
    ctx, P, D = env
    g = inputs.rng(104)
    n = 5
    ct = inputs.uniform_residues(g, (n, 2), P.primes, P.n)
    r = inputs.uniform_below(g, (n, P.n), P.t)
    r[0, :4] = [0, 1, P.t - 1, P.t // 2]
    got = D.U(ctx.mask_add(D.R(ct), TP(r)))
    assert (got == he.mask_add(ct, r, P)).all()
    got2 = D.U(ctx.share_add(D.R(ct), TP(r)))
    assert (got2 == got).all()


# ---------------------------------------------------------------------------------------------
# A3: weight preprocessing

@pytest.mark.parametrize("shape", [(4, 16, 16, 8, 3, 1, 1), (40, 6, 6, 6, 1, 1, 0), (3, 30, 30, 5, 7, 2, 3)])
def test_preprocess_weights_matches_oracle(env, shape):
    ctx, P, D = env
    C, H, W, M, k, st, pad = shape
    plan = ctx.plan(C, H, W, M, k, stride=st, pad=pad)
    opl = oplan(P, ctx, layers.ConvLayer("w", C, H, W, M, k, st, pad))
    g = inputs.rng(105)
    K = inputs.full_range_kernel(g, M, C, k, k)
    w = ctx.preprocess_weights(plan, TP(K))
    wn = D.U(w)
    # lifted coefficient-domain polys (oracle packing + centred lift) ...
    kp = packing.kernel_polys(K, opl, P.n)
    lifted = np.zeros((M, opl.G, P.L, P.n), np.uint64)
    for j, q in enumerate(P.primes):
        for m in range(M):
            for gg in range(opl.G):
                lifted[m, gg, j] = np.array([(int(x) - P.t) % q if x >= P.t // 2 else int(x) % q for x in kp[m, gg]],
                                            np.uint64)
    # ... equal the GPU output brought back by the (separately pinned) GPU inverse NTT
    assert (D.U(ctx.ntt_inv(w.clone())) == lifted).all()
    # and a sample of NTT-domain words equals direct evaluation of the oracle's lifted polys
    ks = g.integers(0, P.n, 16).astype(np.uint32)
    for j in range(P.L):
        assert (wn[0, 0, j, ks] == he.ntt_sampled(lifted[0, 0, j], ks, P, j)).all()
    # idempotent
    assert (D.U(ctx.preprocess_weights(plan, TP(K))) == wn).all()


def test_zero_kernel_gives_zero_weights(env):
    ctx, P, D = env
    plan = ctx.plan(4, 16, 16, 8, 3, pad=1)
    w = ctx.preprocess_weights(plan, torch.zeros((8, 4, 3, 3), dtype=torch.int64, device=DEV))
    assert not D.U(w).any()


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


def _run_layer(ctx, D, lay, ct, x0, K, r, use_x0=True, use_r=True):
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    w = ctx.preprocess_weights(plan, TP(K))
    out = ctx.he_conv2d(plan, D.R(ct), w, x0=TP(x0) if use_x0 else None, r=TP(r) if use_r else None)
    return plan, D.U(out)


@pytest.mark.parametrize("use_x0,use_r", [(True, True), (False, False), (True, False), (False, True)])
def test_he_conv2d_tiny_exact(env, use_x0, use_r):
    ctx, P, D = env
    lay = layers.tiny()[0]
    opl = oplan(P, ctx, lay)
    ct, x0, K, r = _layer_inputs(P, lay, 1, opl)
    _, got = _run_layer(ctx, D, lay, ct, x0, K, r, use_x0, use_r)
    ref = he.server_conv(ct, x0 if use_x0 else None, K, r if use_r else None, opl, P)
    assert (got == ref).all()


@pytest.mark.parametrize("rep", range(3))
def test_stage_calls_read_inputs_written_just_before(env, rep):
    """A stage call whose weights (stage 1) or mask (stage 2) were written by the kernel right
    before it on the stream: secn_preprocess_weights then stage 1, a device copy of r then
    stage 2. Stage calls never read an input before the dependency wait (k_mac used to
    pre-issue weight loads and the tails to load r before griddepcontrol.wait)."""
    ctx, P, D = env
    lay = layers.ConvLayer("pw", 64, 13, 13, 256, 3, 1, 1)  # many m-blocks: weights stream long after launch
    opl = oplan(P, ctx, lay)
    ct, x0, K, r = _layer_inputs(P, lay, 40 + rep, opl)
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    cti, x0t = D.R(ct), TP(x0)
    out = ctx.empty(plan.M * plan.S, 2, ctx.L, ctx.n)
    ws = torch.empty(ctx.workspace_bytes(plan) // 8, dtype=torch.int64, device=DEV)
    w = ctx.empty(plan.M, plan.G, ctx.L, ctx.n)
    w.fill_(-1)
    rt = torch.full((plan.M * plan.S, ctx.n), -1, dtype=torch.int64, device=DEV)
    rsrc = TP(r)
    torch.cuda.synchronize()
    ctx.he_conv2d_stage(0, plan, cti, w, x0t, rt, out, ws)
    ctx.preprocess_weights(plan, TP(K), out=w)  # its last kernel writes w ...
    ctx.he_conv2d_stage(1, plan, cti, w, x0t, rt, out, ws)  # ... and the MAC reads w
    rt.copy_(rsrc)  # a plain kernel writes r ...
    ctx.he_conv2d_stage(2, plan, cti, w, x0t, rt, out, ws)  # ... and the tail reads r
    assert (D.U(out) == he.server_conv(ct, x0, K, r, opl, P)).all()


def test_he_conv2d_stages_equal_fused_call(env):
    ctx, P, D = env
    lay = layers.ConvLayer("st", 20, 30, 30, 6, 3, 1, 1)
    opl = oplan(P, ctx, lay)
    ct, x0, K, r = _layer_inputs(P, lay, 3, opl)
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    w = ctx.preprocess_weights(plan, TP(K))
    cti, x0t, rt = D.R(ct), TP(x0), TP(r)
    fused = D.U(ctx.he_conv2d(plan, cti, w, x0=x0t, r=rt))
    out = ctx.empty(plan.M * plan.S, 2, ctx.L, ctx.n)
    ws = torch.empty(ctx.workspace_bytes(plan) // 8, dtype=torch.int64, device=DEV)
    for s in range(3):
        ctx.he_conv2d_stage(s, plan, cti, w, x0t, rt, out, ws)
    assert (D.U(out) == fused).all()
    # secn_he_conv2d_stage_ex: stage 2 also writes the share, as secn_he_conv2d_ex does
    y0f = torch.full((plan.M, plan.OH, plan.OW), -1, dtype=torch.int64, device=DEV)
    ctx.he_conv2d(plan, cti, w, x0=x0t, r=rt, y0=y0f)
    y0s = torch.full_like(y0f, -2)
    out.zero_()
    for s in range(3):
        ctx.he_conv2d_stage_ex(s, plan, cti, w, x0t, rt, out, y0s, ws)
    assert (D.U(out) == fused).all() and torch.equal(y0s, y0f)


L_ = layers.ConvLayer


@pytest.mark.parametrize("lay", [
    L_("multi_g", 40, 12, 12, 7, 3, 1, 1),       # G > 1
    L_("multi_s", 2, 70, 70, 3, 3, 1, 0),        # S > 4 -> several s-groups
    L_("stride2", 3, 40, 40, 5, 3, 2, 0),        # strided 3x3
    L_("ds", 24, 28, 28, 9, 1, 2, 0),            # decimated 1x1 / stride 2
    L_("k7", 3, 64, 64, 4, 7, 2, 3),             # 7x7 / stride 2 / pad 3
    L_("mtile", 8, 8, 8, 37, 1, 1, 0),           # M not a multiple of the m-tile
    L_("scalar", 1, 1, 1, 1, 1, 1, 0),           # 1x1 input, 1x1 kernel
    L_("g19", 512, 14, 14, 4, 3, 1, 1),          # G = 19 (GMAX 32 variants)
], ids=lambda l: l.name)
def test_he_conv2d_shapes_exact(env, lay):
    ctx, P, D = env
    opl = oplan(P, ctx, lay)
    ct, x0, K, r = _layer_inputs(P, lay, 2, opl)
    _, got = _run_layer(ctx, D, lay, ct, x0, K, r)
    ref = he.server_conv(ct, x0, K, r, opl, P)
    assert (got == ref).all()


_MT32 = {1: (16, 8), 2: (8, 4), 3: (5, 2), 4: (3, 2)}  # k_mac m-block per s-group: (big, small), 32-bit


@pytest.mark.parametrize("sg", [1, 2, 3, 4])
@pytest.mark.parametrize("small", [False, True])
def test_mac_register_blocks_exact(env, sg, small, monkeypatch):
    """Every k_mac register-block instantiation (s-group SG x m-block MT, forced through the
    SECN_MAC_SG / SECN_MAC_MT knobs) on a layer with G = 10, S = 3 (explicit 11 x 28 window),
    exact against the oracle. SG = 3, MT = 2 stages only 12 chunks, fewer than the 16 that give
    every thread an INTT task; its epilogue read past the end of shared memory before the guard
    (found by tools/plan_sweep.py on a ResNet-50 candidate window)."""
    ctx, P, D = env
    if ctx.word_bits == 64 and small:
        pytest.skip("64-bit limbs have one m-block size per s-group")
    lay = L_("cfg", 128, 28, 28, 6, 1, 1, 0)
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=1, pad=0, Hw=11, Ww=28)
    assert (plan.G, plan.S) == (10, 3)
    opl = packing.plan_conv(lay.C, lay.H, lay.W, lay.M, 1, 1, 1, 0, P.n, ctx.coef_words64, Hw=11, Ww=28)
    ct, x0, K, r = _layer_inputs(P, lay, 21, opl)
    monkeypatch.setenv("SECN_MAC_SG", str(sg))
    monkeypatch.setenv("SECN_FUSED", "0")  # the three-kernel path's k_mac
    if ctx.word_bits == 32:
        monkeypatch.setenv("SECN_MAC_MT", str(_MT32[sg][1 if small else 0]))
    kctx = secn_mod().Context(0, word_bits=ctx.word_bits)  # knobs are read at context creation
    w = kctx.preprocess_weights(plan, TP(K))
    got = D.U(kctx.he_conv2d(plan, D.R(ct), w, x0=TP(x0), r=TP(r)))
    kctx.close()
    assert (got == he.server_conv(ct, x0, K, r, opl, P)).all()


def _sampled_check(ctx, P, D, lay, seed, n_samples=3):
    opl = oplan(P, ctx, lay)
    ct, x0, K, r = _layer_inputs(P, lay, seed, opl)
    _, got = _run_layer(ctx, D, lay, ct, x0, K, r)
    g = inputs.rng(seed + 1)
    n_out = opl.M * opl.S
    pick = np.unique(np.concatenate([[0, n_out - 1], g.integers(0, n_out, n_samples)]))
    sel = np.zeros(n_out, np.uint8)
    sel[pick] = 1
    ref = he.server_conv(ct, x0, K, r, opl, P, sel=sel)
    assert (got[pick] == ref[pick]).all(), lay.name


@pytest.mark.parametrize("lay", layers.squeezenet11(), ids=lambda l: l.name)
def test_he_conv2d_squeezenet11_full_size_sampled(env, lay):
    """Every SqueezeNet-1.1 layer at full size, in the launch configuration bench.py times."""
    ctx, P, D = env
    _sampled_check(ctx, P, D, lay, 300 + zlib.crc32(lay.name.encode()) % 1000)


@pytest.mark.parametrize("name", ["conv1", "l1.b0.c2", "l2.b0.ds", "l4.b0.c2", "l4.b2.c3"])
def test_he_conv2d_resnet50_layers_sampled(env, name):
    ctx, P, D = env
    lay = next(l for l in layers.resnet50() if l.name == name)
    _sampled_check(ctx, P, D, lay, 400, n_samples=2)


def test_extract_share_matches_oracle(env):
    ctx, P, D = env
    for lay in [layers.tiny()[0], L_("s2", 3, 40, 40, 5, 3, 2, 0), L_("ds", 24, 28, 28, 9, 1, 2, 0)]:
        plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
        opl = oplan(P, ctx, lay)
        r = inputs.uniform_below(inputs.rng(5), (opl.M * opl.S, P.n), P.t)
        got = UP(ctx.extract_share(plan, TP(r)))
        assert (got == packing.extract((P.t - r) % P.t, opl)).all()


@pytest.mark.parametrize("lay", [layers.tiny()[0], L_("s2", 3, 40, 40, 5, 3, 2, 0), L_("ds", 24, 28, 28, 9, 1, 2, 0),
                                 L_("multi_s", 2, 70, 70, 3, 3, 1, 0), L_("k7", 3, 64, 64, 4, 7, 2, 3)],
                         ids=lambda l: l.name)
def test_he_conv2d_ex_fused_share_matches_oracle(env, lay):
    """secn_he_conv2d_ex: the same ciphertexts as secn_he_conv2d, and y0 equal to the oracle's
    designated-coefficient extraction of (t - r) mod t."""
    ctx, P, D = env
    opl = oplan(P, ctx, lay)
    ct, x0, K, r = _layer_inputs(P, lay, 9, opl)
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    w = ctx.preprocess_weights(plan, TP(K))
    y0 = torch.full((plan.M, plan.OH, plan.OW), -1, dtype=torch.int64, device=DEV)
    out = D.U(ctx.he_conv2d(plan, D.R(ct), w, x0=TP(x0), r=TP(r), y0=y0))
    assert (out == he.server_conv(ct, x0, K, r, opl, P)).all()
    assert (UP(y0) == packing.extract((P.t - r) % P.t, opl)).all()


@pytest.mark.parametrize("lay", [layers.tiny()[0], L_("multi_g", 40, 12, 12, 7, 3, 1, 1), L_("ds", 24, 28, 28, 9, 1, 2, 0)],
                         ids=lambda l: l.name)
def test_he_conv2d_online_weights_match_oracle(env, lay):
    """f4 toggle: weights in coefficient form, transformed inside the call;
    the ciphertexts and the share equal the oracle's (and so the offline-preprocessed path)."""
    ctx, P, D = env
    opl = oplan(P, ctx, lay)
    ct, x0, K, r = _layer_inputs(P, lay, 12, opl)
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    y0 = torch.empty((plan.M, plan.OH, plan.OW), dtype=torch.int64, device=DEV)
    ws = torch.full(((ctx.online_workspace_bytes(plan) + 7) // 8,), -1, dtype=torch.int64, device=DEV)
    out = D.U(ctx.he_conv2d_online(plan, D.R(ct), TP(K), x0=TP(x0), r=TP(r), y0=y0, workspace=ws))
    assert (out == he.server_conv(ct, x0, K, r, opl, P)).all()
    assert (UP(y0) == packing.extract((P.t - r) % P.t, opl)).all()


def test_he_conv2d_ex_needs_r(env):
    ctx, P, D = env
    lay = layers.tiny()[0]
    opl = oplan(P, ctx, lay)
    ct, x0, K, r = _layer_inputs(P, lay, 1, opl)
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    w = ctx.preprocess_weights(plan, TP(K))
    y0 = torch.empty((plan.M, plan.OH, plan.OW), dtype=torch.int64, device=DEV)
    from paper_2506_11586_b200 import secn as m

    with pytest.raises(m.SecnError):
        ctx.he_conv2d(plan, D.R(ct), w, x0=TP(x0), r=None, y0=y0)


def test_end_to_end_decrypts_to_plain_conv(env):
    """Client (oracle harness) encrypts its share; the GPU server path runs; decrypt + the
    GPU-extracted server share reconstruct conv(x0 + x1, K) mod 2^37 exactly."""
    ctx, P, D = env
    lay = L_("e2e", 6, 20, 20, 4, 3, 2, 1)
    opl = oplan(P, ctx, lay)
    g = inputs.rng(77)
    x1 = inputs.uniform_below(g, (lay.C, lay.H, lay.W), P.t)
    x0 = inputs.uniform_below(g, (lay.C, lay.H, lay.W), P.t)
    K = inputs.quantized_kernel(g, lay.M, lay.C, lay.k, lay.k)
    sk = inputs.ternary(g, P.n)
    xin = packing.pack_input(x1, opl, P.n)
    ct = np.stack([he.encrypt(xin[i], sk, inputs.uniform_residues(g, (), P.primes, P.n),
                              inputs.rounded_gaussian(g, P.n), P) for i in range(opl.G * opl.S)])
    r = inputs.uniform_below(g, (opl.M * opl.S, P.n), P.t)
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    w = ctx.preprocess_weights(plan, TP(K))
    y0t = torch.empty((plan.M, plan.OH, plan.OW), dtype=torch.int64, device=DEV)
    out = D.U(ctx.he_conv2d(plan, D.R(ct), w, x0=TP(packing.pack_input(x0, opl, P.n)), r=TP(r), y0=y0t))
    y0 = UP(y0t)
    s_idx, coef = packing.designated_map(opl)
    y1 = np.zeros_like(y0)
    for m in range(opl.M):
        for s in range(opl.S):
            sel = s_idx == s
            if sel.any():
                y1[m][sel] = he.decrypt(out[m * opl.S + s], sk, P, coef[sel])
    y = (y0 + y1) & np.uint64(P.t - 1)
    assert (y == conv.conv2d_mod((x0 + x1) & np.uint64(P.t - 1), K, lay.stride, lay.pad, P.t_bits)).all()


@pytest.mark.parametrize("overlap", ["none", "staged", "free"])
def test_network_step_graph_equals_layerwise(secn, overlap):
    """The bench's step (all SqueezeNet-1.1 layers in one CUDA graph, programmatic dependent
    launches between the kernels; network order, or bench.py --overlap staged / free) gives, on
    every layer, the words of the same layers run one call at a time with a synchronisation after
    each: no cross-layer hazard. Before k_mac released its ring stages through consumer_release
    (proxy fence), the free overlap failed this in every replay."""
    from paper_2506_11586_b200.schedule import GroupRunner, StagedGroupRunner, concurrent_groups
    ctx = secn.Context(0, word_bits=32)
    st = []
    for li, lay in enumerate(layers.squeezenet11()):
        plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
        g = inputs.rng(500 + li)
        ct = torch.from_numpy(inputs.uniform_residues(g, (plan.G * plan.S, 2), ctx.primes, ctx.n)
                              .astype(np.uint32).view(np.int32)).to(DEV)
        d = dict(plan=plan, ct=ct, x0=TP(inputs.uniform_below(g, (plan.G * plan.S, ctx.n), 1 << ctx.t_bits)),
                 r=TP(inputs.uniform_below(g, (plan.M * plan.S, ctx.n), 1 << ctx.t_bits)),
                 out=ctx.empty(plan.M * plan.S, 2, ctx.L, ctx.n),
                 ws=torch.empty(ctx.workspace_bytes(plan) // 8 + 1, dtype=torch.int64, device=DEV),
                 y0=torch.empty((plan.M, plan.OH, plan.OW), dtype=torch.int64, device=DEV))
        d["w"] = ctx.preprocess_weights(plan, TP(inputs.quantized_kernel(g, plan.M, lay.C, lay.k, lay.k)))
        st.append(d)

    def call(d):
        ctx.he_conv2d(d["plan"], d["ct"], d["w"], x0=d["x0"], r=d["r"], out=d["out"], workspace=d["ws"], y0=d["y0"])

    def stage(d, k):
        ctx.he_conv2d_stage_ex(k, d["plan"], d["ct"], d["w"], d["x0"], d["r"], d["out"], d["y0"], d["ws"])

    ref = []
    for d in st:
        call(d)
        torch.cuda.synchronize()
        ref.append((d["out"].clone(), d["y0"].clone()))
    names = [lay.name for lay in layers.squeezenet11()]
    runner = StagedGroupRunner(concurrent_groups(names), DEV)
    free = GroupRunner(concurrent_groups(names), DEV)
    graph = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream(DEV)
    with torch.cuda.graph(graph, stream=cap):
        if overlap == "staged":
            runner(lambda i: call(st[i]), lambda i, k: stage(st[i], k))
        elif overlap == "free":
            free(lambda i: call(st[i]))
        else:
            for d in st:
                call(d)
    for _ in range(10 if overlap == "free" else 3):
        for d in st:
            d["out"].zero_()
            d["y0"].zero_()
        graph.replay()
        torch.cuda.synchronize()
        for d, (o, y) in zip(st, ref):
            assert torch.equal(d["out"], o) and torch.equal(d["y0"], y)
    ctx.close()


def _fuzz_layers(n=20, seed=2026):
    g = np.random.default_rng(seed)
    out = []
    for i in range(n):
        k = int(g.choice([1, 3, 5, 7]))
        st = int(g.choice([1, 2]))
        pad = int(g.integers(0, k // 2 + 1))
        H = int(g.integers(max(k, 2), 41))
        W = int(g.integers(max(k, 2), 41))
        C = int(g.integers(1, 97))
        M = int(g.integers(1, 49))
        out.append(L_(f"fz{i}_c{C}h{H}w{W}m{M}k{k}s{st}p{pad}", C, H, W, M, k, st, pad))
    return out


@pytest.mark.parametrize("rule", ["time", "bytes"])
@pytest.mark.parametrize("lay", _fuzz_layers(), ids=lambda l: l.name)
def test_he_conv2d_ex_random_shapes_exact(env, lay, rule):
    """Seeded random layer geometries (kernel 1-7, stride 1-2, padding, odd sizes), each under the
    time-rule window (polyphase where it wins) and the byte-min window: ciphertexts and the fused
    share y0 equal to the oracle word for word."""
    ctx, P, D = env
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad,
                    rule=secn_mod().PLAN_TIME if rule == "time" else secn_mod().PLAN_BYTES)
    opl = oplan(P, ctx, lay, rule)
    ct, x0, K, r = _layer_inputs(P, lay, 31, opl)
    w = ctx.preprocess_weights(plan, TP(K))
    y0 = torch.full((plan.M, plan.OH, plan.OW), -1, dtype=torch.int64, device=DEV)
    got = D.U(ctx.he_conv2d(plan, D.R(ct), w, x0=TP(x0), r=TP(r), y0=y0))
    assert (got == he.server_conv(ct, x0, K, r, opl, P)).all()
    assert (UP(y0) == packing.extract((P.t - r) % P.t, opl)).all()


def secn_mod():
    from paper_2506_11586_b200 import secn as m
    return m
