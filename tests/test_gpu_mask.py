"""GPU parity of the device-drawn mask (reading R17): secn_mask_draw word for word
against the oracle's Philox4x32-10 draw, and the *_gen entry points (the mask drawn inside the
layer call) against the oracle's server computation with that mask -- whole ciphertexts, the
server share, rank slices of the output channels, and the extracted (LWE) outputs."""
import numpy as np
import pytest
import torch

from oracle import he, packing, philox
from test_gpu_parity import DEV, TP, UP, Dev, _layer_inputs, env, oplan, secn, secn_mod  # noqa: F401  (fixtures)
from workloads import layers

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed,stream,ct0,n_ct", [(0, 0, 0, 1), (0x0123456789ABCDEF, 3, 0, 7),
                                                  (2**64 - 1, 2**32 - 1, 1000, 5), (42, 9, 12345, 300)])
def test_mask_draw_matches_oracle(env, seed, stream, ct0, n_ct):
    ctx, P, D = env
    g = secn_mod().MaskGen(seed=seed, stream=stream, ct0=ct0)
    got = UP(ctx.mask_draw(g, n_ct))
    ref = philox.mask(seed, stream, n_ct, ctx.n, ctx.t_bits, ct0=ct0)
    assert (got == ref).all()


def test_mask_draw_other_ring():
    m = secn_mod()
    c = m.Context(0, log_n=13, primes=(0xFFFFFFFFFFC0001, 0xFFFFFFFFF840001))
    g = m.MaskGen(seed=5, stream=6, ct0=7)
    assert (UP(c.mask_draw(g, 3)) == philox.mask(5, 6, 3, 8192, 37, ct0=7)).all()
    c.close()


@pytest.mark.parametrize("name", ["tiny", "fire9.e3", "conv1"])
def test_he_conv2d_gen_matches_oracle(env, name):
    ctx, P, D = env
    lay = layers.tiny()[0] if name == "tiny" else next(l for l in layers.squeezenet11() if l.name == name)
    opl = oplan(P, ctx, lay)
    ct, x0, K, _ = _layer_inputs(P, lay, 61, opl)
    seed, stream = 0xFEEDFACECAFEBEEF, 17
    r = philox.mask(seed, stream, opl.M * opl.S, P.n, P.t_bits)
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    w = ctx.preprocess_weights(plan, TP(K))
    y0 = torch.full((plan.M, plan.OH, plan.OW), -1, dtype=torch.int64, device=DEV)
    g = secn_mod().MaskGen(seed=seed, stream=stream, ct0=0)
    got = D.U(ctx.he_conv2d_gen(plan, D.R(ct), w, g, x0=TP(x0), y0=y0))
    n_out = opl.M * opl.S
    pick = np.unique(np.array([0, n_out // 2, n_out - 1]))
    sel = np.zeros(n_out, np.uint8)
    sel[pick] = 1
    ref = he.server_conv(ct, x0, K, r, opl, P, sel=sel)
    assert (got[pick] == ref[pick]).all()
    assert (UP(y0) == packing.extract((P.t - r) % P.t, opl)).all()
    # the same call with the oracle's mask passed in as r gives the same words everywhere
    got_r = D.U(ctx.he_conv2d(plan, D.R(ct), w, x0=TP(x0), r=TP(r)))
    assert (got == got_r).all()


@pytest.mark.parametrize("world", [2, 8])
def test_he_conv2d_gen_rank_slices(env, world):
    """Each rank draws only its own output rows (gen.ct0 = m0 * S): together they equal the
    whole layer's mask, so the reassembled shares are the single-GPU ones."""
    from paper_2506_11586_b200 import dist as sdist

    ctx, P, D = env
    lay = next(l for l in layers.squeezenet11() if l.name == "fire2.e3")
    opl = oplan(P, ctx, lay)
    ct, x0, K, _ = _layer_inputs(P, lay, 62, opl)
    seed, stream = 77, 5
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    outs, shares = [], []
    for m0, mc in sdist.m_slices(plan.M, world):
        pl = plan.copy(M=mc)
        w = ctx.preprocess_weights(pl, TP(np.ascontiguousarray(K[m0:m0 + mc])))
        y0 = torch.empty((mc, plan.OH, plan.OW), dtype=torch.int64, device=DEV)
        g = secn_mod().MaskGen(seed=seed, stream=stream, ct0=m0 * plan.S)
        outs.append(D.U(ctx.he_conv2d_gen(pl, D.R(ct), w, g, x0=TP(x0), y0=y0)))
        shares.append(UP(y0))
    r = philox.mask(seed, stream, opl.M * opl.S, P.n, P.t_bits)
    got = np.concatenate(outs)
    pick = np.array([0, got.shape[0] // 2, got.shape[0] - 1])
    sel = np.zeros(got.shape[0], np.uint8)
    sel[pick] = 1
    ref = he.server_conv(ct, x0, K, r, opl, P, sel=sel)
    assert (got[pick] == ref[pick]).all()
    assert (np.concatenate(shares) == packing.extract((P.t - r) % P.t, opl)).all()


def test_he_conv2d_lwe_gen_equals_lwe_with_drawn_mask(env):
    ctx, P, D = env
    lay = next(l for l in layers.squeezenet11() if l.name == "fire5.e3")
    opl = oplan(P, ctx, lay)
    ct, x0, K, _ = _layer_inputs(P, lay, 63, opl)
    seed, stream = 1234, 99
    r = philox.mask(seed, stream, opl.M * opl.S, P.n, P.t_bits)
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    w = ctx.preprocess_weights(plan, TP(K))
    keep = 1 if ctx.L == 2 else 2
    y0a = torch.empty((plan.M, plan.OH, plan.OW), dtype=torch.int64, device=DEV)
    y0b = torch.empty_like(y0a)
    a1, b1 = ctx.he_conv2d_lwe(plan, D.R(ct), w, keep, x0=TP(x0), r=TP(r), y0=y0a)
    g = secn_mod().MaskGen(seed=seed, stream=stream, ct0=0)
    a2, b2 = ctx.he_conv2d_lwe_gen(plan, D.R(ct), w, keep, g, x0=TP(x0), y0=y0b)
    assert torch.equal(a1, a2) and torch.equal(b1, b2) and torch.equal(y0a, y0b)
    assert (UP(y0b) == packing.extract((P.t - r) % P.t, opl)).all()


@pytest.mark.parametrize("name", ["fire9.e3", "conv1", "fire2.sq"])
@pytest.mark.parametrize("src", ["r", "gen"])
def test_mask_encode_then_he_conv2d_em(env, name, src):
    """secn_mask_encode (from r or the generator) + secn_he_conv2d_em equals secn_he_conv2d_ex with
    that r, word for word, and the encoded words are enc_j(r) (the oracle's encoding); also with a
    spatial slice of the outputs and through the LWE form."""
    ctx, P, D = env
    lay = next(l for l in layers.squeezenet11() if l.name == name)
    opl = oplan(P, ctx, lay)
    ct, x0, K, r = _layer_inputs(P, lay, 64, opl)
    seed, stream = 2024, 3
    g = secn_mod().MaskGen(seed=seed, stream=stream, ct0=0)
    if src == "gen":
        r = philox.mask(seed, stream, opl.M * opl.S, P.n, P.t_bits)
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    w = ctx.preprocess_weights(plan, TP(K))
    y0 = torch.full((plan.M, plan.OH, plan.OW), -1, dtype=torch.int64, device=DEV)
    em = ctx.mask_encode(plan, r=TP(r) if src == "r" else None, gen=g if src == "gen" else None, y0=y0)
    emh = D.U(em)
    for j in range(P.L):
        for row in (0, opl.M * opl.S - 1):
            assert (emh[row, j] == he.enc(r[row], P, j)).all()
    assert (UP(y0) == packing.extract((P.t - r) % P.t, opl)).all()
    got = D.U(ctx.he_conv2d_em(plan, D.R(ct), w, em, x0=TP(x0)))
    ref = D.U(ctx.he_conv2d(plan, D.R(ct), w, x0=TP(x0), r=TP(r)))
    assert (got == ref).all()
    keep = 1 if ctx.L == 2 else 2
    a1, b1 = ctx.he_conv2d_lwe(plan, D.R(ct), w, keep, x0=TP(x0), r=TP(r))
    a2, b2 = ctx.he_conv2d_lwe_em(plan, D.R(ct), w, keep, em, x0=TP(x0))
    assert torch.equal(a1, a2) and torch.equal(b1, b2)
    if plan.S > 1:  # a spatial slice: only its blocks' rows are computed (the rest keep their old words)
        pl = plan.copy(s_begin=1, s_count=plan.S - 1)
        em2 = ctx.mask_encode(pl, r=TP(r))
        out = ctx.empty(plan.M * plan.S, 2, ctx.L, ctx.n)
        out.fill_(-1)
        o = D.U(ctx.he_conv2d_em(pl, D.R(ct), w, em2, x0=TP(x0), out=out))
        rows = [m * plan.S + s for m in range(plan.M) for s in range(1, plan.S)]
        assert (o[rows] == ref[rows]).all()
        other = [m * plan.S for m in range(plan.M)]
        assert (o[other] == np.uint64(2**64 - 1) if ctx.word_bits == 64 else o[other] == 2**32 - 1).all()
