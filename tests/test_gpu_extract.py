"""GPU parity of the extracted outputs (reading R16): secn_he_conv2d_lwe and
secn_he_fc_lwe (INTT tail + mask + modulus switch + coefficient extraction, fused) against
oracle/extract.py word for word, and an end-to-end LWE decryption of the GPU outputs."""
import numpy as np
import pytest
import torch

from oracle import conv, extract, fc, he, packing
from workloads import inputs, layers

from test_gpu_parity import DEV, TP, UP, Dev, _layer_inputs, env, oplan, secn  # noqa: F401  (fixtures)

pytestmark = pytest.mark.gpu
L_ = layers.ConvLayer


def _keeps(P):
    return [1] if P.L == 2 else [2, 3]


@pytest.mark.parametrize("lay", [layers.tiny()[0], L_("s2", 3, 40, 40, 5, 3, 2, 0), L_("ds", 24, 28, 28, 9, 1, 2, 0),
                                 L_("multi_s", 2, 70, 70, 3, 3, 1, 0)], ids=lambda l: l.name)
def test_he_conv2d_lwe_matches_oracle(env, lay):
    ctx, P, D = env
    opl = oplan(P, ctx, lay)
    ct, x0, K, r = _layer_inputs(P, lay, 61, opl)
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    w = ctx.preprocess_weights(plan, TP(K))
    full = he.server_conv(ct, x0, K, r, opl, P)
    s_idx, coef = packing.designated_map(opl)
    for keep in _keeps(P):
        y0 = torch.full((plan.M, plan.OH, plan.OW), -1, dtype=torch.int64, device=DEV)
        a, b = ctx.he_conv2d_lwe(plan, D.R(ct), w, keep, x0=TP(x0), r=TP(r), y0=y0)
        ra, rb = extract.server_lwe_outputs(full, keep, P, s_idx, coef, opl.M, opl.S)
        assert (D.U(a) == ra).all(), keep
        assert (D.U(b) == rb).all(), keep
        assert (UP(y0) == packing.extract((P.t - r) % P.t, opl)).all()
        # caller-owned output buffers (the bench's extracted-output e2e leg): same words
        oa, ob = torch.full_like(a, -1), torch.full_like(b, -1)
        a2, b2 = ctx.he_conv2d_lwe(plan, D.R(ct), w, keep, x0=TP(x0), r=TP(r), y0=y0, out=(oa, ob))
        assert a2.data_ptr() == oa.data_ptr() and b2.data_ptr() == ob.data_ptr()
        assert (D.U(oa) == ra).all() and (D.U(ob) == rb).all(), keep


def test_he_conv2d_lwe_end_to_end_decrypt(env):
    """Client encrypts x1; the GPU server returns switched, extracted outputs and y0; LWE
    decryption + y0 = conv(x0 + x1, K) mod 2^37."""
    ctx, P, D = env
    lay = L_("e2e", 6, 20, 20, 4, 3, 2, 1)
    opl = oplan(P, ctx, lay)
    g = inputs.rng(62)
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
    keep = _keeps(P)[0]
    y0t = torch.empty((plan.M, plan.OH, plan.OW), dtype=torch.int64, device=DEV)
    a, b = ctx.he_conv2d_lwe(plan, D.R(ct), w, keep, x0=TP(packing.pack_input(x0, opl, P.n)), r=TP(r), y0=y0t)
    a, b, y0 = D.U(a), D.U(b), UP(y0t)
    Ps = extract.switched_params(P, keep)
    s_idx, coef = packing.designated_map(opl)
    y1 = np.zeros_like(y0)
    for m in range(opl.M):
        for s in range(opl.S):
            sel = s_idx == s
            if sel.any():
                y1[m][sel] = extract.decrypt_lwe(a[m * opl.S + s], b[m][sel], coef[sel], sk, Ps)
    y = (y0 + y1) & np.uint64(P.t - 1)
    assert (y == conv.conv2d_mod((x0 + x1) & np.uint64(P.t - 1), K, lay.stride, lay.pad, P.t_bits)).all()


def test_he_fc_lwe_matches_oracle(env):
    ctx, P, D = env
    p = ctx.fc_plan(300, 50)
    op = fc.FcPlan(p.n_i, p.n_o, p.nib, p.nob, p.G, p.M)
    g = inputs.rng(63)
    ct = inputs.uniform_residues(g, (p.G, 2), P.primes, P.n)
    x0 = inputs.uniform_below(g, (p.G, P.n), P.t)
    Wm = inputs.uniform_below(g, (50, 300), P.t)
    r = inputs.uniform_below(g, (p.M, P.n), P.t)
    w = ctx.fc_preprocess_weights(p, TP(Wm))
    full = fc.server_fc(ct, x0, Wm, r, op, P)
    m_idx, coef = fc.fc_designated(op)
    for keep in _keeps(P):
        y0 = torch.empty((50,), dtype=torch.int64, device=DEV)
        a, b = ctx.he_fc_lwe(p, D.R(ct), w, keep, x0=TP(x0), r=TP(r), y0=y0)
        ms = extract.modswitch(full, keep, P)
        assert (D.U(a) == ms[:, 0]).all()
        assert (D.U(b) == np.stack([ms[m_idx, 1, i, coef] for i in range(keep)], axis=-1)).all()
        assert (UP(y0) == fc.fc_extract((P.t - r) % P.t, op)).all()


def test_lwe_rejects_bad_keep(env):
    ctx, P, D = env
    from paper_2506_11586_b200 import secn as m

    lay = layers.tiny()[0]
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    ct = ctx.empty(plan.G * plan.S, 2, ctx.L, ctx.n)
    w = ctx.empty(plan.M, plan.G, ctx.L, ctx.n)
    for keep in (0, ctx.L):
        with pytest.raises(m.SecnError):
            ctx.he_conv2d_lwe(plan, ct, w, keep)


@pytest.mark.parametrize("lay", __import__("test_gpu_parity")._fuzz_layers(8, seed=77), ids=lambda l: l.name)
def test_he_conv2d_lwe_random_shapes(env, lay):
    """The extracted outputs (modulus switch + designated coefficients) on seeded random layer
    geometries, every keep, against the oracle word for word."""
    ctx, P, D = env
    opl = oplan(P, ctx, lay)
    ct, x0, K, r = _layer_inputs(P, lay, 63, opl)
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    w = ctx.preprocess_weights(plan, TP(K))
    full = he.server_conv(ct, x0, K, r, opl, P)
    s_idx, coef = packing.designated_map(opl)
    for keep in _keeps(P):
        a, b = ctx.he_conv2d_lwe(plan, D.R(ct), w, keep, x0=TP(x0), r=TP(r))
        ra, rb = extract.server_lwe_outputs(full, keep, P, s_idx, coef, opl.M, opl.S)
        assert (D.U(a) == ra).all(), keep
        assert (D.U(b) == rb).all(), keep
