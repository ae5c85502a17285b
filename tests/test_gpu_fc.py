"""GPU parity of the HE fully-connected layer: secn_fc_preprocess_weights and
secn_he_fc through the C ABI against oracle/fc.py, word for word, both residue word sizes."""
import numpy as np
import pytest
import torch

from oracle import fc, he
from oracle.params import Params
from workloads import inputs

from test_gpu_parity import DEV, PRIMES, TP, UP, Dev, env, secn  # noqa: F401  (fixtures)

pytestmark = pytest.mark.gpu


def _inputs(P, p, seed, full=False):
    g = inputs.rng(seed)
    ct = inputs.uniform_residues(g, (p.G, 2), P.primes, P.n)
    x0 = inputs.uniform_below(g, (p.G, P.n), P.t)
    Wm = (inputs.uniform_below(g, (p.n_o, p.n_i), P.t) if full
          else inputs.quantized_kernel(g, p.n_o, p.n_i, 1, 1).reshape(p.n_o, p.n_i))
    r = inputs.uniform_below(g, (p.M, P.n), P.t)
    return ct, x0, Wm, r


def _oplan(ctx, p):
    return fc.FcPlan(p.n_i, p.n_o, p.nib, p.nob, p.G, p.M)


@pytest.mark.parametrize("n_i,n_o,full", [(64, 16, False), (300, 50, True), (100, 37, False), (5000, 3, False),
                                          (7, 900, True)])
def test_he_fc_exact(env, n_i, n_o, full):
    ctx, P, D = env
    p = ctx.fc_plan(n_i, n_o)
    op = fc.plan_fc(n_i, n_o, P.n, ctx.coef_words64)
    assert (p.nib, p.nob, p.G, p.M) == (op.nib, op.nob, op.G, op.M)
    ct, x0, Wm, r = _inputs(P, op, 40 + n_i % 17, full)
    w = ctx.fc_preprocess_weights(p, TP(Wm))
    y0 = torch.full((n_o,), -1, dtype=torch.int64, device=DEV)
    got = D.U(ctx.he_fc(p, D.R(ct), w, x0=TP(x0), r=TP(r), y0=y0))
    assert (got == fc.server_fc(ct, x0, Wm, r, op, P)).all()
    assert (UP(y0) == fc.fc_extract((P.t - r) % P.t, op)).all()


def test_fc_preprocess_weights_matches_oracle(env):
    """The inverse NTT of the preprocessed weights equals the centred lift of the packed matrix."""
    ctx, P, D = env
    p = ctx.fc_plan(300, 50)
    op = _oplan(ctx, p)
    g = inputs.rng(41)
    Wm = inputs.uniform_below(g, (50, 300), P.t)
    w = ctx.fc_preprocess_weights(p, TP(Wm))
    back = D.U(ctx.ntt_inv(w.view(p.M * p.G, ctx.L, ctx.n).clone()))
    raw = fc.fc_weight_polys(Wm, op, P.n).reshape(p.M * p.G, P.n)
    for j, q in enumerate(P.primes):
        lifted = np.where(raw >= P.t // 2, (q - (P.t - raw.astype(object)) % q) % q, raw.astype(object) % q)
        assert (back[:, j] == lifted.astype(np.uint64)).all(), j


def test_he_fc_resnet50_full_size_sampled(env):
    """ResNet-50's fc (2048 -> 1000) at full size, sampled output cts against the oracle."""
    ctx, P, D = env
    p = ctx.fc_plan(2048, 1000)
    op = _oplan(ctx, p)
    ct, x0, Wm, r = _inputs(P, op, 42)
    w = ctx.fc_preprocess_weights(p, TP(Wm))
    y0 = torch.empty((1000,), dtype=torch.int64, device=DEV)
    got = D.U(ctx.he_fc(p, D.R(ct), w, x0=TP(x0), r=TP(r), y0=y0))
    pick = np.array(sorted({0, p.M // 2, p.M - 1}))
    sel = np.zeros(p.M, np.uint8)
    sel[pick] = 1
    ref = fc.server_fc(ct, x0, Wm, r, op, P, sel=sel)
    assert (got[pick] == ref[pick]).all()
    assert (UP(y0) == fc.fc_extract((P.t - r) % P.t, op)).all()


def test_he_fc_end_to_end_decrypts_to_matvec(env):
    """Client (oracle harness) encrypts x1; the GPU server adds x0, multiplies, masks and outputs
    y0; decrypt + y0 = W (x0 + x1) mod 2^37."""
    ctx, P, D = env
    n_i, n_o = 512, 1000
    p = ctx.fc_plan(n_i, n_o)
    op = _oplan(ctx, p)
    g = inputs.rng(43)
    x1 = inputs.uniform_below(g, n_i, P.t)
    x0 = inputs.uniform_below(g, n_i, P.t)
    Wm = inputs.quantized_kernel(g, n_o, n_i, 1, 1).reshape(n_o, n_i)
    sk = inputs.ternary(g, P.n)
    xin = fc.pack_fc_input(x1, op, P.n)
    ct = np.stack([he.encrypt(xin[i], sk, inputs.uniform_residues(g, (), P.primes, P.n),
                              inputs.rounded_gaussian(g, P.n), P) for i in range(op.G)])
    r = inputs.uniform_below(g, (op.M, P.n), P.t)
    w = ctx.fc_preprocess_weights(p, TP(Wm))
    y0t = torch.empty((n_o,), dtype=torch.int64, device=DEV)
    out = D.U(ctx.he_fc(p, D.R(ct), w, x0=TP(fc.pack_fc_input(x0, op, P.n)), r=TP(r), y0=y0t))
    y0 = UP(y0t)
    m_idx, coef = fc.fc_designated(op)
    y1 = np.zeros(n_o, np.uint64)
    for m in range(op.M):
        pick = m_idx == m
        y1[pick] = he.decrypt(out[m], sk, P, coef[pick])
    assert (((y0 + y1) & np.uint64(P.t - 1)) == fc.matvec_mod(Wm, (x0 + x1) & np.uint64(P.t - 1), P.t_bits)).all()


def test_he_fc_rejects_inconsistent_plan(env):
    ctx, P, D = env
    from paper_2506_11586_b200 import secn as m

    p = ctx.fc_plan(64, 16)
    p.G += 1
    ct = ctx.empty(p.G, 2, ctx.L, ctx.n)
    w = ctx.empty(p.M, p.G, ctx.L, ctx.n)
    with pytest.raises(m.SecnError):
        ctx.he_fc(p, ct, w)
