"""Out-of-bounds write check (compute-sanitizer is closed on this GPU pool): every layer's outputs,
workspace, encoded mask and share live inside larger buffers with canary guards; one network step
(all layers, serial) through secn32_he_conv2d (caller mask) and through secn_mask_encode +
secn32_he_conv2d_em (drawn mask, the bench path), and the plain NTT / INTT calls on odd batches
(the TMA-staged engine), must leave every guard intact."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

import __graft_entry__
from paper_2506_11586_b200 import Context, MaskGen
from workloads import inputs, layers

__graft_entry__.build()
ctx = Context(0, word_bits=32)
dev = torch.device("cuda:0")
T = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)  # noqa: E731
GUARD = 1 << 16  # int32 words per guard
CANARY = 0x5A5A5A5A


def guarded(n_words):
    buf = torch.full((n_words + 2 * GUARD,), CANARY, dtype=torch.int32, device=dev)
    return buf, buf[GUARD:GUARD + n_words]


bad = []
for lay in layers.network(sys.argv[1] if len(sys.argv) > 1 else "squeezenet1_1"):
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    g = inputs.rng(7)
    ctn = inputs.uniform_residues(g, (plan.G * plan.S, 2), ctx.primes, ctx.n)
    ct = torch.from_numpy(ctn.astype(np.uint32).view(np.int32)).to(dev)
    x0 = T(inputs.uniform_below(g, (plan.G * plan.S, ctx.n), 1 << ctx.t_bits))
    r = T(inputs.uniform_below(g, (plan.M * plan.S, ctx.n), 1 << ctx.t_bits))
    K = T(inputs.quantized_kernel(g, plan.M, lay.C, lay.k, lay.k))
    w = ctx.preprocess_weights(plan, K)
    n_out = plan.M * plan.S * 2 * ctx.L * ctx.n
    ob, out = guarded(n_out)
    wsw = ctx.workspace_bytes(plan) // 4
    wb, ws = guarded(wsw)
    y0b = torch.full((plan.M * plan.OH * plan.OW + 2 * GUARD,), CANARY, dtype=torch.int64, device=dev)
    y0 = y0b[GUARD:GUARD + plan.M * plan.OH * plan.OW].view(plan.M, plan.OH, plan.OW)
    ctx.he_conv2d(plan, ct, w, x0=x0, r=r, out=out.view(plan.M * plan.S, 2, ctx.L, ctx.n), workspace=ws.view(torch.int64),
                  y0=y0)
    torch.cuda.synchronize()
    for name, b, n in (("out", ob, n_out), ("ws", wb, wsw)):
        lo = int((b[:GUARD] != CANARY).sum())
        hi = int((b[GUARD + n:] != CANARY).sum())
        if lo or hi:
            bad.append((lay.name, name, lo, hi))
    lo = int((y0b[:GUARD] != CANARY).sum()); hi = int((y0b[GUARD + plan.M * plan.OH * plan.OW:] != CANARY).sum())
    if lo or hi:
        bad.append((lay.name, "y0", lo, hi))
    # the bench path: drawn mask encoded into a guarded buffer, then the _em call
    n_em = plan.M * plan.S * ctx.L * ctx.n
    eb, em = guarded(n_em)
    ob.fill_(CANARY)
    wb.fill_(CANARY)
    y0b.fill_(CANARY)
    ctx.mask_encode(plan, gen=MaskGen(seed=5, stream=1, ct0=0), out=em.view(plan.M * plan.S, ctx.L, ctx.n), y0=y0)
    ctx.he_conv2d_em(plan, ct, w, em.view(plan.M * plan.S, ctx.L, ctx.n), x0=x0,
                     out=out.view(plan.M * plan.S, 2, ctx.L, ctx.n), workspace=ws.view(torch.int64))
    torch.cuda.synchronize()
    for name, b, n in (("out_em", ob, n_out), ("ws_em", wb, wsw), ("em", eb, n_em)):
        lo = int((b[:GUARD] != CANARY).sum())
        hi = int((b[GUARD + n:] != CANARY).sum())
        if lo or hi:
            bad.append((lay.name, name, lo, hi))
    lo = int((y0b[:GUARD] != CANARY).sum()); hi = int((y0b[GUARD + plan.M * plan.OH * plan.OW:] != CANARY).sum())
    if lo or hi:
        bad.append((lay.name, "y0_em", lo, hi))
    print(lay.name, "ok" if not bad or bad[-1][0] != lay.name else bad[-1], flush=True)
for n_polys in (1, 7, 301, 1777):  # plain NTT / INTT calls (odd batches take the TMA-staged engine)
    nb, polys = guarded(n_polys * ctx.L * ctx.n)
    polys.random_(0, min(ctx.primes))
    ctx.ntt_fwd(polys.view(n_polys, ctx.L, ctx.n))
    ctx.ntt_inv(polys.view(n_polys, ctx.L, ctx.n))
    torch.cuda.synchronize()
    lo = int((nb[:GUARD] != CANARY).sum()); hi = int((nb[GUARD + n_polys * ctx.L * ctx.n:] != CANARY).sum())
    if lo or hi:
        bad.append(("ntt", n_polys, lo, hi))
    print("ntt", n_polys, "ok" if not (lo or hi) else (lo, hi), flush=True)
print("guard violations:", bad)
