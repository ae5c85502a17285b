"""Times every layer of a network through secn32_he_conv2d under several packing plans (Hw, Ww):
the library's default, and the best few by a simple time model (output / MAC / input limb-polys
and bytes). Usage: python tools/plan_sweep.py [net] [n_candidates]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

import __graft_entry__
from oracle import packing
from paper_2506_11586_b200 import Context
from workloads import inputs, layers

__graft_entry__.build()
net = sys.argv[1] if len(sys.argv) > 1 else "squeezenet1_1"
ncand = int(sys.argv[2]) if len(sys.argv) > 2 else 4
ctx = Context(0, word_bits=32)
dev = torch.device("cuda:0")
L, n = ctx.L, ctx.n
T = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)


def candidates(lay):
    C, H, W, M, k, st, pad = lay.C, lay.H, lay.W, lay.M, lay.k, lay.stride, lay.pad
    out = {}
    for poly in ([False, True] if st > 1 and k > 1 else [False]):
        OH, OW, decim, Hp, Wp, Ph, Pw = packing._geometry(C, H, W, k, k, st, pad, poly)
        ps = st if poly else 1
        Ce, ke = C * ps * ps, -(-k // ps)
        for a in range(ke, Hp + 1):
            for b in range(ke, Wp + 1):
                if a * b > n:
                    continue
                Cw = min(Ce, n // (a * b))
                G = -(-Ce // Cw)
                if G > 32:
                    continue
                S = (-(-Ph // (a - ke + 1))) * (-(-Pw // (b - ke + 1)))
                byt = 16 * n * (2 * G * S + M * G + 2 * M * S) + 8 * n * M * S
                t = 13e-3 * (2 * L * M * S) + 1.3e-3 * (2 * L * M * S * G) + 6e-3 * (2 * L * G * S) + byt / 6450e3 * 0.3
                key = (G, S, poly)  # plans with the same (G, S) cost the same: keep the largest window
                if key not in out or (a * b) > out[key][1] * out[key][2]:
                    out[key] = (t, a, b, poly)
    return sorted(out.values())[:ncand]


def time_plan(plan, lay, g):
    ctn = inputs.uniform_residues(g, (plan.G * plan.S, 2), ctx.primes, n)
    ct = torch.from_numpy(ctn.astype(np.uint32).view(np.int32)).to(dev)
    x0 = T(inputs.uniform_below(g, (plan.G * plan.S, n), 1 << ctx.t_bits))
    K = T(inputs.quantized_kernel(g, plan.M, lay.C, lay.k, lay.k))
    r = T(inputs.uniform_below(g, (plan.M * plan.S, n), 1 << ctx.t_bits))
    w = ctx.preprocess_weights(plan, K)
    out = ctx.empty(plan.M * plan.S, 2, L, n)
    ws = torch.empty(ctx.workspace_bytes(plan) // 8 + 1, dtype=torch.int64, device=dev)
    y0 = torch.empty((plan.M, plan.OH, plan.OW), dtype=torch.int64, device=dev)
    f = lambda: ctx.he_conv2d(plan, ct, w, x0=x0, r=r, out=out, workspace=ws, y0=y0)  # noqa: E731
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream(dev)
    with torch.cuda.graph(gr, stream=s):
        for _ in range(5):
            f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gr.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(4):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 20 * 1e3


def _poly_plan(lay, a, b):
    import ctypes

    from paper_2506_11586_b200 import secn as m

    p = m.Plan(C=lay.C, H=lay.H, W=lay.W, M=lay.M, kh=lay.k, kw=lay.k, stride=lay.stride, pad=lay.pad, Hw=a, Ww=b,
               decim=2)
    m._check(m.lib().secn_conv_plan_ex(ctx.log_n, ctx.coef_words64, 1, ctypes.byref(p)))
    return p


import os  # noqa: E402

FROM = os.environ.get("PLAN_SWEEP_FROM")  # start at this layer (debugging)
VERBOSE = bool(os.environ.get("PLAN_SWEEP_VERBOSE"))
tot_def = tot_best = 0.0
started = FROM is None
for lay in layers.network(net):
    started = started or lay.name == FROM
    if not started:
        continue
    g = inputs.rng(9)
    pdef = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    tdef = time_plan(pdef, lay, g)
    res = [(tdef, pdef.Hw, pdef.Ww, pdef.G, pdef.S, f"default d{pdef.decim}")]
    for tm, a, b, poly in candidates(lay):
        if (a, b, poly) == (pdef.Hw, pdef.Ww, pdef.decim == 2):
            continue
        p = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad, Hw=a, Ww=b)
        if poly:
            from paper_2506_11586_b200.secn import Plan, conv_plan  # noqa: F401
            p = p.copy(decim=2)
            p = conv_plan(lay.C, lay.H, lay.W, lay.M, lay.k, lay.k, lay.stride, lay.pad, ctx.log_n, ctx.coef_words64,
                          a, b) if False else _poly_plan(lay, a, b)
        if VERBOSE:
            print("   timing", lay.name, p, flush=True)
        res.append((time_plan(p, lay, g), a, b, p.G, p.S, f"model {tm:.1f}{' poly' if poly else ''}"))
    best = min(res)
    tot_def += tdef
    tot_best += best[0]
    print(f"{lay.name:10s} " + "  ".join(f"[{tag} Hw={a} Ww={b} G={G} S={S}: {t:6.1f}us]" for t, a, b, G, S, tag in res),
          flush=True)
print(f"total default {tot_def:.1f} us, best-of-candidates {tot_best:.1f} us")
