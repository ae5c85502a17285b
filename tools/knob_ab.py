"""Per-layer A/B of library variants selected by SECN_* knobs (read at context creation): graph-replayed
secn32_he_conv2d_ex device time (median of 15, L2 flushed before each replay) for each variant, and
a bit-exact comparison of every variant's outputs (ciphertexts and shares) with the first's.
Usage: python tools/knob_ab.py [net] [variants...]
  variant = "base" (no knobs) or "K=V,K2=V2" (e.g. SECN_MAC_WS=1); default: base SECN_MAC_WS=1"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

import __graft_entry__
from paper_2506_11586_b200 import Context
from workloads import inputs, layers

__graft_entry__.build()
net_name = sys.argv[1] if len(sys.argv) > 1 else "squeezenet1_1"
variants = sys.argv[2:] or ["base", "SECN_MAC_WS=1"]
net = layers.network(net_name)
dev = torch.device("cuda:0")
big = torch.empty(300 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)


def ctx_for(v):
    for k in [k for k in os.environ if k.startswith("SECN_")]:
        os.environ.pop(k)
    if v != "base":
        for kv in v.split(","):
            k, val = kv.split("=")
            os.environ[k] = val
    return Context(0, word_bits=32)


def graph_of(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    torch.cuda.synchronize()
    return g


def timed(g, reps=15):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        big.add_(1)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


ctxs = {v: ctx_for(v) for v in variants}
base = ctxs[variants[0]]
print(f"{'layer':14s} " + " ".join(f"{v[-12:]:>12s}" for v in variants) + "   (us; 'same' = outputs bit-equal to the first)")
tot = {v: 0.0 for v in variants}
for li, lay in enumerate(net):
    plan = base.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    g = inputs.rng(100 + li)
    ct = inputs.uniform_residues(g, (plan.G * plan.S, 2), base.primes, base.n)
    x0 = inputs.uniform_below(g, (plan.G * plan.S, base.n), 1 << 37)
    K = inputs.quantized_kernel(g, plan.M, lay.C, lay.k, lay.k)
    r = inputs.uniform_below(g, (plan.M * plan.S, base.n), 1 << 37)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)  # noqa: E731
    ctd = torch.from_numpy(ct.astype(np.uint32).view(np.int32)).to(dev)
    x0d, rd, Kd = T(x0), T(r), T(K)
    w = base.preprocess_weights(plan, Kd)
    ref = None
    row = []
    for v in variants:
        c = ctxs[v]
        out = c.empty(plan.M * plan.S, 2, c.L, c.n)
        y0 = torch.empty((plan.M, plan.OH, plan.OW), dtype=torch.int64, device=dev)
        ws = torch.empty(c.workspace_bytes(plan) // 8 + 1, dtype=torch.int64, device=dev)
        fn = lambda: c.he_conv2d(plan, ctd, w, x0=x0d, r=rd, out=out, workspace=ws, y0=y0)  # noqa: E731
        gr = graph_of(fn)
        t = timed(gr)
        tot[v] += t
        same = ""
        if ref is None:
            ref = (out.clone(), y0.clone())
        else:
            same = "same" if torch.equal(out, ref[0]) and torch.equal(y0, ref[1]) else "DIFF"
        row.append(f"{t:12.1f}{same and ' ' + same}")
        del gr
    print(f"{lay.name:14s} G={plan.G:<2d} S={plan.S:<2d} M={plan.M:<4d} " + " ".join(row), flush=True)
print(f"{'sum':14s} " + " ".join(f"{tot[v]:12.1f}" for v in variants))
