"""Per-layer, per-stage device time of the hot path inside CUDA graphs (L2 flushed before each
replay; the graph-launch floor measured with an empty-ish graph is reported separately).
Usage: python tools/layer_times.py [word_bits] [net]"""
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
wb = int(sys.argv[1]) if len(sys.argv) > 1 else 32
net = layers.network(sys.argv[2] if len(sys.argv) > 2 else "squeezenet1_1")
ctx = Context(0, word_bits=wb)
dev = torch.device("cuda:0")
big = torch.empty(300 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)


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


floor = timed(graph_of(lambda: big[:1].add_(1)))
print(f"graph floor (1 tiny kernel): {floor:.1f} us")
R = lambda a: torch.from_numpy(a.view(np.int64) if wb == 64 else a.astype(np.uint32).view(np.int32)).to(dev)  # noqa
P = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)  # noqa
tot = np.zeros(4)
print(f"{'layer':10s} {'fwd':>8s} {'+mac':>8s} {'+inv':>8s} {'+extr':>8s}   (us, cumulative stages, minus floor)")
for li, lay in enumerate(net):
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    g = inputs.rng(li)
    ct = R(inputs.uniform_residues(g, (plan.G * plan.S, 2), ctx.primes, ctx.n))
    x0 = P(inputs.uniform_below(g, (plan.G * plan.S, ctx.n), 1 << 37))
    K = P(inputs.quantized_kernel(g, plan.M, lay.C, lay.k, lay.k))
    r = P(inputs.uniform_below(g, (plan.M * plan.S, ctx.n), 1 << 37))
    w = ctx.preprocess_weights(plan, K)
    out = ctx.empty(plan.M * plan.S, 2, ctx.L, ctx.n)
    ws = torch.empty(ctx.workspace_bytes(plan) // 8, dtype=torch.int64, device=dev)
    y0 = torch.empty((plan.M, plan.OH, plan.OW), dtype=torch.int64, device=dev)
    ts = []
    for upto in range(4):
        def fn(upto=upto):
            for s in range(min(upto + 1, 3)):
                ctx.he_conv2d_stage(s, plan, ct, w, x0, r, out, ws)
            if upto == 3:
                ctx.extract_share(plan, r, out=y0)
        ts.append(timed(graph_of(fn)) - floor)
    tot += np.array(ts)
    print(f"{lay.name:10s} " + " ".join(f"{t:8.1f}" for t in ts))
print(f"{'sum':10s} " + " ".join(f"{t:8.1f}" for t in tot))
