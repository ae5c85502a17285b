"""Times every layer of a network through secn32_he_conv2d under several settings of the libsecn
tuning environment variables (read at every launch), in one process.
Usage: python tools/variant_sweep.py net 'A=1,B=2' 'A=2' ..."""
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
net = sys.argv[1]
variants = [dict(kv.split("=") for kv in v.split(",") if kv) for v in sys.argv[2:]] or [{}]
ctx = Context(0, word_bits=32)
dev = torch.device("cuda:0")
T = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)
g = inputs.rng(5)
rows = []
for lay in layers.network(net):
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    ctn = inputs.uniform_residues(g, (plan.G * plan.S, 2), ctx.primes, ctx.n)
    ct = torch.from_numpy(ctn.astype(np.uint32).view(np.int32)).to(dev)
    x0 = T(inputs.uniform_below(g, (plan.G * plan.S, ctx.n), 1 << ctx.t_bits))
    K = T(inputs.quantized_kernel(g, plan.M, lay.C, lay.k, lay.k))
    r = T(inputs.uniform_below(g, (plan.M * plan.S, ctx.n), 1 << ctx.t_bits))
    w = ctx.preprocess_weights(plan, K)
    out = ctx.empty(plan.M * plan.S, 2, ctx.L, ctx.n)
    ws = torch.empty(ctx.workspace_bytes(plan) // 8 + 1, dtype=torch.int64, device=dev)
    times = []
    ref = None
    for v in variants:
        for k in [k for k in os.environ if k.startswith("SECN_")]:
            os.environ.pop(k, None)
        os.environ.update(v)
        for _ in range(3):
            ctx.he_conv2d(plan, ct, w, x0=x0, r=r, out=out, workspace=ws)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            ctx.he_conv2d(plan, ct, w, x0=x0, r=r, out=out, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 10 * 1e3)
        if os.environ.get("SWEEP_STAGES"):  # per-stage device time (stage calls back to back)
            for st in (0, 1, 2):
                e0.record()
                for _ in range(10):
                    ctx.he_conv2d_stage(st, plan, ct, w, x0, r, out, ws)
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1) / 10 * 1e3)
        got = out.cpu()
        if ref is None:
            ref = got
        elif not torch.equal(ref, got):
            times[-1] = float("nan")  # a variant that changes the result is a bug
    rows.append((lay.name, times))
    print(f"{lay.name:10s} " + " ".join(f"{t:8.1f}" for t in times), flush=True)
tot = np.nansum(np.array([t for _, t in rows]), axis=0)
print("total_us   " + " ".join(f"{t:8.1f}" for t in tot))
print("variants:", sys.argv[2:])
