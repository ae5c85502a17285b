"""Runs one layer through secn32_he_conv2d on seeded inputs and saves the output ciphertexts
(for A/B comparisons of kernel variants, e.g. SECN_NO_FUSE=1 vs the fused path).
Usage: python tools/dump_layer.py layer net out.npy [M_override]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

import __graft_entry__
from paper_2506_11586_b200 import Context
from workloads import inputs, layers

name, net, out = sys.argv[1], sys.argv[2], sys.argv[3]
__graft_entry__.build()
ctx = Context(0, word_bits=32)
lay = next(l for l in layers.network(net) if l.name == name)
M = int(sys.argv[4]) if len(sys.argv) > 4 else lay.M
plan = ctx.plan(lay.C, lay.H, lay.W, M, lay.k, stride=lay.stride, pad=lay.pad)
g = inputs.rng(7)
dev = torch.device("cuda:0")
T = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)
ctn = inputs.uniform_residues(g, (plan.G * plan.S, 2), ctx.primes, ctx.n)
ct = torch.from_numpy(ctn.astype(np.uint32).view(np.int32)).to(dev)
x0 = T(inputs.uniform_below(g, (plan.G * plan.S, ctx.n), 1 << ctx.t_bits))
K = T(inputs.quantized_kernel(g, plan.M, lay.C, lay.k, lay.k))
r = T(inputs.uniform_below(g, (plan.M * plan.S, ctx.n), 1 << ctx.t_bits))
w = ctx.preprocess_weights(plan, K)
import os
if os.environ.get('DUMP_SYNC'):
    torch.cuda.synchronize()
if os.environ.get('DUMP_STAGE01'):
    o = ctx.empty(plan.M * plan.S, 2, ctx.L, ctx.n)
    ws = torch.empty(ctx.workspace_bytes(plan) // 8 + 1, dtype=torch.int64, device=dev)
    for st in (0, 1):
        ctx.he_conv2d_stage(st, plan, ct, w, x0, r, o, ws)
else:
    o = ctx.he_conv2d(plan, ct, w, x0=x0, r=r)
torch.cuda.synchronize()
np.save(out, o.cpu().numpy())
print(name, plan)
