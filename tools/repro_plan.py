"""Runs one he_conv2d call with an explicit packing window (debugging aid).
Usage: python tools/repro_plan.py C H W M k stride pad Hw Ww"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

import __graft_entry__
from paper_2506_11586_b200 import Context
from workloads import inputs

__graft_entry__.build()
C, H, W, M, k, st, pad, Hw, Ww = map(int, sys.argv[1:10])
ctx = Context(0, word_bits=32)
dev = torch.device("cuda:0")
T = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)  # noqa: E731
p = ctx.plan(C, H, W, M, k, stride=st, pad=pad, Hw=Hw, Ww=Ww)
print(p, flush=True)
g = inputs.rng(1)
ct = torch.from_numpy(inputs.uniform_residues(g, (p.G * p.S, 2), ctx.primes, ctx.n).astype(np.uint32).view(np.int32)).to(dev)
w = ctx.preprocess_weights(p, T(inputs.quantized_kernel(g, M, C, k, k)))
torch.cuda.synchronize()
print("weights ok", flush=True)
out = ctx.empty(p.M * p.S, 2, ctx.L, ctx.n)
ws = torch.empty(ctx.workspace_bytes(p) // 8 + 1, dtype=torch.int64, device=dev)
for k_ in range(3):
    ctx.he_conv2d_stage(k_, p, ct, w, None, None, out, ws)
    torch.cuda.synchronize()
    print("stage", k_, "ok", flush=True)
