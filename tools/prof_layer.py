"""Runs one layer of the hot path a few times (for ncu captures of single kernels).
Usage: python tools/prof_layer.py [layer_name] [net] [reps] [word_bits] [mode: full|lwe|em]
(em: the bench step's path -- secn_mask_encode from the generator, then secn[32]_he_conv2d_em)"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

import __graft_entry__
from paper_2506_11586_b200 import Context, MaskGen
from workloads import inputs, layers

name = sys.argv[1] if len(sys.argv) > 1 else "conv10"
net = sys.argv[2] if len(sys.argv) > 2 else "squeezenet1_1"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
wb = int(sys.argv[4]) if len(sys.argv) > 4 else 64
mode = sys.argv[5] if len(sys.argv) > 5 else "full"
__graft_entry__.build()
ctx = Context(0, word_bits=wb)
lay = next(l for l in layers.network(net) if l.name == name)
plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
g = inputs.rng(5)
dev = torch.device("cuda:0")
T = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)
ctn = inputs.uniform_residues(g, (plan.G * plan.S, 2), ctx.primes, ctx.n)
ct = T(ctn) if wb == 64 else torch.from_numpy(ctn.astype(np.uint32).view(np.int32)).to(dev)
x0 = T(inputs.uniform_below(g, (plan.G * plan.S, ctx.n), 1 << ctx.t_bits))
K = T(inputs.quantized_kernel(g, plan.M, lay.C, lay.k, lay.k))
r = T(inputs.uniform_below(g, (plan.M * plan.S, ctx.n), 1 << ctx.t_bits))
w = ctx.preprocess_weights(plan, K)
out = ctx.empty(plan.M * plan.S, 2, ctx.L, ctx.n)
ws = torch.empty(ctx.workspace_bytes(plan) // 8, dtype=torch.int64, device=dev)
y0 = torch.empty((plan.M, plan.OH, plan.OW), dtype=torch.int64, device=dev)


em = ctx.empty(plan.M * plan.S, ctx.L, ctx.n)


def call():
    if mode == "em":
        ctx.mask_encode(plan, gen=MaskGen(seed=77, stream=1, ct0=0), out=em, y0=y0)
        ctx.he_conv2d_em(plan, ct, w, em, x0=x0, out=out, workspace=ws)
    elif mode == "lwe":
        ctx.he_conv2d_lwe(plan, ct, w, ctx.L // 2, x0=x0, r=r, y0=y0)
    else:
        ctx.he_conv2d(plan, ct, w, x0=x0, r=r, out=out, workspace=ws, y0=y0)


for _ in range(reps):
    call()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    call()
e1.record()
torch.cuda.synchronize()
print(name, wb, plan, f"{e0.elapsed_time(e1) / reps:.4f} ms/layer")
