"""One eager step of the bench workload between cudaProfilerStart/Stop, for an ncu capture of every
kernel of the step (run under `ncu --profile-from-start off ...`). Same layers, plans, inputs and
mask schedule as bench.py (SqueezeNet-1.1, 32-bit limbs, device-drawn mask encoded ahead).
Usage: python tools/step_profile.py [net] [word_bits]
Summarise with tools/ncu_step_summary.py."""
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
net = sys.argv[1] if len(sys.argv) > 1 else "squeezenet1_1"
wb = int(sys.argv[2]) if len(sys.argv) > 2 else 32
ctx = Context(0, word_bits=wb)
dev = torch.device("cuda:0")
st = []
for li, lay in enumerate(layers.network(net)):
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    g = inputs.rng(3000 + li)
    ct = inputs.uniform_residues(g, (plan.G * plan.S, 2), ctx.primes, ctx.n)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)  # noqa: E731
    d = {"plan": plan, "name": lay.name,
         "ct": T(ct) if wb == 64 else torch.from_numpy(ct.astype(np.uint32).view(np.int32)).to(dev),
         "x0": T(inputs.uniform_below(g, (plan.G * plan.S, ctx.n), 1 << ctx.t_bits)),
         "gen": MaskGen(seed=77, stream=li, ct0=0)}
    d["w"] = ctx.preprocess_weights(plan, T(inputs.quantized_kernel(g, plan.M, lay.C, lay.k, lay.k)))
    d["em"] = ctx.empty(plan.M * plan.S, ctx.L, ctx.n)
    d["y0"] = torch.empty((plan.M, plan.OH, plan.OW), dtype=torch.int64, device=dev)
    d["out"] = ctx.empty(plan.M * plan.S, 2, ctx.L, ctx.n)
    d["ws"] = torch.empty(ctx.workspace_bytes(plan) // 8 + 1, dtype=torch.int64, device=dev)
    st.append(d)


def step():
    for d in st:
        ctx.mask_encode(d["plan"], gen=d["gen"], out=d["em"], y0=d["y0"])
    for d in st:
        ctx.he_conv2d_em(d["plan"], d["ct"], d["w"], d["em"], x0=d["x0"], out=d["out"], workspace=d["ws"])


for _ in range(3):
    step()
torch.cuda.synchronize()
torch.cuda.profiler.start()
step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("layers:", " ".join(f"{d['name']}:G{d['plan'].G}S{d['plan'].S}M{d['plan'].M}" for d in st))
