"""Stress check of the bench's schedule: the SqueezeNet-1.1 step captured as one CUDA graph
(OVERLAP=staged | none | free, as bench.py --overlap) is replayed REPS times, and after every
replay each layer's ciphertexts and shares are compared with the same layers run one call at a
time. MASK=device runs the bench's default schedule instead: every layer's mask drawn and encoded
at the start on a low-priority side stream (secn_mask_encode), each layer through
secn32_he_conv2d_em on high-priority streams after its mask's event.
Usage: OVERLAP=staged REPS=50 [MASK=device] python tools/staged_stress.py"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

import __graft_entry__
from paper_2506_11586_b200 import Context, MaskGen
from paper_2506_11586_b200.schedule import GroupRunner, StagedGroupRunner, concurrent_groups
from workloads import inputs, layers

__graft_entry__.build()
OVERLAP = os.environ.get("OVERLAP", "free")
REPS = int(os.environ.get("REPS", "50"))
MASK = os.environ.get("MASK", "host")
ctx = Context(0, word_bits=32)
dev = torch.device("cuda:0")
T = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)  # noqa: E731
st = []
for li, lay in enumerate(layers.squeezenet11()):
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    g = inputs.rng(700 + li)
    ct = torch.from_numpy(inputs.uniform_residues(g, (plan.G * plan.S, 2), ctx.primes, ctx.n)
                          .astype(np.uint32).view(np.int32)).to(dev)
    d = dict(plan=plan, ct=ct, x0=T(inputs.uniform_below(g, (plan.G * plan.S, ctx.n), 1 << ctx.t_bits)),
             r=T(inputs.uniform_below(g, (plan.M * plan.S, ctx.n), 1 << ctx.t_bits)),
             out=ctx.empty(plan.M * plan.S, 2, ctx.L, ctx.n),
             ws=torch.empty(ctx.workspace_bytes(plan) // 8 + 1, dtype=torch.int64, device=dev),
             y0=torch.empty((plan.M, plan.OH, plan.OW), dtype=torch.int64, device=dev))
    d["w"] = ctx.preprocess_weights(plan, T(inputs.quantized_kernel(g, plan.M, lay.C, lay.k, lay.k)))
    d["gen"] = MaskGen(seed=99, stream=li, ct0=0)
    d["em"] = ctx.empty(plan.M * plan.S, ctx.L, ctx.n)
    st.append(d)
mstream = torch.cuda.Stream(dev)
mev = [torch.cuda.Event() for _ in st]


def call(i):
    d = st[i]
    if MASK == "device":
        torch.cuda.current_stream().wait_event(mev[i])
        ctx.he_conv2d_em(d["plan"], d["ct"], d["w"], d["em"], x0=d["x0"], out=d["out"], workspace=d["ws"])
    else:
        ctx.he_conv2d(d["plan"], d["ct"], d["w"], x0=d["x0"], r=d["r"], out=d["out"], workspace=d["ws"], y0=d["y0"])


def masks_ahead():
    mstream.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(mstream):
        for i, d in enumerate(st):
            ctx.mask_encode(d["plan"], gen=d["gen"], out=d["em"], y0=d["y0"])
            mev[i].record(mstream)


def stage(i, k):
    d = st[i]
    ctx.he_conv2d_stage_ex(k, d["plan"], d["ct"], d["w"], d["x0"], d["r"], d["out"], d["y0"], d["ws"])


ref = []
if MASK == "device":
    masks_ahead()
    torch.cuda.current_stream().wait_stream(mstream)
for i in range(len(st)):
    call(i)
    torch.cuda.synchronize()
    ref.append((st[i]["out"].clone(), st[i]["y0"].clone()))
names = [lay.name for lay in layers.squeezenet11()]
groups = concurrent_groups(names) if OVERLAP != "none" else [[i] for i in range(len(st))]
hi = -1 if MASK == "device" else 0  # the bench's priorities: chain high, mask side stream default
runner = StagedGroupRunner(groups, dev) if OVERLAP == "staged" else GroupRunner(groups, dev, priority=hi)
graph = torch.cuda.CUDAGraph()
cap = torch.cuda.Stream(dev, priority=hi)
with torch.cuda.graph(graph, stream=cap):
    if MASK == "device":
        masks_ahead()
    if OVERLAP == "staged":
        runner(call, stage)
    else:
        runner(call)
    if MASK == "device":
        torch.cuda.current_stream().wait_stream(mstream)
bad_reps = 0
for rep in range(REPS):
    for d in st:
        d["out"].zero_()
        d["y0"].zero_()
    graph.replay()
    torch.cuda.synchronize()
    bad = [(names[i], int((d["out"] != o).sum()) + int((d["y0"] != y).sum()))
           for i, (d, (o, y)) in enumerate(zip(st, ref)) if not (torch.equal(d["out"], o) and torch.equal(d["y0"], y))]
    if bad:
        bad_reps += 1
        print(f"replay {rep}: {bad}", flush=True)
print(f"OVERLAP={OVERLAP} MASK={MASK}: {bad_reps} of {REPS} replays with wrong words")
