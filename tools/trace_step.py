"""Kernel timeline of one replay of the bench step (CUDA graph of all layers, as bench.py builds it),
recorded with torch.profiler (CUPTI): per kernel its start, duration and the idle gap before it.
Usage: python tools/trace_step.py [net] [word_bits] > timeline.txt"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

import __graft_entry__
from paper_2506_11586_b200 import Context
from paper_2506_11586_b200.schedule import GroupRunner, StagedGroupRunner, concurrent_groups
from workloads import inputs, layers

__graft_entry__.build()
net = sys.argv[1] if len(sys.argv) > 1 else "squeezenet1_1"
wb = int(sys.argv[2]) if len(sys.argv) > 2 else 32
ctx = Context(0, word_bits=wb)
dev = torch.device("cuda:0")
T = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)
st = []
for li, lay in enumerate(layers.network(net)):
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    g = inputs.rng(1000 + li)
    ctn = inputs.uniform_residues(g, (plan.G * plan.S, 2), ctx.primes, ctx.n)
    ct = torch.from_numpy(ctn.astype(np.uint32).view(np.int32) if wb == 32 else ctn.view(np.int64)).to(dev)
    d = dict(lay=lay, plan=plan, ct=ct,
             x0=T(inputs.uniform_below(g, (plan.G * plan.S, ctx.n), 1 << ctx.t_bits)),
             r=T(inputs.uniform_below(g, (plan.M * plan.S, ctx.n), 1 << ctx.t_bits)),
             out=ctx.empty(plan.M * plan.S, 2, ctx.L, ctx.n),
             ws=torch.empty(ctx.workspace_bytes(plan) // 8 + 1, dtype=torch.int64, device=dev),
             y0=torch.empty((plan.M, plan.OH, plan.OW), dtype=torch.int64, device=dev))
    d["w"] = ctx.preprocess_weights(plan, T(inputs.quantized_kernel(g, plan.M, lay.C, lay.k, lay.k)))
    st.append(d)
import os  # noqa: E402

# the bench's schedule (OVERLAP=free, the default | staged | none), as bench.py --overlap
OVERLAP = os.environ.get("OVERLAP", "free")
names = [d["lay"].name for d in st]
groups = concurrent_groups(names) if OVERLAP != "none" else [[i] for i in range(len(st))]
runner = StagedGroupRunner(groups, dev) if OVERLAP == "staged" else GroupRunner(groups, dev)


def call(i):
    d = st[i]
    ctx.he_conv2d(d["plan"], d["ct"], d["w"], x0=d["x0"], r=d["r"], out=d["out"], workspace=d["ws"], y0=d["y0"])


def stage(i, k):
    d = st[i]
    ctx.he_conv2d_stage_ex(k, d["plan"], d["ct"], d["w"], d["x0"], d["r"], d["out"], d["y0"], d["ws"])


def step():
    if OVERLAP == "staged":
        runner(call, stage)
    else:
        runner(call)


for _ in range(3):
    step()
torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()
cap = torch.cuda.Stream(dev)
with torch.cuda.graph(graph, stream=cap):
    step()
for _ in range(5):
    graph.replay()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and "k_" in e.name]
ev.sort(key=lambda e: e.time_range.start)
per_step = len(ev) // 3
last = ev[-per_step:]
t0 = last[0].time_range.start
prev_end = t0
tot = {}
print(f"{'start_us':>9} {'dur_us':>8} {'gap_us':>7}  kernel")
for e in last:
    s, en = e.time_range.start, e.time_range.end
    name = e.name.split("(")[0].replace("void secn::", "")
    print(f"{s - t0:9.1f} {en - s:8.1f} {s - prev_end:7.1f}  {name[:60]}")
    prev_end = max(prev_end, en)
    k = name.split("<")[0]
    tot[k] = tot.get(k, 0.0) + (en - s)
print("step span (us):", round(prev_end - t0, 1), " kernels:", per_step)
print("sum of durations by kernel (us):", {k: round(v, 1) for k, v in tot.items()})
