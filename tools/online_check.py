"""secn32_he_conv2d_online must equal preprocess + secn32_he_conv2d word for word on every layer of
a network (the f4 toggle only moves the weight NTT into the call). Usage: online_check.py [net]"""
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
ctx = Context(0, word_bits=32)
dev = torch.device("cuda:0")
T = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)  # noqa: E731
bad_layers = 0
for lay in layers.network(sys.argv[1] if len(sys.argv) > 1 else "squeezenet1_1"):
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    g = inputs.rng(5)
    ctn = inputs.uniform_residues(g, (plan.G * plan.S, 2), ctx.primes, ctx.n)
    ct = torch.from_numpy(ctn.astype(np.uint32).view(np.int32)).to(dev)
    x0 = T(inputs.uniform_below(g, (plan.G * plan.S, ctx.n), 1 << ctx.t_bits))
    r = T(inputs.uniform_below(g, (plan.M * plan.S, ctx.n), 1 << ctx.t_bits))
    K = T(inputs.quantized_kernel(g, plan.M, lay.C, lay.k, lay.k))
    w = ctx.preprocess_weights(plan, K)
    a = ctx.he_conv2d(plan, ct, w, x0=x0, r=r).clone()
    ws = torch.empty((ctx.online_workspace_bytes(plan) + 7) // 8, dtype=torch.int64, device=dev)
    b = ctx.he_conv2d_online(plan, ct, K, x0=x0, r=r, workspace=ws)
    torch.cuda.synchronize()
    nb = int((a != b).sum())
    bad_layers += nb > 0
    print(f"{lay.name:10s} decim={plan.decim} G={plan.G} S={plan.S} mismatched words {nb}")
print("layers with mismatches:", bad_layers)

# ---- the same comparison inside a CUDA graph of the whole network with the fire-module side
# streams (the bench's online leg)
from paper_2506_11586_b200.schedule import GroupRunner, concurrent_groups  # noqa: E402

net = layers.network(sys.argv[1] if len(sys.argv) > 1 else "squeezenet1_1")
st = []
for li, lay in enumerate(net):
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    g = inputs.rng(100 + li)
    ctn = inputs.uniform_residues(g, (plan.G * plan.S, 2), ctx.primes, ctx.n)
    d = dict(lay=lay, plan=plan, ct=torch.from_numpy(ctn.astype(np.uint32).view(np.int32)).to(dev),
             x0=T(inputs.uniform_below(g, (plan.G * plan.S, ctx.n), 1 << ctx.t_bits)),
             r=T(inputs.uniform_below(g, (plan.M * plan.S, ctx.n), 1 << ctx.t_bits)),
             K=T(inputs.quantized_kernel(g, plan.M, lay.C, lay.k, lay.k)), out=ctx.empty(plan.M * plan.S, 2, ctx.L, ctx.n),
             ws=torch.empty(ctx.workspace_bytes(plan) // 8 + 1, dtype=torch.int64, device=dev),
             ws_on=torch.empty((ctx.online_workspace_bytes(plan) + 7) // 8, dtype=torch.int64, device=dev))
    d["w"] = ctx.preprocess_weights(plan, d["K"])
    st.append(d)
import os  # noqa: E402

runner = GroupRunner([[i] for i in range(len(st))] if os.environ.get("SERIAL") else
                     concurrent_groups([d["lay"].name for d in st]), dev)
from paper_2506_11586_b200.schedule import StagedGroupRunner  # noqa: E402

STAGED_RUNNER = StagedGroupRunner(concurrent_groups([d["lay"].name for d in st]), dev)
for i in range(len(st)):  # serial reference
    ctx.he_conv2d(st[i]["plan"], st[i]["ct"], st[i]["w"], x0=st[i]["x0"], r=st[i]["r"], out=st[i]["out"],
                  workspace=st[i]["ws"])
torch.cuda.synchronize()
ref = [d["out"].clone() for d in st]


def offline_step():
    if os.environ.get("STAGED"):
        from paper_2506_11586_b200.schedule import StagedGroupRunner

        sr = STAGED_RUNNER
        sr(lambda i: ctx.he_conv2d(st[i]["plan"], st[i]["ct"], st[i]["w"], x0=st[i]["x0"], r=st[i]["r"],
                                   out=st[i]["out"], workspace=st[i]["ws"]),
           lambda i, k: ctx.he_conv2d_stage(k, st[i]["plan"], st[i]["ct"], st[i]["w"], st[i]["x0"], st[i]["r"],
                                            st[i]["out"], st[i]["ws"]))
        return
    runner(lambda i: ctx.he_conv2d(st[i]["plan"], st[i]["ct"], st[i]["w"], x0=st[i]["x0"], r=st[i]["r"],
                                   out=st[i]["out"], workspace=st[i]["ws"]))


def online_step():
    runner(lambda i: ctx.he_conv2d_online(st[i]["plan"], st[i]["ct"], st[i]["K"], x0=st[i]["x0"], r=st[i]["r"],
                                          out=st[i]["out"], workspace=st[i]["ws_on"]))


for mode, step in (("offline-eager", offline_step), ("offline-graph", offline_step)) + (
        () if os.environ.get("STAGED") else (("eager", online_step), ("graph", online_step))):
    for d in st:
        d["out"].zero_()
    if mode.endswith("eager"):
        step()
    else:
        gr = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(dev)
        with torch.cuda.graph(gr, stream=cap):
            step()
        for _ in range(3):
            gr.replay()
    torch.cuda.synchronize()
    bad = [(d["lay"].name, int((d["out"] != r0).sum())) for d, r0 in zip(st, ref)]
    print(mode, "layers with mismatches:", [b for b in bad if b[1]])
    for d, r0 in zip(st, ref):
        diff = (d["out"] != r0).reshape(d["out"].shape[0], 2, ctx.L, ctx.n)
        if diff.any():
            per = diff.any(-1).nonzero().cpu().numpy()
            names = [x["lay"].name for x in st]
            partner = None
            if d["lay"].name.endswith(".e3"):
                partner = names.index(d["lay"].name[:-3] + ".e1")
            elif d["lay"].name.endswith(".e1"):
                partner = names.index(d["lay"].name[:-3] + ".e3")
            if partner is not None and ref[partner].shape == r0.shape:
                ctb = int(per[0, 0])
                got_row = d["out"][ctb].cpu()
                print("   first bad ct", ctb, "equals partner ref row:", bool(torch.equal(got_row, ref[partner][ctb].cpu())),
                      "equals partner current row:", bool(torch.equal(got_row, st[partner]["out"][ctb].cpu())),
                      "zero:", bool((got_row == 0).all()))
            print("  ", d["lay"].name, "bad (ct, comp, limb):", len(per), "comps", np.unique(per[:, 1]).tolist(),
                  "limbs", np.unique(per[:, 2]).tolist(), "cts", np.unique(per[:, 0]).tolist()[:20],
                  "coef-fraction", float(diff.float().mean()))
