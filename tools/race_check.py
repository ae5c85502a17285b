"""Concurrency check of the fire-module side streams: e1 and e3 run stage by stage (forward NTT,
MAC, tail) on two streams and every intermediate is compared with a serial run."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

import __graft_entry__
from paper_2506_11586_b200 import Context
from paper_2506_11586_b200.schedule import GroupRunner
from workloads import inputs, layers

__graft_entry__.build()
ctx = Context(0, word_bits=32)
dev = torch.device("cuda:0")
T = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)  # noqa: E731
fire = sys.argv[1] if len(sys.argv) > 1 else "fire3"
MODE = sys.argv[2] if len(sys.argv) > 2 else ""
net = layers.network("squeezenet1_1")
st = []
for li, lay in enumerate([l for l in net if l.name in (fire + ".e1", fire + ".e3", fire + ".sq")]):
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    g = inputs.rng(200 + li)
    ctn = inputs.uniform_residues(g, (plan.G * plan.S, 2), ctx.primes, ctx.n)
    d = dict(lay=lay, plan=plan, ct=torch.from_numpy(ctn.astype(np.uint32).view(np.int32)).to(dev),
             x0=T(inputs.uniform_below(g, (plan.G * plan.S, ctx.n), 1 << ctx.t_bits)),
             r=T(inputs.uniform_below(g, (plan.M * plan.S, ctx.n), 1 << ctx.t_bits)),
             K=T(inputs.quantized_kernel(g, plan.M, lay.C, lay.k, lay.k)), out=ctx.empty(plan.M * plan.S, 2, ctx.L, ctx.n),
             ws=torch.zeros(ctx.workspace_bytes(plan) // 8 + 1, dtype=torch.int64, device=dev))
    d["w"] = ctx.preprocess_weights(d["plan"], d["K"])
    st.append(d)
W0 = [d["w"].clone() for d in st]
BIG_A = torch.ones(1 << 28, dtype=torch.int32, device=dev)
BIG_B = torch.empty_like(BIG_A)
runner = GroupRunner([[0], [1, 2]], dev)  # sq, then e1 | e3
NL = 3


def stage(sts):
    def f(i):
        d = st[i]
        for s_ in sts:
            ctx.he_conv2d_stage(s_, d["plan"], d["ct"], d["w"], d["x0"], d["r"], d["out"], d["ws"])
    return f


# serial reference per stage
refs = {}
for i in range(NL):
    for s_ in (0, 1, 2):
        stage([s_])(i)
        torch.cuda.synchronize()
        refs[(i, s_)] = (st[i]["ws"].clone(), st[i]["out"].clone())
def full(i):
    d = st[i]
    ctx.he_conv2d(d["plan"], d["ct"], d["w"], x0=d["x0"], r=d["r"], out=d["out"], workspace=d["ws"])


def full_mode(i):
    # fork_empty: e3's branch does nothing; fork_copy: e3's branch only copies 1 GiB
    if MODE == "fork_empty" and i == 2:
        return
    if MODE == "fork_copy" and i == 2:
        BIG_B.copy_(BIG_A)
        return
    full(i)


for trial in range(5):
    for d in st:
        d["out"].zero_()
    if trial % 2:
        gr = torch.cuda.CUDAGraph(keep_graph=(trial == 1))
        if trial == 1:
            gr.enable_debug_mode()
        cap = torch.cuda.Stream(dev)
        with torch.cuda.graph(gr, stream=cap):
            runner(full_mode)
        if trial == 1:
            gr.debug_dump("gpurun_out/race_full_graph.dot")
        for d in st:
            d["out"].zero_()
        gr.replay()
    else:
        runner(full_mode)
    torch.cuda.synchronize()
    if trial % 2 and MODE == "classify":
        # classify each wrong (ct, limb) unit of e1 / e3: which known array does it equal?
        L4 = ctx.L
        for i in (1, 2):
            got = st[i]["out"].view(-1, 2, L4, ctx.n).cpu()
            fin = refs[(i, 2)][1].view(-1, 2, L4, ctx.n).cpu()
            mac = refs[(i, 1)][1].view(-1, 2, L4, ctx.n).cpu()
            other = refs[(3 - i, 2)][1].view(-1, 2, L4, ctx.n).cpu()
            for ct_ in range(got.shape[0]):
                for jl in range(L4):
                    g_ = got[ct_, :, jl]
                    if torch.equal(g_, fin[ct_, :, jl]):
                        continue
                    tags = []
                    if torch.equal(g_, mac[ct_, :, jl]): tags.append("=MAC output (Y^ after levels 0-7)")
                    if bool((g_[0] == 0).all()): tags.append("a=0")
                    if ct_ < other.shape[0] and torch.equal(g_, other[ct_, :, jl]): tags.append("=other layer final")
                    nbad = int((g_ != fin[ct_, :, jl]).sum())
                    print(f"   {st[i]['lay'].name} ct {ct_} limb {jl}: {nbad} words differ {tags}")
    for i in range(NL):
        got = st[i]["out"].view(-1, 256).cpu()
        ref_ = refs[(i, 2)][1].view(-1, 256).cpu()
        badc = (got != ref_).any(1).nonzero().flatten().tolist()
        if badc:
            rows = sorted({k // 16 for k in badc})
            print("   ", st[i]["lay"].name, "bad chunks", len(badc), "rows", rows[:12], "etiles", sorted({k % 16 for k in badc})[:16],
                  "words/chunk", [int((got[k] != ref_[k]).sum()) for k in badc[:6]])
    print(f"trial {trial} full calls ({'graph' if trial % 2 else 'eager'}):",
          "; ".join(f"{st[i]['lay'].name}: out bad {int((st[i]['out'] != refs[(i, 2)][1]).sum())}" for i in range(NL)))
for trial in range(4):
    for upto in (0, 1, 2):
        gr = torch.cuda.CUDAGraph()
        if trial == 0 and upto == 2:
            gr.enable_debug_mode()
        cap = torch.cuda.Stream(dev)
        with torch.cuda.graph(gr, stream=cap):
            if MODE == "tails_serial" and upto == 2:
                runner(stage([0, 1]))
                for i in range(NL):
                    stage([2])(i)
            elif MODE == "tails_parallel" and upto == 2:
                runner(stage([0, 1]))
                runner(stage([2]))
            elif MODE == "e1_then_e3tail" and upto == 2:
                # e1 chain on main while e3 runs fwd+mac on the side; e3's tail after the join
                runner(lambda i: stage([0, 1, 2] if i != 2 else [0, 1])(i))
                stage([2])(2)
            elif MODE == "e3mac_vs_copy" and upto == 2:
                BIG_B.copy_(BIG_A)  # main: heavy memory traffic beside e3's forward NTT + MAC
                runner(lambda i: (BIG_B.copy_(BIG_A), BIG_A.copy_(BIG_B), BIG_B.copy_(BIG_A)) if i == 1 else stage([0, 1])(i))
            elif MODE == "e3mac_check" and upto == 2:
                runner(lambda i: stage([0, 1, 2] if i != 2 else [0, 1])(i))
            elif MODE == "e3_serial" and upto == 2:
                stage([0, 1, 2])(0)
                stage([0, 1, 2])(1)
                stage([0, 1, 2])(2)
            else:
                runner(stage(list(range(upto + 1))))
        if trial == 0 and upto == 2:
            gr.debug_dump("gpurun_out/race_graph.dot")
        for d in st:
            d["out"].zero_()
            d["ws"].zero_()
        gr.replay()
        torch.cuda.synchronize()
        msg = []
        for i in range(NL):
            ws_ref, out_ref = refs[(i, upto)]
            if MODE in ("e3mac_check", "e3mac_vs_copy") and upto == 2 and i == 2:
                ws_ref, out_ref = refs[(i, 1)]
            nx = int((st[i]["ws"] != ws_ref).sum())
            if MODE in ("e3mac_check", "e3mac_vs_copy") and upto == 2 and i == 2:
                print("   weights intact:", all(torch.equal(x["w"], w0) for x, w0 in zip(st, W0)))
                got = st[i]["out"].view(-1, 256).cpu()
                ref_ = out_ref.view(-1, 256).cpu()
                badc = (got != ref_).any(1).nonzero().flatten().tolist()
                allref = {tuple(ref_[k].tolist()): k for k in range(ref_.shape[0])}
                e1ref = refs[(1, 1)][1].view(-1, 256).cpu()
                e1map = {tuple(e1ref[k].tolist()): k for k in range(e1ref.shape[0])}
                for k in badc[:6]:
                    row = got[k]
                    nbad = int((row != ref_[k]).sum())
                    print(f"   chunk {k} (row {k // 16}, etile {k % 16}): {nbad}/256 words differ; zero={bool((row == 0).all())}; "
                          f"equals own chunk {allref.get(tuple(row.tolist()))}; equals e1 chunk {e1map.get(tuple(row.tolist()))}")
            ny = int((st[i]["out"] != out_ref).sum()) if upto >= 1 else 0
            msg.append(f"{st[i]['lay'].name}: X^ bad {nx} out bad {ny}")
        print(f"graph trial {trial} stages 0..{upto}:", "; ".join(msg))
