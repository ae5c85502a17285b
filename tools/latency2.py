"""Cold vs hot latency of one small forward-NTT call (16 limb-polys), graph-replayed.
Usage: python tools/latency2.py [word_bits]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch

import __graft_entry__
from paper_2506_11586_b200 import Context

__graft_entry__.build()
wb = int(sys.argv[1]) if len(sys.argv) > 1 else 32
ctx = Context(0, word_bits=wb)
dev = torch.device("cuda:0")
n_ct = 2
nbuf = 64
bufs = [ctx.empty(n_ct, 2, ctx.L, ctx.n).zero_() for _ in range(nbuf)]
outs = [ctx.empty(n_ct, 2, ctx.L, ctx.n) for _ in range(nbuf)]
big = torch.empty(300 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)  # 300 MB > L2


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


def timed(g, reps=20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        big.add_(1)  # flush L2 (also evicts the twiddle tables)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


import paper_2506_11586_b200.secn as S  # noqa: E402
lib = S.lib()
import ctypes  # noqa: E402

def fwd_into(i):
    ws_in, ws_out = bufs[i], outs[i]
    # one forward NTT launch through the stage-0 entry (ct_in -> workspace), no share add
    plan = ctx.plan(1, 1, 1, 1, 1)
    return lambda: ctx.ntt_fwd(ws_in)


g1 = graph_of(lambda: ctx.ntt_fwd(bufs[0]))
print(f"w{wb} 1 fwd NTT call ({n_ct * 2 * ctx.L} limb-polys), cold L2 (flushed): {timed(g1):.2f} us")
g10 = graph_of(lambda: [ctx.ntt_fwd(bufs[i]) for i in range(10)])
print(f"w{wb} 10 fwd NTT calls back to back (different buffers), cold L2: {timed(g10) / 10:.2f} us/call")
# hot: replay without flush
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
g1.replay(); torch.cuda.synchronize()
e0.record()
for _ in range(100):
    g1.replay()
e1.record(); torch.cuda.synchronize()
print(f"w{wb} 1 fwd NTT call, hot, replayed: {e0.elapsed_time(e1) * 10:.2f} us")
g0 = graph_of(lambda: big[:1].add_(1))
print(f"tiny torch kernel, cold: {timed(g0):.2f} us")
