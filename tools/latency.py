"""Launch/latency floors of the hot-path kernels on small batches (graph-replayed, CUDA events).
Usage: python tools/latency.py [word_bits]"""
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
wb = int(sys.argv[1]) if len(sys.argv) > 1 else 32
ctx = Context(0, word_bits=wb)
dev = torch.device("cuda:0")


def timeit(fn, reps=50):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(10):
            fn()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 10 * 1e3  # us per call


g = inputs.rng(1)
for n in (1, 2, 8, 32, 128, 512, 2048):
    x = ctx.empty(n, 2, ctx.L, ctx.n)
    x.copy_(torch.from_numpy(inputs.uniform_residues(g, (n, 2), ctx.primes, ctx.n).astype(
        np.uint64 if wb == 64 else np.uint32).view(np.int64 if wb == 64 else np.int32)))
    r = torch.zeros((n, ctx.n), dtype=torch.int64, device=dev)
    t_f = timeit(lambda: ctx.ntt_fwd(x))
    t_i = timeit(lambda: ctx.ntt_inv(x))
    t_m = timeit(lambda: ctx.mask_add(x, r))
    print(f"w{wb} cts={n:5d} limb-polys={n * 2 * ctx.L:6d}  ntt_fwd {t_f:8.2f} us  ntt_inv {t_i:8.2f} us  mask_add {t_m:7.2f} us")
