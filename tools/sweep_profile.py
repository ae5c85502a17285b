"""One forward and one inverse NTT call per ring degree of the C5 sweep (32-bit limbs, 4 sweep
primes, ~256 MiB per call) between cudaProfilerStart/Stop, for an ncu capture of the NTT engine.
Usage: python tools/sweep_profile.py [word_bits] [MiB] [log_n,...]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch

import __graft_entry__
from paper_2506_11586_b200 import Context

__graft_entry__.build()
wb = int(sys.argv[1]) if len(sys.argv) > 1 else 32
mib = int(sys.argv[2]) if len(sys.argv) > 2 else 256
P = {64: (0xFFFFFFFFFFC0001, 0xFFFFFFFFF840001, 0xFFFFFFFFF6A0001, 0xFFFFFFFFF5A0001),
     32: (0x7E90001, 0x7E00001, 0x7DD0001, 0x7D70001)}[wb]
L = 4 if wb == 32 else 2
jobs = []
logns = tuple(int(v) for v in sys.argv[3].split(",")) if len(sys.argv) > 3 else (12, 13, 14, 15)
for logn in logns:
    ctx = Context(0, log_n=logn, primes=P[:L], word_bits=wb)
    n_polys = (mib << 20) // ((1 << logn) * (wb // 8) * L)
    t = ctx.empty(n_polys, L, 1 << logn)
    t.random_(0, min(P[:L]))
    for _ in range(2):
        ctx.ntt_fwd(t)
        ctx.ntt_inv(t)
    jobs.append((ctx, t))
torch.cuda.synchronize()
torch.cuda.profiler.start()
for ctx, t in jobs:
    ctx.ntt_fwd(t)
    ctx.ntt_inv(t)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
