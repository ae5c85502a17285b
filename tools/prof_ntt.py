"""One large batched INTT / NTT call (for ncu). Usage: python tools/prof_ntt.py [word_bits] [n_ct]"""
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
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
ctx = Context(0, word_bits=wb)
a = inputs.uniform_residues(inputs.rng(1), (n, 2), ctx.primes, ctx.n)
x = torch.from_numpy(a.view(np.int64) if wb == 64 else a.astype(np.uint32).view(np.int32)).cuda()
r = torch.zeros((n, ctx.n), dtype=torch.int64, device="cuda")
for _ in range(3):
    ctx.ntt_fwd(x)
    ctx.ntt_inv(x)
    ctx.mask_add(x, r)
torch.cuda.synchronize()
print("ok", wb, n)
