"""Device time of one batched forward / inverse NTT call (32-bit limbs, N = 4096, L = 4) on a batch
of n_ct ciphertexts (2 L limb-polys each). Usage: python tools/ntt_time.py [n_ct ...]"""
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
ctx = Context(0, word_bits=32)
for n in [int(a) for a in sys.argv[1:]] or [8192, 1024, 32]:
    a = inputs.uniform_residues(inputs.rng(1), (n, 2), ctx.primes, ctx.n)
    x = torch.from_numpy(a.astype(np.uint32).view(np.int32)).cuda()
    ref = x.clone()
    res = {}
    for name, f in (("fwd", ctx.ntt_fwd), ("inv", ctx.ntt_inv)):
        for _ in range(3):
            f(x)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            f(x)
        e1.record()
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / 10 * 1e3
    P = n * 2 * ctx.L
    x.copy_(ref)
    ctx.ntt_fwd(x)
    ctx.ntt_inv(x)
    ok = bool(torch.equal(x, ref))
    print(f"n_ct={n:6d} polys={P:7d} fwd {res['fwd']:8.1f} us ({P / res['fwd']:.1f} M/s, "
          f"{P * 32768 / res['fwd'] / 1e3:.0f} GB/s)  inv {res['inv']:8.1f} us ({P / res['inv']:.1f} M/s)  roundtrip_ok={ok}")
