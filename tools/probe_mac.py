"""Timeline of one k_mac launch from globaltimer probes (a -DSECN_PROBE build of libsecn):
CTA 0's phases and the start/end spread of all CTAs. Usage: python tools/probe_mac.py layer [net]"""
import ctypes
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

from paper_2506_11586_b200 import build as B
from paper_2506_11586_b200 import secn
from workloads import inputs, layers

so = B.PKG / "libsecn_probe.so"
cmd = [B.NVCC, *[f for f in B.FLAGS if f != "-v" and f != "-Xptxas"], "-DSECN_PROBE", "-o", str(so), *map(str, B.SOURCES)]
subprocess.run(cmd, check=True, capture_output=True)
secn._lib = secn.lib(so)
L_ = secn._lib
L_.secn_probe_read.restype = ctypes.c_int
L_.secn_probe_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
name = sys.argv[1]
net = sys.argv[2] if len(sys.argv) > 2 else "squeezenet1_1"
ctx = secn.Context(0, word_bits=32)
dev = torch.device("cuda:0")
T = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)  # noqa: E731
lay = next(l for l in layers.network(net) if l.name == name)
plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
g = inputs.rng(3)
ctn = inputs.uniform_residues(g, (plan.G * plan.S, 2), ctx.primes, ctx.n)
ct = torch.from_numpy(ctn.astype(np.uint32).view(np.int32)).to(dev)
x0 = T(inputs.uniform_below(g, (plan.G * plan.S, ctx.n), 1 << ctx.t_bits))
r = T(inputs.uniform_below(g, (plan.M * plan.S, ctx.n), 1 << ctx.t_bits))
w = ctx.preprocess_weights(plan, T(inputs.quantized_kernel(g, plan.M, lay.C, lay.k, lay.k)))
out = ctx.empty(plan.M * plan.S, 2, ctx.L, ctx.n)
ws = torch.empty(ctx.workspace_bytes(plan) // 8 + 1, dtype=torch.int64, device=dev)
for _ in range(3):
    ctx.he_conv2d(plan, ct, w, x0=x0, r=r, out=out, workspace=ws)
torch.cuda.synchronize()
buf = np.zeros(65536 * 2 + 64, np.uint64)
L_.secn_probe_read(buf.ctypes.data, buf.size)
ph = buf[:8].astype(np.int64)
cta = buf[64:].reshape(-1, 2).astype(np.int64)
cta = cta[cta[:, 0] > 0]
t0 = cta[:, 0].min()
print(name, plan)
print("CTA0 phases (us from its start): init+tw %.2f  xbar %.2f  mac1 %.2f  levels1 %.2f  end %.2f" %
      tuple((ph[k] - ph[0]) / 1e3 for k in (1, 2, 3, 4, 5)))
d = (cta[:, 1] - cta[:, 0]) / 1e3
print(f"CTAs {len(cta)}: span {(cta[:, 1].max() - t0) / 1e3:.2f} us; per-CTA duration mean {d.mean():.2f} "
      f"min {d.min():.2f} max {d.max():.2f} us; start spread {(cta[:, 0].max() - t0) / 1e3:.2f} us")
hist = np.histogram((cta[:, 0] - t0) / 1e3, bins=10)
print("start histogram (us bins):", [f"{b:.1f}:{c}" for b, c in zip(hist[1], hist[0])])
