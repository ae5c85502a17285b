"""Per-layer kernel durations from an ncu launch list (gpu__time_duration.sum CSV) of bench.py:
takes the last complete step (26 layers x 4 launches, in order). Usage: launch_table.py file.csv [net]"""
import collections
import csv
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from workloads import layers  # noqa: E402

lines = open(sys.argv[1]).read().splitlines()
i = [k for k, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[i:]))
hdr = rows[0]
ki, vi, gi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size")
ks = [(r[ki].split("(")[0].replace("void ", "").replace("secn::", ""), float(r[vi]), r[gi]) for r in rows[1:]
      if len(r) > vi and "secn::" in r[ki]]
net = layers.network(sys.argv[2] if len(sys.argv) > 2 else "squeezenet1_1")
step = [k for k in ks if not k[0].startswith("k_pack")][-4 * len(net):]
tot = collections.defaultdict(float)
print(f"{'layer':10s} {'ntt_fwd':>9s} {'mac':>9s} {'ntt_inv':>9s} {'extract':>9s}  (us, warm, serialised)")
for li, l in enumerate(net):
    g = step[li * 4:li * 4 + 4]
    print(f"{l.name:10s} " + " ".join(f"{k[1] / 1e3:9.1f}" for k in g))
    for k in g:
        tot[k[0].split("<")[0]] += k[1] / 1e3
print("totals (us):", {k: round(v, 1) for k, v in tot.items()}, "sum", round(sum(tot.values()), 1))
