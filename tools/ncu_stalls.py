"""Stall-reason breakdown of one kernel from an ncu report's source page.
Usage: python tools/ncu_stalls.py report.ncu-rep kernel_regex"""
import collections
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
num = lambda x: int(x) if x.isdigit() else 0  # noqa: E731
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
byop = collections.defaultdict(collections.Counter)
for r in data:
    t = r[hdr.index("Source")].split()
    if not t:
        continue
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    for h in reasons:
        v = num(r[hdr.index(h)])
        tot[h] += v
        byop[op][h] += v
s = sum(tot.values())
print("stall reasons (all samples):", ", ".join(f"{k[6:]}={v / s:.1%}" for k, v in tot.most_common(8)))
for op in sorted(byop, key=lambda o: -sum(byop[o].values()))[:8]:
    c = byop[op]
    print(f"  {op:10s} {sum(c.values()) / s:6.1%}:", ", ".join(f"{k[6:]}={v / s:.1%}" for k, v in c.most_common(4)))
