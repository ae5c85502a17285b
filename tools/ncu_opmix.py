"""Executed-instruction mix of one kernel from an ncu report's source page (SASS view): warp-level
instructions executed per opcode (and per opcode+modifiers with -v), with their share.
Usage: python tools/ncu_opmix.py report.ncu-rep kernel_regex [-v]"""
import collections
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
verbose = "-v" in sys.argv[3:]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
hdr = rows[hi]
ix, si = hdr.index("Instructions Executed"), hdr.index("Source")
cnt = collections.Counter()
for r in rows[hi + 1:]:
    if len(r) != len(hdr) or not r[ix].isdigit():
        continue
    t = r[si].split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") else t[0]
    cnt[op if verbose else op.split(".")[0]] += int(r[ix])
tot = sum(cnt.values())
print(f"{kre}: {tot / 1e6:.2f} M warp instructions executed")
for op, n in cnt.most_common(25):
    print(f"  {op:28s} {n / 1e6:8.3f} M  {n / tot:6.1%}")
