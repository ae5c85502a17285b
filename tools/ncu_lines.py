"""Executed warp instructions and stall samples per CUDA source line of one kernel, from an ncu
report captured with --import-source on (-lineinfo build): the `cuda,sass` source view groups
each SASS instruction under its source line (inlined helpers under their own file and line).
Usage: python tools/ncu_lines.py report.ncu-rep kernel_regex [top]"""
import collections
import csv
import io
import os
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv", "-k",
                      f"regex:{kre}"], capture_output=True, text=True).stdout
fname, hdr, cur = "?", None, None
inst = collections.Counter()
samp = collections.Counter()
text = {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1])
        continue
    if r[0] == "Line No":
        hdr = r
        ii, si = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        text[cur] = r[1].strip()
        continue
    if cur and r[ii].isdigit():
        inst[cur] += int(r[ii])
        samp[cur] += int(r[si]) if r[si].isdigit() else 0
tot, stot = sum(inst.values()), sum(samp.values()) or 1
print(f"{kre}: {tot / 1e6:.2f} M warp instructions, {stot} stall samples")
for k, n in inst.most_common(top):
    print(f"  {k[0]:>14s}:{k[1]:<5d} {n / tot:6.1%} inst {samp[k] / stot:6.1%} samples  {text.get(k, '')[:90]}")
