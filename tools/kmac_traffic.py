"""Writes profiles/kmac_traffic.json (read by bench.py as roofline.traffic) from an ncu --set full
capture of conv10's MAC launch (tools/gpu_round.sh: conv10_TAG.ncu-rep).
Usage: python tools/kmac_traffic.py report.ncu-rep source_label"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
rep, label = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, r = rows[0], rows[1], rows[2]
SC = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3, "usecond": 1, "nsecond": 1e-3}


def v(name):
    i = hdr.index(name)
    return float(r[i].replace(",", "")) * SC.get(units[i], 1)


# conv10 under the time-rule plan (G = 22, S = 1, M = 1000), 32-bit limbs, L = 4, N = 4096:
# W_b L N (M G [weights] + 2 G S [X^] + 2 M S [Y^ out])
G, S, M, WL, N = 22, 1, 1000, 16, 4096
alg = WL * N * (M * G + 2 * G * S + 2 * M * S)
dram = v("dram__bytes_read.sum") + v("dram__bytes_write.sum")
t = v("gpu__time_duration.sum")
d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("secn::", ""),
     "layer": "squeezenet1_1 conv10 (the step's largest MAC launch; time-rule plan G=22 S=1)",
     "source": label, "dram_bytes_per_launch": int(dram), "algorithmic_bytes_per_launch": alg,
     "fmaheavy_pct_of_peak_elapsed": round(v("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"), 1)
     if "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed" in hdr else None,
     "duration_us_ncu": round(t, 3), "dram_GBps_ncu": round(dram / (t * 1e-6) / 1e9, 1)}
(ROOT / "profiles" / "kmac_traffic.json").write_text(json.dumps(d, indent=1) + "\n")
print(json.dumps(d))
