"""Summary of an ncu capture of one bench step (tools/step_profile.py; gpu_step_ncu.sh): per kernel
family the launch count, summed duration (ncu serialises kernels: cold-cache times), summed DRAM
bytes read + written, warp instructions, issue-slot and pipe utilisation (duration-weighted) and
the dominant stall reasons; then the step's total DRAM traffic.
Usage: python tools/ncu_step_summary.py report.ncu-rep [algorithmic_bytes_per_step]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
alg = float(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].endswith(".json") else None
json_out = next((a for a in sys.argv[2:] if a.endswith(".json")), None)
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
data = rows[2:]


def col(name):
    return hdr.index(name) if name in hdr else None


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3, "msecond": 1e3,
         "usecond": 1, "nsecond": 1e-3}


def num(r, name):
    """the value in base units (bytes; microseconds for durations)"""
    i = col(name)
    if i is None:
        return 0.0
    try:
        return float(r[i].replace(",", "")) * SCALE.get(rows[1][i], 1)
    except ValueError:
        return 0.0


def family(k):
    k = re.sub(r"^void ", "", k)
    return re.sub(r"\(.*", "", k).replace("secn::", "")


fam = collections.OrderedDict()
stall_cols = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
for r in data:
    k = family(r[col("Kernel Name")])
    f = fam.setdefault(k, collections.Counter())
    t = num(r, "gpu__time_duration.sum")
    f["n"] += 1
    f["us"] += t
    f["dram"] += num(r, "dram__bytes_read.sum") + num(r, "dram__bytes_write.sum")
    f["inst"] += num(r, "smsp__inst_executed.sum")
    for m in ("smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
              "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "dram__throughput.avg.pct_of_peak_sustained_elapsed",
              "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct",
              "smsp__sass_average_data_bytes_per_sector_mem_global_op_st.pct"):
        f[m] += num(r, m) * t
    for m in ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum"):
        f[m] += num(r, m)
    for h in stall_cols:
        f[h] += num(r, h) * t
    f["t"] += t

scale = 1
tot_dram = 0.0
print(f"{'kernel':40s} {'n':>4s} {'sum_us':>9s} {'DRAM_MB':>9s} {'Minst':>8s} {'issue%':>7s} {'alu%':>6s} {'fma%':>6s} "
      f"{'warps%':>7s} {'dram%':>6s}  top stalls (per issued instr)")
for k, f in fam.items():
    t = f["t"] or 1
    tot_dram += f["dram"] * scale
    st = sorted(((f[h] / t, h) for h in stall_cols), reverse=True)[:4]
    sts = ", ".join(f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}"
                    for v, h in st)
    print(f"{k[:40]:40s} {int(f['n']):4d} {f['us']:9.1f} {f['dram'] * scale / 1e6:9.1f} {f['inst'] / 1e6:8.2f} "
          f"{f['smsp__issue_active.avg.pct_of_peak_sustained_active'] / t:7.1f} "
          f"{f['sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active'] / t:6.1f} "
          f"{f['sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active'] / t:6.1f} "
          f"{f['sm__warps_active.avg.pct_of_peak_sustained_active'] / t:7.1f} "
          f"{f['dram__throughput.avg.pct_of_peak_sustained_elapsed'] / t:6.1f}  {sts}")
if any(f["smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct"] for f in fam.values()):
    print("global-access sector efficiency (bytes used per sector fetched / stored, %) and shared-memory bank conflicts:")
    for k, f in fam.items():
        t = f["t"] or 1
        print(f"  {k[:40]:40s} ld {f['smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct'] / t:6.1f}  "
              f"st {f['smsp__sass_average_data_bytes_per_sector_mem_global_op_st.pct'] / t:6.1f}  "
              f"conflicts ld {f['l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum'] / 1e6:7.2f} M  "
              f"st {f['l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum'] / 1e6:7.2f} M")
print(f"step DRAM traffic (read + write, all kernels): {tot_dram / 1e9:.3f} GB"
      + (f"; algorithmic bytes {alg / 1e9:.3f} GB; traffic / algorithmic = {tot_dram / alg:.3f}" if alg else ""))

if json_out:  # machine-readable copy for bench.py's roofline block
    import json

    summary = {"source": rep, "step_dram_bytes": tot_dram, "kernels": {}}
    for k, f in fam.items():
        t = f["t"] or 1
        summary["kernels"][k] = {
            "launches": int(f["n"]), "sum_us_ncu": round(f["us"], 1), "dram_bytes": f["dram"],
            "warp_instructions": f["inst"],
            "issue_active_pct": round(f["smsp__issue_active.avg.pct_of_peak_sustained_active"] / t, 1),
            "pipe_alu_pct": round(f["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"] / t, 1),
            "pipe_fma_pct": round(f["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"] / t, 1),
            "warps_active_pct": round(f["sm__warps_active.avg.pct_of_peak_sustained_active"] / t, 1),
            "top_stalls_per_issue": {h.replace("smsp__average_warps_issue_stalled_", "").replace(
                "_per_issue_active.ratio", ""): round(f[h] / t, 2)
                for _, h in sorted(((f[h] / t, h) for h in stall_cols), reverse=True)[:5]}}
    open(json_out, "w").write(json.dumps(summary, indent=1))
