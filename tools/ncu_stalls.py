"""Summarise an ncu report: stall reasons, pipe utilisation, and the top stalled SASS lines.

  python tools/ncu_stalls.py gpurun_out/attn.ncu-rep [n_lines]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h = r[0]
for row in r[2:]:
    d = dict(zip(h, row))
    print(d.get("Kernel Name", "")[:60], "duration(ns)", d.get("gpu__time_duration.sum"))
    items, tot = [], 0.0
    for k, v in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                continue
            items.append((x, k[len("smsp__pcsamp_warps_issue_stalled_"):]))
            tot += x
    for x, k in sorted(items, reverse=True)[:10]:
        print(f"  stall {k:22s} {100 * x / tot:5.1f}%")
    for k in ["smsp__issue_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
              "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
              "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_elapsed.avg.per_second"]:
        print(f"  {k:70s} {d.get(k)}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(src)))
h = r[1]
rows = r[2:]
ia, isrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
tot = sum(int(x[ia] or 0) for x in rows)
for x in sorted(rows, key=lambda x: -int(x[ia] or 0))[:n]:
    print(f"{int(x[ia]):8d} {100 * int(x[ia]) / tot:5.1f}%  {x[0][-5:]}  {x[isrc].strip()[:90]}")
