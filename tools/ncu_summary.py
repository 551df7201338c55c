"""Summarise ncu artifacts into a committed text file under profiles/.

    python tools/ncu_summary.py <launches.csv> <report.ncu-rep> <out.txt> [algorithmic_bytes]

Launch list: per-kernel count, total device time and share (cold, serialised —
compare shares).  Full report: the metrics the roofline uses (tensor pipe,
MUFU/XU, DRAM bytes, duration, registers, occupancy) and the top stall reasons.
"""

import collections
import csv
import io
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    idx = {k: j for j, k in enumerate(h)}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) < len(h):
            continue
        name = r[idx["Kernel Name"]]
        agg[name][0] += 1
        agg[name][1] += float(r[idx["Metric Value"]].replace(",", ""))
    tot = sum(v for _, v in agg.values())
    out = ["launch list (ncu gpu__time_duration.sum, cold + serialised):",
           f"{'count':>6} {'total ms':>10} {'share':>7}  kernel"]
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:15]:
        out.append(f"{n:6d} {v / 1e6:10.3f} {100 * v / tot:6.2f}%  {k[:90]}")
    return out


WANT = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__bytes_read.sum.per_second", "lts__t_bytes.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    vals = {k: (u[i], v[i]) for i, k in enumerate(h)}
    out = [f"kernel: {vals.get('Kernel Name', ('', '?'))[1]}"]
    for k in WANT:
        if k in vals:
            out.append(f"  {k:70s} {vals[k][1]:>18s} {vals[k][0]}")
    stalls = [(float(val[1]), k) for k, val in vals.items()
              if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
              and val[1] not in ("", "n/a")]
    if stalls:
        out.append("  top warp stall reasons (warps per issue-active cycle):")
        for x, k in sorted(stalls, reverse=True)[:8]:
            out.append(f"    {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:28s} {x:8.3f}")
    return out, vals


def main():
    lcsv, rep, out_path = sys.argv[1:4]
    alg = float(sys.argv[4]) if len(sys.argv) > 4 else None
    lines = launches(lcsv) + [""]
    rl, vals = report(rep)
    lines += rl
    try:
        rd = float(vals["dram__bytes_read.sum"][1].replace(",", ""))
        wr = float(vals["dram__bytes_write.sum"][1].replace(",", ""))
        unit = vals["dram__bytes_read.sum"][0]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        traffic = (rd + wr) * scale
        lines.append(f"  DRAM traffic per launch: {traffic / 1e9:.3f} GB")
        if alg:
            lines.append(f"  algorithmic bytes per launch: {alg / 1e9:.3f} GB  (traffic / algorithmic = {traffic / alg:.2f})")
    except Exception as e:  # pragma: no cover
        lines.append(f"  (no DRAM bytes: {e})")
    with open(out_path, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
