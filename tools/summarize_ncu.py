"""Summarise ncu outputs (gpurun_out/) into tracked text under profiles/.

    python tools/summarize_ncu.py launches <launches.csv> <out.md>
    python tools/summarize_ncu.py kernels <report.ncu-rep> <out.md> [label]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn_smem"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall_lsb"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall_bar"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
    ("smsp__inst_executed.sum", "inst"),
]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values())
    with open(out, "w") as f:
        f.write(f"# Launch list: {path.split('/')[-1]}\n\n")
        f.write("ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised:"
                " compare shares, not absolutes)\n\n")
        f.write("| launches | total us | share | mean us | kernel |\n|---:|---:|---:|---:|---|\n")
        for k, (cnt, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"| {cnt} | {us:.1f} | {100 * us / tot:.1f}% | {us / cnt:.1f} | `{k}` |\n")
        f.write(f"\nTotal: {sum(v[0] for v in agg.values())} launches, {tot / 1e3:.2f} ms\n")


def kernels(rep, out, label=""):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = [(hdr.index(m), short) for m, short in METRICS if m in hdr]
    ki = hdr.index("Kernel Name")
    with open(out, "w") as f:
        f.write(f"# ncu --set full: {rep.split('/')[-1]} {label}\n\n")
        f.write("| kernel | " + " | ".join(f"{s} [{units[i]}]" for i, s in idx) + " |\n")
        f.write("|---|" + "---:|" * len(idx) + "\n")
        for r in rows[2:]:
            name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
            f.write(f"| `{name}` | " + " | ".join(r[i] for i, _ in idx) + " |\n")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        kernels(sys.argv[2], sys.argv[3], " ".join(sys.argv[4:]))
