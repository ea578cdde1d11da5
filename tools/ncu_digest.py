"""Digest of one ncu report (raw metrics + SASS opcode mix + hottest stall lines).

    python tools/ncu_digest.py <report.ncu-rep> [top]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


rows = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
d = dict(zip(rows[0], rows[2]))
for k in ["gpu__time_duration.sum", "smsp__inst_executed.sum",
          "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
          "launch__block_size", "launch__grid_size", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "dram__throughput.avg.pct_of_peak_sustained_elapsed",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]:
    print(f"{k:70s} {d.get(k)}")
for k in rows[0]:
    if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio"):
        try:
            if float(d[k]) > 0.1:
                print(f"  stall {k.replace('smsp__average_warps_issue_stalled_', ''):50s} {d[k]}")
        except ValueError:
            pass
rows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
hdr = rows[1]
ia, isrc, iss = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index(
    "Warp Stall Sampling (All Samples)")
data = [(r[isrc], int(r[ia] or 0), int(r[iss] or 0)) for r in rows[2:]
        if len(r) > ia and r[ia].strip().isdigit()]  # multi-kernel reports repeat headers
tot, tots = sum(x[1] for x in data), sum(x[2] for x in data)
print("total inst", tot, "samples", tots)
op, ops = collections.Counter(), collections.Counter()
for src, ex, ss in data:
    w = src.split()
    o = (w[1] if w[0].startswith("@") else w[0]).split(".")[0]
    op[o] += ex
    ops[o] += ss
for o, c in op.most_common(top):
    print(f"  {o:12s} {c:10d} {100 * c / tot:5.1f}%  samples {ops[o]}")
print("--- hottest stall lines")
for src, ex, ss in sorted(data, key=lambda x: -x[2])[:top]:
    print(f"  {ss:5d} {ex:9d} {src}")
