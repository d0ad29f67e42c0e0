"""Summarise an ncu capture exported by tools/ncu_capture.sh (raw + source CSVs)."""
import collections
import csv
import re
import sys

tag = sys.argv[1]
base = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
rows = list(csv.reader(open(f"{base}/{tag}_raw.csv")))
hdr, units, vals = rows[0], rows[1], rows[2]
d = dict(zip(hdr, vals))
u = dict(zip(hdr, units))
keys = ["Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
for k in keys:
    if k in d:
        print(f"{k:60s} {d[k]} {u.get(k, '')}")
stall = [(k, float(d[k] or 0)) for k in hdr
         if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
stall.sort(key=lambda x: -x[1])
print("stalls per issue:", ", ".join(f"{k[34:-23]}={v:.2f}" for k, v in stall[:8]))
try:
    srows = list(csv.reader(open(f"{base}/{tag}_source.csv")))
    h = srows[1]
    iS, iE = h.index("Source"), h.index("Instructions Executed")
    cnt = collections.Counter()
    tot = 0
    for r in srows[2:]:
        if len(r) <= iE:
            continue
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[iS].strip())
        n = int(r[iE] or 0)
        cnt[m.group(2) if m else r[iS]] += n
        tot += n
    print("instr mix:", ", ".join(f"{op}={n / tot * 100:.1f}%" for op, n in cnt.most_common(16)))
except FileNotFoundError:
    pass
