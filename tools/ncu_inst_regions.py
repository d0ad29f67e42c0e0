"""Group an ncu SASS source export by execution count (dev tool): shows how the
executed instructions split between the pair loop, per-tile and per-chunk code.

    python tools/ncu_inst_regions.py gpurun_out/<tag>_source.csv
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
by = collections.defaultdict(lambda: [0, 0, 0, collections.Counter()])
tot_i = tot_s = 0
for r in rows[2:]:
    try:
        n = int(r[ix["Instructions Executed"]] or 0)
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, IndexError):
        continue
    if n == 0:
        continue
    op = r[ix["Source"]].strip().split()
    op = op[1] if op and op[0].startswith("@") else (op[0] if op else "?")
    g = by[n]
    g[0] += 1
    g[1] += n
    g[2] += s
    g[3][op.split(".")[0]] += n
    tot_i += n
    tot_s += s
print(f"total executed warp-instructions {tot_i}, samples {tot_s}")
for n, (k, ins, s, ops) in sorted(by.items(), key=lambda kv: -kv[1][1])[:14]:
    print(f"exec={n:>9} sass_lines={k:>4} inst={ins / tot_i:6.1%} samples={s / max(tot_s, 1):6.1%}  "
          + ", ".join(f"{o}:{c // n}" for o, c in ops.most_common(9)))
