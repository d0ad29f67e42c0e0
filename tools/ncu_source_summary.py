"""Per-instruction stall summary of an ncu --page source --csv export (SASS view).

    python tools/ncu_source_summary.py gpurun_out/<tag>_source.csv [top]
Prints total samples per stall reason and the top instructions by samples with
their dominant stall reasons.
"""
import collections
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
hdr = rows[1]
data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
items = []
for r in data:
    try:
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    per = {h: int(r[ix[h]] or 0) for h in stalls}
    tot.update(per)
    items.append((s, r[ix["Address"]][-5:], r[ix["Source"]].strip(), per))
T = sum(tot.values())
print(f"total samples {T}")
for k, v in tot.most_common(12):
    print(f"  {k:28s} {v:8d} {100*v/T:5.1f}%")
print("top instructions:")
for s, a, src, per in sorted(items, reverse=True)[:top]:
    dom = ", ".join(f"{k[6:]}={v}" for k, v in sorted(per.items(), key=lambda kv: -kv[1])[:3] if v)
    print(f"{s:6d} {a} {src[:60]:60s} {dom}")
