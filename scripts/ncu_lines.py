"""Aggregate an `ncu --page source --print-source cuda,sass --csv` dump by CUDA source line."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
by = collections.defaultdict(lambda: [0.0, 0.0, ""])
hdr = None
cur = None
fname = ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        li, ls = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) <= ls:
        continue
    if r[0].strip().isdigit():
        cur = (fname, int(r[0]))
        if r[1].strip():
            by[cur][2] = r[1].strip()[:85]
    try:
        by[cur][0] += float(r[li] or 0)
        by[cur][1] += float(r[ls] or 0)
    except ValueError:
        pass
tot = sum(v[0] for v in by.values()) or 1
ts = sum(v[1] for v in by.values()) or 1
for k, v in sorted(by.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{k[0][:12]}:{k[1]:<4d} inst {v[0] / tot * 100:5.1f}% stall {v[1] / ts * 100:5.1f}%  {v[2]}")
