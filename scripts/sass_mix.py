"""Opcode mix + stall hot spots from an `ncu --page source --csv --print-source sass` dump."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
per = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr = rows[1]
si, ie, ss = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
cnt, stall = collections.Counter(), collections.Counter()
tot = 0
for r in rows[2:]:
    try:
        n = float(r[ie])
    except (ValueError, IndexError):
        continue
    toks = r[si].strip().split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    cnt[op] += n
    stall[op] += float(r[ss] or 0)
    tot += n
ts = sum(stall.values())
for op, n in cnt.most_common(30):
    print(f"{op:10s} {n / tot * 100:5.1f}% inst  {stall[op] / ts * 100:5.1f}% stall-samples  {n / per:9.1f} per unit")
