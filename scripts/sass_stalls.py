"""Stall-reason totals per hot SASS block of an `ncu --page source --print-source sass --csv` dump."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
hdr = rows[1]
iex = hdr.index("Instructions Executed")
isrc = hdr.index("Source")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = [r for r in rows[2:] if len(r) > iex]
# contiguous blocks with the same execution count
blocks, cur = [], None
for i, r in enumerate(data):
    e = float(r[iex] or 0)
    if cur and e == cur[2]:
        cur[1] = i
    else:
        if cur:
            blocks.append(cur)
        cur = [i, i, e]
blocks.append(cur)
tot = sum(float(r[hdr.index(h)] or 0) for r in data for h in reasons) or 1
blocks.sort(key=lambda b: -sum(float(data[i][hdr.index(h)] or 0) for i in range(b[0], b[1] + 1) for h in reasons))
for b in blocks[: int(sys.argv[2]) if len(sys.argv) > 2 else 6]:
    c = collections.Counter()
    for i in range(b[0], b[1] + 1):
        for h in reasons:
            c[h[6:]] += float(data[i][hdr.index(h)] or 0)
    s = sum(c.values())
    print(f"[{b[0]}-{b[1]}] n={b[1] - b[0] + 1} exec={b[2]:.3g} stalls={s / tot * 100:.1f}%: " +
          ", ".join(f"{k} {v / s * 100:.0f}%" for k, v in c.most_common(6)) + f"  | {data[b[0]][isrc][:40]}")
