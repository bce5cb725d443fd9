"""Per-opcode and per-block instruction/stall totals from `ncu --page source --print-source sass --csv`."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
hdr = rows[1]
ia, isrc, ist, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
ith = hdr.index("Avg. Threads Executed")
data = []
for r in rows[2:]:
    if len(r) <= iex:
        continue
    try:
        data.append((int(r[ia], 16), r[isrc].strip(), float(r[ist] or 0), float(r[iex] or 0), float(r[ith] or 0)))
    except ValueError:
        pass
tot = sum(d[3] for d in data)
tst = sum(d[2] for d in data)
print(f"total warp-instr {tot:.3e}, stall samples {tst:.0f}")
op = collections.Counter()
ops = collections.Counter()
for d in data:
    o = d[1].split()[0] if d[1] else "?"
    if o.startswith("@"):
        o = d[1].split()[1]
    o = o.split(".")[0]
    op[o] += d[3]
    ops[o] += d[2]
for o, v in op.most_common(30):
    print(f"  {o:12s} {v / tot * 100:5.1f}% inst  {ops[o] / tst * 100:5.1f}% stall")
# blocks: split where executed count changes
print("hot blocks (contiguous same-count runs):")
blocks = []
cur = None
for i, d in enumerate(data):
    if cur and d[3] == cur[2]:
        cur[1] = i
        cur[3] += d[2]
    else:
        if cur:
            blocks.append(cur)
        cur = [i, i, d[3], d[2]]
blocks.append(cur)
blocks.sort(key=lambda b: -(b[1] - b[0] + 1) * b[2])
for b in blocks[:25]:
    n = b[1] - b[0] + 1
    print(f"  [{b[0]:5d}-{b[1]:5d}] n={n:4d} exec/inst={b[2]:.3e} share={n * b[2] / tot * 100:5.1f}% stall={b[3] / tst * 100:5.1f}% thr={data[b[0]][4]:.1f}  {data[b[0]][1][:60]}")
