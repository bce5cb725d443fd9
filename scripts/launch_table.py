"""Per-kernel launch table (count, total, average, share) from an
`ncu --metrics gpu__time_duration.sum --csv --log-file X` launch list."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    name = r[ik].split("(")[0][:60]
    v = float(r[iv].replace(",", ""))
    unit = r[hdr.index("Metric Unit")]
    ms = v / 1e6 if unit in ("ns", "nsecond") else (v / 1e3 if unit in ("us", "usecond") else v)
    c, t = agg.get(name, (0, 0.0))
    agg[name] = (c + 1, t + ms)
tot = sum(t for _, t in agg.values())
print(f"{'kernel':60s} {'launches':>9s} {'total_ms':>10s} {'avg_ms':>9s} {'share':>6s}")
for name, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{name:60s} {c:9d} {t:10.3f} {t / c:9.4f} {t / tot * 100:5.1f}%")
