"""Summarize an `ncu --metrics gpu__time_duration.sum --csv` launch list: per kernel count, mean and
total (cold, serialized per-launch times: shares, not absolute step times)."""
import collections, csv, sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ik, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
agg = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) <= iv or r[im] != "gpu__time_duration.sum":
        continue
    name = r[ik].split("(")[0]
    v = float(r[iv].replace(",", ""))
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
unit = "ns" if max(a[1] for a in agg.values()) > 1e5 else "us"
print(f"{'kernel':60s} {'n':>5s} {'mean_us':>10s} {'total_us':>11s} {'share':>6s}")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    sc = 1e-3 if unit == "ns" else 1.0
    print(f"{k[:60]:60s} {n:5d} {t / n * sc:10.1f} {t * sc:11.1f} {t / tot * 100:5.1f}%")
