"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    v *= {"msecond": 1e3, "ms": 1e3, "usecond": 1.0, "us": 1.0, "nsecond": 1e-3, "ns": 1e-3}.get(r[ui], 1.0)
    name = r[ki]
    name = name[:100]
    agg.setdefault(name, []).append(v)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{len(v):4d} x {sum(v)/len(v):9.2f} us  share {sum(v)/tot*100:5.1f}%  {k}")
print(f"total {tot:.1f} us over {sum(len(v) for v in agg.values())} launches")
