"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel launches, total ms, share."""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
agg = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) < len(h) or r[h.index("Metric Name")] != "gpu__time_duration.sum":
        continue
    nm = r[h.index("Kernel Name")].split("(")[0][:70]
    v = float(r[h.index("Metric Value")].replace(",", ""))
    v *= {"ns": 1e-6, "us": 1e-3, "ms": 1, "s": 1e3}.get(r[h.index("Metric Unit")], 1)
    agg.setdefault(nm, []).append(v)
skip = [k for k in agg if "fma_peak" in k]
tot = sum(sum(v) for k, v in agg.items() if k not in skip)
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))[: int(sys.argv[2]) if len(sys.argv) > 2 else 16]:
    if k in skip:
        continue
    print("%-70s %4d %10.3f ms  %5.1f%%" % (k, len(v), sum(v), 100 * sum(v) / tot))
