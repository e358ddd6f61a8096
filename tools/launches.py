"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram__bytes_*])."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
tscale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
bscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("void ", "").replace("hb::", "").replace("<unnamed>::", "")
    name = name.replace("unnamed>::", "")
    v = float(r[vi].replace(",", ""))
    if r[mi] == "gpu__time_duration.sum":
        agg[name][0] += 1
        agg[name][1] += v * tscale.get(r[ui], 1.0)
    elif r[mi].startswith("dram__bytes"):
        agg[name][2] += v * bscale.get(r[ui], 1.0)
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':40s} {'launches':>8s} {'total_ms':>9s} {'avg_us':>8s} {'share':>6s} {'MB/launch':>10s} {'GB/s':>7s}")
for k, (n, t, by) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    bw = by / (t * 1e-6) / 1e9 if t > 0 else 0
    print(f"{k[:40]:40s} {n:8d} {t / 1e3:9.3f} {t / n:8.2f} {t / tot:6.3f} {by / n / 1e6:10.3f} {bw:7.0f}")
