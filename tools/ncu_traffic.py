"""Summarise an ncu report into profiles/ncu_traffic.json: per kernel class, the
average DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) and
duration, as read by bench.py for roofline.traffic.

   python tools/ncu_traffic.py <report.ncu-rep | raw-page.csv> <source description>
"""
import csv
import io
import json
import os
import subprocess
import sys

CLASSES = [("k_coarse", "coarse_solve"), ("k_down", "vcycle_down"), ("k_up_", "vcycle_up"),
           ("k_adots", "krylov_adots"), ("k_update", "krylov_update"), ("k_restart", "krylov_restart"),
           ("k_finalize", "krylov_finalize"), ("k_conv", "conv3x3"), ("k_maxpool", "net_io"),
           ("k_upsample", "net_io"), ("k_pack", "net_io"), ("k_unpack", "net_io")]


def classify(name):
    base = name.split("(")[0].split("::")[-1].split("<")[0]
    for pre, cls in CLASSES:
        if base.startswith(pre):
            return cls
    return None


def main():
    rep, source = sys.argv[1], sys.argv[2]
    if rep.endswith(".csv"):  # a raw-page export (ncu -i rep --page raw --csv --metrics ...)
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                              "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                             capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    units = rows[1]
    k_name = h.index("Kernel Name")
    i_rd, i_wr, i_t = (h.index(m) for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    tscale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}
    agg = {}
    for r in rows[2:]:
        cls = classify(r[k_name])
        if cls is None:
            continue
        by = float(r[i_rd]) * scale.get(units[i_rd], 1) + float(r[i_wr]) * scale.get(units[i_wr], 1)
        us = float(r[i_t]) * tscale.get(units[i_t], 1.0)
        a = agg.setdefault(cls, {"launches": 0, "bytes": 0.0, "us": 0.0, "kernels": set()})
        a["launches"] += 1
        a["bytes"] += by
        a["us"] += us
        a["kernels"].add(r[k_name].split("(")[0][-60:])
    res = {"source": source, "classes": {}}
    for cls, a in agg.items():
        res["classes"][cls] = {"launches_captured": a["launches"], "dram_bytes_per_launch": a["bytes"] / a["launches"],
                               "ncu_us_per_launch": a["us"] / a["launches"], "kernels": sorted(a["kernels"])}
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
    with open(path, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
