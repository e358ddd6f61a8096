"""Per-source-line warp-stall summary of an ncu report (needs -lineinfo).

  python tools/srcprof.py report.ncu-rep kernel_regex [top]
"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv", "-k",
                      f"regex:{kre}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
files = []
cur = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1]
    elif len(r) > 5 and r[0] == "Line No":
        hdr = r
    elif len(r) > 7 and r[0].isdigit() and cur:
        try:
            files.append((cur.split("/")[-1], int(r[0]), r[1], int(r[4] or 0), int(r[7] or 0)))
        except ValueError:
            pass
tot = sum(f[3] for f in files) or 1
print(f"total stall samples {tot}")
for f in sorted(files, key=lambda x: -x[3])[:top]:
    print(f"{100 * f[3] / tot:5.1f}% {f[0]}:{f[1]:<4d} inst={f[4]:<8d} {f[2].strip()[:90]}")
