import csv, io, subprocess, sys
rep, out = sys.argv[1], sys.argv[2]
keep = {"Duration", "Memory Throughput", "DRAM Throughput", "Achieved Occupancy", "Registers Per Thread",
        "Compute (SM) Throughput", "Issue Slots Busy", "Executed Ipc Active", "L2 Hit Rate", "Theoretical Occupancy",
        "Grid Size", "Block Size", "Dynamic Shared Memory Per Block"}
txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(txt)))
h = r[0]
ki, mi, ui, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value"), h.index("ID")
w = csv.writer(open(out, "w"))
w.writerow(["ID", "Kernel", "Metric", "Unit", "Value"])
for row in r[1:]:
    if len(row) > vi and row[mi] in keep:
        w.writerow([row[ii], row[ki][:70], row[mi], row[ui], row[vi]])
# dram bytes per launch from raw page
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hh = rr[0]
for row in rr[2:]:
    w.writerow([row[hh.index("ID")], row[hh.index("Kernel Name")][:70], "dram__bytes_read.sum", rr[1][hh.index("dram__bytes_read.sum")], row[hh.index("dram__bytes_read.sum")]])
    w.writerow([row[hh.index("ID")], row[hh.index("Kernel Name")][:70], "dram__bytes_write.sum", rr[1][hh.index("dram__bytes_write.sum")], row[hh.index("dram__bytes_write.sum")]])
