"""Condense an ncu --set full report (one kernel) into the metrics DESIGN.md cites."""
import csv, subprocess, sys
rep, title = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
keep = ("Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "Compute (SM) Throughput",
        "Achieved Occupancy", "Registers Per Thread", "Grid Size", "Block Size", "Cluster Size",
        "Warp Cycles Per Issued Instruction", "Executed Ipc Active", "Issue Slots Busy",
        "Dynamic Shared Memory Per Block", "Static Shared Memory Per Block")
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
name = None
print(f"# {title}")
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if name is None:
        name = d.get("Kernel Name"); print(f"# kernel: {name}")
    if d.get("Metric Name") in keep:
        print(f"{d['Section Name']:40s} {d['Metric Name']:38s} {d['Metric Unit']:>10s} {d['Metric Value']:>14s}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                     capture_output=True, text=True).stdout.splitlines()
h, u, v = list(csv.reader(raw[-3:]))
for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
    i = h.index(k)
    print(f"{'raw':40s} {k:38s} {u[i]:>10s} {v[i]:>14s}")
