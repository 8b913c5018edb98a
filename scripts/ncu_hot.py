"""Top SASS lines by warp-stall samples from `ncu -i rep --page source --csv`."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                     text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
iS = h.index("Warp Stall Sampling (All Samples)")
iSrc = h.index("Source")
iE = h.index("Instructions Executed")
data = []
tot = 0
for r in rows[1:]:
    try:
        s = int(r[iS])
    except (ValueError, IndexError):
        continue
    tot += s
    data.append((s, r[0], r[iSrc].strip(), r[iE]))
print("total samples", tot)
for s, a, src, e in sorted(data, reverse=True)[:top]:
    print(f"{s:7d} {100*s/tot:5.1f}% {a[-5:]} {e:>9} {src}")
