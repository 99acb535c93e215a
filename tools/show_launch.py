"""Print the tail of an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import csv
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
hdr = rows[0]
ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
seq = [(r[ik].split("(")[0][-44:], float(r[iv].replace(",", ""))) for r in rows[1:]]
a = int(sys.argv[2]) if len(sys.argv) > 2 else -40
b = int(sys.argv[3]) if len(sys.argv) > 3 else -25
for name, v in seq[a:b]:
    print(f"{name:46s} {v / 1e3:10.1f} us")
