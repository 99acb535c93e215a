"""Hot SASS instructions of an ncu report (--set full --import-source on): stall samples and
executed instructions per address, plus the stall mix.

    python tools/ncu_sass_hot.py report.ncu-rep [kernel-regex] [top]"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."
top = int(sys.argv[3]) if len(sys.argv) > 3 else 60
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = txt.split('"Kernel Name"')
for b in blocks[1:]:
    name = b.split("\n", 1)[0]
    if not re.search(kre, name):
        continue
    rows = list(csv.reader(io.StringIO(b.split("\n", 1)[1])))
    h = rows[0]
    ia, isrc, ismp, iex = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), \
        h.index("Instructions Executed")
    stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    data = []
    for r in rows[1:]:
        if len(r) < len(h):
            continue
        try:
            data.append((int(r[ia], 16), r[isrc], float(r[ismp] or 0), float(r[iex] or 0),
                         {h[i]: float(r[i] or 0) for i in stall_cols}))
        except ValueError:
            pass
    S = sum(d[2] for d in data)
    E = sum(d[3] for d in data)
    print(f"{name[:100]}  samples {S:.0f}  instructions {E:.3e}")
    tot = {}
    for d in data:
        for k, v in d[4].items():
            tot[k] = tot.get(k, 0) + v
    print("  stalls:", ", ".join(f"{k[6:]} {v / S:.1%}" for k, v in sorted(tot.items(), key=lambda t: -t[1])[:10]))
    for d in sorted(data, key=lambda t: -t[2])[:top]:
        st = sorted(d[4].items(), key=lambda t: -t[1])[:2]
        print(f"  {d[0]:05x} {d[2] / S:6.2%} ex {d[3]:.2e}  {d[1][:60]:60s} " + " ".join(f"{k[6:]}={v:.0f}" for k, v in st))
