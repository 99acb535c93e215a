"""Summarise an ncu report (``--set full``) into the JSON kept under profiles/.

    python tools/ncu_summary.py gpurun_out/x.ncu-rep profiles/r01_ncu_<name>.json [workload]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
        "launch__block_size", "sm__cycles_elapsed.avg.per_second"]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
              "usecond": 1e-6, "nsecond": 1e-9, "msecond": 1e-3}


def main(rep, out, workload=""):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        d = {"kernel": r[head.index("Kernel Name")]}
        for k in KEYS:
            if k in head:
                i = head.index(k)
                v = r[i].replace(",", "")
                try:
                    d[k] = float(v) * UNIT_SCALE.get(units[i], 1.0) if units[i] in UNIT_SCALE else float(v)
                    d[k + ".unit"] = "byte" if units[i].endswith("byte") else (
                        "s" if units[i] in UNIT_SCALE else units[i])
                except ValueError:
                    d[k] = v
        if "dram__bytes_read.sum" in d and "dram__bytes_write.sum" in d:
            d["traffic_bytes"] = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
        launches.append(d)
    with open(out, "w") as fh:
        json.dump({"report": rep.split("/")[-1], "workload": workload, "launches": launches}, fh, indent=1)
    for d in launches:
        print(d["kernel"][:60], f"{d.get('gpu__time_duration.sum', 0) * 1e6:.1f} us",
              f"traffic {d.get('traffic_bytes', 0) / 1e6:.1f} MB")


if __name__ == "__main__":
    main(*sys.argv[1:])
