"""Per-kernel duration and DRAM traffic of one iteration's four pass kernels from an ncu report.

usage: ncu_traffic.py REPORT DTYPE [OUT_JSON [CONFIG]]
The report is `ncu --set full --cache-control none --clock-control none -k regex:kb_pass_ -s 4
-c 4 python tools/one_iter.py DTYPE` (the second iteration, warm L2 as inside a solve). With
OUT_JSON the iteration's bytes are merged into that file under DTYPE (bench.py reads it as the
roofline "traffic" field).
"""
import csv
import json
import os
import subprocess
import sys

rep, dtype = sys.argv[1], sys.argv[2]
# REPORT may also be the saved `ncu -i REPORT --page raw --csv` text (*.csv)
raw = open(rep).read() if rep.endswith(".csv") else subprocess.run(
    ["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TSCALE = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}


def val(d, key):
    u = units[hdr.index(key)]
    v = float(d[key].replace(",", ""))
    return v * SCALE.get(u, 1) if "bytes" in key else v * TSCALE.get(u, 1)


out = []
for row in data:
    d = dict(zip(hdr, row))
    nbytes = val(d, "dram__bytes_read.sum") + val(d, "dram__bytes_write.sum")
    out.append({"kernel": d.get("Kernel Name", "")[:48], "us": round(val(d, "gpu__time_duration.sum"), 2),
                "dram_bytes": int(nbytes)})
for o in out:
    print(f"{o['kernel']:48s} {o['us']:8.2f} us  {o['dram_bytes'] / 1e6:8.2f} MB")
total = sum(o["dram_bytes"] for o in out)
print("iteration dram bytes", total)
if len(sys.argv) > 3:
    path = sys.argv[3]
    cur = {}
    if os.path.exists(path):
        with open(path) as f:
            cur = json.load(f)
    cur[dtype] = total
    cur.setdefault("_per_kernel", {})[dtype] = out
    cfgname = sys.argv[4] if len(sys.argv) > 4 else "cfg2"
    cur["_source"] = ("ncu --set full --cache-control none --clock-control none, tools/one_iter.py "
                      f"(second iteration of {cfgname}), dram__bytes_read.sum + dram__bytes_write.sum")
    with open(path, "w") as f:
        json.dump(cur, f, indent=1)
