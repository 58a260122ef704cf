"""Stall samples of one kernel aggregated by SASS address bucket (find where warps spend time)."""
import csv
import subprocess
import sys
from collections import defaultdict

rep, regex = sys.argv[1], sys.argv[2]
bucket = int(sys.argv[3], 0) if len(sys.argv) > 3 else 0x200
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{regex}",
                      "--launch-count", "1", "--print-source", "sass"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
hdr = rows[0]
data = [dict(zip(hdr, r)) for r in rows[1:] if len(r) == len(hdr) and r[0].startswith("0x")]
tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
agg = defaultdict(lambda: [0, 0, defaultdict(int)])
for d in data:
    a = int(d["Address"], 16) if "Address" in d else int(d[hdr[0]], 16)
    b = a // bucket * bucket
    s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    agg[b][0] += s
    agg[b][1] += int(d["Instructions Executed"] or 0)
    op = d["Source"].split()
    op = (op[1] if op and op[0].startswith("@") and len(op) > 1 else (op[0] if op else "?")).split(".")[0]
    agg[b][2][op] += s
print("total samples", tot)
for b in sorted(agg):
    s, n, ops = agg[b]
    if s * 100 >= tot:
        top = sorted(ops.items(), key=lambda kv: -kv[1])[:4]
        print(f"{b:#07x} {100.0 * s / tot:5.1f}% exec={n:9d} ", " ".join(f"{k}:{v}" for k, v in top))
