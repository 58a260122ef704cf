"""Top SASS instructions by stall samples for one kernel of an ncu report (needs --set full)."""
import csv
import subprocess
import sys

rep, regex = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{regex}",
                      "--launch-skip", skip, "--launch-count", "1", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
hdr = rows[0]
data = [dict(zip(hdr, r)) for r in rows[1:] if len(r) == len(hdr) and r[0].startswith("0x")]
tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
print("total samples", tot, "instructions", len(data))
# group by opcode
from collections import Counter
byop = Counter()
cnt = Counter()
for d in data:
    op = d["Source"].split()[0] if d["Source"].split() else "?"
    if op.startswith("@"):
        op = d["Source"].split()[1]
    byop[op.split(".")[0]] += int(d["Warp Stall Sampling (All Samples)"] or 0)
    cnt[op.split(".")[0]] += int(d["Instructions Executed"] or 0)
print("samples by opcode:", byop.most_common(12))
print("executed by opcode:", cnt.most_common(12))
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = Counter()
for d in data:
    for h in stall_cols:
        agg[h] += int(d[h] or 0)
print("stalls:", agg.most_common(8))
top = sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:25]
for d in top:
    st = sorted(((int(d[h] or 0), h) for h in stall_cols), reverse=True)[:3]
    print(d["Warp Stall Sampling (All Samples)"], d["Source"].strip()[:60], st)
