"""Stall samples per CUDA source line of one kernel (ncu --set full report, -lineinfo build)."""
import csv
import subprocess
import sys

rep, regex = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{regex}",
                      "--launch-skip", skip, "--launch-count", "1", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
agg, files, fname = {}, {}, None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 5 or not r[0].isdigit():
        continue
    key = (fname, int(r[0]), r[1].strip()[:90])
    try:
        agg[key] = agg.get(key, 0) + int(r[4] or 0)
    except ValueError:
        pass
tot = sum(agg.values())
print("total samples", tot)
for (f, ln, src), v in sorted(agg.items(), key=lambda x: -x[1])[:int(sys.argv[4]) if len(sys.argv) > 4 else 30]:
    if v:
        print(f"{v:6d} {100 * v / tot:5.1f}%  {f}:{ln}  {src}")
