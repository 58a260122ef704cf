"""Per-source-line stall samples and executed instructions of one kernel launch in an ncu report
(--set full, -lineinfo build):  ncu_src_lines.py report.ncu-rep <kernel regex> [skip] [top]"""
import csv
import subprocess
import sys

rep, regex = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{regex}",
                      "--launch-skip", skip, "--launch-count", "1", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
fname, hdr = None, None
samples, inst = {}, {}
for r in csv.reader(out):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 2 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or not r[0].isdigit():
        continue
    key = (fname, int(r[0]), r[1].strip()[:80])
    try:
        samples[key] = samples.get(key, 0) + int(r[4] or 0)
        inst[key] = inst.get(key, 0) + int(r[7] or 0)
    except ValueError:
        pass
ts, ti = max(1, sum(samples.values())), max(1, sum(inst.values()))
print(f"samples {ts}  warp instructions {ti}")
for k, v in sorted(samples.items(), key=lambda x: -x[1])[:top]:
    print(f"{v:6d} {100 * v / ts:5.1f}%  inst {100 * inst[k] / ti:5.1f}%  {k[0]}:{k[1]}  {k[2]}")
