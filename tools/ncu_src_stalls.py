"""Top SASS instructions of one kernel by warp-stall samples, with their source line and leading
stall reasons (ncu --set full --import-source on, -lineinfo build):
ncu_src_stalls.py report.ncu-rep <kernel regex> [top] [source-line filter]"""
import csv, subprocess, sys
rep, regex = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{regex}",
                      "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout.splitlines()
hdr, rows, fname = None, [], ""
for r in csv.reader(out):
    if len(r) >= 2 and r[0] == "File Name":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[2]:
        continue
    d = dict(zip(range(len(hdr)), r))
    rows.append((fname, r[0], r[1], r[2], r[3], r))
def num(x):
    try:
        return float(x)
    except (TypeError, ValueError):
        return 0.0
si = hdr.index("Warp Stall Sampling (All Samples)")
stall_idx = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(num(r[5][si]) for r in rows) or 1
print(f"total samples {tot:.0f}")
for fn, ln, src, addr, sass, r in sorted(rows, key=lambda x: -num(x[5][si]))[:top]:
    parts = sorted(((num(r[i]), hdr[i][6:]) for i in stall_idx if num(r[i]) > 0), reverse=True)[:3]
    print(f"{100 * num(r[si]) / tot:5.1f}% {fn}:{ln:>4} {sass.strip()[:48]:48s} | {src.strip()[:50]:50s} | "
          + " ".join(f"{n}={v:.0f}" for v, n in parts))
