"""Summarise an ncu report (--set full): duration, throughput, occupancy, pipe use, top stalls."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
KEYS = [
    ("gpu__time_duration.sum", "dur"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64pipe%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fmapipe%"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("dram__bytes_read.sum", "dramR"),
    ("dram__bytes_write.sum", "dramW"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "bankconf"),
]
for row in data:
    d = dict(zip(hdr, row))
    name = d.get("Kernel Name", "")[:60]
    parts = []
    for k, short in KEYS:
        v = d.get(k)
        if v not in (None, "", "n/a"):
            u = units[hdr.index(k)]
            parts.append(f"{short}={v}{'' if u in ('', '%') else u}")
    stalls = []
    for k, v in d.items():
        if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
            try:
                stalls.append((float(v), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    # tensor-pipe evidence (tcgen05 / DMMA / HMMA issue and activity): every pct-of-peak metric
    # whose name mentions the tensor pipes, so the summary shows tensor utilisation directly
    tens = []
    for k, v in d.items():
        lk = k.lower()
        if (("pipe_tensor_cycles_active" in lk or "inst_executed_pipe_tc.avg" in lk
             or "inst_executed_pipe_tmem.avg" in lk or "subpipe_hmma.avg" in lk or "subpipe_dmma.avg" in lk)
                and "pct" in lk and v not in ("", "n/a")):
            tens.append(f"{k.replace('TPC.TriageCompute.', '')}={v}")
    print(name)
    print("   ", " ".join(parts))
    if tens:
        print("    tensor:", " ".join(sorted(tens)))
    print("    stalls:", ", ".join(f"{n}={v:.2f}" for v, n in stalls[:6]))
