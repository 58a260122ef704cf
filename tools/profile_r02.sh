#!/bin/bash
# Round-2 profiling set (run on the GPU box from the repo root; text summaries under
# gpurun_out/prof2/): 1. bench.py (exit 0 without ncu) 2. its ncu launch list 3. --set full of
# the cfg1 whole-solve persistent kernel.
set -u
out=gpurun_out/prof2
mkdir -p $out
python bench.py --steps 5 --warmup 3 --no-variants > $out/bench.json 2> $out/bench.err; echo "bench rc $?"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:kb_ -c 700 --csv --log-file $out/launches_cfg5.csv \
  python bench.py --steps 2 --warmup 1 --no-variants --no-cpu-baseline > $out/ncu_launch.log 2>&1
echo "launch list rc $?"
python tools/launch_summary.py $out/launches_cfg5.csv > $out/launches_cfg5_summary.txt 2>&1
ncu --set full --import-source on --cache-control none --clock-control none -k regex:kb_solve_persistent -c 1 \
  -o $out/persist_cfg1 python tools/one_iter.py float64 20 cfg1 > $out/persist.log 2>&1; echo "persist rc $?"
python tools/ncu_summary.py $out/persist_cfg1.ncu-rep > $out/persist_cfg1_summary.txt 2>&1
python tools/ncu_src_lines.py $out/persist_cfg1.ncu-rep kb_solve_persistent 0 30 > $out/persist_cfg1_lines.txt 2>&1
rm -f $out/persist_cfg1.ncu-rep
ls -la $out
