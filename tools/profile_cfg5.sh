#!/bin/bash
# ncu --set full of one cfg5 fp32 iteration's four pass kernels (tcgen05) -> text summaries.
set -u
out=gpurun_out/prof5
mkdir -p $out
python tools/one_iter.py float32 2 cfg5 > $out/run.log 2>&1; echo "plain rc $?"
ncu --set full --import-source on --cache-control none --clock-control none -k regex:kb_pass_ -s 4 -c 4 \
  -o $out/iter_cfg5 python tools/one_iter.py float32 2 cfg5 > $out/ncu.log 2>&1; echo "ncu rc $?"
python tools/ncu_summary.py $out/iter_cfg5.ncu-rep > $out/iter_cfg5_summary.txt 2>&1
ncu -i $out/iter_cfg5.ncu-rep --page raw --csv > $out/iter_cfg5_raw.csv 2>&1
python tools/ncu_src_lines.py $out/iter_cfg5.ncu-rep kb_pass_sum_tc 1 30 > $out/iter_cfg5_sum_lines.txt 2>&1
python tools/ncu_src_lines.py $out/iter_cfg5.ncu-rep kb_pass_split_tc 0 30 > $out/iter_cfg5_split_lines.txt 2>&1
rm -f $out/iter_cfg5.ncu-rep
ls -la $out
