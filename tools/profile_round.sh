#!/bin/bash
# Round profiling set (run on the GPU box from the repo root; writes text summaries under
# gpurun_out/prof/, keeps only the cfg2 fp64 report to stay under gpurun's 64 MiB merge limit):
#  1. bench.py (exit 0 without ncu), 2. its ncu launch list, 3. --set full captures of one
#  iteration's four pass kernels at cfg2 fp64 / fp32, cfg4 fp32 and cfg3 (batch) fp32.
set -u
out=gpurun_out/prof
mkdir -p $out
python bench.py --steps 2 --warmup 1 > $out/bench.json 2> $out/bench.err; echo "bench rc $?"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:kb_ -c 400 --csv --log-file $out/launches_cfg2.csv \
  python bench.py --steps 2 --warmup 1 --no-variants --no-cpu-baseline > $out/ncu_launch.log 2>&1
echo "launch list rc $?"
python tools/launch_summary.py $out/launches_cfg2.csv > $out/launches_cfg2_summary.txt 2>&1
FULL="ncu --set full --import-source on --cache-control none --clock-control none -k regex:kb_pass_ -s 4 -c 4"
cap() {  # name, command...
  local name=$1; shift
  $FULL -o $out/$name "$@" > $out/$name.log 2>&1; echo "$name rc $?"
  python tools/ncu_summary.py $out/$name.ncu-rep > $out/${name}_summary.txt 2>&1
}
cap iter_cfg2_float64 python tools/one_iter.py float64 3 cfg2
python tools/ncu_traffic.py $out/iter_cfg2_float64.ncu-rep float64 $out/traffic_cfg2.json cfg2 > $out/traffic_cfg2_f64.txt 2>&1
python tools/ncu_src_lines.py $out/iter_cfg2_float64.ncu-rep kb_pass_sum_dmma 1 30 > $out/iter_cfg2_float64_update_lines.txt 2>&1
cap iter_cfg2_float32 python tools/one_iter.py float32 3 cfg2
python tools/ncu_traffic.py $out/iter_cfg2_float32.ncu-rep float32 $out/traffic_cfg2.json cfg2 > $out/traffic_cfg2_f32.txt 2>&1
rm -f $out/iter_cfg2_float32.ncu-rep
cap iter_cfg4_float32 python tools/one_iter.py float32 3 cfg4
python tools/ncu_traffic.py $out/iter_cfg4_float32.ncu-rep float32 $out/traffic_cfg4.json cfg4 > $out/traffic_cfg4_f32.txt 2>&1
python tools/ncu_src_lines.py $out/iter_cfg4_float32.ncu-rep kb_pass_sum_tc 1 30 > $out/iter_cfg4_float32_update_lines.txt 2>&1
rm -f $out/iter_cfg4_float32.ncu-rep
cap iter_cfg3_float32 python tools/one_iter_batch.py float32 3 512
python tools/ncu_traffic.py $out/iter_cfg3_float32.ncu-rep float32 $out/traffic_cfg3.json cfg3 > $out/traffic_cfg3_f32.txt 2>&1
rm -f $out/iter_cfg3_float32.ncu-rep
ls -la $out
