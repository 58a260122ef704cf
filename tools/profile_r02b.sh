#!/bin/bash
# Round-2 (second half) evidence, run on the GPU box from the repo root -> gpurun_out/prof3/:
# 1. bench.py (exits 0 without ncu) 2. its launch list 3. ncu --set full of one cfg5 and one cfg3
# iteration (the 128-output single-accumulator sum pass) 4. the opt-in one-sweep kernel at cfg5.
set -u
out=gpurun_out/prof3
mkdir -p $out
python bench.py --steps 3 --warmup 3 --no-variants > $out/bench.json 2> $out/bench.err; echo "bench rc $?"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:kb_ -c 700 --csv --log-file $out/launches_cfg5.csv \
  python bench.py --steps 2 --warmup 1 --no-variants --no-cpu-baseline > $out/ncu_launch.log 2>&1
echo "launch list rc $?"
python tools/launch_summary.py $out/launches_cfg5.csv > $out/launches_cfg5_summary.txt 2>&1
for cfg in cfg5 cfg3; do
  if [ $cfg = cfg3 ]; then runner=tools/one_iter_batch.py; arg=512; else runner=tools/one_iter.py; arg=$cfg; fi
  python $runner float32 2 $arg > $out/run_$cfg.log 2>&1; echo "plain $cfg rc $?"
  ncu --set full --import-source on --cache-control none --clock-control none -k regex:kb_pass_ -s 4 -c 4 \
    -o $out/iter_$cfg python $runner float32 2 $arg > $out/ncu_$cfg.log 2>&1; echo "ncu $cfg rc $?"
  python tools/ncu_summary.py $out/iter_$cfg.ncu-rep > $out/iter_${cfg}_summary.txt 2>&1
  ncu -i $out/iter_$cfg.ncu-rep --page raw --csv > $out/iter_${cfg}_raw.csv 2>&1
  python tools/ncu_src_lines.py $out/iter_$cfg.ncu-rep kb_pass_sum_tc1 1 30 > $out/iter_${cfg}_sum_lines.txt 2>&1
  rm -f $out/iter_$cfg.ncu-rep
done
KB_FUSED=1 python tools/one_iter.py float32 2 cfg5 > $out/run_fused.log 2>&1; echo "plain fused rc $?"
KB_FUSED=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
  --cache-control none --clock-control none -k regex:kb_fused -s 2 -c 2 --csv --log-file $out/fused_cfg5.csv \
  python tools/one_iter.py float32 2 cfg5 > $out/ncu_fused.log 2>&1; echo "ncu fused rc $?"
ls -la $out
