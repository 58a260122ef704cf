#!/bin/bash
# Round-2 final ncu captures of the configs not re-captured since round 1: one iteration's four
# kernels of cfg2 (fp64 DMMA, fp32 mma.sync + tcgen05) and cfg4 (tcgen05) with --set full
# (tensor-pipe counters, DRAM bytes), after each plain run exited 0 -> gpurun_out/prof5/
set -u
out=gpurun_out/prof5
mkdir -p $out
for spec in "cfg2 float64" "cfg2 float32" "cfg4 float32"; do
  set -- $spec; cfg=$1; dt=$2; tag=${cfg}_${dt}
  python tools/one_iter.py $dt 2 $cfg > $out/run_$tag.log 2>&1; echo "plain $tag rc $?"
  ncu --set full --import-source on --cache-control none --clock-control none -k regex:kb_pass_ -s 4 -c 4 \
    -o $out/iter_$tag python tools/one_iter.py $dt 2 $cfg > $out/ncu_$tag.log 2>&1; echo "ncu $tag rc $?"
  python tools/ncu_summary.py $out/iter_$tag.ncu-rep > $out/iter_${tag}_summary.txt 2>&1
  python tools/ncu_traffic.py $out/iter_$tag.ncu-rep $dt $out/traffic_$cfg.json $cfg > $out/iter_${tag}_traffic.txt 2>&1
  rm -f $out/iter_$tag.ncu-rep
done
ls -la $out
