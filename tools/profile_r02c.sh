#!/bin/bash
# Round-2 final evidence, run on the GPU box from the repo root -> gpurun_out/prof4/:
# 1. pytest -m gpu, smoke 2. bench.py both arms (exit 0 without ncu) 3. the row-block path at N=1
# (direct and under torch.distributed.run) 4. launch list of the bench command 5. ncu --set full of
# the cfg1 whole-solve kernel (kb_solve_persistent2).
set -u
out=gpurun_out/prof4
mkdir -p $out
nvidia-smi > $out/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > $out/pytest_gpu.log 2>&1; echo "pytest rc $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc $?"
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err; echo "ref rc $?"
timeout 600 python bench.py --row-blocks --steps 2 --warmup 3 --no-cpu-baseline > $out/bench_rowblocks.json 2> $out/bench_rowblocks.err; echo "row-blocks rc $?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 1 --steps 2 --warmup 3 --no-variants --no-cpu-baseline > $out/bench_torchrun1.json 2> $out/bench_torchrun1.err; echo "torchrun rc $?"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:kb_ -c 700 --csv --log-file $out/launches_cfg5.csv \
  python bench.py --steps 2 --warmup 1 --no-variants --no-cpu-baseline > $out/ncu_launch.log 2>&1
echo "launch list rc $?"
python tools/launch_summary.py $out/launches_cfg5.csv > $out/launches_cfg5_summary.txt 2>&1
python tools/one_iter.py float64 20 cfg1 > $out/run_cfg1.log 2>&1; echo "plain cfg1 rc $?"
ncu --set full --import-source on --cache-control none --clock-control none -k regex:kb_solve_persistent -c 1 \
  -o $out/persist2_cfg1 python tools/one_iter.py float64 20 cfg1 > $out/ncu_cfg1.log 2>&1; echo "ncu cfg1 rc $?"
python tools/ncu_summary.py $out/persist2_cfg1.ncu-rep > $out/persist2_cfg1_summary.txt 2>&1
python tools/ncu_src_lines.py $out/persist2_cfg1.ncu-rep kb_solve_persistent2 0 30 > $out/persist2_cfg1_lines.txt 2>&1
rm -f $out/persist2_cfg1.ncu-rep
ls -la $out
