# cfg1 persist2 A/B over the synchronisation modes (KB_PERSIST2_SYNC), parity first
set -u
out=gpurun_out/p2c; mkdir -p $out
for sync in grid counter flags; do
  KB_PERSIST2_SYNC=$sync timeout 600 python -m pytest tests/test_gpu_persist2.py tests/test_gpu_projection.py "tests/test_gpu_fullsize.py::test_cfg1_against_the_references_own_solution" -x -q > $out/pytest_$sync.log 2>&1; echo "pytest $sync rc $?"
done
run() { (cd $1 && env $2 timeout 200 python bench.py --config cfg1 --no-variants --no-cpu-baseline --steps 30 2>/dev/null) | python -c "import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', d['value'], d['ms_per_step'], d['e2e']['value'])"; }
for rep in 1 2 3; do
  for sync in grid counter flags; do
    run . KB_PERSIST2_SYNC=$sync
  done
done
