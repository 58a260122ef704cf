# cfg1: second whole-solve kernel (kb_persist2.cuh) parity + A/B against the first form
set -u
out=gpurun_out/p2; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_persist2.py tests/test_gpu_projection.py "tests/test_gpu_fullsize.py::test_cfg1_against_the_references_own_solution" -x -q > $out/pytest.log 2>&1; echo "pytest rc $?"
for v in "KB_PERSIST2=0" "KB_PERSIST_RB=1" "KB_PERSIST_RB=2" "KB_PERSIST2=1"; do
  env $v timeout 200 python bench.py --config cfg1 --no-variants --no-cpu-baseline --steps 20 2>>$out/bench.err | python -c "import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'], d['engines'][0], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
