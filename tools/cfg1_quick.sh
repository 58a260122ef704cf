set -u
timeout 600 python -m pytest tests/test_gpu_persist2.py tests/test_gpu_projection.py "tests/test_gpu_fullsize.py::test_cfg1_against_the_references_own_solution" tests/test_gpu_configs.py -x -q 2>&1 | tail -2
for rep in 1 2 3; do
timeout 200 python bench.py --config cfg1 --no-variants --no-cpu-baseline --steps 30 2>/dev/null | python -c "import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'])"
done
