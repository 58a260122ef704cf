# cfg4: slot sum pass (default) vs single- / two-accumulator 128-output sum pass: full-length error and rate
set -u
for v in "KB_NONE=0" "KB_TC_SUM1=2" "KB_TC_SUM1=1"; do
  echo "== $v"
  env $v timeout 300 python tools/fullsize_err.py cfg4_float32 2>&1 | tail -1
  env $v timeout 300 python bench.py --config cfg4 --no-variants --no-cpu-baseline --steps 5 2>/dev/null | python -c "import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['iteration']['per_kernel_ms'], d['clocks']['sm_mhz'])"
done
