# cfg1 A/B of the whole-solve persistent kernel settings (bench.py cfg1 line per setting)
for v in "KB_PERSIST=0" "KB_PERSIST_SYNC=flags" "KB_PERSIST_RB=1" "KB_PERSIST_RB=2" "KB_PERSIST_RB=4"; do
  env $v timeout 200 python bench.py --config cfg1 --no-variants --no-cpu-baseline --steps 20 2>/dev/null | python -c "import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['value'], d['engines'][0], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
