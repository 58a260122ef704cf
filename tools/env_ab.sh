#!/bin/bash
# A/B of environment settings on bench.py:  tools/env_ab.sh "<bench args>" rounds "VAR=a" "VAR=b" ...
args=$1
rounds=$2
shift 2
for i in $(seq "$rounds"); do
  for v in "$@"; do
    env $v timeout 300 python bench.py $args --no-variants --no-cpu-baseline 2>/dev/null |
      python -c "import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$v', round(d['value'],1), [round(x*1e3,1) for x in r.get('iteration',{}).get('per_kernel_ms',[])], r['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
