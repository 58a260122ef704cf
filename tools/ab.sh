#!/bin/bash
# A/B timing on the GPU box: runs bench.py for one config in the working tree and in each
# tmp_variants/<name>, alternating, and prints value + per-kernel ms + clocks per run.
#   tools/ab.sh "<bench args>" rounds name1 name2 ...   ("." = the working tree)
args=$1
rounds=$2
shift 2
for i in $(seq "$rounds"); do
  for d in "$@"; do
    dir=.
    [ "$d" != "." ] && dir=tmp_variants/$d
    (cd "$dir" && timeout 300 python bench.py $args --no-variants --no-cpu-baseline 2>/dev/null |
      python -c "import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$d', round(d['value'],1), [round(x*1e3,1) for x in r.get('iteration',{}).get('per_kernel_ms',[])], r['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])")
  done
done
