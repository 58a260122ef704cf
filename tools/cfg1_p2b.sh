# cfg1 persist2: staging-piece / Z-padding A/B (tmp_variants built by tools/variant.sh), same box
set -u
run() { (cd $1 && env $2 timeout 200 python bench.py --config cfg1 --no-variants --no-cpu-baseline --steps 30 2>/dev/null) | python -c "import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', d['value'], d['ms_per_step'], d['roofline']['frac'])"; }
for rep in 1 2; do
run . KB_PERSIST_RB=2
for v in orig np8 np4 p4; do run tmp_variants/$v KB_PERSIST_RB=2; done
run tmp_variants/orig KB_PERSIST_RB=1
done
