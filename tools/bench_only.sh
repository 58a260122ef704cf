set -u
out=gpurun_out/b2; mkdir -p $out
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc $?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/b2/bench.json').read().strip().splitlines()[-1])
print('cfg5', d['value'], d['e2e']['value'], d['ms_per_step'], d['clocks'])
for k,v in d['variants'].items(): print(k, v['value'], v['e2e'], v['per_kernel_ms'])
PY
