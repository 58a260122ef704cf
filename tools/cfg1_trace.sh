# cfg1 persist2: clock64 timeline of the middle CTA's middle iteration (KB_P2_TRACE build in tmp_variants/trace)
set -u
cd tmp_variants/trace
for sync in grid flags; do
  for rb in 2 1; do
    echo "== sync $sync RB $rb"
    KB_P2_TRACE=1 KB_PERSIST2_SYNC=$sync KB_PERSIST_RB=$rb timeout 200 python bench.py --config cfg1 --no-variants --no-cpu-baseline --steps 3 2>&1 | grep "p2 trace" | tail -3
  done
done
