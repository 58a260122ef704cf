# cfg1 persist2: clock64 timeline of the middle iteration over all CTAs (KB_P2_TRACE build in tmp_variants/trace)
set -u
cd tmp_variants/trace
for sync in grid flags; do
  echo "== sync $sync"
  KB_P2_TRACE=1 KB_PERSIST2_SYNC=$sync timeout 200 python bench.py --config cfg1 --no-variants --no-cpu-baseline --steps 3 2>&1 | grep "p2 trace" | tail -2
done
