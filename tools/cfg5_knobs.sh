# cfg5: per-kernel times (split fwd, residual sum, split adj, update sum) under the existing knobs
for v in "KB_NONE=0" "KB_TC_SPLIT_EPI=4" "KB_TC1_NST=4" "KB_TC1_NST=6" "KB_RING_STAGES=6" "KB_TC_G=2" "KB_AXIS_SWAP=0" "KB_PDL=0" "KB_NONE=1"; do
  echo -n "$v  "; env $v timeout 300 python tools/time_kernels.py cfg5 float32 2>/dev/null | tail -1
done
