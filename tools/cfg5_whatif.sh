# what-if timing of cfg5's four pass kernels with profiling switches (KB_DEBUG_MODE bits in the
# tcgen05 kernels: 1 skip MMAs, 2 skip the sum epilogue's loads/stores, 4 skip the A conversion)
for d in 0 1 2 4 5 6 7; do
  KB_DEBUG_MODE=$d timeout 300 python tools/time_kernels.py cfg5 float32 2>/dev/null | tail -1
done
