set -u
out=gpurun_out/v1; mkdir -p $out
nvidia-smi > $out/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 > $out/pytest_gpu.log 2>&1; echo "pytest rc $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc $?"
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err; echo "ref rc $?"
