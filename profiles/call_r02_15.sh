set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/c15_gpu_tests.txt 2>&1
tail -5 gpurun_out/c15_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c15_smoke.txt 2>&1
timeout 600 python bench.py --config C3 --windows 8192 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c15_bench_c3.log 2>&1
grep -h '^{' gpurun_out/c15_bench_c3.log | cut -c1-300
