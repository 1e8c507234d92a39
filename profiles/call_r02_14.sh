set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/c14_gpu_tests.txt 2>&1
tail -3 gpurun_out/c14_gpu_tests.txt
timeout 600 python bench.py --config C3 --windows 8192 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c14_bench_c3.log 2>&1
timeout 600 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c14_bench_c2.log 2>&1
grep -h '^{' gpurun_out/c14_bench_c3.log gpurun_out/c14_bench_c2.log | cut -c1-300
