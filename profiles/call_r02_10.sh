set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -k "not bench_instances" > gpurun_out/c10_gpu_tests.txt 2>&1
tail -15 gpurun_out/c10_gpu_tests.txt
