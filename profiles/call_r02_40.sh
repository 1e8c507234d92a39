set -x
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/c40_gpu_tests.txt 2>&1
tail -3 gpurun_out/c40_gpu_tests.txt
