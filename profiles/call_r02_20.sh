set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/c20_gpu_tests.txt 2>&1
tail -5 gpurun_out/c20_gpu_tests.txt
VARIANTS="base new" bash profiles/ab_lean.sh > gpurun_out/ab_lean3.txt 2>&1
tail -6 gpurun_out/ab_lean3.txt
