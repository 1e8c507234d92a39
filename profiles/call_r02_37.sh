set -x
mkdir -p gpurun_out
timeout 900 python -m pytest -m gpu -x -q tests/test_gpu_parity.py -k "golden or random" > gpurun_out/c37_gpu_tests.txt 2>&1
tail -3 gpurun_out/c37_gpu_tests.txt
VARIANTS="base c7" bash profiles/ab_lean.sh > gpurun_out/ab_lean16.txt 2>&1
tail -4 gpurun_out/ab_lean16.txt
