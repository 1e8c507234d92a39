set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest -m gpu -x -q tests/test_gpu_parity.py tests/test_bench_instances.py tests/test_item_split.py tests/test_sim_span_seam.py > gpurun_out/c64_gpu_tests.txt 2>&1
tail -3 gpurun_out/c64_gpu_tests.txt
VARIANTS="base new" bash profiles/ab_lean.sh > gpurun_out/ab_lean35.txt 2>&1
tail -4 gpurun_out/ab_lean35.txt
