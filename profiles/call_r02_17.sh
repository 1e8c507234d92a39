set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cli_gpu.py tests/test_distributed.py tests/test_reference_suite.py -m gpu -x -q > gpurun_out/c17_tests.txt 2>&1
tail -3 gpurun_out/c17_tests.txt
VARIANTS="base ctas6 cap16 cap4 mspread" bash profiles/ab_lean.sh > gpurun_out/ab_lean.txt 2>&1
tail -12 gpurun_out/ab_lean.txt
