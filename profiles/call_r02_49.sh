set -x
mkdir -p gpurun_out
GLSIM_LIB=libglsim_cuda_sp2.so timeout 900 python -m pytest -m gpu -x -q tests/test_gpu_parity.py tests/test_bench_instances.py > gpurun_out/c49_gpu_tests.txt 2>&1
tail -3 gpurun_out/c49_gpu_tests.txt
VARIANTS="base sp2" bash profiles/ab_lean.sh > gpurun_out/ab_lean23.txt 2>&1
tail -4 gpurun_out/ab_lean23.txt
