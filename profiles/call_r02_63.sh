set -x
mkdir -p gpurun_out
GLSIM_LIB=libglsim_cuda_c8c7.so timeout 900 python -m pytest -m gpu -x -q tests/test_gpu_parity.py > gpurun_out/c63_gpu_tests.txt 2>&1
tail -3 gpurun_out/c63_gpu_tests.txt
VARIANTS="base c8c7" bash profiles/ab_lean.sh > gpurun_out/ab_lean34.txt 2>&1
tail -4 gpurun_out/ab_lean34.txt
