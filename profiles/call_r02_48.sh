set -x
GLSIM_LIB=libglsim_cuda_m60.so timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/m60.log 2>&1
tail -5 gpurun_out/m60.log
