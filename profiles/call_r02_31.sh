set -x
mkdir -p gpurun_out
timeout 600 python bench.py --config C3 --windows 4096 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c31_pre.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gate_eval_lean --launch-skip 41 --launch-count 3 -f -o gpurun_out/k4_c3_v4 python bench.py --config C3 --windows 4096 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c31_ncu.log 2>&1
tail -2 gpurun_out/c31_ncu.log
