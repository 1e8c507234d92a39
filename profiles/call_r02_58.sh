set -x
mkdir -p gpurun_out
timeout 600 python bench.py --config C3 --windows 4096 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c58_pre.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gate_eval_lean --launch-skip 42 --launch-count 2 -f -o gpurun_out/k4_c3_v6 python bench.py --config C3 --windows 4096 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c58_ncu.log 2>&1
tail -2 gpurun_out/c58_ncu.log
