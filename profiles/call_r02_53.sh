set -x
mkdir -p gpurun_out
timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c53_pre.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:stim_segment --launch-count 1 -f -o gpurun_out/k1_c3_final python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c53_ncu.log 2>&1
tail -2 gpurun_out/c53_ncu.log
