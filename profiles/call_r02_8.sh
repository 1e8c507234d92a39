set -x
mkdir -p gpurun_out
timeout 600 python bench.py --config C3 --windows 4096 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c8_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gate_eval -s 41 -c 1 -o gpurun_out/c8_k4_c3 python bench.py --config C3 --windows 4096 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c8_ncu.log 2>&1
timeout 600 python bench.py --config C2 --windows 4096 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c8_plain2.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gate_eval -s 41 -c 1 -o gpurun_out/c8_k4_c2 python bench.py --config C2 --windows 4096 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c8_ncu2.log 2>&1
