set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "stats_then_arena or arena_comes" > gpurun_out/c18_tests.txt 2>&1
tail -3 gpurun_out/c18_tests.txt
timeout 600 python bench.py --config C3 --windows 4096 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c18_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gate_eval -s 41 -c 1 -o gpurun_out/c18_k4_c3 python bench.py --config C3 --windows 4096 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c18_ncu.log 2>&1
