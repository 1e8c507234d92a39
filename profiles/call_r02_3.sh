set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_synth_device.py -m gpu -x -q > gpurun_out/c3_synth_tests.txt 2>&1
tail -3 gpurun_out/c3_synth_tests.txt
timeout 600 python bench.py --config C3 --windows 4096 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c3_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gate_eval -s 41 -c 1 -o gpurun_out/c3_k4_c3 python bench.py --config C3 --windows 4096 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c3_ncu.log 2>&1
timeout 900 python bench.py > gpurun_out/c3_bench_default.log 2>&1
tail -c 2000 gpurun_out/c3_bench_default.log
