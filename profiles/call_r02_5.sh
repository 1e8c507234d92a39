set -x
mkdir -p gpurun_out
timeout 600 python bench.py --config C3 --windows 4096 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c5_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gate_eval -s 41 -c 1 -o gpurun_out/c5_k4_c3 python bench.py --config C3 --windows 4096 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c5_ncu.log 2>&1
timeout 2400 python -m pytest tests/test_reference_suite.py tests/test_synth_device.py tests/test_distributed.py -m gpu -x -q > gpurun_out/c5_tests.txt 2>&1
tail -30 gpurun_out/c5_tests.txt
