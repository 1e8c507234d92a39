set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest -m gpu -x -q tests/test_sim_span_seam.py tests/test_synth_device.py tests/test_vcd_writer.py tests/test_netlist_reader.py > gpurun_out/c21_gpu_tests.txt 2>&1
tail -3 gpurun_out/c21_gpu_tests.txt
timeout 600 python bench.py --config C3 --windows 4096 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c21_pre.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gate_eval_lean --launch-skip 40 --launch-count 1 -f -o gpurun_out/k4_c3_cur python bench.py --config C3 --windows 4096 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c21_ncu.log 2>&1
tail -3 gpurun_out/c21_ncu.log
