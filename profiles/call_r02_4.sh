set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/c4_gpu_tests.txt 2>&1
tail -5 gpurun_out/c4_gpu_tests.txt
timeout 300 python profiles/prof_phases.py C3 4096 > gpurun_out/c4_prof_c3.txt 2>&1
timeout 300 python profiles/prof_phases.py C2 2048 > gpurun_out/c4_prof_c2.txt 2>&1
timeout 600 python bench.py --config C3 --windows 8192 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c4_bench_c3.log 2>&1
timeout 600 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c4_bench_c2.log 2>&1
timeout 600 python bench.py --config C4 --windows 1024 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c4_bench_c4.log 2>&1
cat gpurun_out/c4_prof_c3.txt
