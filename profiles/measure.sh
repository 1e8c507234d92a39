# Round measurement pass (run on the GPU box from the repo root):
#   bench lines for C2 (default, with CPU baseline), the reference arm, C3 and
#   C4 slices; the K4 launch list with DRAM bytes; one ncu --set full capture
#   of a C2 K4 launch (k = 2 group of a middle level).
set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
timeout 900 python bench.py --config C3 --windows 8192 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C3.log 2>&1
timeout 900 python bench.py --config C4 --windows 1024 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -c 100 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu1.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gate_eval -s 41 -c 1 -o gpurun_out/prof_k4_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu2.log 2>&1
tail -c 300 gpurun_out/bench_default.log
