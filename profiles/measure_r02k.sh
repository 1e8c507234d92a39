# Round-2 final measurement pass (second kernel revision of the round) (GPU box, repo root): bench lines for every config,
# the reference arm, and the K4 launch list of the default (C3) bench.
set -x
mkdir -p gpurun_out
lscpu > gpurun_out/m11_lscpu.txt 2>&1
timeout 1200 python bench.py > gpurun_out/m11_default.log 2>&1
timeout 1200 python bench.py --impl reference > gpurun_out/m11_reference.log 2>&1
timeout 900 python bench.py --config C2 --steps 10 > gpurun_out/m11_c2.log 2>&1
timeout 900 python bench.py --config C1 --steps 10 > gpurun_out/m11_c1.log 2>&1
timeout 1200 python bench.py --config C4 --steps 3 > gpurun_out/m11_c4.log 2>&1
for v in C5 C5-pct0 C5-avg C5-avg-pct0; do
  timeout 900 python bench.py --config $v --windows 16384 --steps 3 > gpurun_out/m11_$v.log 2>&1
done
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:gate_eval -c 100 --csv --log-file gpurun_out/m11_launches_c3.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/m11_ncu_c3.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:gate_eval -c 80 --csv --log-file gpurun_out/m11_launches_c2.csv python bench.py --config C2 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/m11_ncu_c2.log 2>&1
grep -h '^{' gpurun_out/m11_*.log | cut -c1-200
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gate_eval_lean --launch-skip 41 --launch-count 1 -f -o gpurun_out/m11_k4_full python bench.py --config C3 --windows 4096 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/m11_ncu_full.log 2>&1
tail -2 gpurun_out/m11_ncu_full.log
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/m11_gpu_tests.txt 2>&1
tail -2 gpurun_out/m11_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/m11_smoke.txt 2>&1
tail -2 gpurun_out/m11_smoke.txt
