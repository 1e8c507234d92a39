set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/c1_smi.txt 2>&1
lscpu > gpurun_out/c1_lscpu.txt 2>&1; free -g >> gpurun_out/c1_lscpu.txt
timeout 300 python profiles/prof_phases.py C3 4096 > gpurun_out/c1_prof_c3.txt 2>&1
timeout 300 python profiles/prof_phases.py C2 2048 > gpurun_out/c1_prof_c2.txt 2>&1
timeout 300 python profiles/prof_phases.py C4 512 > gpurun_out/c1_prof_c4.txt 2>&1
timeout 600 python bench.py --config C3 --windows 4096 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c1_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gate_eval -s 41 -c 1 -o gpurun_out/c1_k4_c3 python bench.py --config C3 --windows 4096 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c1_ncu.log 2>&1
tail -5 gpurun_out/c1_prof_c3.txt
