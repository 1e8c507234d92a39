set -x
mkdir -p gpurun_out
VARIANTS="base c9 c10" bash profiles/ab_lean.sh > gpurun_out/ab_lean10.txt 2>&1
tail -6 gpurun_out/ab_lean10.txt
