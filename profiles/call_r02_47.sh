set -x
VARIANTS="base m60" bash profiles/ab_full_c3.sh > gpurun_out/ab_full1.txt 2>&1
tail -3 gpurun_out/ab_full1.txt
