# A/B of the K4 head item sizing with the tail split on (dev helper):
# tpi = min(GS_ITEM_CAP, n * Tc / (GS_ITEM_DIV * warps))
mkdir -p gpurun_out
r() { timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 "$@" | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), round(d['roofline']['frac'],4))"; }
for cfg in "" "--config C3 --windows 8192" "--config C3 --windows 2048"; do
  for v in "4 8" "4 12"; do set -- $v; echo -n "[$cfg] div=$1 cap=$2 "; GS_ITEM_DIV=$1 GS_ITEM_CAP=$2 r $cfg; done
done
