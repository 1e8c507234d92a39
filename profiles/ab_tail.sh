# A/B of the K4 tail split on the bench configs (dev helper):
# GS_TAIL_DIV (1 = off, 2, 4: tail item = tpi / div tiles),
# GS_TAIL_FRAC (split only when the tail is <= 1/frac of the tiles; 1 = always),
# GS_TAIL_MULT (tail = about MULT head items' worth of tiles per warp)
mkdir -p gpurun_out
r() { timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 "$@" | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), round(d['roofline']['frac'],4))"; }
for cfg in "" "--config C3 --windows 8192" "--config C3 --windows 2048"; do
  for i in 1 2; do
    for v in "2 2 1" "2 2 2" "3 2 1" "3 2 2" "4 2 2"; do set -- $v; echo -n "[$cfg] div=$1 frac=$2 mult=$3 "; GS_TAIL_DIV=$1 GS_TAIL_FRAC=$2 GS_TAIL_MULT=$3 r $cfg; done
  done
done
