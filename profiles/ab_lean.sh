# A/B of lean-kernel build variants (paper_2203_06117_b200/libglsim_cuda_<v>.so),
# interleaved rounds; one JSON line per run into gpurun_out/ab_lean.jsonl
mkdir -p gpurun_out
: > gpurun_out/ab_lean.jsonl
for r in 1 2 3; do
  for v in $VARIANTS; do
    for c in "C3 --windows 8192" "C2"; do
      line=$(GLSIM_LIB=libglsim_cuda_$v.so timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | grep '^{')
      echo "{\"variant\": \"$v\", \"round\": $r, \"run\": $line}" >> gpurun_out/ab_lean.jsonl
    done
  done
done
python - <<'PY'
import json, collections, statistics
d = collections.defaultdict(list)
for l in open("gpurun_out/ab_lean.jsonl"):
    try:
        x = json.loads(l)
    except Exception:
        continue
    r = x["run"]
    d[(x["variant"], r["config"]["workload"][:2])].append(r["roofline"]["k4_ms_per_step"])
for k, v in sorted(d.items()):
    print(k, "k4 ms", [round(a, 2) for a in v], "median", round(statistics.median(v), 2))
PY
